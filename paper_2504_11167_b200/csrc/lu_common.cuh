// Device helpers shared by the band LU kernels (band_lu.cu, band_lu_piv.cu).
#pragma once

#include "lrs_internal.h"
#include "scalar.cuh"

namespace lrs {

// In-place inverses of the LU factors held in the 128 x 128 smem tile A: threads 0..255
// invert U (upper, non-unit, LAPACK dtrti2 'U'), threads 256..511 invert L (unit lower,
// dtrti2 'L' 'U'); disjoint triangles.  part: 4 x 128 doubles of scratch.
__device__ __forceinline__ void diag_inverses(double* A, double* part, int tid) {
  const int i = tid & (NB - 1);
  const int half = tid >> 8;           // 0: U, 1: L
  const int q = (tid >> 7) & 1;        // k-phase
  double* pq = part + (half * 2 + q) * NB;
  for (int s = 0; s < NB; ++s) {
    // phase 1: partial triangular mat-vec products (reads only)
    double ujj_inv = 0.0;
    if (half == 0) {
      const int j = s;
      // t_i = sum_{k=i}^{j-1} invU[i][k] * U[k][j]   for i < j
      double t = 0.0;
      if (i < j)
        for (int kk = i + q; kk < j; kk += 2) t = fma(A[kk * NB + i], A[j * NB + kk], t);
      pq[i] = t;
      ujj_inv = 1.0 / A[j * NB + j];
    } else {
      const int j = NB - 1 - s;
      // t_i = sum_{k=j+1}^{i-1} invL[i][k] * L[k][j]   for i > j
      double t = 0.0;
      if (i > j)
        for (int kk = j + 1 + q; kk < i; kk += 2) t = fma(A[kk * NB + i], A[j * NB + kk], t);
      pq[i] = t;
    }
    __syncthreads();
    // phase 2: write column j (disjoint addresses; no reads of other threads' outputs)
    if (q == 0) {
      if (half == 0) {
        const int j = s;
        if (i < j) A[j * NB + i] = -ujj_inv * (part[i] + part[NB + i]);
        else if (i == j) A[j * NB + j] = ujj_inv;
      } else {
        const int j = NB - 1 - s;
        if (i > j) A[j * NB + i] = -(A[j * NB + i] + part[2 * NB + i] + part[3 * NB + i]);
      }
    }
    __syncthreads();
  }
}


// complex in-place inverses of the LU factors of a 128 x 128 tile (any memory space): threads
// 0..255 invert U (ztrti2 'U'), threads 256..511 invert L (unit lower); part: 4 x 128 scratch
__device__ __forceinline__ void diag_inverses_z(zc* A, zc* part, int tid) {
  const int i = tid & (NB - 1);
  const int half = tid >> 8, q = (tid >> 7) & 1;
  zc* pq = part + (half * 2 + q) * NB;
  for (int s = 0; s < NB; ++s) {
    zc ujj_inv = {0.0, 0.0};
    if (half == 0) {
      const int j = s;
      zc t = {0.0, 0.0};
      if (i < j)
        for (int kk = i + q; kk < j; kk += 2) t = s_fma(A[kk * NB + i], A[j * NB + kk], t);
      pq[i] = t;
      ujj_inv = s_inv(A[j * NB + j]);
    } else {
      const int j = NB - 1 - s;
      zc t = {0.0, 0.0};
      if (i > j)
        for (int kk = j + 1 + q; kk < i; kk += 2) t = s_fma(A[kk * NB + i], A[j * NB + kk], t);
      pq[i] = t;
    }
    __syncthreads();
    if (q == 0) {
      if (half == 0) {
        const int j = s;
        if (i < j) A[j * NB + i] = s_neg(s_mul(ujj_inv, s_add(part[i], part[NB + i])));
        else if (i == j) A[j * NB + j] = ujj_inv;
      } else {
        const int j = NB - 1 - s;
        if (i > j)
          A[j * NB + i] = s_neg(s_add(A[j * NB + i], s_add(part[2 * NB + i], part[3 * NB + i])));
      }
    }
    __syncthreads();
  }
}

}  // namespace lrs
