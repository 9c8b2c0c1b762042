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

// Symmetric blocks (g.sym): with A_i = A_i^T (plain transpose, also for complex blocks) and
// no interchanges the trailing matrix stays symmetric, so U_KJ = inv(L_KK) A_KJ =
// diag(U_KK) L_JK^T: the U panel of step K is the transposed L panel with row a scaled by
// u_aa (the diagonal tile holds 1 / u_aa on the diagonal of inv(U_KK)).  The upper trailing
// tiles are then never read, and every trailing update forms the lower tiles only (half the
// GEMM work of the LU).  One CTA per panel tile, 32 x 32 blocks transposed through shared
// memory.
template <class S>
__global__ void __launch_bounds__(256) lu_mirror_kernel(BandGeom g, S* tiles, int K) {
  __shared__ S blk[32][33];
  __shared__ S d[NB];
  const int p = blockIdx.y, T = g.T[p], J = K + 1 + blockIdx.x;
  if (J >= T) return;
  const int64_t base = g.tbase[p];
  const S* dg = tiles + (base + (int64_t)K * g.W + g.wl) * TILE_ELEMS;
  const S* src = tiles + (base + (int64_t)J * g.W + (K - J + g.wl)) * TILE_ELEMS;  // L_JK
  S* dst = tiles + (base + (int64_t)K * g.W + (J - K + g.wl)) * TILE_ELEMS;        // U_KJ
  if (threadIdx.x < NB) d[threadIdx.x] = s_inv(dg[threadIdx.x * NB + threadIdx.x]);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int bb = 0; bb < 16; ++bb) {
    const int a0 = (bb >> 2) * 32, b0 = (bb & 3) * 32;  // block of U: rows a0.., columns b0..
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q)  // L_JK[b0 + tx][a0 + ty + 8 q]
      blk[ty + 8 * q][tx] = src[(int64_t)(a0 + ty + 8 * q) * NB + b0 + tx];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q)  // U_KJ[a0 + tx][b0 + ty + 8 q] = u_aa L_JK[b][a]
      dst[(int64_t)(b0 + ty + 8 * q) * NB + a0 + tx] = s_mul(d[a0 + tx], blk[tx][ty + 8 * q]);
  }
}

}  // namespace lrs
