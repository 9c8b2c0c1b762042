// CSR SpMV (K11) and the coupling SpMMs of the randomized spike SVD (K6).
//
// spmv follows reference proj/core/src/matrix.cpp:121-136: every output row
// sums its entries in ascending column order (one thread per row walks the
// row sequentially), so the summation order is the reference's.
#include "common.cuh"
#include "lrs_internal.h"
#include "kernels.h"

namespace lrs {

template <int NR>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t n, const int* __restrict__ rp,
                                                   const int* __restrict__ ci,
                                                   const double* __restrict__ va,
                                                   const double* __restrict__ x, int64_t ldx,
                                                   double* __restrict__ y, int64_t ldy, int nrhs,
                                                   int mode, const double* __restrict__ b,
                                                   int64_t ldb, int64_t row_lo) {
  const int64_t row = row_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  double acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.0;
  const int s = rp[row], e = rp[row + 1];
  for (int q = s; q < e; ++q) {
    const double v = va[q];
    const int64_t c = ci[q];
#pragma unroll
    for (int j = 0; j < NR; ++j)
      if (j < nrhs) acc[j] = fma(v, x[c + j * ldx], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (j >= nrhs) break;
    double* yo = y + row + j * ldy;
    if (mode == 0) *yo = acc[j];
    else if (mode == 1) *yo += acc[j];
    else *yo = b[row + j * ldb] - acc[j];
  }
}

void launch_spmv(Ctx* c, const Mat* m, const double* x, int64_t ldx, double* y, int64_t ldy,
                 int nrhs, int mode, const double* b, int64_t ldb, int64_t row_lo,
                 int64_t row_hi) {
  const int64_t n = row_hi < 0 ? m->n : row_hi;  // rows [row_lo, n)
  if (n <= row_lo || nrhs == 0) return;
  for (int j0 = 0; j0 < nrhs; j0 += MAX_RHS) {
    const int nr = nrhs - j0 < MAX_RHS ? nrhs - j0 : MAX_RHS;
    dim3 grid((unsigned)((n - row_lo + 255) / 256));
    const double* xj = x + j0 * ldx;
    double* yj = y + j0 * ldy;
    const double* bj = b ? b + j0 * ldb : nullptr;
    ProfScope ps_(c, K_SPMV);
#define LRS_SPMV(NRV)                                                                     \
  spmv_kernel<NRV><<<grid, 256, 0, c->stream>>>(n, m->row_ptr.get(), m->col_idx.get(),    \
                                                m->vals.get(), xj, ldx, yj, ldy, nr, mode, bj, \
                                                ldb, row_lo)
    if (nr == 1) LRS_SPMV(1);
    else if (nr <= 2) LRS_SPMV(2);
    else if (nr <= 4) LRS_SPMV(4);
    else if (nr <= 8) LRS_SPMV(8);
    else LRS_SPMV(16);
#undef LRS_SPMV
    LRS_LAUNCHED(c);
  }
}

// out[dst0 + (row - r0), j] = sum_{col in [c0, c0+b)} A[row, col] * X[col - c0, j]
// for row in [r0, r0 + b): the coupling block B_i / C_i (or their transposes,
// using the CSR of A^T) applied to a b x ncols block, written into a padded
// n_i x ncols right-hand side.
__global__ void __launch_bounds__(256) coupling_kernel(const CoupleJob* __restrict__ jobs,
                                                       const int* __restrict__ rp,
                                                       const int* __restrict__ ci,
                                                       const double* __restrict__ va) {
  const CoupleJob jb = jobs[blockIdx.y];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= jb.b * jb.ncols) return;
  const int64_t rr = t % jb.b;
  const int j = (int)(t / jb.b);
  const int64_t row = jb.r0 + rr;
  double acc = 0.0;
  const int s = rp[row], e = rp[row + 1];
  for (int q = s; q < e; ++q) {
    const int64_t col = ci[q];
    if (col < jb.c0 || col >= jb.c0 + jb.b) continue;
    acc = fma(va[q], jb.X[(col - jb.c0) + j * jb.ldx], acc);
  }
  jb.out[jb.dst0 + rr + j * jb.ldo] = acc;
}

void launch_coupling(Ctx* c, const Mat* m, bool transposed, const CoupleJob* d_jobs, int njobs,
                     int64_t b, int ncols) {
  if (njobs == 0) return;
  dim3 grid((unsigned)((b * ncols + 255) / 256), (unsigned)njobs);
  ProfScope ps_(c, K_SETUP);
  coupling_kernel<<<grid, 256, 0, c->stream>>>(
      d_jobs, transposed ? m->trow_ptr.get() : m->row_ptr.get(),
      transposed ? m->tcol_idx.get() : m->col_idx.get(),
      transposed ? m->tvals.get() : m->vals.get());
  LRS_LAUNCHED(c);
}

}  // namespace lrs
