// CSR SpMV (K11) and the coupling SpMMs of the randomized spike SVD (K6), real and
// complex.
//
// spmv follows reference proj/core/src/matrix.cpp:121-136: every output row
// sums its entries in ascending column order (one thread per row walks the
// row sequentially), so the summation order is the reference's.
//
// spmv_staged_kernel (default): a CTA owns 256 consecutive rows; their nonzeros, one
// contiguous range of col_idx / values, are staged through shared memory in chunks of
// SPMV_CAP entries with coalesced loads (a warp reads 32 consecutive 8-byte values and
// 4-byte indices), then each thread sums its own row from shared memory in ascending
// column order -- the one-thread-per-row kernel's summation order, without its strided
// per-thread loads (27-point rows put a warp's loads ~216 B apart).  LRS_SPMV_SCALAR=1
// selects the one-thread-per-row kernel.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

__device__ __forceinline__ double kv_sum(double v) { return warp_sum(v); }
__device__ __forceinline__ zc kv_sum(zc v) { return warp_sum_z(v); }

template <int NR, class S>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t n, const int* __restrict__ rp,
                                                   const int* __restrict__ ci,
                                                   const S* __restrict__ va,
                                                   const S* __restrict__ x, int64_t ldx,
                                                   S* __restrict__ y, int64_t ldy, int nrhs,
                                                   int mode, const S* __restrict__ b,
                                                   int64_t ldb, int64_t row_lo) {
  const int64_t row = row_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  S acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = s_zero(S());
  const int s = rp[row], e = rp[row + 1];
  for (int q = s; q < e; ++q) {
    const S v = va[q];
    const int64_t c = ci[q];
#pragma unroll
    for (int j = 0; j < NR; ++j)
      if (j < nrhs) acc[j] = s_fma(v, x[c + j * ldx], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (j >= nrhs) break;
    S* yo = y + row + j * ldy;
    if (mode == 0) *yo = acc[j];
    else if (mode == 1) *yo = s_add(*yo, acc[j]);
    else *yo = s_sub(b[row + j * ldb], acc[j]);
  }
}

constexpr int SPMV_ROWS = 256;
constexpr int SPMV_CAP = 4096;  // staged nonzeros per chunk: 48 KB (real), 80 KB (complex)

template <int NR, class S>
__global__ void __launch_bounds__(SPMV_ROWS) spmv_staged_kernel(
    int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const S* __restrict__ va,
    const S* __restrict__ x, int64_t ldx, S* __restrict__ y, int64_t ldy, int nrhs, int mode,
    const S* __restrict__ b, int64_t ldb, int64_t row_lo) {
  extern __shared__ __align__(16) unsigned char spmv_sm[];
  S* sv = reinterpret_cast<S*>(spmv_sm);
  int* sc = reinterpret_cast<int*>(sv + SPMV_CAP);
  const int64_t r0 = row_lo + (int64_t)blockIdx.x * SPMV_ROWS;
  const int64_t r1 = r0 + SPMV_ROWS < n ? r0 + SPMV_ROWS : n;
  const int64_t row = r0 + threadIdx.x;
  const int q0 = rp[r0], q1 = rp[r1];
  const int s = row < r1 ? rp[row] : q1, e = row < r1 ? rp[row + 1] : q1;
  S acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = s_zero(S());
  for (int base = q0; base < q1; base += SPMV_CAP) {
    const int cnt = q1 - base < SPMV_CAP ? q1 - base : SPMV_CAP;
    for (int t = threadIdx.x; t < cnt; t += SPMV_ROWS) {
      sv[t] = va[base + t];
      sc[t] = ci[base + t];
    }
    __syncthreads();
    const int a = s > base ? s : base, z = e < base + cnt ? e : base + cnt;
    for (int q = a; q < z; ++q) {
      const S v = sv[q - base];
      const int64_t col = sc[q - base];
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (j < nrhs) acc[j] = s_fma(v, x[col + j * ldx], acc[j]);
    }
    __syncthreads();
  }
  if (row >= r1) return;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (j >= nrhs) break;
    S* yo = y + row + j * ldy;
    if (mode == 0) *yo = acc[j];
    else if (mode == 1) *yo = s_add(*yo, acc[j]);
    else *yo = s_sub(b[row + j * ldb], acc[j]);
  }
}

template <class S>
static void spmv_t(Ctx* c, const Mat* m, const S* x, int64_t ldx, S* y, int64_t ldy, int nrhs,
                   int mode, const S* b, int64_t ldb, int64_t row_lo, int64_t row_hi) {
  const int64_t n = row_hi < 0 ? m->n : row_hi;  // rows [row_lo, n)
  if (n <= row_lo || nrhs == 0) return;
  const S* va = reinterpret_cast<const S*>(m->vals.get());
  for (int j0 = 0; j0 < nrhs; j0 += MAX_RHS) {
    const int nr = nrhs - j0 < MAX_RHS ? nrhs - j0 : MAX_RHS;
    dim3 grid((unsigned)((n - row_lo + 255) / 256));
    const S* xj = x + j0 * ldx;
    S* yj = y + j0 * ldy;
    const S* bj = b ? b + j0 * ldb : nullptr;
    ProfScope ps_(c, K_SPMV);
    static const bool scalar = std::getenv("LRS_SPMV_SCALAR") && std::getenv("LRS_SPMV_SCALAR")[0] == '1';
    constexpr size_t smem = (sizeof(S) + sizeof(int)) * SPMV_CAP;
#define LRS_SPMV(NRV)                                                                          \
  do {                                                                                         \
    if (scalar) {                                                                              \
      spmv_kernel<NRV, S><<<grid, 256, 0, c->stream>>>(n, m->row_ptr.get(), m->col_idx.get(),  \
                                                       va, xj, ldx, yj, ldy, nr, mode, bj, ldb, \
                                                       row_lo);                                \
    } else {                                                                                   \
      static bool attr_ = false;                                                               \
      if (!attr_) {                                                                            \
        LRS_CUDA(cudaFuncSetAttribute(spmv_staged_kernel<NRV, S>,                              \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        attr_ = true;                                                                          \
      }                                                                                        \
      spmv_staged_kernel<NRV, S><<<grid, SPMV_ROWS, smem, c->stream>>>(                        \
          n, m->row_ptr.get(), m->col_idx.get(), va, xj, ldx, yj, ldy, nr, mode, bj, ldb,      \
          row_lo);                                                                             \
    }                                                                                          \
  } while (0)
    if (nr == 1) LRS_SPMV(1);
    else if (nr <= 2) LRS_SPMV(2);
    else if (nr <= 4) LRS_SPMV(4);
    else if (nr <= 8) LRS_SPMV(8);
    else LRS_SPMV(16);
#undef LRS_SPMV
    LRS_LAUNCHED(c);
  }
}

void launch_spmv(Ctx* c, const Mat* m, const double* x, int64_t ldx, double* y, int64_t ldy,
                 int nrhs, int mode, const double* b, int64_t ldb, int64_t row_lo,
                 int64_t row_hi) {
  spmv_t<double>(c, m, x, ldx, y, ldy, nrhs, mode, b, ldb, row_lo, row_hi);
}

void launch_spmv_z(Ctx* c, const Mat* m, const zc* x, int64_t ldx, zc* y, int64_t ldy, int nrhs,
                   int mode, const zc* b, int64_t ldb, int64_t row_lo, int64_t row_hi) {
  spmv_t<zc>(c, m, x, ldx, y, ldy, nrhs, mode, b, ldb, row_lo, row_hi);
}

// ---- SpMV with the BiCGStab omega dots in its epilogue --------------------------------
// y = A x over one deterministic reduction chunk per CTA (the partition-aligned 2048-row
// chunks of the Krylov dots), then the chunk partials of [X^H y, y^H y] -- the t^H s and
// t^H t of BiCGStab's omega -- in the SAME per-thread row order and reduction tree as
// multidot_partial_kernel (krylov.cu): thread tid < 256 chains rows r0 + tid + 256 i in
// order, then a warp sum and the fixed-order sum over the 8 warps.  The partials are
// therefore bit-identical to the unfused SpMV + multidot, and one pass over t (and the
// launch of the dot kernel) disappears.  The SpMV half uses all SPMVD_THREADS threads
// with the staged coalesced nonzero loads of spmv_staged_kernel; each row's sum is in
// ascending column order (matrix.cpp:127-136), so y equals the plain SpMV bitwise.
constexpr int DOT_THREADS = 256;  // KV_THREADS of krylov.cu
// SpMV threads per CTA: 1024 for one or two columns; wider blocks keep 256 (register budget)
template <int NR, class S>
constexpr int spmvd_threads() { return NR * sizeof(S) <= 16 ? 1024 : DOT_THREADS; }

template <int NR, class S>
__global__ void __launch_bounds__(spmvd_threads<NR, S>()) spmv_dot2_kernel(
    const int64_t* __restrict__ cstart, const int* __restrict__ rp, const int* __restrict__ ci,
    const S* __restrict__ va, const S* __restrict__ x, int64_t ldx, S* y, int64_t ldy, int nrhs,
    const S* X, int64_t ldX, S* __restrict__ partial) {
  constexpr int SPMVD_THREADS = spmvd_threads<NR, S>();
  extern __shared__ __align__(16) unsigned char spmv_sm[];
  S* sv = reinterpret_cast<S*>(spmv_sm);
  int* sc = reinterpret_cast<int*>(sv + SPMV_CAP);
  __shared__ S red[DOT_THREADS / 32][NR];
  const int cidx = blockIdx.x, tid = threadIdx.x;
  const int64_t c0 = cstart[cidx], c1 = cstart[cidx + 1];
  for (int64_t r0 = c0; r0 < c1; r0 += SPMVD_THREADS) {
    const int64_t r1 = r0 + SPMVD_THREADS < c1 ? r0 + SPMVD_THREADS : c1;
    const int64_t row = r0 + tid;
    const int q0 = rp[r0], q1 = rp[r1];
    const int s = row < r1 ? rp[row] : q1, e = row < r1 ? rp[row + 1] : q1;
    S acc[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) acc[j] = s_zero(S());
    for (int base = q0; base < q1; base += SPMV_CAP) {
      const int cnt = q1 - base < SPMV_CAP ? q1 - base : SPMV_CAP;
      for (int t = tid; t < cnt; t += SPMVD_THREADS) {
        sv[t] = va[base + t];
        sc[t] = ci[base + t];
      }
      __syncthreads();
      const int a = s > base ? s : base, z = e < base + cnt ? e : base + cnt;
      for (int q = a; q < z; ++q) {
        const S v = sv[q - base];
        const int64_t col = sc[q - base];
#pragma unroll
        for (int j = 0; j < NR; ++j)
          if (j < nrhs) acc[j] = s_fma(v, x[col + j * ldx], acc[j]);
      }
      __syncthreads();
    }
    if (row < r1)
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (j < nrhs) y[row + j * ldy] = acc[j];
  }
  __syncthreads();  // the CTA's own y stores are visible to the CTA after the barrier
  if (tid >= DOT_THREADS) return;
  const int lane = tid & 31, w = tid >> 5;
  S d0[NR], d1[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) d0[j] = d1[j] = s_zero(S());
  for (int64_t row = c0 + tid; row < c1; row += DOT_THREADS) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j >= nrhs) break;
      const S yv = y[row + j * ldy];
      d0[j] = s_cfma(X[row + j * ldX], yv, d0[j]);
      d1[j] = s_cfma(yv, yv, d1[j]);
    }
  }
#pragma unroll
  for (int qq = 0; qq < 2; ++qq) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const S v = kv_sum(qq == 0 ? d0[j] : d1[j]);
      if (lane == 0) red[w][j] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(DOT_THREADS) : "memory");
    if (tid < nrhs) {
      S v = s_zero(S());
      for (int ww = 0; ww < DOT_THREADS / 32; ++ww) v = s_add(v, red[ww][tid]);
      partial[((int64_t)cidx * 2 + qq) * nrhs + tid] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(DOT_THREADS) : "memory");
  }
}

template <class S>
void launch_spmv_dot2_t(Ctx* c, const Mat* m, const Chunks& ch, const S* x, int64_t ldx, S* y,
                        int64_t ldy, int nrhs, const S* X, int64_t ldX, S* partial) {
  if (ch.nchunks == 0 || nrhs == 0) return;
  if (nrhs > MAX_RHS) throw LrsError(LRS_ERR_PARAMETER, "fused SpMV-dot batch > MAX_RHS");
  const S* va = reinterpret_cast<const S*>(m->vals.get());
  constexpr size_t smem = (sizeof(S) + sizeof(int)) * SPMV_CAP;
  {
    ProfScope ps_(c, K_SPMV);
#define LRS_SPMVD(NRV)                                                                         \
  do {                                                                                         \
    static bool attr_ = false;                                                                 \
    if (!attr_) {                                                                              \
      LRS_CUDA(cudaFuncSetAttribute(spmv_dot2_kernel<NRV, S>,                                  \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  \
      attr_ = true;                                                                            \
    }                                                                                          \
    spmv_dot2_kernel<NRV, S><<<ch.nchunks, spmvd_threads<NRV, S>(), smem, c->stream>>>(                  \
        ch.start, m->row_ptr.get(), m->col_idx.get(), va, x, ldx, y, ldy, nrhs, X, ldX,        \
        partial);                                                                              \
  } while (0)
    if (nrhs == 1) LRS_SPMVD(1);
    else if (nrhs <= 2) LRS_SPMVD(2);
    else if (nrhs <= 4) LRS_SPMVD(4);
    else if (nrhs <= 8) LRS_SPMVD(8);
    else LRS_SPMVD(16);
#undef LRS_SPMVD
    LRS_LAUNCHED(c);
  }
}
template void launch_spmv_dot2_t<double>(Ctx*, const Mat*, const Chunks&, const double*, int64_t,
                                         double*, int64_t, int, const double*, int64_t, double*);
template void launch_spmv_dot2_t<zc>(Ctx*, const Mat*, const Chunks&, const zc*, int64_t, zc*,
                                     int64_t, int, const zc*, int64_t, zc*);

// out[dst0 + (row - r0), j] = sum_{col in [c0, c0+b)} A[row, col] * X[col - c0, j]
// for row in [r0, r0 + b): the coupling block B_i / C_i (or their transposes,
// using the CSR of A^T; conjugated for the complex adjoint) applied to a b x ncols
// block, written into a padded n_i x ncols right-hand side.
template <class S>
__global__ void __launch_bounds__(256) coupling_kernel(const CoupleJobT<S>* __restrict__ jobs,
                                                       const int* __restrict__ rp,
                                                       const int* __restrict__ ci,
                                                       const S* __restrict__ va, int conj,
                                                       int accumulate) {
  const CoupleJobT<S> jb = jobs[blockIdx.y];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= jb.b * jb.ncols) return;
  const int64_t rr = t % jb.b;
  const int j = (int)(t / jb.b);
  const int64_t row = jb.r0 + rr;
  S acc = s_zero(S());
  const int s = rp[row], e = rp[row + 1];
  for (int q = s; q < e; ++q) {
    const int64_t col = ci[q];
    if (col < jb.c0 || col >= jb.c0 + jb.b) continue;
    const S v = conj ? s_conj(va[q]) : va[q];
    acc = s_fma(v, jb.X[(col - jb.c0) + j * jb.ldx], acc);
  }
  S* o = jb.out + jb.dst0 + rr + j * jb.ldo;
  *o = accumulate ? s_add(*o, acc) : acc;
}

template <class S>
void launch_coupling_t(Ctx* c, const Mat* m, bool transposed, const CoupleJobT<S>* d_jobs,
                       int njobs, int64_t b, int ncols, bool accumulate) {
  if (njobs == 0) return;
  dim3 grid((unsigned)((b * ncols + 255) / 256), (unsigned)njobs);
  ProfScope ps_(c, K_SETUP);
  const double* vals = transposed ? m->tvals.get() : m->vals.get();
  coupling_kernel<S><<<grid, 256, 0, c->stream>>>(
      d_jobs, transposed ? m->trow_ptr.get() : m->row_ptr.get(),
      transposed ? m->tcol_idx.get() : m->col_idx.get(), reinterpret_cast<const S*>(vals),
      transposed && IsC<S>::value ? 1 : 0, accumulate ? 1 : 0);
  LRS_LAUNCHED(c);
}
template void launch_coupling_t<double>(Ctx*, const Mat*, bool, const CoupleJobT<double>*, int,
                                        int64_t, int, bool);
template void launch_coupling_t<zc>(Ctx*, const Mat*, bool, const CoupleJobT<zc>*, int, int64_t,
                                    int, bool);

}  // namespace lrs
