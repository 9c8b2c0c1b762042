// Krylov vector kernels (K12 of SURVEY.md 2.3) for bicgstab
// and GMRES(m), real and complex: column-batched, per-column scalars,
// Hermitian dot products, and deterministic reductions -- every dot product is summed
// per partition-aligned chunk in a fixed tree, per partition over its chunks in order,
// then over the GLOBAL partitions in order, so the result does not
// depend on launch geometry or on the number of GPUs.
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

constexpr int KV_THREADS = 256;

__device__ __forceinline__ double kv_warp_sum(double v) { return warp_sum(v); }
__device__ __forceinline__ zc kv_warp_sum(zc v) { return warp_sum_z(v); }

// Each pass over the chunk's rows serves QB vectors X_q at once, so Y (the GMRES w, bigger
// than L2 for the 16-column complex batches of c5) is read once per QB vectors instead of
// once per vector (measured on c5: 340 -> 319 ms of Krylov kernels per 80 GMRES steps;
// splitting the 16 columns over two CTAs per chunk was slower, 427 ms).  Per (q, column)
// the row order of each thread's sum and the reduction tree are those of one vector at a
// time: the results are bit-identical.
template <int NR, int QB, class S>
__global__ void __launch_bounds__(KV_THREADS) multidot_partial_kernel(
    const int64_t* __restrict__ cstart, const S* __restrict__ X, int64_t ldx, int64_t strideX,
    int nvec, const S* __restrict__ Y, int64_t ldy, int nrhs, S* __restrict__ partial) {
  __shared__ S red[KV_THREADS / 32][NR];
  const int c = blockIdx.x;
  const int64_t r0 = cstart[c], r1 = cstart[c + 1];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int q0 = 0; q0 < nvec; q0 += QB) {
    S acc[QB][NR];
#pragma unroll
    for (int qq = 0; qq < QB; ++qq)
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[qq][j] = s_zero(S());
    for (int64_t row = r0 + tid; row < r1; row += KV_THREADS) {
      S y[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) y[j] = j < nrhs ? Y[row + j * ldy] : s_zero(S());
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) {
        if (q0 + qq >= nvec) break;
        const S* Xq = X + (q0 + qq) * strideX;
#pragma unroll
        for (int j = 0; j < NR; ++j)
          if (j < nrhs) acc[qq][j] = s_cfma(Xq[row + j * ldx], y[j], acc[qq][j]);
      }
    }
#pragma unroll
    for (int qq = 0; qq < QB; ++qq) {
      if (q0 + qq >= nvec) break;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const S s = kv_warp_sum(acc[qq][j]);
        if (lane == 0) red[w][j] = s;
      }
      __syncthreads();
      if (tid < nrhs) {
        S s = s_zero(S());
        for (int ww = 0; ww < KV_THREADS / 32; ++ww) s = s_add(s, red[ww][tid]);
        partial[((int64_t)c * nvec + q0 + qq) * nrhs + tid] = s;
      }
      __syncthreads();
    }
  }
}

// persum[p][o] = sum of the chunk partials of local partition p, in chunk order
// (o indexes doubles: a complex output is two independent sums)
__global__ void multidot_partition_kernel(const int* __restrict__ part_first, int Pl, int nout,
                                          const double* __restrict__ partial,
                                          double* __restrict__ persum) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x, p = blockIdx.y;
  if (o >= nout || p >= Pl) return;
  double s = 0.0;
  for (int c = part_first[p]; c < part_first[p + 1]; ++c) s += partial[(int64_t)c * nout + o];
  persum[(int64_t)p * nout + o] = s;
}

// out[o] = sum over ranks r, partitions p < counts[r] (global partition order)
__global__ void partition_total_kernel(const double* __restrict__ blocks,
                                       const int* __restrict__ counts, int nranks, int pmax,
                                       int nout, double* __restrict__ out) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nout) return;
  double s = 0.0;
  for (int rk = 0; rk < nranks; ++rk)
    for (int p = 0; p < counts[rk]; ++p) s += blocks[((int64_t)rk * pmax + p) * nout + o];
  out[o] = s;
}

template <class S>
void launch_multidot_partition_t(Ctx* c, const Chunks& ch, const S* X, int64_t ldx,
                                 int64_t strideX, int nvec, const S* Y, int64_t ldy, int nrhs,
                                 S* partial, S* persum) {
  if (nvec == 0 || nrhs == 0) return;
  ProfScope ps_(c, K_KRYLOV);
  if (nrhs == 1)
    multidot_partial_kernel<1, 8, S><<<ch.nchunks, KV_THREADS, 0, c->stream>>>(
        ch.start, X, ldx, strideX, nvec, Y, ldy, nrhs, partial);
  else
    multidot_partial_kernel<MAX_RHS, sizeof(S) == 16 ? 2 : 4, S><<<ch.nchunks, KV_THREADS, 0,
                                                                 c->stream>>>(
        ch.start, X, ldx, strideX, nvec, Y, ldy, nrhs, partial);
  LRS_LAUNCHED(c);
  const int nout = nvec * nrhs * (int)(sizeof(S) / sizeof(double));
  multidot_partition_kernel<<<dim3((nout + 127) / 128, ch.Pl), 128, 0, c->stream>>>(
      ch.part_first, ch.Pl, nout, reinterpret_cast<const double*>(partial),
      reinterpret_cast<double*>(persum));
  LRS_LAUNCHED(c);
}

void launch_multidot_persum(Ctx* c, const Chunks& ch, int nout, const double* partial,
                            double* persum) {
  if (nout == 0) return;
  ProfScope ps_(c, K_KRYLOV);
  multidot_partition_kernel<<<dim3((nout + 127) / 128, ch.Pl), 128, 0, c->stream>>>(
      ch.part_first, ch.Pl, nout, partial, persum);
  LRS_LAUNCHED(c);
}

void launch_partition_total(Ctx* c, const double* blocks, const int* counts, int nranks,
                            int pmax, int nout, double* out) {
  if (nout == 0) return;
  ProfScope ps_(c, K_KRYLOV);
  partition_total_kernel<<<(nout + 127) / 128, 128, 0, c->stream>>>(blocks, counts, nranks, pmax,
                                                                     nout, out);
  LRS_LAUNCHED(c);
}

// Column-masked BLAS-1 updates; a, b per column, act[j] != 0 selects columns.
//  0: X = Y + a (X - b Z)      (BiCGStab p)
//  1: W = Y - a Z              (BiCGStab s = r - alpha v; r = s - omega t)
//  2: X = X + a Y + b Z        (BiCGStab x)
//  3: W = X + a Y              (half-step candidate x + alpha phat)
//  4: W = a Y                  (scale: GMRES basis normalisation)
//  5: W = Y                    (copy)
template <class S>
__global__ void __launch_bounds__(KV_THREADS) axpby_kernel(int64_t n, int nrhs, int op,
                                                           ColScalT<S> a, ColScalT<S> b,
                                                           ColScal act, S* X, int64_t ldx,
                                                           const S* Y, int64_t ldy, const S* Z,
                                                           int64_t ldz, S* W, int64_t ldw) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  // compile-time column indices into the by-value scalar arrays: a runtime index would copy
  // the 3 x 16 parameters into local memory in every thread
#pragma unroll
  for (int j = 0; j < MAX_RHS; ++j) {
    if (j >= nrhs) break;
    if (act.v[j] == 0.0) continue;
    const S aj = a.v[j], bj = b.v[j];
    switch (op) {
      case 0: {
        S* xp = X + row + j * ldx;
        *xp = s_add(Y[row + j * ldy], s_mul(aj, s_sub(*xp, s_mul(bj, Z[row + j * ldz]))));
      } break;
      case 1: W[row + j * ldw] = s_sub(Y[row + j * ldy], s_mul(aj, Z[row + j * ldz])); break;
      case 2: {
        S* xp = X + row + j * ldx;
        *xp = s_add(s_add(*xp, s_mul(aj, Y[row + j * ldy])), s_mul(bj, Z[row + j * ldz]));
      } break;
      case 3: W[row + j * ldw] = s_add(X[row + j * ldx], s_mul(aj, Y[row + j * ldy])); break;
      case 4: W[row + j * ldw] = s_mul(aj, Y[row + j * ldy]); break;
      default: W[row + j * ldw] = Y[row + j * ldy]; break;
    }
  }
}

template <class S>
void launch_axpby_cols_t(Ctx* c, int64_t n, int nrhs, int op, const ColScalT<S>& a,
                         const ColScalT<S>& b, const ColScal& act, S* X, int64_t ldx, const S* Y,
                         int64_t ldy, const S* Z, int64_t ldz, S* W, int64_t ldw) {
  if (n == 0 || nrhs == 0) return;
  ProfScope ps_(c, K_KRYLOV);
  axpby_kernel<S><<<(unsigned)((n + KV_THREADS - 1) / KV_THREADS), KV_THREADS, 0, c->stream>>>(
      n, nrhs, op, a, b, act, X, ldx, Y, ldy, Z, ldz, W, ldw);
  LRS_LAUNCHED(c);
}

template <class S>
__global__ void __launch_bounds__(KV_THREADS) multi_axpy_kernel(int64_t n, int nrhs,
                                                                const S* __restrict__ V,
                                                                int64_t ldv, int64_t strideV,
                                                                int nvec, const S* __restrict__ y,
                                                                double sign, S* x, int64_t ldx) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  for (int j = 0; j < nrhs; ++j) {
    S s = s_zero(S());
    for (int q = 0; q < nvec; ++q) s = s_fma(V[q * strideV + row + j * ldv], y[q * nrhs + j], s);
    x[row + j * ldx] = s_add(x[row + j * ldx], s_scale(s, sign));
  }
}

template <class S>
void launch_multi_axpy_t(Ctx* c, int64_t n, int nrhs, const S* V, int64_t ldv, int64_t strideV,
                         int nvec, const S* y_dev, double sign, S* x, int64_t ldx) {
  if (n == 0 || nrhs == 0 || nvec == 0) return;
  ProfScope ps_(c, K_KRYLOV);
  multi_axpy_kernel<S><<<(unsigned)((n + KV_THREADS - 1) / KV_THREADS), KV_THREADS, 0,
                         c->stream>>>(n, nrhs, V, ldv, strideV, nvec, y_dev, sign, x, ldx);
  LRS_LAUNCHED(c);
}

#define LRS_INST(S)                                                                             \
  template void launch_multidot_partition_t<S>(Ctx*, const Chunks&, const S*, int64_t, int64_t, \
                                               int, const S*, int64_t, int, S*, S*);            \
  template void launch_axpby_cols_t<S>(Ctx*, int64_t, int, int, const ColScalT<S>&,             \
                                       const ColScalT<S>&, const ColScal&, S*, int64_t,         \
                                       const S*, int64_t, const S*, int64_t, S*, int64_t);      \
  template void launch_multi_axpy_t<S>(Ctx*, int64_t, int, const S*, int64_t, int64_t, int,     \
                                       const S*, double, S*, int64_t);
LRS_INST(double)
LRS_INST(zc)
#undef LRS_INST

}  // namespace lrs
