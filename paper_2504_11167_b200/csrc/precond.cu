// Interface Woodbury solve (K9) and low-rank recovery (K10) of apply_precond_T
// (SURVEY.md Appendix A.1/A.3), real and complex.
//
// Per interface i (partitions i, i+1), from the D-stage output y:
//   m_W = vW y_{i,b},  m_T = vT y_{i+1,t}                      (the two C1 messages)
//   vTz = m_T - E S_W m_W,  h = H^-1 (S_T vTz)
//   cT  = vTz + E S_W h          (= vT x_{i+1,t}, the C2 message to partition i)
//   cW  = m_W - K S_T cT         (= vW x_{i,b},  the C2 message to partition i+1)
// and the recovery x_p = y_p - uW_p (S_W cW) - uT_p (S_T cT).  This is the
// algebra of the oracle's literal W1-W3 + recovery with the reduced-solution
// tips eliminated (x_{i,b} = g_{i,b} - uTb S_T cT), so no b x n_rhs tip is
// ever formed; results agree with the oracle to roundoff.
//
// Multi-GPU: each side of a cross-GPU interface computes only its own message
// (m_W on the GPU of partition i, m_T on the GPU of partition i+1); the two
// r x n_rhs messages are exchanged (C1), after which both GPUs run the same
// deterministic r x r algebra and each keeps the half its recovery needs -- so
// the C2 messages never cross the link.
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

constexpr int IA_THREADS = 256;
constexpr int IA_ROWS = 256;  // tip rows per partial-dot CTA

__device__ __forceinline__ double warp_sum_s(double v) { return warp_sum(v); }
__device__ __forceinline__ zc warp_sum_s(zc v) { return warp_sum_z(v); }

// part[((job*2 + which)*nchunk + chunk)] = r x nrhs partial dots of v^T with y over a
// 256-row slice (which 0: m_W from y_{i,b}, 1: m_T from y_{i+1,t}); only local sides.
template <class S>
__global__ void __launch_bounds__(IA_THREADS) iface_dots_kernel(const IfaceApplyJobT<S>* jobs,
                                                                int r, int64_t k, const S* y,
                                                                int64_t ldy, int nrhs, S* part) {
  __shared__ S red[IA_THREADS / 32][MAX_RHS];
  const int job = blockIdx.y >> 1, which = blockIdx.y & 1, chunk = blockIdx.x;
  const int nchunk = gridDim.x;
  const IfaceApplyJobT<S> jb = jobs[job];
  if (which == 0 ? !jb.has_left : !jb.has_right) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t row = (int64_t)chunk * IA_ROWS + tid;
  const bool valid = row < k;
  const S* vt = which ? jb.vtT : jb.vtW;
  const S* yy = y + (which ? jb.yt_row : jb.yb_row);
  S yv[MAX_RHS];
#pragma unroll
  for (int j = 0; j < MAX_RHS; ++j) yv[j] = (valid && j < nrhs) ? yy[row + j * ldy] : s_zero(S());
  S* out = part + ((size_t)(job * 2 + which) * nchunk + chunk) * r * MAX_RHS;
  for (int a = 0; a < r; ++a) {
    const S v = valid ? vt[row + a * k] : s_zero(S());
#pragma unroll
    for (int j = 0; j < MAX_RHS; ++j) {
      if (j >= nrhs) break;
      const S s = warp_sum_s(s_mul(v, yv[j]));
      if (lane == 0) red[w][j] = s;
    }
    __syncthreads();
    if (tid < nrhs) {
      S s = s_zero(S());
      for (int q = 0; q < IA_THREADS / 32; ++q) s = s_add(s, red[q][tid]);
      out[a + tid * r] = s;
    }
    __syncthreads();
  }
}

// One right-hand side (the Krylov hot path): the same partial dots -- per row one product,
// a warp sum, the 8 warp sums in order, so bitwise the values of iface_dots_kernel -- but
// every thread loads its IA_AB columns of v at once and the warp sums of all r columns go
// to shared memory before ONE barrier (iface_dots_kernel waits on a barrier per column, so
// its v loads run one DRAM round trip at a time).
constexpr int IA_AB = 16;  // columns of v in flight per thread
template <class S>
__global__ void __launch_bounds__(IA_THREADS) iface_dots1_kernel(const IfaceApplyJobT<S>* jobs,
                                                                 int r, int64_t k, const S* y,
                                                                 S* part) {
  extern __shared__ __align__(16) unsigned char ia1_raw[];
  S* red = reinterpret_cast<S*>(ia1_raw);  // [IA_THREADS / 32][r]
  const int job = blockIdx.y >> 1, which = blockIdx.y & 1, chunk = blockIdx.x;
  const int nchunk = gridDim.x;
  const IfaceApplyJobT<S> jb = jobs[job];
  if (which == 0 ? !jb.has_left : !jb.has_right) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t row = (int64_t)chunk * IA_ROWS + tid;
  const bool valid = row < k;
  const S* vt = which ? jb.vtT : jb.vtW;
  const S yv = valid ? y[(which ? jb.yt_row : jb.yb_row) + row] : s_zero(S());
  for (int a0 = 0; a0 < r; a0 += IA_AB) {
    S v[IA_AB];
#pragma unroll
    for (int u = 0; u < IA_AB; ++u)
      v[u] = (valid && a0 + u < r) ? vt[row + (a0 + u) * k] : s_zero(S());
#pragma unroll
    for (int u = 0; u < IA_AB; ++u) {
      if (a0 + u >= r) break;
      const S sm = warp_sum_s(s_mul(v[u], yv));
      if (lane == 0) red[w * r + a0 + u] = sm;
    }
  }
  __syncthreads();
  S* out = part + ((size_t)(job * 2 + which) * nchunk + chunk) * r * MAX_RHS;
  for (int a = tid; a < r; a += IA_THREADS) {
    S sm = s_zero(S());
    for (int q = 0; q < IA_THREADS / 32; ++q) sm = s_add(sm, red[q * r + a]);
    out[a] = sm;
  }
}

// msg[which] = sum over chunks (fixed order) of the local partial messages
template <class S>
__global__ void iface_reduce_kernel(const IfaceApplyJobT<S>* jobs, int r, int nrhs, int nchunk,
                                    const S* part) {
  const IfaceApplyJobT<S> jb = jobs[blockIdx.x];
  for (int o = threadIdx.x; o < 2 * r * nrhs; o += blockDim.x) {
    const int which = o / (r * nrhs), aj = o % (r * nrhs);
    if (which == 0 ? !jb.has_left : !jb.has_right) continue;
    const S* pp = part + (size_t)(blockIdx.x * 2 + which) * nchunk * r * MAX_RHS + aj;
    S s = s_zero(S());
    for (int c = 0; c < nchunk; ++c) s = s_add(s, pp[(size_t)c * r * MAX_RHS]);
    jb.msg[which * r * MAX_RHS + aj] = s;
  }
}

template <class S>
__global__ void __launch_bounds__(IA_THREADS) iface_solve_kernel(const IfaceApplyJobT<S>* jobs,
                                                                 int r, int nrhs) {
  extern __shared__ __align__(16) unsigned char ism_raw[];
  S* mW = reinterpret_cast<S*>(ism_raw);  // r x nrhs
  S* mT = mW + r * nrhs;
  S* vTz = mT + r * nrhs;
  S* h = vTz + r * nrhs;
  S* cT = h + r * nrhs;
  S* tmp = cT + r * nrhs;
  const IfaceApplyJobT<S> jb = jobs[blockIdx.x];
  const int tid = threadIdx.x;
  for (int o = tid; o < r * nrhs; o += IA_THREADS) {
    mW[o] = jb.msg[o];
    mT[o] = jb.msg[r * MAX_RHS + o];
  }
  __syncthreads();
  const int nout = r * nrhs;
  // vTz = mT - E (sW .* mW)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    S s = mT[e];
    for (int c = 0; c < r; ++c) s = s_sub(s, s_mul(jb.E[a + c * r], s_scale(mW[c + j * r], jb.sW[c])));
    vTz[e] = s;
  }
  __syncthreads();
  // h = Hinv (sT .* vTz)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    S s = s_zero(S());
    for (int c = 0; c < r; ++c) s = s_add(s, s_mul(jb.Hinv[a + c * r], s_scale(vTz[c + j * r], jb.sT[c])));
    h[e] = s;
  }
  __syncthreads();
  // cT = vTz + E (sW .* h)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    S s = vTz[e];
    for (int c = 0; c < r; ++c) s = s_add(s, s_mul(jb.E[a + c * r], s_scale(h[c + j * r], jb.sW[c])));
    cT[e] = s;
  }
  __syncthreads();
  // cW = mW - K (sT .* cT)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    S s = mW[e];
    for (int c = 0; c < r; ++c) s = s_sub(s, s_mul(jb.K[a + c * r], s_scale(cT[c + j * r], jb.sT[c])));
    tmp[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r;
    if (jb.has_left) jb.scT[e] = s_scale(cT[e], jb.sT[a]);
    if (jb.has_right) jb.scW[e] = s_scale(tmp[e], jb.sW[a]);
  }
}

template <class S>
void launch_iface_messages_t(Ctx* c, const IfaceApplyJobT<S>* d_jobs, int njobs, int r, int64_t k,
                             const S* y, int64_t ldy, int nrhs, S* work) {
  if (njobs == 0) return;
  const int nchunk = (int)((k + IA_ROWS - 1) / IA_ROWS);
  ProfScope ps_(c, K_IFACE);
  if (nrhs == 1)
    iface_dots1_kernel<S><<<dim3(nchunk, 2 * njobs), IA_THREADS,
                            sizeof(S) * (IA_THREADS / 32) * r, c->stream>>>(d_jobs, r, k, y, work);
  else
    iface_dots_kernel<S><<<dim3(nchunk, 2 * njobs), IA_THREADS, 0, c->stream>>>(d_jobs, r, k, y,
                                                                                ldy, nrhs, work);
  LRS_LAUNCHED(c);
  iface_reduce_kernel<S><<<njobs, 128, 0, c->stream>>>(d_jobs, r, nrhs, nchunk, work);
  LRS_LAUNCHED(c);
}

template <class S>
void launch_iface_solve_t(Ctx* c, const IfaceApplyJobT<S>* d_jobs, int njobs, int r, int nrhs) {
  if (njobs == 0) return;
  ProfScope ps_(c, K_IFACE);
  const size_t smem = sizeof(S) * 6 * r * nrhs;
  iface_solve_kernel<S><<<njobs, IA_THREADS, smem, c->stream>>>(d_jobs, r, nrhs);
  LRS_LAUNCHED(c);
}

size_t iface_work_doubles(int njobs, int r, int64_t k) {
  return (size_t)njobs * 2 * ((k + IA_ROWS - 1) / IA_ROWS) * r * MAX_RHS;
}

// x[row, j] = y[row, j] - sum_a uW[row, a] scW_p[a, j] - sum_a uT[row, a] scT_p[a, j]
// for the local rows; scT / scW: one r x MAX_RHS block per GLOBAL partition (scT of the
// last partition and scW of the first are never read).
template <class S, int NRC>
__global__ void __launch_bounds__(256) recovery_kernel(BandGeom g, int64_t n, int64_t row_lo,
                                                       int64_t row_hi, const S* y, int64_t ldy,
                                                       S* x, int64_t ldx, int nrhs,
                                                       const S* __restrict__ uT,
                                                       const S* __restrict__ uW, int r,
                                                       const S* __restrict__ scT,
                                                       const S* __restrict__ scW) {
  const int64_t row = row_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= row_hi) return;
  int lo = 0, hi = g.P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g.off[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  const int pg = g.p0 + lo;
  const bool hasW = pg > 0, hasT = pg < g.Pg - 1;
  // NRC: compile-time bound of the column loops (1 for the Krylov hot path), so acc[] stays
  // in registers
  S acc[NRC];
#pragma unroll
  for (int j = 0; j < NRC; ++j)
    if (j < nrhs) acc[j] = y[row + j * ldy];
  if (hasW) {
    const S* sc = scW + (int64_t)pg * r * MAX_RHS;
    for (int a = 0; a < r; ++a) {
      const S u = uW[row + a * n];
#pragma unroll
      for (int j = 0; j < NRC; ++j)
        if (j < nrhs) acc[j] = s_sub(acc[j], s_mul(u, sc[a + j * r]));
    }
  }
  if (hasT) {
    const S* sc = scT + (int64_t)pg * r * MAX_RHS;
    for (int a = 0; a < r; ++a) {
      const S u = uT[row + a * n];
#pragma unroll
      for (int j = 0; j < NRC; ++j)
        if (j < nrhs) acc[j] = s_sub(acc[j], s_mul(u, sc[a + j * r]));
    }
  }
#pragma unroll
  for (int j = 0; j < NRC; ++j)
    if (j < nrhs) x[row + j * ldx] = acc[j];
}

template <class S>
void launch_recovery_t(Ctx* c, const BandGeom& g, int64_t n, int64_t row_lo, int64_t row_hi,
                       const S* y, int64_t ldy, S* x, int64_t ldx, int nrhs, const S* uT,
                       const S* uW, int r, const S* scT, const S* scW) {
  if (row_hi <= row_lo) return;
  ProfScope ps_(c, K_RECOVERY);
  const unsigned grid = (unsigned)((row_hi - row_lo + 255) / 256);
  if (nrhs == 1)
    recovery_kernel<S, 1><<<grid, 256, 0, c->stream>>>(g, n, row_lo, row_hi, y, ldy, x, ldx, nrhs,
                                                       uT, uW, r, scT, scW);
  else
    recovery_kernel<S, MAX_RHS><<<grid, 256, 0, c->stream>>>(g, n, row_lo, row_hi, y, ldy, x, ldx,
                                                             nrhs, uT, uW, r, scT, scW);
  LRS_LAUNCHED(c);
}

#define LRS_INST(S)                                                                              \
  template void launch_iface_messages_t<S>(Ctx*, const IfaceApplyJobT<S>*, int, int, int64_t,    \
                                           const S*, int64_t, int, S*);                          \
  template void launch_iface_solve_t<S>(Ctx*, const IfaceApplyJobT<S>*, int, int, int);          \
  template void launch_recovery_t<S>(Ctx*, const BandGeom&, int64_t, int64_t, int64_t, const S*, \
                                     int64_t, S*, int64_t, int, const S*, const S*, int,         \
                                     const S*, const S*);
LRS_INST(double)
LRS_INST(zc)
#undef LRS_INST

}  // namespace lrs
