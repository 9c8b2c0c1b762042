// Reduced-system kernels of LR-SPIKE-I and LR-SPIKE-OTF.
//
// A ReducedVector is stored compactly as a 2 k Pg x n_rhs column-major
// block: partition i's top tip x_{i,t} in rows [2ki, 2ki + k), its bottom tip x_{i,b} in
// rows [2ki + k, 2k(i+1)).  Tips may overlap in the n-layout when n_i < 2k; in the compact
// layout they are separate unknowns, as in the SPEC.
//
//   tips_gather  : r = [x +] tips(y)                 (n-layout -> compact)
//   tips_lowrank : out = in + sign (uW_tip scW + uT_tip scT), per tip with a term mask:
//                  matvec_lowrank uses both terms on both tips (sign +), the truncated
//                  preconditioner the W term on top tips and the T term on bottom tips
//                  (sign -), i.e. x_{i+1,t} = g_{i+1,t} - uW_t S_W cW, x_{i,b} = g_{i,b} -
//                  uT_b S_T cT (the elimination in precond.cu)
//   iface_scale  : scW_{i+1} = S_W m_W, scT_i = S_T m_T from the two messages of interface
//                  i (the compressed messages of matvec_lowrank and of the recovery)
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

// one thread per (compact row, column); local partitions only
template <class S>
__global__ void __launch_bounds__(256) tips_gather_kernel(BandGeom g, int64_t k, const S* y,
                                                          int64_t ldy, const S* x, S* r,
                                                          int64_t ldr, int nrhs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = 2 * k;
  if (t >= per * g.P * nrhs) return;
  const int j = (int)(t / (per * g.P));
  const int64_t e = t % (per * g.P);
  const int p = (int)(e / per);
  const int64_t q = e % per;
  const int64_t row = q < k ? g.off[p] + q : g.off[p] + g.size[p] - per + q;
  const int64_t cr = (int64_t)(g.p0 + p) * per + q;
  S v = y[row + j * ldy];
  if (x) v = s_add(x[cr + j * ldr], v);
  r[cr + j * ldr] = v;
}

template <class S>
void launch_tips_gather_t(Ctx* c, const BandGeom& g, int64_t k, const S* y, int64_t ldy,
                          const S* x, S* r, int64_t ldr, int nrhs) {
  const int64_t tot = 2 * k * g.P * nrhs;
  if (tot == 0) return;
  ProfScope ps_(c, K_IFACE);
  tips_gather_kernel<S><<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(g, k, y, ldy, x, r,
                                                                              ldr, nrhs);
  LRS_LAUNCHED(c);
}

// mode 0 (matvec_lowrank): both terms on every tip row; mode 1 (truncated precond): W
// term on top rows, T term on bottom rows.  sign: +1 / -1.
template <class S, int NRC>
__global__ void __launch_bounds__(256) tips_lowrank_kernel(BandGeom g, int64_t n, int64_t k,
                                                           const S* in, S* out, int64_t ldr,
                                                           int nrhs, const S* __restrict__ uT,
                                                           const S* __restrict__ uW, int r,
                                                           const S* __restrict__ scT,
                                                           const S* __restrict__ scW, int mode,
                                                           double sign) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = 2 * k;
  if (t >= per * g.P) return;
  const int p = (int)(t / per);
  const int64_t q = t % per;
  const int pg = g.p0 + p;
  const bool top = q < k;
  const int64_t urow = top ? g.off[p] + q : g.off[p] + g.size[p] - per + q;
  const int64_t cr = (int64_t)pg * per + q;
  const bool useW = pg > 0 && (mode == 0 || top);
  const bool useT = pg < g.Pg - 1 && (mode == 0 || !top);
  // NRC: compile-time bound of the column loops, so acc[] / d[] stay in registers
  S acc[NRC];
#pragma unroll
  for (int j = 0; j < NRC; ++j)
    if (j < nrhs) acc[j] = in[cr + j * ldr];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    if (side == 0 ? !useW : !useT) continue;
    const S* sc = (side == 0 ? scW : scT) + (int64_t)pg * r * MAX_RHS;
    const S* u = side == 0 ? uW : uT;
    S d[NRC];
#pragma unroll
    for (int j = 0; j < NRC; ++j) d[j] = s_zero(S());
    for (int a = 0; a < r; ++a) {
      const S ua = u[urow + a * n];
#pragma unroll
      for (int j = 0; j < NRC; ++j)
        if (j < nrhs) d[j] = s_fma(ua, sc[a + j * r], d[j]);
    }
#pragma unroll
    for (int j = 0; j < NRC; ++j)
      if (j < nrhs) acc[j] = s_add(acc[j], s_scale(d[j], sign));
  }
#pragma unroll
  for (int j = 0; j < NRC; ++j)
    if (j < nrhs) out[cr + j * ldr] = acc[j];
}

template <class S>
void launch_tips_lowrank_t(Ctx* c, const BandGeom& g, int64_t n, int64_t k, const S* in, S* out,
                           int64_t ldr, int nrhs, const S* uT, const S* uW, int r, const S* scT,
                           const S* scW, int mode, double sign) {
  const int64_t tot = 2 * k * g.P;
  if (tot == 0 || nrhs == 0) return;
  ProfScope ps_(c, K_RECOVERY);
  const unsigned grid = (unsigned)((tot + 255) / 256);
  if (nrhs == 1)
    tips_lowrank_kernel<S, 1><<<grid, 256, 0, c->stream>>>(g, n, k, in, out, ldr, nrhs, uT, uW, r,
                                                          scT, scW, mode, sign);
  else
    tips_lowrank_kernel<S, MAX_RHS><<<grid, 256, 0, c->stream>>>(g, n, k, in, out, ldr, nrhs, uT,
                                                                uW, r, scT, scW, mode, sign);
  LRS_LAUNCHED(c);
}

template <class S>
__global__ void iface_scale_kernel(const IfaceApplyJobT<S>* jobs, int r, int nrhs) {
  const IfaceApplyJobT<S> jb = jobs[blockIdx.x];
  for (int e = threadIdx.x; e < r * nrhs; e += blockDim.x) {
    const int a = e % r;
    jb.scW[e] = s_scale(jb.msg[e], jb.sW[a]);                 // S_W (vW x_{i,b})
    jb.scT[e] = s_scale(jb.msg[r * MAX_RHS + e], jb.sT[a]);   // S_T (vT x_{i+1,t})
  }
}

template <class S>
void launch_iface_scale_t(Ctx* c, const IfaceApplyJobT<S>* d_jobs, int njobs, int r, int nrhs) {
  if (njobs == 0) return;
  ProfScope ps_(c, K_IFACE);
  iface_scale_kernel<S><<<njobs, 128, 0, c->stream>>>(d_jobs, r, nrhs);
  LRS_LAUNCHED(c);
}

// *flag = 1 if a local row holds an entry outside its own partition's columns (some
// coupling block B_i / C_i is structurally nonzero); CSR columns are sorted, so the
// first and last entry of the row decide.
__global__ void coupling_present_kernel(const int* __restrict__ rp, const int* __restrict__ ci,
                                        BandGeom g, int64_t row_lo, int64_t row_hi, int* flag) {
  const int64_t row = row_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= row_hi) return;
  const int s = rp[row], e = rp[row + 1];
  if (s == e) return;
  int lo = 0, hi = g.P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g.off[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  if (ci[s] < g.off[lo] || ci[e - 1] >= g.off[lo] + g.size[lo]) atomicExch(flag, 1);
}

void launch_coupling_present(Ctx* c, const Mat* m, const BandGeom& g, int64_t row_lo,
                             int64_t row_hi, int* d_flag) {
  if (row_hi <= row_lo) return;
  ProfScope ps_(c, K_SETUP);
  coupling_present_kernel<<<(unsigned)((row_hi - row_lo + 255) / 256), 256, 0, c->stream>>>(
      m->row_ptr.get(), m->col_idx.get(), g, row_lo, row_hi, d_flag);
  LRS_LAUNCHED(c);
}

#define LRS_INST(S)                                                                             \
  template void launch_tips_gather_t<S>(Ctx*, const BandGeom&, int64_t, const S*, int64_t,      \
                                        const S*, S*, int64_t, int);                            \
  template void launch_tips_lowrank_t<S>(Ctx*, const BandGeom&, int64_t, int64_t, const S*, S*, \
                                         int64_t, int, const S*, const S*, int, const S*,       \
                                         const S*, int, double);                                \
  template void launch_iface_scale_t<S>(Ctx*, const IfaceApplyJobT<S>*, int, int, int);
LRS_INST(double)
LRS_INST(zc)
#undef LRS_INST

}  // namespace lrs
