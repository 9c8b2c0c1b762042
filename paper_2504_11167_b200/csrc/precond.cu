// Interface Woodbury solve (K9) and low-rank recovery (K10) of apply_precond_T
// (SURVEY.md Appendix A.1/A.3).
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
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

constexpr int IA_THREADS = 256;

__global__ void __launch_bounds__(IA_THREADS) iface_apply_kernel(const IfaceApplyJob* jobs, int r,
                                                                 int64_t k, const double* y,
                                                                 int64_t ldy, int nrhs) {
  extern __shared__ double ism[];
  double* mW = ism;              // r x nrhs
  double* mT = mW + r * nrhs;
  double* vTz = mT + r * nrhs;
  double* h = vTz + r * nrhs;
  double* cT = h + r * nrhs;
  double* tmp = cT + r * nrhs;
  const IfaceApplyJob jb = jobs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = IA_THREADS / 32;
  // 2 r nrhs dot products of length k, one warp each
  for (int o = w; o < 2 * r * nrhs; o += nw) {
    const int which = o / (r * nrhs), aj = o % (r * nrhs);
    const int a = aj % r, j = aj / r;
    const double* vt = which ? jb.vtT : jb.vtW;
    const double* yy = y + (which ? jb.yt_row : jb.yb_row) + j * ldy;
    double s = 0.0;
    for (int64_t row = lane; row < k; row += 32) s = fma(vt[row + a * k], yy[row], s);
    s = warp_sum(s);
    if (lane == 0) (which ? mT : mW)[a + j * r] = s;
  }
  __syncthreads();
  const int nout = r * nrhs;
  // vTz = mT - E (sW .* mW)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    double s = mT[e];
    for (int c = 0; c < r; ++c) s -= jb.E[a + c * r] * (jb.sW[c] * mW[c + j * r]);
    vTz[e] = s;
  }
  __syncthreads();
  // h = Hinv (sT .* vTz)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    double s = 0.0;
    for (int c = 0; c < r; ++c) s += jb.Hinv[a + c * r] * (jb.sT[c] * vTz[c + j * r]);
    h[e] = s;
  }
  __syncthreads();
  // cT = vTz + E (sW .* h)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    double s = vTz[e];
    for (int c = 0; c < r; ++c) s += jb.E[a + c * r] * (jb.sW[c] * h[c + j * r]);
    cT[e] = s;
  }
  __syncthreads();
  // cW = mW - K (sT .* cT)
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r, j = e / r;
    double s = mW[e];
    for (int c = 0; c < r; ++c) s -= jb.K[a + c * r] * (jb.sT[c] * cT[c + j * r]);
    tmp[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < nout; e += IA_THREADS) {
    const int a = e % r;
    jb.scT[e] = jb.sT[a] * cT[e];
    jb.scW[e] = jb.sW[a] * tmp[e];
  }
}

void launch_iface_apply(Ctx* c, const IfaceApplyJob* d_jobs, int njobs, int r, int64_t k,
                        const double* y, int64_t ldy, int nrhs) {
  if (njobs == 0) return;
  const size_t smem = sizeof(double) * 6 * r * nrhs;
  ProfScope ps_(c, K_IFACE);
  iface_apply_kernel<<<njobs, IA_THREADS, smem, c->stream>>>(d_jobs, r, k, y, ldy, nrhs);
  LRS_LAUNCHED(c);
}

// x[row, j] = y[row, j] - sum_a uW[row, a] scW_p[a, j] - sum_a uT[row, a] scT_p[a, j]
// scT / scW: per partition r x MAX_RHS blocks (scT of the last partition and scW of the
// first are never read).
__global__ void __launch_bounds__(256) recovery_kernel(BandGeom g, int64_t n, const double* y,
                                                       int64_t ldy, double* x, int64_t ldx,
                                                       int nrhs, const double* __restrict__ uT,
                                                       const double* __restrict__ uW, int r,
                                                       const double* __restrict__ scT,
                                                       const double* __restrict__ scW) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  int lo = 0, hi = g.P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g.off[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  const int p = lo;
  const bool hasW = p > 0, hasT = p < g.P - 1;
  double acc[MAX_RHS];
  for (int j = 0; j < nrhs; ++j) acc[j] = y[row + j * ldy];
  if (hasW) {
    const double* sc = scW + (int64_t)p * r * MAX_RHS;
    for (int a = 0; a < r; ++a) {
      const double u = uW[row + a * n];
      for (int j = 0; j < nrhs; ++j) acc[j] -= u * sc[a + j * r];
    }
  }
  if (hasT) {
    const double* sc = scT + (int64_t)p * r * MAX_RHS;
    for (int a = 0; a < r; ++a) {
      const double u = uT[row + a * n];
      for (int j = 0; j < nrhs; ++j) acc[j] -= u * sc[a + j * r];
    }
  }
  for (int j = 0; j < nrhs; ++j) x[row + j * ldx] = acc[j];
}

void launch_recovery(Ctx* c, const BandGeom& g, int64_t n, const double* y, int64_t ldy, double* x,
                     int64_t ldx, int nrhs, const double* uT, const double* uW, int r,
                     const double* scT, const double* scW) {
  if (n == 0) return;
  ProfScope ps_(c, K_RECOVERY);
  recovery_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(g, n, y, ldy, x, ldx, nrhs,
                                                                      uT, uW, r, scT, scW);
  LRS_LAUNCHED(c);
}

}  // namespace lrs
