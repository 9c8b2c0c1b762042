// Small dense kernels of the setup (K7/K8 of SURVEY.md 2.3): Householder QR of
// tall-skinny blocks (orth() of the randomized spike SVD),
// one-sided Jacobi SVD of the l x l R factor, the small GEMMs that form u and
// v, and the per-interface Woodbury setup of build_truncated_precond
// (G = K^-1 explicit, H = G - S_T vT uW S_W, cond_1 estimate).
// All run on the GPU, one CTA per job; nothing here falls back to the host.
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

// ---------------------------------------------------------------------------------------
// Householder QR (LAPACK dgeqr2 + dorg2r semantics, no column pivoting).
// ---------------------------------------------------------------------------------------
constexpr int QR_THREADS = 512;
constexpr int QR_CB = 8;  // columns per reduction batch

__global__ void __launch_bounds__(QR_THREADS) householder_qr_kernel(const QrJob* jobs, int l) {
  extern __shared__ double qsm[];
  double* tau = qsm;                 // l
  double* red = tau + l;             // (QR_THREADS/32) * QR_CB
  double* wv = red + (QR_THREADS / 32) * QR_CB;  // QR_CB
  const QrJob jb = jobs[blockIdx.x];
  double* A = jb.A;
  const int64_t m = jb.m, ld = jb.ld;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = QR_THREADS / 32;

  // apply H_j = I - tau v v^T (v_j = 1, v_i = A[i][j] for i > j) to columns [c0, c0+cb)
  auto apply_reflector = [&](int j, int c0, int cb, double tj) {
    double part[QR_CB];
#pragma unroll
    for (int u = 0; u < QR_CB; ++u) part[u] = 0.0;
    for (int64_t i = j + tid; i < m; i += QR_THREADS) {
      const double vi = (i == j) ? 1.0 : A[i + j * ld];
#pragma unroll
      for (int u = 0; u < QR_CB; ++u)
        if (u < cb) part[u] = fma(vi, A[i + (c0 + u) * ld], part[u]);
    }
#pragma unroll
    for (int u = 0; u < QR_CB; ++u) {
      const double s = warp_sum(part[u]);
      if (lane == 0) red[w * QR_CB + u] = s;
    }
    __syncthreads();
    if (tid < cb) {
      double s = 0.0;
      for (int q = 0; q < nw; ++q) s += red[q * QR_CB + tid];
      wv[tid] = s * tj;
    }
    __syncthreads();
    for (int64_t i = j + tid; i < m; i += QR_THREADS) {
      const double vi = (i == j) ? 1.0 : A[i + j * ld];
#pragma unroll
      for (int u = 0; u < QR_CB; ++u)
        if (u < cb) A[i + (c0 + u) * ld] -= vi * wv[u];
    }
    __syncthreads();
  };

  for (int j = 0; j < l; ++j) {
    double ss = 0.0;
    for (int64_t i = j + 1 + tid; i < m; i += QR_THREADS) {
      const double v = A[i + j * ld];
      ss = fma(v, v, ss);
    }
    ss = block_sum(ss, red);
    const double alpha = A[j + j * ld];
    const double xnorm = sqrt(ss);
    double tj = 0.0, scal = 1.0, beta = alpha;
    if (xnorm != 0.0) {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (tj != 0.0)
      for (int64_t i = j + 1 + tid; i < m; i += QR_THREADS) A[i + j * ld] *= scal;
    __syncthreads();
    if (tid == 0) {
      A[j + j * ld] = beta;
      tau[j] = tj;
    }
    __syncthreads();
    if (tj != 0.0)
      for (int c0 = j + 1; c0 < l; c0 += QR_CB) apply_reflector(j, c0, min(QR_CB, l - c0), tj);
  }
  if (jb.R) {
    for (int e = tid; e < l * l; e += QR_THREADS) {
      const int r = e % l, c = e / l;
      jb.R[e] = (r <= c) ? A[r + c * ld] : 0.0;
    }
  }
  __syncthreads();
  // form Q explicitly (dorg2r): right to left
  for (int j = l - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (j < l - 1 && tj != 0.0)
      for (int c0 = j + 1; c0 < l; c0 += QR_CB) apply_reflector(j, c0, min(QR_CB, l - c0), tj);
    for (int64_t i = tid; i < m; i += QR_THREADS) {
      double v;
      if (i < j) v = 0.0;
      else if (i == j) v = 1.0 - tj;
      else v = -tj * A[i + j * ld];
      A[i + j * ld] = v;
    }
    __syncthreads();
  }
}

void launch_householder_qr(Ctx* c, const QrJob* d_jobs, int njobs, int l) {
  if (njobs == 0) return;
  const size_t smem = sizeof(double) * (l + (QR_THREADS / 32) * QR_CB + QR_CB);
  ProfScope ps_(c, K_SETUP);
  householder_qr_kernel<<<njobs, QR_THREADS, smem, c->stream>>>(d_jobs, l);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi SVD of an l x l matrix R: R V = U diag(sigma).
// Round-robin pair ordering, one warp per pair, converged when a sweep makes no
// rotation with |c| > 1e-15 sqrt(a b).  Results sorted by sigma descending.
// ---------------------------------------------------------------------------------------
constexpr int SVD_THREADS = 256;
constexpr int SVD_MAXL = 96;

__global__ void __launch_bounds__(SVD_THREADS) jacobi_svd_kernel(const SvdJob* jobs, int l) {
  extern __shared__ double ssm[];
  const int L2 = (l + 1) & ~1;  // even number of slots (dummy column if l is odd)
  double* R = ssm;              // L2 x L2 column-major (padded rows/cols zero)
  double* V = R + L2 * L2;
  double* sg = V + L2 * L2;     // L2
  int* pos = reinterpret_cast<int*>(sg + L2);  // L2 tournament slots
  int* order = pos + L2;
  int* rotated = order + L2;
  const SvdJob jb = jobs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = SVD_THREADS / 32;
  for (int e = tid; e < L2 * L2; e += SVD_THREADS) {
    const int r = e % L2, c = e / L2;
    R[e] = (r < l && c < l) ? jb.R[r + c * l] : 0.0;
    V[e] = (r == c) ? 1.0 : 0.0;
  }
  for (int e = tid; e < L2; e += SVD_THREADS) pos[e] = e;
  __syncthreads();
  const int npairs = L2 / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) *rotated = 0;
    __syncthreads();
    for (int round = 0; round < L2 - 1; ++round) {
      for (int pr = w; pr < npairs; pr += nw) {
        int p = pos[pr], q = pos[L2 - 1 - pr];
        if (p > q) { const int t = p; p = q; q = t; }
        double a = 0, b = 0, cc = 0;
        for (int r = lane; r < L2; r += 32) {
          const double x = R[r + p * L2], y = R[r + q * L2];
          a = fma(x, x, a);
          b = fma(y, y, b);
          cc = fma(x, y, cc);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        cc = warp_sum(cc);
        if (fabs(cc) > 1e-15 * sqrt(a * b) && cc != 0.0) {
          const double zeta = (b - a) / (2.0 * cc);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          for (int r = lane; r < L2; r += 32) {
            const double x = R[r + p * L2], y = R[r + q * L2];
            R[r + p * L2] = cs * x - sn * y;
            R[r + q * L2] = sn * x + cs * y;
            const double vx = V[r + p * L2], vy = V[r + q * L2];
            V[r + p * L2] = cs * vx - sn * vy;
            V[r + q * L2] = sn * vx + cs * vy;
          }
          if (lane == 0) *rotated = 1;
        }
      }
      __syncthreads();
      // rotate tournament positions (slot 0 fixed)
      if (tid == 0) {
        const int last = pos[L2 - 1];
        for (int e = L2 - 1; e > 1; --e) pos[e] = pos[e - 1];
        pos[1] = last;
      }
      __syncthreads();
    }
    const int any = *rotated;
    __syncthreads();
    if (!any) break;
  }
  // singular values and ordering
  for (int c = w; c < L2; c += nw) {
    double s = 0.0;
    for (int r = lane; r < L2; r += 32) s = fma(R[r + c * L2], R[r + c * L2], s);
    s = warp_sum(s);
    if (lane == 0) sg[c] = sqrt(s);
  }
  __syncthreads();
  if (tid == 0) {
    for (int c = 0; c < l; ++c) order[c] = c;
    for (int a = 0; a < l; ++a) {  // stable selection sort, descending
      int best = a;
      for (int b = a + 1; b < l; ++b)
        if (sg[order[b]] > sg[order[best]]) best = b;
      const int t = order[best];
      for (int b = best; b > a; --b) order[b] = order[b - 1];
      order[a] = t;
    }
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += SVD_THREADS) {
    const int r = e % l, c = e / l;
    const int src = order[c];
    const double s = sg[src];
    jb.V[r + c * l] = V[r + src * L2];
    jb.U[r + c * l] = s > 0.0 ? R[r + src * L2] / s : (r == c ? 1.0 : 0.0);
  }
  for (int c = tid; c < l; c += SVD_THREADS) jb.sigma[c] = sg[order[c]];
}

void launch_jacobi_svd(Ctx* c, const SvdJob* d_jobs, int njobs, int l) {
  if (njobs == 0) return;
  if (l > SVD_MAXL) throw LrsError(LRS_ERR_PARAMETER, "n_svd + oversample > 96 not supported");
  const int L2 = (l + 1) & ~1;
  const size_t smem = sizeof(double) * (2 * L2 * L2 + L2) + sizeof(int) * (2 * L2 + 1);
  static bool attr = false;
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * (2 * 96 * 96 + 96) + sizeof(int) * 200)));
    attr = true;
  }
  ProfScope ps_(c, K_SETUP);
  jacobi_svd_kernel<<<njobs, SVD_THREADS, smem, c->stream>>>(d_jobs, l);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// C (m x n) = op(A) (m x k) * B (k x n); k, n <= 128 (B staged in shared memory).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) small_gemm_kernel(const GemmJob* jobs) {
  extern __shared__ double gsm[];
  const GemmJob jb = jobs[blockIdx.y];
  for (int e = threadIdx.x; e < jb.k * jb.n; e += blockDim.x) {
    const int r = e % jb.k, c = e / jb.k;
    gsm[e] = jb.B[r + c * jb.ldb];
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= jb.m) return;
  for (int c = 0; c < jb.n; ++c) {
    double s = 0.0;
    for (int kk = 0; kk < jb.k; ++kk) {
      const double a = jb.transA ? jb.A[kk + i * jb.lda] : jb.A[i + kk * jb.lda];
      s = fma(a, gsm[kk + c * jb.k], s);
    }
    jb.C[i + c * jb.ldc] = s;
  }
}

void launch_small_gemm(Ctx* c, const GemmJob* d_jobs, int njobs, int64_t max_m, int max_n) {
  if (njobs == 0 || max_m == 0) return;
  (void)max_n;
  static bool attr = false;
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(small_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * 128 * 128)));
    attr = true;
  }
  dim3 grid((unsigned)((max_m + 255) / 256), (unsigned)njobs);
  ProfScope ps_(c, K_SETUP);
  small_gemm_kernel<<<grid, 256, sizeof(double) * 128 * 128, c->stream>>>(d_jobs);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// Interface setup: K = vW uTb, E = vT uWt, G = K^-1, H = G - S_T E S_W, Hinv = H^-1,
// cond_1 of K and H.  Degenerate interfaces (a spike with all sigma = 0)
// are the identity: Hinv = 0, cond = 1.
// ---------------------------------------------------------------------------------------
constexpr int IF_THREADS = 256;

// Gauss-Jordan inverse with partial pivoting of an r x r matrix in shared memory.
// M is r x 2r column-major [A | I]; returns 0 on an exact zero pivot.
__device__ int gj_inverse(double* M, int r, int* piv_row) {
  const int tid = threadIdx.x;
  const int ld = r;
  __shared__ int s_ok;
  if (tid == 0) s_ok = 1;
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    if (tid == 0) {
      int best = j;
      double bv = fabs(M[j + j * ld]);
      for (int i = j + 1; i < r; ++i)
        if (fabs(M[i + j * ld]) > bv) { bv = fabs(M[i + j * ld]); best = i; }
      *piv_row = best;
      if (bv == 0.0) s_ok = 0;
    }
    __syncthreads();
    if (!s_ok) return 0;
    const int pr = *piv_row;
    if (pr != j)
      for (int c = tid; c < 2 * r; c += blockDim.x) {
        const double t = M[j + c * ld];
        M[j + c * ld] = M[pr + c * ld];
        M[pr + c * ld] = t;
      }
    __syncthreads();
    const double d = 1.0 / M[j + j * ld];
    __syncthreads();
    for (int c = tid; c < 2 * r; c += blockDim.x) M[j + c * ld] *= d;
    __syncthreads();
    for (int e = tid; e < r * 2 * r; e += blockDim.x) {
      const int i = e % r, c = e / r;
      if (i != j && c != j) M[i + c * ld] -= M[i + j * ld] * M[j + c * ld];
    }
    __syncthreads();
    for (int i = tid; i < r; i += blockDim.x)
      if (i != j) M[i + j * ld] = 0.0;
    __syncthreads();
  }
  return 1;
}

__device__ double norm1(const double* A, int r, int ld, double* red) {
  // max column sum of |A|, columns handled by threads, reduced by thread 0
  const int tid = threadIdx.x;
  for (int c = tid; c < r; c += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < r; ++i) s += fabs(A[i + c * ld]);
    red[c] = s;
  }
  __syncthreads();
  double mx = 0.0;
  for (int c = 0; c < r; ++c) mx = fmax(mx, red[c]);
  __syncthreads();
  return mx;
}

__global__ void __launch_bounds__(IF_THREADS) iface_setup_kernel(const IfaceSetupJob* jobs, int r,
                                                                 int64_t k) {
  extern __shared__ double fsm[];
  double* Ks = fsm;            // r x r
  double* Es = Ks + r * r;     // r x r
  double* M = Es + r * r;      // r x 2r
  double* red = M + 2 * r * r; // r
  __shared__ int piv;
  const IfaceSetupJob jb = jobs[blockIdx.x];
  const int tid = threadIdx.x;
  // K[a][c] = sum_row vtW[row, a] uTb[row, c];  E[a][c] = sum_row vtT[row, a] uWt[row, c]
  for (int e = tid; e < 2 * r * r; e += IF_THREADS) {
    const int which = e / (r * r), ac = e % (r * r);
    const int a = ac % r, c = ac / r;
    const double* vt = which ? jb.vtT : jb.vtW;
    const double* u = which ? jb.uWt : jb.uTb;
    const int64_t ldu = which ? jb.ld_uW : jb.ld_uT;
    double s = 0.0;
    for (int64_t row = 0; row < k; ++row) s = fma(vt[row + a * k], u[row + c * ldu], s);
    (which ? Es : Ks)[a + c * r] = s;
  }
  __syncthreads();
  bool degenerate = true;
  {
    bool anyT = false, anyW = false;
    for (int a = 0; a < r; ++a) {
      anyT |= jb.sT[a] != 0.0;
      anyW |= jb.sW[a] != 0.0;
    }
    degenerate = !(anyT && anyW);
  }
  for (int e = tid; e < r * r; e += IF_THREADS) {
    jb.K[e] = Ks[e];
    jb.E[e] = Es[e];
  }
  if (degenerate) {
    for (int e = tid; e < r * r; e += IF_THREADS) jb.Hinv[e] = 0.0;
    if (tid == 0) {
      jb.cond[0] = jb.cond[1] = 1.0;
      *jb.degenerate = 1;
    }
    return;
  }
  // G = K^-1
  for (int e = tid; e < 2 * r * r; e += IF_THREADS) {
    const int i = e % r, c = e / r;
    M[e] = (c < r) ? Ks[i + c * r] : (i == c - r ? 1.0 : 0.0);
  }
  __syncthreads();
  const double nK = norm1(Ks, r, r, red);
  const int okK = gj_inverse(M, r, &piv);
  double condK = INFINITY;
  if (okK) condK = nK * norm1(M + r * r, r, r, red);
  // H = G - S_T E S_W   (store H in Ks, G no longer needed afterwards)
  for (int e = tid; e < r * r; e += IF_THREADS) {
    const int a = e % r, c = e / r;
    Ks[e] = okK ? M[r * r + e] - jb.sT[a] * Es[e] * jb.sW[c] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < 2 * r * r; e += IF_THREADS) {
    const int i = e % r, c = e / r;
    M[e] = (c < r) ? Ks[i + c * r] : (i == c - r ? 1.0 : 0.0);
  }
  __syncthreads();
  const double nH = norm1(Ks, r, r, red);
  const int okH = okK ? gj_inverse(M, r, &piv) : 0;
  double condH = INFINITY;
  if (okH) condH = nH * norm1(M + r * r, r, r, red);
  for (int e = tid; e < r * r; e += IF_THREADS) jb.Hinv[e] = okH ? M[r * r + e] : 0.0;
  if (tid == 0) {
    jb.cond[0] = isfinite(condK) ? condK : INFINITY;
    jb.cond[1] = isfinite(condH) ? condH : INFINITY;
    *jb.degenerate = 0;
  }
}

void launch_iface_setup(Ctx* c, const IfaceSetupJob* d_jobs, int njobs, int r, int64_t k) {
  if (njobs == 0) return;
  const size_t smem = sizeof(double) * (4 * r * r + r);
  static bool attr = false;
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(iface_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * (4 * 64 * 64 + 64))));
    attr = true;
  }
  ProfScope ps_(c, K_SETUP);
  iface_setup_kernel<<<njobs, IF_THREADS, smem, c->stream>>>(d_jobs, r, k);
  LRS_LAUNCHED(c);
}

__global__ void sigma_trunc_kernel(const SigmaJob* jobs, int r, int* flag) {
  const SigmaJob jb = jobs[blockIdx.x];
  const double s0 = jb.sig[0];
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    const double s = jb.sig[j];
    const bool drop = (s0 == 0.0) || (s < 1e-14 * s0);
    jb.dst[j] = drop ? 0.0 : s;
    if (drop) atomicExch(flag, 1);
  }
}

void launch_sigma_trunc(Ctx* c, const SigmaJob* d_jobs, int njobs, int r, int* d_flag) {
  if (njobs == 0) return;
  ProfScope ps_(c, K_SETUP);
  sigma_trunc_kernel<<<njobs, 64, 0, c->stream>>>(d_jobs, r, d_flag);
  LRS_LAUNCHED(c);
}

}  // namespace lrs
