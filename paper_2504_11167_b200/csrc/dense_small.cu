// Small dense kernels of the setup (K7/K8 of SURVEY.md 2.3), real and complex:
// Householder QR of tall-skinny blocks (orth() of the randomized spike SVD,
// SPEC.md:289, :310; LAPACK geqr2 + ung2r semantics), one-sided Jacobi SVD of the
// l x l R factor, the small GEMMs that form u and v, and the per-interface Woodbury
// setup of build_truncated_precond (G = K^-1 explicit,
// H = G - S_T vT uW S_W, cond_1 estimate).  All on the GPU, one CTA per job.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

__device__ __forceinline__ double ds_warp_sum(double v) { return warp_sum(v); }
__device__ __forceinline__ zc ds_warp_sum(zc v) { return warp_sum_z(v); }

// ---------------------------------------------------------------------------------------
// Householder QR.  Reflector j: H_j = I - tau_j v v^H (v_j = 1); the factorization
// applies H_j^H (coefficient conj(tau)), the explicit Q applies H_j (coefficient tau).
// ---------------------------------------------------------------------------------------
constexpr int QR_THREADS = 512;
constexpr int SVD_MAXL = 96;
constexpr int QR_CB = 8;  // columns per reduction batch

template <class S>
__global__ void __launch_bounds__(QR_THREADS) householder_qr_kernel(const QrJobT<S>* jobs, int l) {
  extern __shared__ __align__(16) unsigned char qsm_raw[];
  S* tau = reinterpret_cast<S*>(qsm_raw);   // l
  S* red = tau + l;                         // (QR_THREADS/32) * QR_CB
  S* wv = red + (QR_THREADS / 32) * QR_CB;  // QR_CB
  double* rs = reinterpret_cast<double*>(wv + QR_CB);  // QR_THREADS/32 real partials
  const QrJobT<S> jb = jobs[blockIdx.x];
  S* A = jb.A;
  const int64_t m = jb.m, ld = jb.ld;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = QR_THREADS / 32;

  // A[j:, c0:c0+cb] -= v (coef * (v^H A[j:, c]))
  auto apply_reflector = [&](int j, int c0, int cb, S coef) {
    S part[QR_CB];
#pragma unroll
    for (int u = 0; u < QR_CB; ++u) part[u] = s_zero(S());
    for (int64_t i = j + tid; i < m; i += QR_THREADS) {
      const S vi = (i == j) ? s_real<S>(1.0) : A[i + j * ld];
#pragma unroll
      for (int u = 0; u < QR_CB; ++u)
        if (u < cb) part[u] = s_cfma(vi, A[i + (c0 + u) * ld], part[u]);
    }
#pragma unroll
    for (int u = 0; u < QR_CB; ++u) {
      const S s = ds_warp_sum(part[u]);
      if (lane == 0) red[w * QR_CB + u] = s;
    }
    __syncthreads();
    if (tid < cb) {
      S s = s_zero(S());
      for (int q = 0; q < nw; ++q) s = s_add(s, red[q * QR_CB + tid]);
      wv[tid] = s_mul(coef, s);
    }
    __syncthreads();
    for (int64_t i = j + tid; i < m; i += QR_THREADS) {
      const S vi = (i == j) ? s_real<S>(1.0) : A[i + j * ld];
#pragma unroll
      for (int u = 0; u < QR_CB; ++u)
        if (u < cb) A[i + (c0 + u) * ld] = s_sub(A[i + (c0 + u) * ld], s_mul(vi, wv[u]));
    }
    __syncthreads();
  };

  for (int j = 0; j < l; ++j) {
    double ss = 0.0;
    for (int64_t i = j + 1 + tid; i < m; i += QR_THREADS) ss += s_abs2(A[i + j * ld]);
    ss = block_sum(ss, rs);
    const S alpha = A[j + j * ld];
    const double xnorm = sqrt(ss);
    S tj = s_zero(S()), scal = s_real<S>(1.0), beta = alpha;
    const double alphi = IsC<S>::value ? reinterpret_cast<const double*>(&alpha)[1] : 0.0;
    const double alphr = reinterpret_cast<const double*>(&alpha)[0];
    if (xnorm != 0.0 || alphi != 0.0) {  // LAPACK larfg
      const double b = -copysign(sqrt(alphr * alphr + alphi * alphi + ss), alphr);
      beta = s_real<S>(b);
      S t;
      if constexpr (IsC<S>::value) t = S{(b - alphr) / b, -alphi / b};
      else t = (b - alphr) / b;
      tj = t;
      scal = s_inv(s_sub(alpha, beta));
    }
    if (!s_iszero(tj))
      for (int64_t i = j + 1 + tid; i < m; i += QR_THREADS) A[i + j * ld] = s_mul(A[i + j * ld], scal);
    __syncthreads();
    if (tid == 0) {
      A[j + j * ld] = beta;
      tau[j] = tj;
    }
    __syncthreads();
    if (!s_iszero(tj))
      for (int c0 = j + 1; c0 < l; c0 += QR_CB)
        apply_reflector(j, c0, min(QR_CB, l - c0), s_conj(tj));
  }
  if (jb.R) {
    for (int e = tid; e < l * l; e += QR_THREADS) {
      const int r = e % l, c = e / l;
      jb.R[e] = (r <= c) ? A[r + c * ld] : s_zero(S());
    }
  }
  __syncthreads();
  // form Q explicitly (ung2r): right to left
  for (int j = l - 1; j >= 0; --j) {
    const S tj = tau[j];
    if (j < l - 1 && !s_iszero(tj))
      for (int c0 = j + 1; c0 < l; c0 += QR_CB) apply_reflector(j, c0, min(QR_CB, l - c0), tj);
    for (int64_t i = tid; i < m; i += QR_THREADS) {
      S v;
      if (i < j) v = s_zero(S());
      else if (i == j) v = s_sub(s_real<S>(1.0), tj);
      else v = s_neg(s_mul(tj, A[i + j * ld]));
      A[i + j * ld] = v;
    }
    __syncthreads();
  }
}

// Cluster variant: QRC CTAs per job (one thread-block cluster), each owning a contiguous
// slice of the rows, so a spike's QR streams through QRC SMs instead of one.  Every column
// reduction is a block reduction followed by a fixed-rank-order sum of the QRC block
// partials read through distributed shared memory (deterministic, identical on every CTA
// of the cluster).  Rank 0 owns rows 0..l-1 (requires ceil(m / QRC) >= l).
constexpr int QRC = 8;

template <class S>
__global__ void __cluster_dims__(QRC, 1, 1) __launch_bounds__(QR_THREADS)
    householder_qr_cluster_kernel(const QrJobT<S>* jobs, int l) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  constexpr int NW = QR_THREADS / 32;
  __shared__ S wred[NW][QR_CB];
  __shared__ S slot[2][QR_CB + 1];  // block partials (double buffered) + alpha broadcast
  __shared__ S tot[QR_CB + 1];
  __shared__ S tau[SVD_MAXL];
  const QrJobT<S> jb = jobs[blockIdx.x / QRC];
  S* A = jb.A;
  const int64_t m = jb.m, ld = jb.ld;
  const int64_t rows_per = (m + QRC - 1) / QRC;
  const int64_t r0 = crank * rows_per, r1 = min(m, r0 + rows_per);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int par = 0;
  // tot[u] = sum over the cluster of every thread's part[u], u < cb; tot[QR_CB] = the
  // value rank 0 passed as bcast (when given)
  auto cluster_sum = [&](const S* part, int cb, const S* bcast) {
#pragma unroll
    for (int u = 0; u < QR_CB; ++u)
      if (u < cb) {
        const S v = ds_warp_sum(part[u]);
        if (lane == 0) wred[w][u] = v;
      }
    __syncthreads();
    if (tid < cb) {
      S v = s_zero(S());
      for (int q = 0; q < NW; ++q) v = s_add(v, wred[q][tid]);
      slot[par][tid] = v;
    }
    if (bcast && crank == 0 && tid == 0) slot[par][QR_CB] = *bcast;
    cluster.sync();
    if (tid < cb) {
      S v = s_zero(S());
      for (int rk = 0; rk < QRC; ++rk) v = s_add(v, *cluster.map_shared_rank(&slot[par][tid], rk));
      tot[tid] = v;
    }
    if (bcast && tid == 0) tot[QR_CB] = *cluster.map_shared_rank(&slot[par][QR_CB], 0);
    __syncthreads();
    par ^= 1;
  };
  // A[j:, c0:c0+cb] -= v (coef * (v^H A[j:, c])) on this CTA's rows
  auto apply_reflector = [&](int j, int c0, int cb, S coef) {
    S part[QR_CB];
#pragma unroll
    for (int u = 0; u < QR_CB; ++u) part[u] = s_zero(S());
    for (int64_t i = (r0 > (int64_t)j ? r0 : (int64_t)j) + tid; i < r1; i += QR_THREADS) {
      const S vi = (i == j) ? s_real<S>(1.0) : A[i + j * ld];
#pragma unroll
      for (int u = 0; u < QR_CB; ++u)
        if (u < cb) part[u] = s_cfma(vi, A[i + (c0 + u) * ld], part[u]);
    }
    cluster_sum(part, cb, nullptr);
    S wv[QR_CB];
#pragma unroll
    for (int u = 0; u < QR_CB; ++u) wv[u] = u < cb ? s_mul(coef, tot[u]) : s_zero(S());
    for (int64_t i = (r0 > (int64_t)j ? r0 : (int64_t)j) + tid; i < r1; i += QR_THREADS) {
      const S vi = (i == j) ? s_real<S>(1.0) : A[i + j * ld];
#pragma unroll
      for (int u = 0; u < QR_CB; ++u)
        if (u < cb) A[i + (c0 + u) * ld] = s_sub(A[i + (c0 + u) * ld], s_mul(vi, wv[u]));
    }
    __syncthreads();
  };

  for (int j = 0; j < l; ++j) {
    S ss[QR_CB];
    ss[0] = s_zero(S());
    double acc = 0.0;
    for (int64_t i = (r0 > (int64_t)(j + 1) ? r0 : (int64_t)(j + 1)) + tid; i < r1; i += QR_THREADS) acc += s_abs2(A[i + j * ld]);
    ss[0] = s_real<S>(acc);
    S alpha_own = s_zero(S());
    if (crank == 0) alpha_own = A[j + j * ld];
    cluster_sum(ss, 1, &alpha_own);
    const double sq = reinterpret_cast<const double*>(&tot[0])[0];
    const S alpha = tot[QR_CB];
    const double xnorm = sqrt(sq);
    const double alphr = reinterpret_cast<const double*>(&alpha)[0];
    const double alphi = IsC<S>::value ? reinterpret_cast<const double*>(&alpha)[1] : 0.0;
    S tj = s_zero(S()), scal = s_real<S>(1.0), beta = alpha;
    if (xnorm != 0.0 || alphi != 0.0) {  // LAPACK larfg
      const double b = -copysign(sqrt(alphr * alphr + alphi * alphi + sq), alphr);
      beta = s_real<S>(b);
      S t;
      if constexpr (IsC<S>::value) t = S{(b - alphr) / b, -alphi / b};
      else t = (b - alphr) / b;
      tj = t;
      scal = s_inv(s_sub(alpha, beta));
    }
    if (!s_iszero(tj))
      for (int64_t i = (r0 > (int64_t)(j + 1) ? r0 : (int64_t)(j + 1)) + tid; i < r1; i += QR_THREADS)
        A[i + j * ld] = s_mul(A[i + j * ld], scal);
    __syncthreads();
    if (tid == 0) {
      if (crank == 0) A[j + j * ld] = beta;
      tau[j] = tj;
    }
    __syncthreads();
    if (!s_iszero(tj))
      for (int c0 = j + 1; c0 < l; c0 += QR_CB) apply_reflector(j, c0, min(QR_CB, l - c0), s_conj(tj));
  }
  if (jb.R && crank == 0) {
    for (int e = tid; e < l * l; e += QR_THREADS) {
      const int r = e % l, c = e / l;
      jb.R[e] = (r <= c) ? A[r + c * ld] : s_zero(S());
    }
  }
  __syncthreads();
  for (int j = l - 1; j >= 0; --j) {
    const S tj = tau[j];
    if (j < l - 1 && !s_iszero(tj))
      for (int c0 = j + 1; c0 < l; c0 += QR_CB) apply_reflector(j, c0, min(QR_CB, l - c0), tj);
    for (int64_t i = r0 + tid; i < r1; i += QR_THREADS) {
      S v;
      if (i < j) v = s_zero(S());
      else if (i == j) v = s_sub(s_real<S>(1.0), tj);
      else v = s_neg(s_mul(tj, A[i + j * ld]));
      A[i + j * ld] = v;
    }
    __syncthreads();
  }
  cluster.sync();  // no CTA leaves while another may still read its shared memory
}

template <class S>
void launch_householder_qr_t(Ctx* c, const QrJobT<S>* d_jobs, int njobs, int l, int64_t min_m) {
  if (njobs == 0) return;
  if (l <= SVD_MAXL && (min_m + QRC - 1) / QRC >= l && min_m >= 2048) {
    ProfScope ps_(c, K_SETUP);
    householder_qr_cluster_kernel<S><<<njobs * QRC, QR_THREADS, 0, c->stream>>>(d_jobs, l);
    LRS_LAUNCHED(c);
    return;
  }
  const size_t smem = sizeof(S) * (l + (QR_THREADS / 32) * QR_CB + QR_CB) +
                      sizeof(double) * (QR_THREADS / 32);
  ProfScope ps_(c, K_SETUP);
  householder_qr_kernel<S><<<njobs, QR_THREADS, smem, c->stream>>>(d_jobs, l);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi SVD of an l x l matrix R: R V = U diag(sigma).
// Round-robin pair ordering, one warp per pair, converged when a sweep makes no
// rotation with |c| > 1e-15 sqrt(a b).  Complex: column q is first turned by the phase
// of c = p^H q (a unitary diagonal factor, accumulated in V) so the rotation is real.
// Results sorted by sigma descending.
// ---------------------------------------------------------------------------------------
constexpr int SVD_THREADS = 256;

template <class S>
__global__ void __launch_bounds__(SVD_THREADS) jacobi_svd_kernel(const SvdJobT<S>* jobs, int l) {
  extern __shared__ __align__(16) unsigned char ssm_raw[];
  const int L2 = (l + 1) & ~1;  // even number of slots (dummy column if l is odd)
  S* R = reinterpret_cast<S*>(ssm_raw);  // L2 x L2 column-major (padded rows/cols zero)
  S* V = R + L2 * L2;
  double* sg = reinterpret_cast<double*>(V + L2 * L2);  // L2
  int* pos = reinterpret_cast<int*>(sg + L2);
  int* order = pos + L2;
  int* rotated = order + L2;
  S* scr = reinterpret_cast<S*>(ssm_raw + ((sizeof(S) * 2 * L2 * L2 + sizeof(double) * L2 +
                                            sizeof(int) * (2 * L2 + 1) + 15) & ~size_t(15)));
  const SvdJobT<S> jb = jobs[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = SVD_THREADS / 32;
  for (int e = tid; e < L2 * L2; e += SVD_THREADS) {
    const int r = e % L2, c = e / L2;
    R[e] = (r < l && c < l) ? jb.R[r + c * l] : s_zero(S());
    V[e] = (r == c) ? s_real<S>(1.0) : s_zero(S());
  }
  for (int e = tid; e < L2; e += SVD_THREADS) pos[e] = e;
  // ||R||_F^2: columns below 1e-100 ||R||_F count as converged (zero).  A rank-deficient R
  // (a collapsed spike) has more columns than its rank, and Jacobi keeps
  // shrinking the surplus ones pair against pair -- left alone they reach the denormal range,
  // where the phase cc / |cc| overflowed into NaN.
  double* fro = sg;  // scratch until the singular values are formed
  if (w == 0) {
    double t = 0.0;
    for (int e = lane; e < L2 * L2; e += 32) t += s_abs2(R[e]);
    t = warp_sum(t);
    if (lane == 0) fro[0] = t;
  }
  __syncthreads();
  const double tiny = 1e-200 * fro[0];
  __syncthreads();
  const int npairs = L2 / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) *rotated = 0;
    __syncthreads();
    for (int round = 0; round < L2 - 1; ++round) {
      for (int pr = w; pr < npairs; pr += nw) {
        int p = pos[pr], q = pos[L2 - 1 - pr];
        if (p > q) { const int t = p; p = q; q = t; }
        double a = 0, b = 0;
        S cc = s_zero(S());
        for (int r = lane; r < L2; r += 32) {
          const S x = R[r + p * L2], y = R[r + q * L2];
          a += s_abs2(x);
          b += s_abs2(y);
          cc = s_cfma(x, y, cc);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        cc = ds_warp_sum(cc);
        const double cabs = s_abs(cc);
        if (cabs > 1e-15 * sqrt(a * b) && cabs != 0.0 && a > tiny && b > tiny) {
          const double zeta = (b - a) / (2.0 * cabs);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          const S ph = s_unit_phase(s_conj(cc), cabs);  // q~ = ph q, p^H q~ = |c|
          for (int r = lane; r < L2; r += 32) {
            const S x = R[r + p * L2], y = s_mul(ph, R[r + q * L2]);
            R[r + p * L2] = s_sub(s_scale(x, cs), s_scale(y, sn));
            R[r + q * L2] = s_add(s_scale(x, sn), s_scale(y, cs));
            const S vx = V[r + p * L2], vy = s_mul(ph, V[r + q * L2]);
            V[r + p * L2] = s_sub(s_scale(vx, cs), s_scale(vy, sn));
            V[r + q * L2] = s_add(s_scale(vx, sn), s_scale(vy, cs));
          }
          if (lane == 0) *rotated = 1;
        }
      }
      __syncthreads();
      if (tid == 0) {  // rotate tournament positions (slot 0 fixed)
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
  for (int c = w; c < L2; c += nw) {
    double s = 0.0;
    for (int r = lane; r < L2; r += 32) s += s_abs2(R[r + c * L2]);
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
  // U = R / sigma in place; the null columns (sigma^2 <= tiny: a rank-deficient R, whose
  // surplus columns took no rotations) get an orthonormal completion instead, in output
  // order -- as LAPACK's singular vectors of a zero singular value -- so u and v stay
  // orthonormal and the interface matrices K = vW uT of build_truncated_precond stay
  // invertible (the spike operators u S v do not depend on the completion).
  for (int e = tid; e < L2 * l; e += SVD_THREADS) {
    const int r = e % L2, c = e / L2;
    if (sg[c] * sg[c] > tiny) R[r + c * L2] = s_scale(R[r + c * L2], 1.0 / sg[c]);
  }
  __syncthreads();
  for (int oc = 0; oc < l; ++oc) {
    const int src = order[oc];
    if (sg[src] * sg[src] > tiny) continue;
    if (w == 0) {  // e_j with the largest residual against the output columns before oc
      double best = -1.0;
      int bj = 0;
      for (int j = lane; j < l; j += 32) {
        double res = 1.0;
        for (int q = 0; q < oc; ++q) res -= s_abs2(R[j + order[q] * L2]);
        if (res > best) { best = res; bj = j; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oj = __shfl_down_sync(0xffffffffu, bj, o);
        if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
      }
      if (lane == 0) *rotated = bj;
    }
    __syncthreads();
    const int jbest = *rotated;
    S* x = R + src * L2;
    for (int r = tid; r < L2; r += SVD_THREADS) {  // e_j - U (U^H e_j)
      S v = (r == jbest) ? s_real<S>(1.0) : s_zero(S());
      for (int q = 0; q < oc; ++q)
        v = s_sub(v, s_mul(R[r + order[q] * L2], s_conj(R[jbest + order[q] * L2])));
      x[r] = r < l ? v : s_zero(S());
    }
    __syncthreads();
    for (int q = tid; q < oc; q += SVD_THREADS) {  // second Gram-Schmidt pass: coefficients
      S cq = s_zero(S());
      for (int r = 0; r < l; ++r) cq = s_cfma(R[r + order[q] * L2], x[r], cq);
      scr[q] = cq;
    }
    __syncthreads();
    double nrm = 0.0;
    for (int r = tid; r < l; r += SVD_THREADS) {
      S v = x[r];
      for (int q = 0; q < oc; ++q) v = s_sub(v, s_mul(R[r + order[q] * L2], scr[q]));
      x[r] = v;
      nrm += s_abs2(v);
    }
    nrm = block_sum(nrm, reinterpret_cast<double*>(scr));
    for (int r = tid; r < l; r += SVD_THREADS) x[r] = s_scale(x[r], 1.0 / sqrt(nrm));
    __syncthreads();
  }
  for (int e = tid; e < l * l; e += SVD_THREADS) {
    const int r = e % l, c = e / l;
    const int src = order[c];
    jb.V[r + c * l] = V[r + src * L2];
    jb.U[r + c * l] = R[r + src * L2];
  }
  for (int c = tid; c < l; c += SVD_THREADS) jb.sigma[c] = sg[order[c]];
}

template <class S>
void launch_jacobi_svd_t(Ctx* c, const SvdJobT<S>* d_jobs, int njobs, int l) {
  if (njobs == 0) return;
  if (l > SVD_MAXL) throw LrsError(LRS_ERR_PARAMETER, "n_svd + oversample > 96 not supported");
  const int L2 = (l + 1) & ~1;
  const size_t smem = ((sizeof(S) * 2 * L2 * L2 + sizeof(double) * L2 + sizeof(int) * (2 * L2 + 1) +
                       15) & ~size_t(15)) + sizeof(S) * L2 + sizeof(double) * 32;
  if (smem > 227 * 1024)  // complex: l <= 84
    throw LrsError(LRS_ERR_PARAMETER, "n_svd + oversample too large for the shared-memory SVD");
  static size_t attr = 0;
  if (smem > attr) {
    LRS_CUDA(cudaFuncSetAttribute(jacobi_svd_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = smem;
  }
  ProfScope ps_(c, K_SETUP);
  jacobi_svd_kernel<S><<<njobs, SVD_THREADS, smem, c->stream>>>(d_jobs, l);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// C (m x n) = A (m x k) * B (k x n); k x n <= 96 x 64 (B staged in shared memory)
// ---------------------------------------------------------------------------------------
template <class S>
__global__ void __launch_bounds__(256) small_gemm_kernel(const GemmJobT<S>* jobs) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  S* gsm = reinterpret_cast<S*>(gsm_raw);
  const GemmJobT<S> jb = jobs[blockIdx.y];
  for (int e = threadIdx.x; e < jb.k * jb.n; e += blockDim.x) {
    const int r = e % jb.k, c = e / jb.k;
    gsm[e] = jb.B[r + c * jb.ldb];
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= jb.m) return;
  for (int c = 0; c < jb.n; ++c) {
    S s = s_zero(S());
    for (int kk = 0; kk < jb.k; ++kk) s = s_fma(jb.A[i + kk * jb.lda], gsm[kk + c * jb.k], s);
    jb.C[i + c * jb.ldc] = jb.conjC ? s_conj(s) : s;
  }
}

template <class S>
void launch_small_gemm_t(Ctx* c, const GemmJobT<S>* d_jobs, int njobs, int64_t max_m, int max_n) {
  if (njobs == 0 || max_m == 0) return;
  (void)max_n;
  const size_t smem = sizeof(S) * 96 * 64;
  static bool attr = false;
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(small_gemm_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  ProfScope ps_(c, K_SETUP);
  dim3 grid((unsigned)((max_m + 255) / 256), (unsigned)njobs);
  small_gemm_kernel<S><<<grid, 256, smem, c->stream>>>(d_jobs);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// Interface setup: K = vW uTb, E = vT uWt, G = K^-1, H = G - S_T E S_W, Hinv = H^-1,
// cond_1 of K and H.  Degenerate interfaces (a spike with all sigma = 0)
// are the identity: Hinv = 0, cond = 1.
// ---------------------------------------------------------------------------------------
constexpr int IF_THREADS = 256;

// Gauss-Jordan inverse with partial pivoting (largest |a|) of an r x r matrix in shared
// memory.  M is r x 2r column-major [A | I]; returns 0 on an exact zero pivot.
template <class S>
__device__ int gj_inverse(S* M, int r, int* piv_row) {
  const int tid = threadIdx.x;
  const int ld = r;
  __shared__ int s_ok;
  if (tid == 0) s_ok = 1;
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    if (tid == 0) {
      int best = j;
      double bv = s_abs(M[j + j * ld]);
      for (int i = j + 1; i < r; ++i)
        if (s_abs(M[i + j * ld]) > bv) { bv = s_abs(M[i + j * ld]); best = i; }
      *piv_row = best;
      if (bv == 0.0) s_ok = 0;
    }
    __syncthreads();
    if (!s_ok) return 0;
    const int pr = *piv_row;
    if (pr != j)
      for (int c = tid; c < 2 * r; c += blockDim.x) {
        const S t = M[j + c * ld];
        M[j + c * ld] = M[pr + c * ld];
        M[pr + c * ld] = t;
      }
    __syncthreads();
    const S d = s_inv(M[j + j * ld]);
    __syncthreads();
    for (int c = tid; c < 2 * r; c += blockDim.x) M[j + c * ld] = s_mul(M[j + c * ld], d);
    __syncthreads();
    for (int e = tid; e < r * 2 * r; e += blockDim.x) {
      const int i = e % r, c = e / r;
      if (i != j && c != j) M[i + c * ld] = s_sub(M[i + c * ld], s_mul(M[i + j * ld], M[j + c * ld]));
    }
    __syncthreads();
    for (int i = tid; i < r; i += blockDim.x)
      if (i != j) M[i + j * ld] = s_zero(S());
    __syncthreads();
  }
  return 1;
}

template <class S>
__device__ double norm1(const S* A, int r, int ld, double* red) {
  // max column sum of |A|, columns handled by threads, reduced by thread 0
  const int tid = threadIdx.x;
  for (int c = tid; c < r; c += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < r; ++i) s += s_abs(A[i + c * ld]);
    red[c] = s;
  }
  __syncthreads();
  double mx = 0.0;
  for (int c = 0; c < r; ++c) mx = fmax(mx, red[c]);
  __syncthreads();
  return mx;
}

template <class S>
__global__ void __launch_bounds__(IF_THREADS) iface_setup_kernel(const IfaceSetupJobT<S>* jobs,
                                                                 int r, int64_t k) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  S* Ks = reinterpret_cast<S*>(fsm_raw);  // r x r
  S* Es = Ks + r * r;                      // r x r
  S* M = Es + r * r;                       // r x 2r
  double* red = reinterpret_cast<double*>(M + 2 * r * r);  // r
  __shared__ int piv;
  const IfaceSetupJobT<S> jb = jobs[blockIdx.x];
  const int tid = threadIdx.x;
  // K[a][c] = sum_row vtW[row, a] uTb[row, c];  E[a][c] = sum_row vtT[row, a] uWt[row, c]
  // The k rows stream through shared memory in tiles of KT rows (coalesced column reads;
  // the staging area is M, free until the inverses), IF_ACC entries per thread per pass;
  // each entry still sums its rows in ascending order.
  {
    constexpr int IF_ACC = 8;
    const int KT = r >= 2 ? min(16, r / 2) : 1;
    S* st = r >= 2 ? M : M + 2 * r * r;  // [4][KT][r]: vtW, uTb, vtT, uWt rows
    for (int e0 = 0; e0 < 2 * r * r; e0 += IF_THREADS * IF_ACC) {
      S acc[IF_ACC];
#pragma unroll
      for (int j = 0; j < IF_ACC; ++j) acc[j] = s_zero(S());
      for (int64_t r0 = 0; r0 < k; r0 += KT) {
        const int kt = (int)(k - r0 < KT ? k - r0 : KT);
        __syncthreads();
        for (int xx = tid; xx < 4 * KT * r; xx += IF_THREADS) {
          const int which = xx / (KT * r), rem = xx % (KT * r), col = rem / KT, rr = rem % KT;
          const S* src = which == 0   ? jb.vtW + (int64_t)col * k
                         : which == 1 ? jb.uTb + (int64_t)col * jb.ld_uT
                         : which == 2 ? jb.vtT + (int64_t)col * k
                                      : jb.uWt + (int64_t)col * jb.ld_uW;
          st[(which * KT + rr) * r + col] = rr < kt ? src[r0 + rr] : s_zero(S());
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < IF_ACC; ++j) {
          const int e = e0 + tid + j * IF_THREADS;
          if (e < 2 * r * r) {
            const int which = e / (r * r), ac = e % (r * r), a = ac % r, c = ac / r;
            const S* V = st + (which ? 2 : 0) * KT * r;
            const S* U = st + (which ? 3 : 1) * KT * r;
            for (int rr = 0; rr < kt; ++rr) acc[j] = s_fma(V[rr * r + a], U[rr * r + c], acc[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < IF_ACC; ++j) {
        const int e = e0 + tid + j * IF_THREADS;
        if (e < 2 * r * r) {
          const int which = e / (r * r), ac = e % (r * r), a = ac % r, c = ac / r;
          (which ? Es : Ks)[a + c * r] = acc[j];
        }
      }
    }
  }
  __syncthreads();
  bool anyT = false, anyW = false;
  for (int a = 0; a < r; ++a) {
    anyT |= jb.sT[a] != 0.0;
    anyW |= jb.sW[a] != 0.0;
  }
  const bool degenerate = !(anyT && anyW);
  for (int e = tid; e < r * r; e += IF_THREADS) {
    jb.K[e] = Ks[e];
    jb.E[e] = Es[e];
  }
  if (degenerate) {
    for (int e = tid; e < r * r; e += IF_THREADS) jb.Hinv[e] = s_zero(S());
    if (tid == 0) {
      jb.cond[0] = jb.cond[1] = 1.0;
      *jb.degenerate = 1;
    }
    return;
  }
  // G = K^-1
  for (int e = tid; e < 2 * r * r; e += IF_THREADS) {
    const int i = e % r, c = e / r;
    M[e] = (c < r) ? Ks[i + c * r] : (i == c - r ? s_real<S>(1.0) : s_zero(S()));
  }
  __syncthreads();
  const double nK = norm1(Ks, r, r, red);
  const int okK = gj_inverse(M, r, &piv);
  double condK = INFINITY;
  if (okK) condK = nK * norm1(M + r * r, r, r, red);
  // H = G - S_T E S_W   (stored in Ks; G is no longer needed afterwards)
  for (int e = tid; e < r * r; e += IF_THREADS) {
    const int a = e % r, c = e / r;
    Ks[e] = okK ? s_sub(M[r * r + e], s_scale(Es[e], jb.sT[a] * jb.sW[c])) : s_zero(S());
  }
  __syncthreads();
  for (int e = tid; e < 2 * r * r; e += IF_THREADS) {
    const int i = e % r, c = e / r;
    M[e] = (c < r) ? Ks[i + c * r] : (i == c - r ? s_real<S>(1.0) : s_zero(S()));
  }
  __syncthreads();
  const double nH = norm1(Ks, r, r, red);
  const int okH = okK ? gj_inverse(M, r, &piv) : 0;
  double condH = INFINITY;
  if (okH) condH = nH * norm1(M + r * r, r, r, red);
  for (int e = tid; e < r * r; e += IF_THREADS) jb.Hinv[e] = okH ? M[r * r + e] : s_zero(S());
  if (tid == 0) {
    jb.cond[0] = isfinite(condK) ? condK : INFINITY;
    jb.cond[1] = isfinite(condH) ? condH : INFINITY;
    *jb.degenerate = 0;
  }
}

template <class S>
void launch_iface_setup_t(Ctx* c, const IfaceSetupJobT<S>* d_jobs, int njobs, int r, int64_t k) {
  if (njobs == 0) return;
  const size_t smem = sizeof(S) * (4 * r * r + 4) + sizeof(double) * r;
  if (smem > 227 * 1024)  // real: r <= 85, complex: r <= 60
    throw LrsError(LRS_ERR_PARAMETER, "n_svd too large for the shared-memory interface setup");
  static size_t attr = 0;
  if (smem > attr) {
    LRS_CUDA(cudaFuncSetAttribute(iface_setup_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = smem;
  }
  ProfScope ps_(c, K_SETUP);
  iface_setup_kernel<S><<<njobs, IF_THREADS, smem, c->stream>>>(d_jobs, r, k);
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

template <class S>
__global__ void scale_cols_kernel(const ScaleColsJobT<S>* jobs, int64_t m, int ncols) {
  const ScaleColsJobT<S> jb = jobs[blockIdx.x];
  for (int64_t e = threadIdx.x; e < m * ncols; e += blockDim.x) {
    const int64_t i = e % m;
    const int j = (int)(e / m);
    jb.X[i + j * jb.ld] = s_scale(jb.X[i + j * jb.ld], jb.s[j]);
  }
}

template <class S>
void launch_scale_cols_t(Ctx* c, const ScaleColsJobT<S>* d_jobs, int njobs, int64_t m, int ncols) {
  if (njobs == 0) return;
  ProfScope ps_(c, K_SETUP);
  scale_cols_kernel<S><<<njobs, 256, 0, c->stream>>>(d_jobs, m, ncols);
  LRS_LAUNCHED(c);
}

#define LRS_INST(S)                                                                          \
  template void launch_scale_cols_t<S>(Ctx*, const ScaleColsJobT<S>*, int, int64_t, int);    \
  template void launch_householder_qr_t<S>(Ctx*, const QrJobT<S>*, int, int, int64_t);       \
  template void launch_jacobi_svd_t<S>(Ctx*, const SvdJobT<S>*, int, int);                   \
  template void launch_small_gemm_t<S>(Ctx*, const GemmJobT<S>*, int, int64_t, int);         \
  template void launch_iface_setup_t<S>(Ctx*, const IfaceSetupJobT<S>*, int, int, int64_t);
LRS_INST(double)
LRS_INST(zc)
#undef LRS_INST

}  // namespace lrs
