// Band LU with partial pivoting (LAPACK dgbtrf / zgbtrf semantics) and the
// matching solves (dgbtrs / zgbtrs), for blocks the no-interchange path of band_lu.cu (or
// band_lu_z.cu) rejects.  Every kernel is templated on the scalar (double, or zc for
// complex128: pivot magnitude |Re| + |Im| as izamax, adjoint solves conjugate).
//
// Storage: the same tiles as band_lu.cu with the upper band widened to ku + kl (the fill
// of the row interchanges): wu' = ceil((ku + kl) / 128) tile columns.  Step K:
//   lu_panel_piv : the tall panel (rows K*128 .. (K+1+wl)*128 of column tile K) factored
//                  column by column with partial pivoting by a 16-CTA cluster (rows split
//                  over the CTAs; pivot search = block argmax + fixed-rank-order reduction
//                  over distributed shared memory, first maximum wins as in idamax).  The
//                  interchanges are applied across the panel's 128 columns (so the panel
//                  holds P_K-permuted L, like dgetrf on the panel) and recorded in ipiv;
//                  the composed row permutation of the step is stored for the solves.
//   diag_invert  : inv(L_KK) strictly below, inv(U_KK) on/above the diagonal (as always)
//   swap_trail   : the step's interchanges on the trailing tile columns K+1 .. K+wu'
//   then the DMMA kernels of band_lu.cu (band_lu_z.cu): U_KJ = inv(L_KK) A_KJ and the
//   trailing update.
// Solves: L (forward) and L^T (backward) step by step with the interleaved permutations
// (dgbtrs); U and U^T with the dataflow kernels of band_solve.cu over the wider band.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"
#include "lu_common.cuh"

namespace lrs {

namespace cg = cooperative_groups;

constexpr int PIV_CL = 16;       // CTAs per partition (non-portable cluster size)
constexpr int PIV_THREADS = 512;
constexpr int PIV_MAXPERM = 2 * NB;  // rows moved by one step's 128 interchanges
constexpr int PIV_MAXROWS = 1664;    // panel rows per CTA: (wl + 1) * 128 / 16, wl <= 207

__device__ __forceinline__ bool piv_better(double v, int i, double bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

template <class S>
__global__ void __cluster_dims__(PIV_CL, 1, 1) __launch_bounds__(PIV_THREADS, 1)
    lu_panel_piv_kernel(BandGeom g, S* tiles, int K, int* ipiv, int* perm, int* status) {
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int p = blockIdx.x / PIV_CL;
  const int T = g.T[p];
  if (K >= T) return;  // the whole cluster returns together
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NW = PIV_THREADS / 32;
  __shared__ double wv[NW];
  __shared__ int wi[NW];
  __shared__ double slot_v[2];
  __shared__ int slot_i[2];
  __shared__ S urow[NB];
  __shared__ S lcol[PIV_MAXROWS];
  __shared__ int s_piv;
  __shared__ double s_pv;
  const int64_t base = g.tbase[p];
  const int r0 = K * NB;
  const int Ilast = min(T - 1, K + g.wl);
  const int rend = (Ilast + 1) * NB;
  const int H = rend - r0;
  const int per = (H + PIV_CL - 1) / PIV_CL;
  const int slo = r0 + crank * per, shi = min(rend, slo + per);
  auto el = [&](int r, int c) -> S* {
    const int I = r >> 7;
    return tiles + (base + (int64_t)I * g.W + (K - I + g.wl)) * TILE_ELEMS + (r & (NB - 1)) +
           (int64_t)c * NB;
  };
  int* piv = ipiv + g.fbase[p] * NB;
  int par = 0;
  for (int c = 0; c < NB; ++c) {
    const int j = r0 + c;
    // ---- pivot search: first max |a_rj|, r >= j ----------------------------------------
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int r = max(j, slo) + tid; r < shi; r += PIV_THREADS) {
      const double v = s_abs1(*el(r, c));
      if (piv_better(v, r, bv, bi)) bv = v, bi = r;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (piv_better(ov, oi, bv, bi)) bv = ov, bi = oi;
    }
    if (lane == 0) wv[w] = bv, wi[w] = bi;
    __syncthreads();
    if (tid == 0) {
      double v = -1.0;
      int ii = 0x7fffffff;
      for (int q = 0; q < NW; ++q)
        if (piv_better(wv[q], wi[q], v, ii)) v = wv[q], ii = wi[q];
      slot_v[par] = v;
      slot_i[par] = ii;
    }
    cluster.sync();
    if (tid == 0) {
      double v = -1.0;
      int ii = 0x7fffffff;
      for (int rk = 0; rk < PIV_CL; ++rk) {
        const double ov = *cluster.map_shared_rank(&slot_v[par], rk);
        const int oi = *cluster.map_shared_rank(&slot_i[par], rk);
        if (piv_better(ov, oi, v, ii)) v = ov, ii = oi;
      }
      s_piv = ii;
      s_pv = v;
    }
    __syncthreads();
    const int prow = s_piv;
    if (crank == 0) {
      if (tid == 0) {
        piv[j] = prow;
        if (s_pv == 0.0) atomicMin(&status[2 * p + 1], j);
      }
      if (prow != j && tid < NB) {  // interchange across the panel's columns
        S* a = el(j, tid);
        S* b = el(prow, tid);
        const S t = *a;
        *a = *b;
        *b = t;
      }
    }
    cluster.sync();
    par ^= 1;
    // ---- scale the column and rank-1 update of this CTA's rows ------------------------
    if (tid < NB) urow[tid] = tid > c ? *el(j, tid) : s_zero(S{});
    __syncthreads();
    const S pv = *el(j, c);
    const int ra = max(j + 1, slo), nr = max(0, shi - ra);
    if (!s_iszero(pv) && nr > 0) {  // ?gbtf2 skips scaling / update on an exact zero pivot
      const S inv = s_inv(pv);        // ?scal by 1 / pivot
      for (int e = tid; e < nr; e += PIV_THREADS) {
        S* lr = el(ra + e, c);
        const S l = s_mul(*lr, inv);
        *lr = l;
        lcol[e] = l;
      }
      __syncthreads();
      // (row, column) pairs over all threads: consecutive threads take consecutive rows
      const int ncols = NB - 1 - c, tot = nr * ncols;
      for (int e = tid; e < tot; e += PIV_THREADS) {
        const int rr = e % nr, c2 = c + 1 + e / nr;
        const S l = lcol[rr];
        if (!s_iszero(l)) {
          S* a = el(ra + rr, c2);
          *a = s_fma(s_neg(l), urow[c2], *a);
        }
      }
    }
    __syncthreads();
  }
  // ---- the step's composed permutation: new x[dst] = old x[src] (rank 0) ---------------
  if (crank == 0) {
    extern __shared__ int idx[];  // H entries
    for (int e = tid; e < H; e += PIV_THREADS) idx[e] = r0 + e;
    __syncthreads();
    if (tid == 0) {
      for (int c = 0; c < NB; ++c) {
        const int a = c, b = piv[r0 + c] - r0;
        const int t = idx[a];
        idx[a] = idx[b];
        idx[b] = t;
      }
      int* pl = perm + ((int64_t)g.fbase[p] + K) * (2 * PIV_MAXPERM + 1);
      int cnt = 0;
      for (int e = 0; e < H; ++e)
        if (idx[e] != r0 + e) {
          pl[1 + 2 * cnt] = r0 + e;     // dst
          pl[2 + 2 * cnt] = idx[e];     // src
          ++cnt;
        }
      pl[0] = cnt;
    }
  }
  cluster.sync();
}

// inv(L_KK) / inv(U_KK) of the factored diagonal tile, in place
__global__ void __launch_bounds__(512, 1) diag_invert_kernel(BandGeom g, double* tiles, int K) {
  extern __shared__ double sm[];
  double* A = sm;
  double* part = sm + TILE_ELEMS;
  const int p = blockIdx.x;
  if (K >= g.T[p]) return;
  double* gt = tiles + (g.tbase[p] + (int64_t)K * g.W + g.wl) * TILE_ELEMS;
  for (int e = threadIdx.x; e < TILE_ELEMS; e += 512) A[e] = gt[e];
  __syncthreads();
  diag_inverses(A, part, threadIdx.x);
  for (int e = threadIdx.x; e < TILE_ELEMS; e += 512) gt[e] = A[e];
}
// complex: the same inverses (ztrti2 'U' / 'L' 'U') on the tile in global memory
__global__ void __launch_bounds__(512, 1) diag_invert_z_kernel(BandGeom g, zc* tiles, int K) {
  __shared__ zc part[4 * NB];
  const int p = blockIdx.x;
  if (K >= g.T[p]) return;
  diag_inverses_z(tiles + (g.tbase[p] + (int64_t)K * g.W + g.wl) * TILE_ELEMS, part, threadIdx.x);
}

// the step's interchanges on tile columns K+1 .. K+wu, applied as the composed
// permutation (new row dst = old row src): gather all moved rows, then scatter.
template <class S>
__global__ void __launch_bounds__(NB) swap_trailing_kernel(BandGeom g, S* tiles, int K,
                                                           const int* perm) {
  constexpr int CW = sizeof(S) == 8 ? 16 : 8;  // columns moved per round (static smem)
  const int p = blockIdx.y;
  const int T = g.T[p];
  const int J = K + 1 + blockIdx.x;
  if (K >= T || J >= T) return;
  __shared__ S vals[PIV_MAXPERM][CW + 1];
  __shared__ int dst[PIV_MAXPERM], src[PIV_MAXPERM];
  const int tid = threadIdx.x;
  const int64_t base = g.tbase[p];
  const int* pl = perm + ((int64_t)g.fbase[p] + K) * (2 * PIV_MAXPERM + 1);
  const int cnt = pl[0];
  for (int e = tid; e < cnt; e += NB) dst[e] = pl[1 + 2 * e], src[e] = pl[2 + 2 * e];
  __syncthreads();
  auto el = [&](int r, int col) -> S* {
    const int I = r >> 7;
    return tiles + (base + (int64_t)I * g.W + (J - I + g.wl)) * TILE_ELEMS + (r & (NB - 1)) +
           (int64_t)col * NB;
  };
  for (int c0 = 0; c0 < NB; c0 += CW) {  // CW columns at a time
    for (int e = tid; e < cnt * CW; e += NB) vals[e / CW][e % CW] = *el(src[e / CW], c0 + e % CW);
    __syncthreads();
    for (int e = tid; e < cnt * CW; e += NB) *el(dst[e / CW], c0 + e % CW) = vals[e / CW][e % CW];
    __syncthreads();
  }
}

template <class S>
void lu_panel_piv_t(Ctx* c, cudaStream_t s, const BandGeom& g, S* tiles, int K, int* ipiv,
                    int* perm, int* status) {
  constexpr bool CPLX = IsC<S>::value;
  const size_t smem = sizeof(int) * (size_t)(g.wl + 1) * NB;
  static bool attrs = false;
  if (!attrs) {
    LRS_CUDA(cudaFuncSetAttribute(lu_panel_piv_kernel<S>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    LRS_CUDA(cudaFuncSetAttribute(lu_panel_piv_kernel<S>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(int) * 200 * NB)));
    if (!CPLX)
      LRS_CUDA(cudaFuncSetAttribute(diag_invert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(sizeof(double) * (TILE_ELEMS + 4 * NB))));
    attrs = true;
  }
  if ((g.wl + 1) * NB > PIV_CL * PIV_MAXROWS || g.wl + 1 > 200)
    throw LrsError(LRS_ERR_PARAMETER, "pivoting LU: lower band > 199 tiles");
  {
    ProfScope ps_(c, K_LU_DIAG, s);
    lu_panel_piv_kernel<S><<<g.P * PIV_CL, PIV_THREADS, smem, s>>>(g, tiles, K, ipiv, perm,
                                                                   status);
    LRS_LAUNCHED(c);
  }
  {
    ProfScope ps_(c, K_LU_DIAG, s);
    if constexpr (CPLX)
      diag_invert_z_kernel<<<g.P, 512, 0, s>>>(g, tiles, K);
    else
      diag_invert_kernel<<<g.P, 512, sizeof(double) * (TILE_ELEMS + 4 * NB), s>>>(g, tiles, K);
    LRS_LAUNCHED(c);
  }
  if (g.wu > 0) {
    ProfScope ps_(c, K_LU_PANEL, s);
    swap_trailing_kernel<S><<<dim3(g.wu, g.P), NB, 0, s>>>(g, tiles, K, perm);
    LRS_LAUNCHED(c);
  }
}

void launch_lu_panel_piv(Ctx* c, cudaStream_t s, const BandGeom& g, double* tiles, int K, int* ipiv,
                         int* perm, int* status) {
  lu_panel_piv_t(c, s, g, tiles, K, ipiv, perm, status);
}
void launch_lu_panel_piv_z(Ctx* c, cudaStream_t s, const BandGeom& g, zc* tiles, int K, int* ipiv,
                           int* perm, int* status) {
  lu_panel_piv_t(c, s, g, tiles, K, ipiv, perm, status);
}

size_t piv_perm_ints(int64_t total_rowtiles) { return (size_t)total_rowtiles * (2 * PIV_MAXPERM + 1); }

// ---------------------------------------------------------------------------------------
// Solves with the interleaved interchanges (dgbtrs), step by step.
// Forward L, step K:  x <- P_K x (rows of the panel);  x_K <- inv(L_KK) x_K  (piv_fwd_a),
//                     x_I -= L_IK x_K, I = K+1 .. K+wl                      (piv_fwd_b)
// Backward L^T (L^H for complex), step K: x_K -= sum_I L_IK^H x_I; x_K <- inv(L_KK)^H x_K;
//                     x <- P_K^T x
// x: global-row layout (partition offset off_p), nrhs columns with leading dimension ld.
// ---------------------------------------------------------------------------------------
constexpr int PIV_COLS = 4;  // right-hand-side columns per CTA of the solve kernels

template <class S>
__global__ void __launch_bounds__(NB) piv_fwd_a_kernel(BandGeom g, const S* tiles, int K,
                                                      const int* perm, S* x, int64_t ld,
                                                      int nrhs, int p_only) {
  x += (int64_t)blockIdx.z * PIV_COLS * ld;
  nrhs = min(PIV_COLS, nrhs - (int)blockIdx.z * PIV_COLS);
  const int p = p_only >= 0 ? p_only : blockIdx.x;
  if (K >= g.T[p]) return;
  __shared__ S xs[NB];
  __shared__ int pl_dst[PIV_MAXPERM], pl_src[PIV_MAXPERM];
  __shared__ S pv[PIV_MAXPERM];
  const int tid = threadIdx.x;
  const int64_t off = g.off[p], size = g.size[p];
  const int* pl = perm + ((int64_t)g.fbase[p] + K) * (2 * PIV_MAXPERM + 1);
  const int cnt = pl[0];
  for (int e = tid; e < cnt; e += NB) pl_dst[e] = pl[1 + 2 * e], pl_src[e] = pl[2 + 2 * e];
  const S* Lt = tiles + (g.tbase[p] + (int64_t)K * g.W + g.wl) * TILE_ELEMS;
  const int64_t row = (int64_t)K * NB + tid;
  __syncthreads();
  for (int j = 0; j < nrhs; ++j) {
    S* xj = x + off + (int64_t)j * ld;
    for (int e = tid; e < cnt; e += NB) pv[e] = pl_src[e] < size ? xj[pl_src[e]] : s_zero(S{});
    __syncthreads();
    for (int e = tid; e < cnt; e += NB)
      if (pl_dst[e] < size) xj[pl_dst[e]] = pv[e];
    __syncthreads();
    xs[tid] = row < size ? xj[row] : s_zero(S{});
    __syncthreads();
    S v = xs[tid];  // unit diagonal
    for (int k = 0; k < tid; ++k) v = s_fma(Lt[tid + k * NB], xs[k], v);
    if (row < size) xj[row] = v;
    __syncthreads();
  }
}

template <class S>
__global__ void __launch_bounds__(NB) piv_fwd_b_kernel(BandGeom g, const S* tiles, int K,
                                                      S* x, int64_t ld, int nrhs, int p_only) {
  x += (int64_t)blockIdx.z * PIV_COLS * ld;
  nrhs = min(PIV_COLS, nrhs - (int)blockIdx.z * PIV_COLS);
  const int p = p_only >= 0 ? p_only : blockIdx.y;
  const int T = g.T[p];
  const int I = K + 1 + blockIdx.x;
  if (K >= T || I >= T) return;
  __shared__ S xs[NB];
  const int tid = threadIdx.x;
  const int64_t off = g.off[p], size = g.size[p];
  const S* L = tiles + (g.tbase[p] + (int64_t)I * g.W + (K - I + g.wl)) * TILE_ELEMS;
  const int64_t row = (int64_t)I * NB + tid, rk = (int64_t)K * NB + tid;
  for (int j = 0; j < nrhs; ++j) {
    S* xj = x + off + (int64_t)j * ld;
    xs[tid] = rk < size ? xj[rk] : s_zero(S{});
    __syncthreads();
    S acc = s_zero(S{});
    for (int k = 0; k < NB; ++k) acc = s_fma(L[tid + k * NB], xs[k], acc);
    if (row < size) xj[row] = s_sub(xj[row], acc);
    __syncthreads();
  }
}

template <class S>
__global__ void __launch_bounds__(NB) piv_bwd_kernel(BandGeom g, const S* tiles, int K,
                                                    const int* perm, S* x, int64_t ld,
                                                    int nrhs, int p_only) {
  x += (int64_t)blockIdx.z * PIV_COLS * ld;
  nrhs = min(PIV_COLS, nrhs - (int)blockIdx.z * PIV_COLS);
  const int p = p_only >= 0 ? p_only : blockIdx.x;
  const int T = g.T[p];
  if (K >= T) return;
  __shared__ S xs[NB];
  __shared__ int pl_dst[PIV_MAXPERM], pl_src[PIV_MAXPERM];
  __shared__ S pv[PIV_MAXPERM];
  const int tid = threadIdx.x;
  const int64_t off = g.off[p], size = g.size[p];
  const int Ilast = min(T - 1, K + g.wl);
  const int* pl = perm + ((int64_t)g.fbase[p] + K) * (2 * PIV_MAXPERM + 1);
  const int cnt = pl[0];
  for (int e = tid; e < cnt; e += NB) pl_dst[e] = pl[1 + 2 * e], pl_src[e] = pl[2 + 2 * e];
  const int64_t base = g.tbase[p];
  const S* Lt = tiles + (base + (int64_t)K * g.W + g.wl) * TILE_ELEMS;
  const int64_t rk = (int64_t)K * NB + tid;
  __syncthreads();
  for (int j = 0; j < nrhs; ++j) {
    S* xj = x + off + (int64_t)j * ld;
    // x_K[m] -= sum_I sum_r conj(L_IK[r][m]) x_I[r]
    S v = rk < size ? xj[rk] : s_zero(S{});
    for (int I = K + 1; I <= Ilast; ++I) {
      const S* L = tiles + (base + (int64_t)I * g.W + (K - I + g.wl)) * TILE_ELEMS;
      const int64_t r0 = (int64_t)I * NB;
      S acc = s_zero(S{});
      for (int r = 0; r < NB; ++r) {
        const S xr = r0 + r < size ? xj[r0 + r] : s_zero(S{});
        acc = s_cfma(L[r + tid * NB], xr, acc);
      }
      v = s_sub(v, acc);
    }
    xs[tid] = v;
    __syncthreads();
    // x_K <- inv(L_KK)^H x_K: v_m = x_m + sum_{i > m} conj(invL[i][m]) x_i
    S u = xs[tid];
    for (int i = tid + 1; i < NB; ++i) u = s_cfma(Lt[i + tid * NB], xs[i], u);
    if (rk < size) xj[rk] = u;
    __syncthreads();
    // x <- P_K^T x: new x[src] = old x[dst]
    for (int e = tid; e < cnt; e += NB) pv[e] = pl_dst[e] < size ? xj[pl_dst[e]] : s_zero(S{});
    __syncthreads();
    for (int e = tid; e < cnt; e += NB)
      if (pl_src[e] < size) xj[pl_src[e]] = pv[e];
    __syncthreads();
  }
}

template <class S>
void piv_lsolve_t(Ctx* c, const BandGeom& g, const S* tiles, const int* perm, int Tmax,
                  bool transposed, S* x, int64_t ld, int nrhs, int p_only) {
  if (nrhs == 0) return;
  const int np = p_only >= 0 ? 1 : g.P;
  const unsigned nz = (unsigned)((nrhs + PIV_COLS - 1) / PIV_COLS);
  ProfScope ps_(c, c->in_setup ? K_SPIKE_SOLVE : (transposed ? K_SOLVE_ADJ : K_SOLVE));
  if (!transposed) {
    for (int K = 0; K < Tmax; ++K) {
      piv_fwd_a_kernel<S><<<dim3(np, 1, nz), NB, 0, c->stream>>>(g, tiles, K, perm, x, ld, nrhs,
                                                                 p_only);
      LRS_LAUNCHED(c);
      if (g.wl > 0) {
        piv_fwd_b_kernel<S><<<dim3(g.wl, np, nz), NB, 0, c->stream>>>(g, tiles, K, x, ld, nrhs,
                                                                      p_only);
        LRS_LAUNCHED(c);
      }
    }
  } else {
    for (int K = Tmax - 1; K >= 0; --K) {
      piv_bwd_kernel<S><<<dim3(np, 1, nz), NB, 0, c->stream>>>(g, tiles, K, perm, x, ld, nrhs,
                                                               p_only);
      LRS_LAUNCHED(c);
    }
  }
}

void launch_piv_lsolve(Ctx* c, const BandGeom& g, const double* tiles, const int* perm, int Tmax,
                       bool transposed, double* x, int64_t ld, int nrhs, int p_only) {
  piv_lsolve_t(c, g, tiles, perm, Tmax, transposed, x, ld, nrhs, p_only);
}
void launch_piv_lsolve_z(Ctx* c, const BandGeom& g, const zc* tiles, const int* perm, int Tmax,
                         bool transposed, zc* x, int64_t ld, int nrhs, int p_only) {
  piv_lsolve_t(c, g, tiles, perm, Tmax, transposed, x, ld, nrhs, p_only);
}

}  // namespace lrs
