// Complex128 tiled band LU (config 5: the FEAST shifted systems z I - A).
//
// Same storage and algorithm as band_lu.cu with complex tiles (128 x 128 complex =
// 256 KB): the diagonal tile is factored in place in global memory (it no longer fits
// the 227 KB of shared memory; it is L2-resident and off the critical path thanks to
// the look-ahead), and the tile GEMMs run on the FP64 tensor cores as four real
// DMMA.8x8x4 products per complex product, each CTA computing half a tile (128 x 64)
// so the complex accumulators fit the same 64-register budget as the real kernel.
// The pivot rule is LAPACK zgbtrf's: izamax, i.e. first max |Re| + |Im|.
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"
#include "lu_common.cuh"

namespace lrs {

__device__ __forceinline__ int find_partition_z(const int64_t* off, int P, int64_t row) {
  int lo = 0, hi = P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) extract_tiles_z_kernel(
    int64_t n, const int* __restrict__ rp, const int* __restrict__ ci, const zc* __restrict__ va,
    BandGeom g, zc* tiles, int64_t k, int64_t row_lo, int64_t row_hi, unsigned long long* bad) {
  const int64_t row = row_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= row_hi) return;
  const int p = find_partition_z(g.off, g.P, row);
  const int pg = g.p0 + p;
  const int64_t o = g.off[p], s = g.size[p];
  const int64_t li = row - o;
  const int I = (int)(li / NB);
  for (int q = rp[row]; q < rp[row + 1]; ++q) {
    const int64_t col = ci[q];
    bool ok;
    if (col >= o && col < o + s) {
      const int64_t lj = col - o;
      const int d = (int)(lj / NB) - I;
      ok = d >= -g.wl && d <= g.wu;
      if (ok)
        tiles[(g.tbase[p] + (int64_t)I * g.W + (d + g.wl)) * TILE_ELEMS + (lj % NB) * NB +
              (li % NB)] = va[q];
    } else if (pg + 1 < g.Pg && col >= o + s && col < g.goff[pg + 2]) {
      ok = row >= o + s - k && col < o + s + k;
    } else if (pg > 0 && col < o && col >= g.goff[pg - 1]) {
      ok = row < o + k && col >= o - k;
    } else {
      ok = false;
    }
    if (!ok) atomicMin(bad, (unsigned long long)(row * n + col));
  }
}

__global__ void pad_diag_z_kernel(BandGeom g, zc* tiles) {
  const int p = blockIdx.x;
  const int64_t s = g.size[p];
  for (int64_t li = s + threadIdx.x; li < (int64_t)g.T[p] * NB; li += blockDim.x) {
    const int I = (int)(li / NB);
    tiles[(g.tbase[p] + (int64_t)I * g.W + g.wl) * TILE_ELEMS + (li % NB) * NB + (li % NB)] =
        zc{1.0, 0.0};
  }
}

void launch_extract_tiles_z(Ctx* c, const Mat* m, const BandGeom& g, zc* tiles, int64_t k,
                            int64_t row_lo, int64_t row_hi, unsigned long long* d_bad) {
  ProfScope ps_(c, K_SETUP);
  if (row_hi > row_lo) {
    extract_tiles_z_kernel<<<(unsigned)((row_hi - row_lo + 255) / 256), 256, 0, c->stream>>>(
        m->n, m->row_ptr.get(), m->col_idx.get(), reinterpret_cast<const zc*>(m->vals.get()), g,
        tiles, k, row_lo, row_hi, d_bad);
    LRS_LAUNCHED(c);
  }
  pad_diag_z_kernel<<<g.P, 128, 0, c->stream>>>(g, tiles);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// diagonal tile: unblocked LU with the izamax rule + in-place triangular inverses, in
// global memory (one CTA of 512 threads per partition)
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1) lu_diag_z_kernel(BandGeom g, zc* tiles, int K,
                                                           int* status) {
  __shared__ zc part[4 * NB];
  const int p = blockIdx.x;
  if (K >= g.T[p]) return;
  const int tid = threadIdx.x;
  zc* A = tiles + (g.tbase[p] + (int64_t)K * g.W + g.wl) * TILE_ELEMS;
  const int col0 = K * NB;
  const int i = tid & (NB - 1), cg = tid >> 7;
  for (int j = 0; j < NB; ++j) {
    const zc piv = A[j * NB + j];
    if (cg == 0 && i > j) {
      const zc a = A[j * NB + i];
      if (s_abs1(a) > s_abs1(piv)) atomicMin(&status[2 * p], col0 + j);  // zgbtrf would swap
      A[j * NB + i] = s_div(a, piv);
    }
    if (tid == 0 && s_iszero(piv)) atomicMin(&status[2 * p + 1], col0 + j);
    __syncthreads();
    if (i > j) {
      const zc nl = s_neg(A[j * NB + i]);
      for (int c = j + 1 + cg; c < NB; c += 4) A[c * NB + i] = s_fma(nl, A[c * NB + j], A[c * NB + i]);
    }
    __syncthreads();
  }
  diag_inverses_z(A, part, tid);
}

// ---------------------------------------------------------------------------------------
// complex tile GEMM on DMMA: C(128 x 64 half tile) = / -= A(128 x 128) B(128 x 64)
// ---------------------------------------------------------------------------------------
constexpr int ZG_THREADS = 256;
#ifndef LRS_ZGEMM_3M
#define LRS_ZGEMM_3M 1
#endif
constexpr int ZKC = 16;
constexpr int ZAS_LD = NB + 2;   // 130 complex: conflict-free 16-byte fragment loads
constexpr int ZBS_LD = ZKC + 4;  // 20
constexpr int ZAS_STAGE = ZKC * ZAS_LD;
constexpr int ZBS_STAGE = 64 * ZBS_LD;
constexpr size_t ZGEMM_SMEM = sizeof(zc) * 2 * (ZAS_STAGE + ZBS_STAGE);
constexpr int ZMASK_NONE = 0, ZMASK_UNIT_LOWER = 1, ZMASK_UPPER = 2;

__device__ __forceinline__ void zgemm_load_chunk(const zc* __restrict__ A, const zc* __restrict__ B,
                                                 zc* As, zc* Bs, int kc, int nbase, int tid) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {  // A: 16 k x 128 m
    const int idx = tid + ZG_THREADS * q;
    const int k = idx >> 7, m = idx & 127;
    cp_async16(As + k * ZAS_LD + m, A + (int64_t)(kc * ZKC + k) * NB + m);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // B: 64 n x 16 k
    const int idx = tid + ZG_THREADS * q;
    const int nn = idx >> 4, kk = idx & 15;
    cp_async16(Bs + nn * ZBS_LD + kk, B + (int64_t)(nbase + nn) * NB + kc * ZKC + kk);
  }
  cp_async_commit();
}

template <int MODE, int maskA, int maskB>
__device__ __forceinline__ void ztile_gemm(const zc* A, const zc* B, zc* C, int nbase, zc* sm,
                                           int* piv_status, int col0, const zc* diag) {
  zc* As = sm;
  zc* Bs = sm + 2 * ZAS_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = w >> 1;  // 2 x 4 warps: 64 rows x 16 columns each
  const int g = lane >> 2, t = lane & 3;
  constexpr int NK = NB / ZKC;
  double ar[2][8][2], ai[2][8][2];  // [n tile][m tile][pair] real / imaginary parts
  // 3M form (LRS_ZGEMM_3M): q1 = sum br ar, q2 = sum bi ai, q3 = sum (br + bi)(ar + ai);
  // C = (ar + q1 - q2, ai + q3 - q1 - q2): three DMMAs per complex product instead of four
  double q1[LRS_ZGEMM_3M ? 2 : 1][8][2], q2[LRS_ZGEMM_3M ? 2 : 1][8][2],
      q3[LRS_ZGEMM_3M ? 2 : 1][8][2];
  if (LRS_ZGEMM_3M) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 2; ++e) q1[j][i][e] = q2[j][i][e] = q3[j][i][e] = 0.0;
  }
  zgemm_load_chunk(A, B, As, Bs, 0, nbase, tid);
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (MODE == 1 && !LRS_ZGEMM_3M) {  // (3M: C is added in the epilogue)
          const zc v = C[(int64_t)(nbase + 16 * wn + 8 * j + g) * NB + 64 * wm + 8 * i + 2 * t + e];
          ar[j][i][e] = v.x;
          ai[j][i][e] = v.y;
        } else {
          ar[j][i][e] = ai[j][i][e] = 0.0;
        }
      }
#pragma unroll 1
  for (int kc = 0; kc < NK; ++kc) {
    const int st = kc & 1;
    if (kc + 1 < NK) {
      zgemm_load_chunk(A, B, As + (st ^ 1) * ZAS_STAGE, Bs + (st ^ 1) * ZBS_STAGE, kc + 1, nbase, tid);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const zc* as = As + st * ZAS_STAGE;
    const zc* bs = Bs + st * ZBS_STAGE;
#pragma unroll
    for (int k4 = 0; k4 < ZKC / 4; ++k4) {
      const int kk = k4 * 4 + t;
      const int kg = kc * ZKC + kk;
      double far_[8], fai[8], fbr[2], fbi[2];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = 64 * wm + 8 * i + g;
        zc v = as[kk * ZAS_LD + m];
        if (maskA == ZMASK_UNIT_LOWER) v = m > kg ? v : (m == kg ? zc{1.0, 0.0} : zc{0.0, 0.0});
        far_[i] = MODE == 1 ? -v.x : v.x;
        fai[i] = MODE == 1 ? -v.y : v.y;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int nn = 16 * wn + 8 * j + g;
        zc v = bs[nn * ZBS_LD + kk];
        if (maskB == ZMASK_UPPER) v = kg <= nbase + nn ? v : zc{0.0, 0.0};
        fbr[j] = v.x;
        fbi[j] = v.y;
      }
      if (LRS_ZGEMM_3M) {
        double fas[8], fbs[2];
#pragma unroll
        for (int i = 0; i < 8; ++i) fas[i] = far_[i] + fai[i];
#pragma unroll
        for (int j = 0; j < 2; ++j) fbs[j] = fbr[j] + fbi[j];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            dmma_8x8x4(q1[j & (LRS_ZGEMM_3M ? 1 : 0)][i][0], q1[j & (LRS_ZGEMM_3M ? 1 : 0)][i][1],
                       fbr[j], far_[i]);
            dmma_8x8x4(q2[j & (LRS_ZGEMM_3M ? 1 : 0)][i][0], q2[j & (LRS_ZGEMM_3M ? 1 : 0)][i][1],
                       fbi[j], fai[i]);
            dmma_8x8x4(q3[j & (LRS_ZGEMM_3M ? 1 : 0)][i][0], q3[j & (LRS_ZGEMM_3M ? 1 : 0)][i][1],
                       fbs[j], fas[i]);
          }
      } else {
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            // C^T = B^T A^T, complex: re += br ar - bi ai ; im += br ai + bi ar
            dmma_8x8x4(ar[j][i][0], ar[j][i][1], fbr[j], far_[i]);
            dmma_8x8x4(ar[j][i][0], ar[j][i][1], -fbi[j], fai[i]);
            dmma_8x8x4(ai[j][i][0], ai[j][i][1], fbr[j], fai[i]);
            dmma_8x8x4(ai[j][i][0], ai[j][i][1], fbi[j], far_[i]);
          }
      }
    }
    __syncthreads();
  }
  if (MODE == 0 && maskB == ZMASK_UPPER) {
    // in-place L_IK = A_IK inv(U_KK): both half-tile CTAs (a cluster of 2) read all of A_IK
    // before either writes its half
    // a launch without the 2-CTA cluster attribute would make the barrier a no-op and
    // bring the write-after-read race back silently: refuse to run instead
    uint32_t ncta;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
    if (ncta != 2) __trap();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                     "memory");
  }
  int bad_col = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int nn = nbase + 16 * wn + 8 * j + g;
    zc u = {1.0, 0.0};
    if (MODE == 0 && piv_status) u = s_inv(diag[(int64_t)nn * NB + nn]);  // u_nn of this column
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        zc v = {ar[j][i][e], ai[j][i][e]};
        if (LRS_ZGEMM_3M) {
          const int jj = j & (LRS_ZGEMM_3M ? 1 : 0);
          const double a1 = q1[jj][i][e], a2 = q2[jj][i][e], a3 = q3[jj][i][e];
          if (MODE == 1) v = C[(int64_t)nn * NB + 64 * wm + 8 * i + 2 * t + e];
          v = {v.x + (a1 - a2), v.y + (a3 - (a1 + a2))};
        }
        C[(int64_t)nn * NB + 64 * wm + 8 * i + 2 * t + e] = v;
        // izamax: the panel entry a_ij = l_ij u_jj would out-rank u_jj
        if (MODE == 0 && piv_status && s_abs1(s_mul(v, u)) > s_abs1(u))
          bad_col = min(bad_col, col0 + nn);
      }
  }
  if (piv_status && bad_col != 0x7fffffff) atomicMin(piv_status, bad_col);
}

template <int KIND>
__global__ void __launch_bounds__(ZG_THREADS, 1) lu_zgemm_kernel(BandGeom g, zc* tiles, int K,
                                                                 int* status) {
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  zc* sm = reinterpret_cast<zc*>(zsm_raw);
  const int p = blockIdx.y;
  const int T = g.T[p];
  if (K >= T) return;
  const int64_t base = g.tbase[p];
  auto tile = [&](int I, int J) -> zc* {
    return tiles + (base + (int64_t)I * g.W + (J - I + g.wl)) * TILE_ELEMS;
  };
  const int x = blockIdx.x >> 1, nbase = (blockIdx.x & 1) * 64;  // two half tiles per tile
  if (KIND == 0) {
    if (x < g.wl) {
      const int I = K + 1 + x;
      if (I >= T) return;
      ztile_gemm<0, ZMASK_NONE, ZMASK_UPPER>(tile(I, K), tile(K, K), tile(I, K), nbase, sm,
                                             &status[2 * p], K * NB, tile(K, K));
    } else {
      const int J = K + 1 + (x - g.wl);
      if (J >= T) return;
      ztile_gemm<0, ZMASK_UNIT_LOWER, ZMASK_NONE>(tile(K, K), tile(K, J), tile(K, J), nbase, sm,
                                                  nullptr, 0, nullptr);
    }
  } else if (KIND == 5) {  // U_KJ only (the pivoting path factors L_IK in its panel)
    const int J = K + 1 + x;
    if (J >= T) return;
    ztile_gemm<0, ZMASK_UNIT_LOWER, ZMASK_NONE>(tile(K, K), tile(K, J), tile(K, J), nbase, sm,
                                                nullptr, 0, nullptr);
  } else if (KIND == 1) {
    const int I = K + 2 + x / (g.wu - 1);
    const int J = K + 2 + x % (g.wu - 1);
    if (I >= T || J >= T) return;
    ztile_gemm<1, ZMASK_NONE, ZMASK_NONE>(tile(I, K), tile(K, J), tile(I, J), nbase, sm, nullptr, 0,
                                          nullptr);
  } else {
    int I, J;
    if (x < g.wl) {
      I = K + 1 + x;
      J = K + 1;
    } else {
      I = K + 1;
      J = K + 2 + (x - g.wl);
    }
    if (I >= T || J >= T) return;
    ztile_gemm<1, ZMASK_NONE, ZMASK_NONE>(tile(I, K), tile(K, J), tile(I, J), nbase, sm, nullptr, 0,
                                          nullptr);
  }
}

static void z_diag(Ctx* c, cudaStream_t s, const BandGeom& g, void* tiles, int K, int* status) {
  lu_diag_z_kernel<<<g.P, 512, 0, s>>>(g, static_cast<zc*>(tiles), K, status);
}

static void z_gemm(Ctx* c, cudaStream_t s, const BandGeom& g, void* tiles, int K, int* status,
                   int kind) {
  zc* t = static_cast<zc*>(tiles);
  if (kind == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (g.sym ? g.wl : g.wl + g.wu), g.P);  // sym: the L panel only
    cfg.blockDim = dim3(ZG_THREADS);
    cfg.dynamicSmemBytes = ZGEMM_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;  // the two half-tile CTAs of a tile
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LRS_CUDA(cudaLaunchKernelEx(&cfg, lu_zgemm_kernel<0>, g, t, K, status));
    if (g.sym && g.wu > 0) {
      lu_mirror_kernel<zc><<<dim3(g.wu, g.P), 256, 0, s>>>(g, t, K);
      LRS_LAUNCHED(c);
    }
  }
  else if (kind == 5)
    lu_zgemm_kernel<5><<<dim3(2 * g.wu, g.P), ZG_THREADS, ZGEMM_SMEM, s>>>(g, t, K, status);
  else if (kind == 1)
    lu_zgemm_kernel<1><<<dim3(2 * (g.wl - 1) * (g.wu - 1), g.P), ZG_THREADS, ZGEMM_SMEM, s>>>(
        g, t, K, status);
  else
    lu_zgemm_kernel<2><<<dim3(2 * (g.sym ? g.wl : g.wl + g.wu - 1), g.P), ZG_THREADS, ZGEMM_SMEM,
                         s>>>(g, t, K, status);
}

static void zgemm_attrs() {
  static bool attr = false;
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(lu_zgemm_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ZGEMM_SMEM));
    LRS_CUDA(cudaFuncSetAttribute(lu_zgemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ZGEMM_SMEM));
    LRS_CUDA(cudaFuncSetAttribute(lu_zgemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ZGEMM_SMEM));
    LRS_CUDA(cudaFuncSetAttribute(lu_zgemm_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ZGEMM_SMEM));
    attr = true;
  }
}

// The complex LU: with a band of >= 3 tiles each side, steps in pairs whose two-step updates
// run realified on the INT8 tensor cores (lu_i8_gemm_kernel<.., true>: C_re -= [Ar Ai][Br; -Bi],
// C_im -= [Ar Ai][Bi; Br], exact integer slices as in the real LU); otherwise (or with
// LRS_LU_I8=0, or when the panel buffers do not fit) single steps with the 3M DMMA update.
// Returns the steps per INT8 update (2) or 0.
int launch_band_lu_z(Ctx* c, const BandGeom& g0, zc* tiles, int Tmax, int* status, bool sym,
                     bool* sym_used) {
  zgemm_attrs();
  BandGeom g = g0;
  g.sym = 0;
  if (sym_used) *sym_used = false;
  LuKernels L{z_diag, z_gemm};
  DevBuf<uint8_t> buf;
  I8Panel pn[2];
  const char* e = std::getenv("LRS_LU_I8");
  const bool want = !(e && e[0] == '0') && g.wl >= 3 && g.wu >= 3;
  if (want && lu_i8_bytes_fit(2 * lu_i8_panel_bytes_z(g))) {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t a = al((size_t)g.P * g.wl * 2 * lu_i8_chunk_bytes(2)),
                 b = al((size_t)g.P * g.wu * 4 * lu_i8_chunk_bytes(2)),
                 ea = al(sizeof(int) * g.P * g.wl * NB), eb = al(sizeof(int) * g.P * g.wu * NB);
    buf.alloc(2 * (a + b + ea + eb));
    uint8_t* q = buf.get();
    for (int k = 0; k < 2; ++k) {
      pn[k].A = q;
      pn[k].B = q + a;
      pn[k].ea = reinterpret_cast<int*>(q + a + b);
      pn[k].eb = reinterpret_cast<int*>(q + a + b + ea);
      q += a + b + ea + eb;
    }
    L.pairs = true;
    L.i8 = pn;
    L.steps = 2;
    L.cplx = true;
    // complex symmetric blocks (A == A^T, not Hermitian): the symmetric schedule of band_lu.cu
    if (sym && lu_sym_wanted(g)) {
      g.sym = 1;
      if (sym_used) *sym_used = true;
    }
  }
  run_band_lu(c, g, tiles, Tmax, status, L);
  return L.i8 ? 2 : 0;
}

// Partial-pivoting complex band LU (zgbtrf): the panel kernels of band_lu_piv.cu, then
// U_KJ and the trailing update on the complex DMMA kernels; one stream, no look-ahead.
void launch_band_lu_piv_z(Ctx* c, const BandGeom& g, zc* tiles, int Tmax, int* status, int* ipiv,
                          int* perm) {
  zgemm_attrs();
  cudaStream_t s = c->stream;
  for (int K = 0; K < Tmax; ++K) {
    launch_lu_panel_piv_z(c, s, g, tiles, K, ipiv, perm, status);
    if (g.wu > 0) {
      ProfScope ps_(c, K_LU_PANEL, s);
      z_gemm(c, s, g, tiles, K, status, 5);
      LRS_LAUNCHED(c);
    }
    if (g.wl > 0 && g.wu > 0) {
      {
        ProfScope ps_(c, K_LU_PANEL, s);
        z_gemm(c, s, g, tiles, K, status, 2);
        LRS_LAUNCHED(c);
      }
      if (g.wl > 1 && g.wu > 1) {
        ProfScope ps_(c, K_LU_UPDATE, s);
        z_gemm(c, s, g, tiles, K, status, 1);
        LRS_LAUNCHED(c);
      }
    }
  }
}

}  // namespace lrs
