// Tiled band LU of the diagonal blocks A_p (K1/K2 of SURVEY.md 2.3).
//
// Implements factorize_block with LAPACK dgbtrf's pivot
// rule: the pivot of column j is the first max |a_ij|, i >= j.  This kernel
// set is the no-interchange path: it evaluates that rule for every column and
// records the first column whose rule would pick a row other than the
// diagonal (status[2p]); the host then raises LRS_ERR_NOT_IMPLEMENTED instead
// of returning factors that differ from LAPACK's.  Column-diagonally-dominant
// blocks (c1-c3) never interchange.
//
// Storage: partition p owns T_p row tiles of NB = 128 rows; row tile I stores
// the W = wl + wu + 1 tiles (I, I-wl) .. (I, I+wu) contiguously, each tile a
// column-major 128 x 128 block.  After factorization the off-diagonal tiles
// hold L (below) and U (above); the diagonal tile holds inv(L_II) strictly
// below and inv(U_II) on/above the diagonal (used by the apply kernels).
//
// Per step K (all partitions in one launch each):
//   lu_diag   : LU of tile (K,K) in shared memory + in-place triangular inverses
//   lu_gemm<0>: L_IK = A_IK inv(U_KK), U_KJ = inv(L_KK) A_KJ (DMMA tiles)
//   lu_gemm<1>: A_IJ -= L_IK U_KJ for the wl x wu trailing tiles (DMMA tiles)
#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"
#include "lu_common.cuh"

namespace lrs {

__device__ __forceinline__ int find_partition(const int64_t* off, int P, int64_t row) {
  int lo = 0, hi = P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) extract_tiles_kernel(int64_t n, const int* __restrict__ rp,
                                                            const int* __restrict__ ci,
                                                            const double* __restrict__ va,
                                                            BandGeom g, double* tiles, int64_t k,
                                                            int64_t row_lo, int64_t row_hi,
                                                            unsigned long long* bad) {
  const int64_t row = row_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= row_hi) return;
  const int p = find_partition(g.off, g.P, row);
  const int pg = g.p0 + p;  // global partition of this row
  const int64_t o = g.off[p], s = g.size[p];
  const int64_t li = row - o;
  const int I = (int)(li / NB);
  for (int q = rp[row]; q < rp[row + 1]; ++q) {
    const int64_t col = ci[q];
    bool ok;
    if (col >= o && col < o + s) {
      const int64_t lj = col - o;
      const int J = (int)(lj / NB);
      const int d = J - I;
      ok = d >= -g.wl && d <= g.wu;
      if (ok)
        tiles[(g.tbase[p] + (int64_t)I * g.W + (d + g.wl)) * TILE_ELEMS + (lj % NB) * NB +
              (li % NB)] = va[q];
    } else if (pg + 1 < g.Pg && col >= o + s && col < g.goff[pg + 2]) {
      ok = row >= o + s - k && col < o + s + k;  // B_p corner
    } else if (pg > 0 && col < o && col >= g.goff[pg - 1]) {
      ok = row < o + k && col >= o - k;  // C_p corner
    } else {
      ok = false;
    }
    if (!ok) atomicMin(bad, (unsigned long long)(row * n + col));
  }
}

__global__ void pad_diag_kernel(BandGeom g, double* tiles) {
  const int p = blockIdx.x;
  const int64_t s = g.size[p];
  const int T = g.T[p];
  for (int64_t li = s + threadIdx.x; li < (int64_t)T * NB; li += blockDim.x) {
    const int I = (int)(li / NB);
    tiles[(g.tbase[p] + (int64_t)I * g.W + g.wl) * TILE_ELEMS + (li % NB) * NB + (li % NB)] = 1.0;
  }
}

void launch_extract_tiles(Ctx* c, const Mat* m, const BandGeom& g, double* tiles, int64_t k,
                          int64_t row_lo, int64_t row_hi, unsigned long long* d_bad) {
  ProfScope ps_(c, K_SETUP);
  if (row_hi > row_lo) {
    extract_tiles_kernel<<<(unsigned)((row_hi - row_lo + 255) / 256), 256, 0, c->stream>>>(
        m->n, m->row_ptr.get(), m->col_idx.get(), m->vals.get(), g, tiles, k, row_lo, row_hi,
        d_bad);
    LRS_LAUNCHED(c);
  }
  pad_diag_kernel<<<g.P, 128, 0, c->stream>>>(g, tiles);
  LRS_LAUNCHED(c);
}

// ---------------------------------------------------------------------------------------
// lu_diag: one CTA (512 threads) per partition factors tile (K,K) with the tile held in
// registers: thread t owns rows (t & 31) + 32 r (r = 0..3) and columns (t >> 5) + 16 c
// (c = 0..7), both cyclic so every warp keeps work until the last steps.  Step j of the
// right-looking LU (no interchanges; dgbtrf's pivot rule checked per column) publishes
// column j of L and row j of U through a double-buffered shared vector pair and applies
// the rank-1 update in registers: one barrier per step, no shared-memory round trip of
// the trailing matrix.  The inverses follow the same pattern (rows of inv(L) forward and
// rows of inv(U) backward in the same sweep): the tile leaves with inv(L_KK) strictly
// below and inv(U_KK) on/above the diagonal.  Register blocks are indexed with
// compile-time r / c only (the step loops are unrolled over 16- / 32-step blocks).
// ---------------------------------------------------------------------------------------
constexpr int DIAG_THREADS = 512;
#ifndef LRS_DIAG_EXP
#define LRS_DIAG_EXP 0  // 1: skip the inverses (timing only, wrong factors)
#endif
constexpr size_t DIAG_SMEM = sizeof(double) * (TILE_ELEMS + 4 * NB);

__global__ void __launch_bounds__(DIAG_THREADS, 1) lu_diag_kernel(BandGeom g, double* tiles,
                                                                  int K, int* status) {
  extern __shared__ double sm[];
  double* A = sm;                   // the LU factors (column-major), read by the inverses
  double* vec = sm + TILE_ELEMS;    // [2 buffers][2 vectors][128]
  const int p = blockIdx.x;
  if (K >= g.T[p]) return;
  const int tid = threadIdx.x, lane = tid & 31, tc = tid >> 5;
  double* gt = tiles + (g.tbase[p] + (int64_t)K * g.W + g.wl) * TILE_ELEMS;
  const int col0 = K * NB;
  double a[4][8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r][c] = gt[(tc + 16 * c) * NB + lane + 32 * r];

  // ---- LU: step j = 16 jb + jj; column j lives in register column jb of warp jj ------
#pragma unroll
  for (int jb = 0; jb < 8; ++jb) {
    constexpr int dummy = 0;
    (void)dummy;
    const int rs = jb >> 1;  // register row block of row j
    for (int jj = 0; jj < 16; ++jj) {
      const int j = 16 * jb + jj;
      double* lcol = vec + (j & 1) * 2 * NB;
      double* urow = lcol + NB;
      if (tc == jj) {  // the warp owning column j: multipliers below the pivot
        const double piv = __shfl_sync(0xffffffffu, a[rs][jb], j & 31);
        const double rpiv = 1.0 / piv;  // dgbtf2 scales the column by 1 / pivot (dscal)
#pragma unroll
        for (int r = rs; r < 4; ++r) {
          const int i = lane + 32 * r;
          if (i > j) {
            const double v = a[r][jb];
            if (fabs(v) > fabs(piv)) atomicMin(&status[2 * p], col0 + j);  // dgbtrf would swap
            a[r][jb] = v * rpiv;
            lcol[i] = a[r][jb];
          }
        }
        if (lane == 0 && piv == 0.0) atomicMin(&status[2 * p + 1], col0 + j);
      }
      if (lane == (j & 31)) {  // row j of U, right of the pivot
#pragma unroll
        for (int c = jb; c < 8; ++c)
          if (tc + 16 * c > j) urow[tc + 16 * c] = a[rs][c];
      }
      __syncthreads();
      double l[4], u[8];
#pragma unroll
      for (int r = rs; r < 4; ++r) l[r] = (lane + 32 * r > j) ? lcol[lane + 32 * r] : 0.0;
#pragma unroll
      for (int c = jb; c < 8; ++c) u[c] = (tc + 16 * c > j) ? urow[tc + 16 * c] : 0.0;
#pragma unroll
      for (int r = rs; r < 4; ++r)
#pragma unroll
        for (int c = jb; c < 8; ++c) a[r][c] = fma(-l[r], u[c], a[r][c]);
    }
  }
  // the factors to shared memory (columns of L and U for the inverse sweeps)
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) A[(tc + 16 * c) * NB + lane + 32 * r] = a[r][c];
  // inverse registers: identity (strictly lower part: inv(L); upper incl. diagonal: the
  // right-hand side of U Y = I, turned into inv(U) row by row)
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) a[r][c] = (lane + 32 * r == tc + 16 * c) ? 1.0 : 0.0;
  __syncthreads();

#if LRS_DIAG_EXP == 1
  return;  // timing experiment: LU only
#endif
  // ---- inverses: step s forward for L (row s of inv(L) final), backward for U (row
  // k = 127 - s of inv(U) final after the division by u_kk) ----------------------------
#pragma unroll
  for (int sb = 0; sb < 4; ++sb) {
    constexpr int dummy = 0;
    (void)dummy;
    const int rb = 3 - sb;  // register row block of row k
    for (int ss = 0; ss < 32; ++ss) {
      const int s = 32 * sb + ss, k = NB - 1 - s;
      double* xrow = vec + (s & 1) * 2 * NB;
      double* yrow = xrow + NB;
      if (lane == ss) {  // row s of inv(L): columns < s final, X[s][s] = 1
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int m = tc + 16 * c;
          if (m < s) xrow[m] = a[sb][c];
          else if (m == s) xrow[m] = 1.0;  // (s, s) holds the U side
        }
      }
      if (lane == (k & 31)) {  // row k of inv(U): scale the finished right-hand side
        const double rkk = 1.0 / A[k * NB + k];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int m = tc + 16 * c;
          if (m >= k) {
            a[rb][c] = a[rb][c] * rkk;
            yrow[m] = a[rb][c];
          }
        }
      }
      __syncthreads();
      // Only the register blocks the step can touch, classified at compile time: the X
      // update needs rows i > s (r >= sb) and columns m <= s (c <= 2 sb + 1), the Y update
      // rows i < k (r <= rb) and columns m >= k (c >= 2 rb); block (r, c) is entirely
      // lower (i > m) when 32 r - 16 c >= 16, entirely upper when c >= 2 r + 2.
      double lv[4], uv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = lane + 32 * r;
        lv[r] = (r >= sb && i > s) ? A[s * NB + i] : 0.0;  // L[i][s]
        uv[r] = (r <= rb && i < k) ? A[k * NB + i] : 0.0;  // U[i][k]
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int m = tc + 16 * c;
        const bool cx = c <= 2 * sb + 1, cy = c >= 2 * rb;
        const double xv = (cx && m <= s) ? xrow[m] : 0.0;
        const double yv = (cy && m >= k) ? yrow[m] : 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const bool lower = 32 * r - 16 * c >= 16, upper = c >= 2 * r + 2;
          const bool ex = cx && r >= sb && !upper, ey = cy && r <= rb && !lower;
          if (ex && ey) {
            const int i = lane + 32 * r;
            if (i > m) a[r][c] = fma(-lv[r], xv, a[r][c]);  // X[i][m] -= L[i][s] X[s][m]
            else a[r][c] = fma(-uv[r], yv, a[r][c]);        // Y[i][m] -= U[i][k] Y[k][m]
          } else if (ex) {
            if (lower || lane + 32 * r > m) a[r][c] = fma(-lv[r], xv, a[r][c]);
          } else if (ey) {
            if (upper || lane + 32 * r <= m) a[r][c] = fma(-uv[r], yv, a[r][c]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) gt[(tc + 16 * c) * NB + lane + 32 * r] = a[r][c];
}

// ---------------------------------------------------------------------------------------
// DMMA tile GEMM: C(128x128) = / -= A(128x128) * B(128x128), all tiles column-major.
// A tile update is split over GEMM_SPLIT CTAs by columns (CN = 128 / GEMM_SPLIT each);
// every warp owns 64 x 32 outputs = 8 x 4 DMMA.8x8x4 accumulators, the warps of a CTA
// laid out 2 (M) x (CN / 32) (N).  With GEMM_SPLIT = 2 two CTAs share an SM, so one's
// C load / store overlaps the other's DMMA stream.  K is streamed in 4 chunks of 32 via
// cp.async, double buffered.  Shared layouts are padded so fragment loads are bank-
// conflict free: As[k][m] with row stride 132, Bs[n][k] with row stride 36.
// ---------------------------------------------------------------------------------------
#ifndef LRS_GEMM_SPLIT
#define LRS_GEMM_SPLIT 2
#endif
constexpr int GEMM_SPLIT = LRS_GEMM_SPLIT;
static_assert(GEMM_SPLIT == 1 || GEMM_SPLIT == 2, "column split");
constexpr int GEMM_THREADS = 256 / GEMM_SPLIT;
constexpr int GEMM_CN = NB / GEMM_SPLIT;     // tile columns per CTA
constexpr int GEMM_WN = GEMM_CN / 32;        // warps along N
constexpr int KC = 32;
constexpr int AS_LD = NB + 4;   // 132
constexpr int BS_LD = KC + 4;   // 36
constexpr int AS_STAGE = KC * AS_LD;
constexpr int BS_STAGE = GEMM_CN * BS_LD;
#ifndef LRS_GEMM_STAGES
#define LRS_GEMM_STAGES 2  // measured: 2 stages 0.328 s vs 3 stages 0.363 s (c2 LU)
#endif
constexpr int GEMM_STAGES = LRS_GEMM_STAGES;
static_assert(GEMM_STAGES >= 2 && GEMM_STAGES <= 3, "pipeline depth");
constexpr size_t GEMM_SMEM = sizeof(double) * GEMM_STAGES * (AS_STAGE + BS_STAGE);

#ifndef LRS_LU_PERSISTENT
#define LRS_LU_PERSISTENT 0  // measured: persistent 0.311 s (TPC 2) vs 0.308 s per-tile CTAs
#endif
#ifndef LRS_LU_PAIRS
#define LRS_LU_PAIRS 1  // two-step (rank-256) trailing updates
#endif
#ifndef LRS_REST_TPC
#define LRS_REST_TPC 4
#endif
#ifndef LRS_C_EPILOGUE
#define LRS_C_EPILOGUE 1  // measured c2 LU 0.308 s vs 0.315 s with the C preload
#endif

constexpr int MASK_NONE = 0, MASK_UNIT_LOWER = 1, MASK_UPPER = 2;

__device__ __forceinline__ void gemm_load_chunk(const double* __restrict__ A,
                                                const double* __restrict__ B, double* As,
                                                double* Bs, int kc, int tid) {
  constexpr int QA = KC * NB / 2 / GEMM_THREADS;       // 16-byte copies per thread (A)
  constexpr int QB = GEMM_CN * KC / 2 / GEMM_THREADS;  // (B)
#pragma unroll
  for (int q = 0; q < QA; ++q) {
    const int idx = tid + GEMM_THREADS * q;
    const int k = idx >> 6, m2 = (idx & 63) * 2;
    cp_async16(As + k * AS_LD + m2, A + (int64_t)(kc * KC + k) * NB + m2);
  }
#pragma unroll
  for (int q = 0; q < QB; ++q) {
    const int idx = tid + GEMM_THREADS * q;
    const int nn = idx >> 4, k2 = (idx & 15) * 2;
    cp_async16(Bs + nn * BS_LD + k2, B + (int64_t)nn * NB + kc * KC + k2);
  }
  cp_async_commit();
}

// The DMMA computes the transposed product C^T = B^T A^T: the B tile supplies the
// "A" fragments and the A tile the "B" fragments, so each lane's accumulator pair
// (c0, c1) is C[m][n], C[m+1][n] -- adjacent in the column-major tile -- and the C
// tile moves as 16-byte vectors.  MODE 1 accumulates -C + A B from the negated C and
// stores the negation: bitwise the same as C - A B (round-to-nearest is sign
// symmetric) without negating every A fragment.  h: the CTA's column block.
template <int MODE, int maskA, int maskB>  // MODE 0: C = A*B, 1: C -= A*B
__device__ __forceinline__ void tile_gemm(const double* A, const double* B, double* C, double* sm,
                                          int* piv_status, int col0, int h) {
  double* As = sm;
  double* Bs = sm + GEMM_STAGES * AS_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = w >> 1;
  const int g = lane >> 2, t = lane & 3;
  const int n0 = h * GEMM_CN;
  B += (int64_t)n0 * NB;
  C += (int64_t)n0 * NB;
  constexpr int NK = NB / KC;
  double acc[4][8][2];  // [n tile j][m tile i][pair]: C[m0 + 2t + e][n0 + g]
  constexpr int DIST = GEMM_STAGES - 1;  // prefetch distance in chunks
#pragma unroll
  for (int s = 0; s < DIST; ++s) gemm_load_chunk(A, B, As + s * AS_STAGE, Bs + s * BS_STAGE, s, tid);
  // MODE 1 (C_EPI = 0) accumulates straight into C: the C fragments load while the first
  // operand chunks are in flight and the epilogue is a plain store.  C_EPI = 1: the TMA
  // engine prefetches the C block into L2 now and the epilogue forms C - A B.
  constexpr bool C_EPI = MODE == 1 && LRS_C_EPILOGUE;
  if (C_EPI && tid == 0) bulk_prefetch_l2(C, sizeof(double) * NB * GEMM_CN);
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 1 && !C_EPI) {
        const double2 v = *reinterpret_cast<const double2*>(
            C + (int64_t)(32 * wn + 8 * j + g) * NB + 64 * wm + 8 * i + 2 * t);
        acc[j][i][0] = -v.x;
        acc[j][i][1] = -v.y;
      } else {
        acc[j][i][0] = acc[j][i][1] = 0.0;
      }
    }
  // B = inv(U) (upper): the output columns n0 .. n0+CN-1 take only k < n0 + CN (the other
  // K chunks are exact zeros), so the first column block stops early
  const int nk = (MODE == 0 && maskB == MASK_UPPER) ? (n0 + GEMM_CN + KC - 1) / KC : NK;
#pragma unroll 1
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + DIST < nk) {
      const int s2 = (kc + DIST) % GEMM_STAGES;
      gemm_load_chunk(A, B, As + s2 * AS_STAGE, Bs + s2 * BS_STAGE, kc + DIST, tid);
    }
    // chunk kc has landed once at most min(DIST, nk-1-kc) younger groups are pending
    const int pend = min(DIST, nk - 1 - kc);
    if (pend >= 2) cp_async_wait<2>();
    else if (pend == 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const int st = kc % GEMM_STAGES;
    const double* as = As + st * AS_STAGE;
    const double* bs = Bs + st * BS_STAGE;
#pragma unroll
    for (int k4 = 0; k4 < KC / 4; ++k4) {
      const int kk = k4 * 4 + t;
      const int kg = kc * KC + kk;
      double fa[8], fb[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {  // A[m][k], m = 64 wm + 8 i + g
        const int m = 64 * wm + 8 * i + g;
        double v = as[kk * AS_LD + m];
        if (maskA == MASK_UNIT_LOWER) v = m > kg ? v : (m == kg ? 1.0 : 0.0);
        fa[i] = v;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // B[k][n], n = 32 wn + 8 j + g (tile column n0 + n)
        const int nn = 32 * wn + 8 * j + g;
        double v = bs[nn * BS_LD + kk];
        if (maskB == MASK_UPPER) v = kg <= n0 + nn ? v : 0.0;
        fb[j] = v;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[j][i][0], acc[j][i][1], fb[j], fa[i]);
    }
    __syncthreads();
  }
  if (MODE == 0 && maskB == MASK_UPPER && GEMM_SPLIT == 2) {
    // L_IK = A_IK inv(U_KK) is formed in place and each half-tile CTA reads all of A_IK:
    // the two halves (a cluster of 2) write only after both have read their operands
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
  for (int j = 0; j < 4; ++j) {
    const int nn = 32 * wn + 8 * j + g;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double2 v;
      double2* cp = reinterpret_cast<double2*>(C + (int64_t)nn * NB + 64 * wm + 8 * i + 2 * t);
      if (C_EPI) {
        v = *cp;
        v.x -= acc[j][i][0];
        v.y -= acc[j][i][1];
      } else {
        v.x = MODE == 1 ? -acc[j][i][0] : acc[j][i][0];
        v.y = MODE == 1 ? -acc[j][i][1] : acc[j][i][1];
      }
      *cp = v;
      if (MODE == 0 && piv_status && (fabs(v.x) > 1.0 || fabs(v.y) > 1.0))
        bad_col = min(bad_col, col0 + n0 + nn);
    }
  }
  if (piv_status && bad_col != 0x7fffffff) atomicMin(piv_status, bad_col);
}

// Two-step trailing update C -= A0 B0 + A1 B1 (the rank-128 updates of steps K and K+1
// in one pass over C: half the C traffic and one prologue/epilogue per 2 x 128 of K).
// kbeg = 1 skips step K where its L / U tile lies outside the band.  Same fragments and
// pipeline as tile_gemm; C is prefetched into L2 and subtracted in the epilogue.
__device__ __forceinline__ void tile_gemm_pair(const double* A0, const double* B0,
                                               const double* A1, const double* B1, double* C,
                                               double* sm, int kbeg, int h) {
  double* As = sm;
  double* Bs = sm + GEMM_STAGES * AS_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = w >> 1;
  const int g = lane >> 2, t = lane & 3;
  const int n0 = h * GEMM_CN;
  B0 += (int64_t)n0 * NB;
  B1 += (int64_t)n0 * NB;
  C += (int64_t)n0 * NB;
  constexpr int NK = NB / KC;
  const int q0 = kbeg * NK, q1 = 2 * NK;
  auto load = [&](int q, int st) {
    const double* A = q < NK ? A0 : A1;
    const double* B = q < NK ? B0 : B1;
    gemm_load_chunk(A, B, As + st * AS_STAGE, Bs + st * BS_STAGE, q % NK, tid);
  };
  if (tid == 0) bulk_prefetch_l2(C, sizeof(double) * NB * GEMM_CN);
  double acc[4][8][2];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[j][i][0] = acc[j][i][1] = 0.0;
  load(q0, 0);
#pragma unroll 1
  for (int q = q0; q < q1; ++q) {
    const int st = (q - q0) & 1;
    if (q + 1 < q1) {
      load(q + 1, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + st * AS_STAGE;
    const double* bs = Bs + st * BS_STAGE;
#pragma unroll
    for (int k4 = 0; k4 < KC / 4; ++k4) {
      const int kk = k4 * 4 + t;
      double fa[8], fb[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) fa[i] = as[kk * AS_LD + 64 * wm + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = bs[(32 * wn + 8 * j + g) * BS_LD + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[j][i][0], acc[j][i][1], fb[j], fa[i]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int nn = 32 * wn + 8 * j + g;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double2* cp = reinterpret_cast<double2*>(C + (int64_t)nn * NB + 64 * wm + 8 * i + 2 * t);
      double2 v = *cp;
      v.x -= acc[j][i][0];
      v.y -= acc[j][i][1];
      *cp = v;
    }
  }
}

template <int KIND>
__global__ void __launch_bounds__(GEMM_THREADS, GEMM_SPLIT) lu_gemm_kernel(BandGeom g, double* tiles,
                                                                           int K, int* status,
                                                                           int m = 0) {
  extern __shared__ double sm[];
  const int p = blockIdx.y;
  const int T = g.T[p];
  if (K >= T) return;
  const int64_t base = g.tbase[p];
  auto tile = [&](int I, int J) -> double* {
    return tiles + (base + (int64_t)I * g.W + (J - I + g.wl)) * TILE_ELEMS;
  };
  const int x = blockIdx.x / GEMM_SPLIT, h = blockIdx.x % GEMM_SPLIT;
  if (KIND == 5) {
    // pivoting path: only U_KJ = inv(L_KK) A_KJ (the panel kernel produced L_IK)
    const int J = K + 1 + x;
    if (J >= T) return;
    tile_gemm<0, MASK_UNIT_LOWER, MASK_NONE>(tile(K, K), tile(K, J), tile(K, J), sm, nullptr, 0,
                                             h);
  } else if (KIND == 0) {
    if (x < g.wl) {
      const int I = K + 1 + x;
      if (I >= T) return;
      // L_IK = A_IK * inv(U_KK); |l| > 1 means dgbtrf would have interchanged rows
      tile_gemm<0, MASK_NONE, MASK_UPPER>(tile(I, K), tile(K, K), tile(I, K), sm, &status[2 * p],
                                          K * NB, h);
    } else {
      const int J = K + 1 + (x - g.wl);
      if (J >= T) return;
      tile_gemm<0, MASK_UNIT_LOWER, MASK_NONE>(tile(K, K), tile(K, J), tile(K, J), sm, nullptr, 0,
                                               h);
    }
  } else if (KIND == 1) {
    // trailing update away from the next pivot row/column: I, J >= K + 2
    const int I = K + 2 + x / (g.wu - 1);
    const int J = K + 2 + x % (g.wu - 1);
    if (I >= T || J >= T) return;
    tile_gemm<1, MASK_NONE, MASK_NONE>(tile(I, K), tile(K, J), tile(I, J), sm, nullptr, 0, h);
  } else if (KIND == 6) {
    // quad schedule, inside the look-ahead quad: step K applied to rows / columns
    // K+1 .. K+m only -- columns K+1..K+m (I = K+1..K+wl) and rows K+1..K+m
    // (J = K+m+1..K+wu); the rest of the trailing matrix waits for the bulk update
    int I, J;
    if (x < m * g.wl) {
      I = K + 1 + x % g.wl;
      J = K + 1 + x / g.wl;
    } else {
      const int y = x - m * g.wl;
      I = K + 1 + y / (g.wu - m);
      J = K + m + 1 + y % (g.wu - m);
    }
    if (I >= T || J >= T) return;
    tile_gemm<1, MASK_NONE, MASK_NONE>(tile(I, K), tile(K, J), tile(I, J), sm, nullptr, 0, h);
  } else if (KIND == 2) {
    // look-ahead part of the trailing update: column K+1 (I = K+1..K+wl) and row K+1
    // (J = K+2..K+wu), i.e. everything diag/panel of step K+1 needs
    int I, J;
    if (x < g.wl) {
      I = K + 1 + x;
      J = K + 1;
    } else {
      I = K + 1;
      J = K + 2 + (x - g.wl);
    }
    if (I >= T || J >= T) return;
    tile_gemm<1, MASK_NONE, MASK_NONE>(tile(I, K), tile(K, J), tile(I, J), sm, nullptr, 0, h);
  } else {
    // two-step updates with steps K and K+1 (K + 1 < T), look-ahead depth 2:
    //   KIND 3 (look-ahead): columns K+2 (I = K+2..K+1+wl), K+3 (I = K+3..K+1+wl) and rows
    //                        K+2 (J = K+3..K+1+wu), K+3 (J = K+4..K+1+wu)
    //   KIND 4 (bulk):       I = K+4..K+1+wl, J = K+4..K+1+wu
    int I, J;
    if (KIND == 3) {
      int y = x;
      if (y < g.wl) {
        I = K + 2 + y;
        J = K + 2;
      } else if ((y -= g.wl) < g.wl - 1) {
        I = K + 3 + y;
        J = K + 3;
      } else if ((y -= g.wl - 1) < g.wu - 1) {
        I = K + 2;
        J = K + 3 + y;
      } else {
        y -= g.wu - 1;
        I = K + 3;
        J = K + 4 + y;
      }
    } else if (g.sym) {
      // symmetric blocks: the lower triangle of the bulk window, row-major (x = a (a+1)/2 + b)
      int a = (int)((sqrtf(8.0f * (float)x + 1.0f) - 1.0f) * 0.5f);
      while ((a + 1) * (a + 2) / 2 <= x) ++a;
      while (a * (a + 1) / 2 > x) --a;
      I = K + 4 + a;
      J = K + 4 + (x - a * (a + 1) / 2);
    } else {
      I = K + 4 + x / (g.wu - 2);
      J = K + 4 + x % (g.wu - 2);
    }
    if (K + 1 >= T || I >= T || J >= T) return;
    const int kbeg = (I - K > g.wl || J - K > g.wu) ? 1 : 0;
    tile_gemm_pair(kbeg ? nullptr : tile(I, K), kbeg ? nullptr : tile(K, J), tile(I, K + 1),
                   tile(K + 1, J), tile(I, J), sm, kbeg, h);
  }
}

// Persistent bulk trailing update (kind 1): GEMM_SPLIT CTAs per SM loop over the
// half-tiles (p, I, J, h), I, J >= K + 2, with the cp.async double buffer running ACROSS
// tiles -- chunk 0 of the next tile lands while the last chunk of the current one is
// multiplied, and the next tile's C block is prefetched into L2 a whole tile ahead -- so
// no CTA start-up or operand-latency bubble separates consecutive tiles.  Arithmetic is
// tile_gemm<1> with LRS_C_EPILOGUE (C - A B formed in the epilogue).
__global__ void __launch_bounds__(GEMM_THREADS, GEMM_SPLIT)
    lu_rest_kernel(BandGeom g, double* tiles, int K, int total) {
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + GEMM_STAGES * AS_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w & 1, wn = w >> 1;
  const int gq = lane >> 2, tq = lane & 3;
  const int wu1 = g.wu - 1, per_p = (g.wl - 1) * wu1 * GEMM_SPLIT;
  struct Job { const double* A; const double* B; double* C; };
  auto decode = [&](int f, Job& jb) -> bool {
    const int p = f / per_p, r = f % per_p;
    const int x = r / GEMM_SPLIT, h = r % GEMM_SPLIT;
    const int T = g.T[p];
    const int I = K + 2 + x / wu1, J = K + 2 + x % wu1;
    if (I >= T || J >= T) return false;
    const int64_t base = g.tbase[p];
    auto tile = [&](int a, int b) { return tiles + (base + (int64_t)a * g.W + (b - a + g.wl)) * TILE_ELEMS; };
    jb.A = tile(I, K);
    jb.B = tile(K, J) + (int64_t)h * GEMM_CN * NB;
    jb.C = tile(I, J) + (int64_t)h * GEMM_CN * NB;
    return true;
  };
  auto next_valid = [&](int f, Job& jb) -> int {
    while (f < total && !decode(f, jb)) f += gridDim.x;
    return f;
  };
  Job cur, nxt;
  int f = next_valid(blockIdx.x, cur);
  if (f >= total) return;
  if (tid == 0) bulk_prefetch_l2(cur.C, sizeof(double) * NB * GEMM_CN);
  gemm_load_chunk(cur.A, cur.B, As, Bs, 0, tid);
  constexpr int NK = NB / KC;
  int q = 0;  // global chunk counter (stage = q % 2)
  while (true) {
    const int fn = next_valid(f + gridDim.x, nxt);
    const bool has_next = fn < total;
    if (has_next && tid == 0) bulk_prefetch_l2(nxt.C, sizeof(double) * NB * GEMM_CN);
    double acc[4][8][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[j][i][0] = acc[j][i][1] = 0.0;
#pragma unroll 1
    for (int kc = 0; kc < NK; ++kc, ++q) {
      const int s2 = (q + 1) & 1;
      bool issued = true;
      if (kc + 1 < NK) gemm_load_chunk(cur.A, cur.B, As + s2 * AS_STAGE, Bs + s2 * BS_STAGE, kc + 1, tid);
      else if (has_next) gemm_load_chunk(nxt.A, nxt.B, As + s2 * AS_STAGE, Bs + s2 * BS_STAGE, 0, tid);
      else issued = false;
      if (issued) cp_async_wait<1>();
      else cp_async_wait<0>();
      __syncthreads();
      const double* as = As + (q & 1) * AS_STAGE;
      const double* bs = Bs + (q & 1) * BS_STAGE;
#pragma unroll
      for (int k4 = 0; k4 < KC / 4; ++k4) {
        const int kk = k4 * 4 + tq;
        double fa[8], fb[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) fa[i] = as[kk * AS_LD + 64 * wm + 8 * i + gq];
#pragma unroll
        for (int j = 0; j < 4; ++j) fb[j] = bs[(32 * wn + 8 * j + gq) * BS_LD + kk];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[j][i][0], acc[j][i][1], fb[j], fa[i]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nn = 32 * wn + 8 * j + gq;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double2* cp = reinterpret_cast<double2*>(cur.C + (int64_t)nn * NB + 64 * wm + 8 * i + 2 * tq);
        double2 v = *cp;
        v.x -= acc[j][i][0];
        v.y -= acc[j][i][1];
        *cp = v;
      }
    }
    if (!has_next) break;
    f = fn;
    cur = nxt;
  }
}

static bool g_lu_attr_set = false;

static void lu_attrs() {
  if (g_lu_attr_set) return;
  LRS_CUDA(cudaFuncSetAttribute(lu_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)DIAG_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_gemm_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_rest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_gemm_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_gemm_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_gemm_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  LRS_CUDA(cudaFuncSetAttribute(lu_gemm_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
  g_lu_attr_set = true;
}

// LRS_LU_SKIP (timing experiments only, wrong factors): 4 drops the bulk two-step update,
// 1 drops everything else (diag, panels, look-ahead updates)
#ifndef LRS_LU_SKIP
#define LRS_LU_SKIP 0
#endif
static void real_diag(Ctx* c, cudaStream_t s, const BandGeom& g, void* tiles, int K, int* status) {
  if (LRS_LU_SKIP == 1) return;
  lu_diag_kernel<<<g.P, DIAG_THREADS, DIAG_SMEM, s>>>(
      g, static_cast<double*>(tiles), K, status);
}
static void real_gemm(Ctx* c, cudaStream_t s, const BandGeom& g, void* tiles, int K, int* status,
                      int kind) {
  double* t = static_cast<double*>(tiles);
  constexpr int S = GEMM_SPLIT;
  if ((LRS_LU_SKIP == 4 && kind == 4) || (LRS_LU_SKIP == 1 && kind != 4)) return;
  if (kind > 60) {  // kind 60 + m: rows / columns K+1 .. K+m with step K (quad look-ahead)
    const int m = kind - 60;
    // (symmetric blocks: the column part only, x < m wl)
    lu_gemm_kernel<6><<<dim3(S * m * (g.sym ? g.wl : g.wl + g.wu - m), g.P), GEMM_THREADS,
                        GEMM_SMEM, s>>>(g, t, K, status, m);
  } else if (kind == 0) {
    // the two half-tile CTAs of a tile form a cluster (tile_gemm's in-place L panel)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S * (g.sym ? g.wl : g.wl + g.wu), g.P);  // sym: the L panel only
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = GEMM_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LRS_CUDA(cudaLaunchKernelEx(&cfg, lu_gemm_kernel<0>, g, t, K, status, 0));
    if (g.sym && g.wu > 0) {
      lu_mirror_kernel<double><<<dim3(g.wu, g.P), 256, 0, s>>>(g, t, K);
      LRS_LAUNCHED(c);
    }
  }
  else if (kind == 1 && LRS_LU_PERSISTENT) {
    // each CTA takes at most LRS_REST_TPC half-tiles and retires, so the high-priority
    // look-ahead kernels (next / diag / panel of step K+1) still get SMs mid-update
    static const int tpc = std::getenv("LRS_REST_TPC") ? std::atoi(std::getenv("LRS_REST_TPC"))
                                                         : LRS_REST_TPC;
    const int total = S * (g.wl - 1) * (g.wu - 1) * g.P;
    const int grid = std::max(1, std::min(total, (total + tpc - 1) / tpc));
    lu_rest_kernel<<<grid, GEMM_THREADS, GEMM_SMEM, s>>>(g, t, K, total);
  } else if (kind == 1)
    lu_gemm_kernel<1><<<dim3(S * (g.wl - 1) * (g.wu - 1), g.P), GEMM_THREADS, GEMM_SMEM, s>>>(
        g, t, K, status);
  else if (kind == 2)
    lu_gemm_kernel<2><<<dim3(S * (g.sym ? g.wl : g.wl + g.wu - 1), g.P), GEMM_THREADS, GEMM_SMEM,
                        s>>>(g, t, K, status);
  else if (kind == 5)
    lu_gemm_kernel<5><<<dim3(S * g.wu, g.P), GEMM_THREADS, GEMM_SMEM, s>>>(g, t, K, status);
  else if (kind == 3)  // (symmetric blocks: columns K+2, K+3 only, the first 2 wl - 1 items)
    lu_gemm_kernel<3><<<dim3(S * (g.sym ? 2 * g.wl - 1 : 2 * g.wl + 2 * g.wu - 4), g.P),
                        GEMM_THREADS, GEMM_SMEM, s>>>(g, t, K, status);
  else  // (symmetric blocks: the lower triangle of the bulk window)
    lu_gemm_kernel<4><<<dim3(S * (g.sym ? (g.wl - 2) * (g.wl - 1) / 2 : (g.wl - 2) * (g.wu - 2)),
                             g.P), GEMM_THREADS, GEMM_SMEM, s>>>(g, t, K, status);
}

static void lu_diag_panel(Ctx* c, cudaStream_t s, const BandGeom& g, void* tiles, int K,
                          int* status, const LuKernels& L) {
  {
    ProfScope ps_(c, K_LU_DIAG, s);
    L.diag(c, s, g, tiles, K, status);
    LRS_LAUNCHED(c);
  }
  if (g.wl + g.wu > 0) {
    ProfScope ps_(c, K_LU_PANEL, s);
    L.gemm(c, s, g, tiles, K, status, 0);
    LRS_LAUNCHED(c);
  }
}

// Partial-pivoting band LU (band_lu_piv.cu for the panel; the DMMA kernels above for
// U_KJ and the trailing update).  One stream, no look-ahead: the interchanges of step K
// touch the tiles the trailing update of step K-1 writes.
void launch_band_lu_piv(Ctx* c, const BandGeom& g, double* tiles, int Tmax, int* status,
                        int* ipiv, int* perm) {
  lu_attrs();
  cudaStream_t s = c->stream;
  for (int K = 0; K < Tmax; ++K) {
    launch_lu_panel_piv(c, s, g, tiles, K, ipiv, perm, status);
    if (g.wu > 0) {
      ProfScope ps_(c, K_LU_PANEL, s);
      real_gemm(c, s, g, tiles, K, status, 5);
      LRS_LAUNCHED(c);
    }
    if (g.wl > 0 && g.wu > 0) {
      {
        ProfScope ps_(c, K_LU_PANEL, s);
        real_gemm(c, s, g, tiles, K, status, 2);
        LRS_LAUNCHED(c);
      }
      if (g.wl > 1 && g.wu > 1) {
        ProfScope ps_(c, K_LU_UPDATE, s);
        real_gemm(c, s, g, tiles, K, status, 1);
        LRS_LAUNCHED(c);
      }
    }
  }
}

bool lu_real_pairs(const BandGeom& g) {
  return lu_uses_pairs(g, LuKernels{real_diag, real_gemm, LRS_LU_PAIRS != 0});
}

// The two-step updates (kinds 3 / 4) run integer-sliced on the INT8 tensor cores (lu_i8.cu)
// unless LRS_LU_I8=0, the band is too narrow for the pair schedule, or the two panel
// buffers do not fit the free device memory (driver free + the pool's cached blocks, which
// an allocation releases on failure) with 2 GB to spare.
bool lu_i8_bytes_fit(size_t bytes) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
  const size_t avail = fr + pool_cached_bytes(), margin = size_t(2) << 30;
  return avail > margin && bytes < avail - margin;
}
static bool lu_i8_fits(const BandGeom& g, int steps) {
  // quads also hold the pair buffer of their look-ahead
  return lu_i8_bytes_fit(2 * lu_i8_panel_bytes(g, steps) +
                         (steps == 4 ? lu_i8_panel_bytes(g, 2) : 0));
}
static bool lu_i8_wanted(const BandGeom& g, const LuKernels& L) {
  const char* e = std::getenv("LRS_LU_I8");
  if (e && e[0] == '0') return false;
  return lu_uses_pairs(g, L);
}
// Quads: the INT8 bulk update runs four steps (K = 512) per launch (band >= 8 tiles each
// side), half the C traffic, TMEM drains and pass hand-offs per MMA, but the look-ahead
// inside the quad (DMMA, 6 tile-steps per column of the band per quad instead of 2 per
// pair) and four serial diagonal factorizations per quad lengthen the critical stream.
// They pay when the bulk launch is large against that chain: measured (profiles/
// r02_lu_variants_*.jsonl) c3 at P = 64 (305k tiles per quad launch, 2060 per SM) LU
// 1.167 s vs 1.237 s with pairs; c2 (6.3k tiles, 42 per SM) 0.162 s vs 0.152 s with the
// all-DMMA look-ahead inside the quad.  With the pair-form look-ahead (run_band_lu) quads
// are level with pairs on c2 or ahead (session 4: 0.148 vs 0.146 s; session 5's boxes:
// 0.166 vs 0.181 s), so quads when the first bulk launch holds >= LRS_QUAD_TILES_PER_SM
// (40) tiles per SM; LRS_LU_QUAD=0 / 1 forces pairs / quads.
static int lu_i8_steps(const BandGeom& g, int num_sms) {
  if (!(g.wl >= 8 && g.wu >= 8)) return 2;
  const char* e = std::getenv("LRS_LU_QUAD");
  if (e && e[0] == '1') return 4;
  if (e && e[0] == '0') return 2;
  const char* t = std::getenv("LRS_QUAD_TILES_PER_SM");
  const double per_sm = t ? std::atof(t) : 40.0;
  const double tiles = (double)g.P * (g.wl - 4) * (g.wu - 4);
  return tiles >= per_sm * num_sms ? 4 : 2;
}

// The symmetric schedule rides on the pair / quad schedules (the DMMA kinds 0, 2, 3, 4, 60+m
// and the INT8 kinds 3, 4 know g.sym); LRS_LU_SYM=0 switches it off.
bool lu_sym_wanted(const BandGeom& g) {
  const char* e = std::getenv("LRS_LU_SYM");
  if (e && e[0] == '0') return false;
  return g.wl == g.wu && !lu_i8_2sm();
}

int launch_band_lu(Ctx* c, const BandGeom& g0, double* tiles, int Tmax, int* status, bool sym,
                   bool* sym_used) {
  lu_attrs();
  BandGeom g = g0;
  g.sym = 0;
  if (sym_used) *sym_used = false;
  LuKernels L{real_diag, real_gemm, LRS_LU_PAIRS != 0};
  DevBuf<uint8_t> buf;
  I8Panel pn[3];  // [0], [1]: the bulk update's buffers (alternating); [2]: the quad
                  // look-ahead's pair update (steps = 4 only)
  int steps = lu_i8_steps(g, c->num_sms);
  if (steps == 4 && !lu_i8_fits(g, 4)) steps = 2;
  if (lu_i8_wanted(g, L) && lu_i8_fits(g, steps)) {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t a = al((size_t)g.P * g.wl * TILE_ELEMS * steps * 8),
                 b = al((size_t)g.P * g.wu * TILE_ELEMS * steps * 8),
                 ea = al(sizeof(int) * g.P * g.wl * NB), eb = al(sizeof(int) * g.P * g.wu * NB);
    // the pair buffer of the quad look-ahead: half the A / B panel bytes of a quad buffer
    const size_t a2 = al((size_t)g.P * g.wl * TILE_ELEMS * 2 * 8),
                 b2 = al((size_t)g.P * g.wu * TILE_ELEMS * 2 * 8);
    const size_t extra = steps == 4 ? a2 + b2 + ea + eb : 0;
    buf.alloc(2 * (a + b + ea + eb) + extra);
    uint8_t* q = buf.get();
    for (int k = 0; k < 2; ++k) {
      pn[k].A = q;
      pn[k].B = q + a;
      pn[k].ea = reinterpret_cast<int*>(q + a + b);
      pn[k].eb = reinterpret_cast<int*>(q + a + b + ea);
      q += a + b + ea + eb;
    }
    if (steps == 4) {
      pn[2].A = q;
      pn[2].B = q + a2;
      pn[2].ea = reinterpret_cast<int*>(q + a2 + b2);
      pn[2].eb = reinterpret_cast<int*>(q + a2 + b2 + ea);
    }
    L.i8 = pn;
    L.steps = steps;
  }
  // the symmetric schedule needs the pair / quad form (INT8, or the DMMA two-step kinds 3 / 4)
  if (sym && lu_sym_wanted(g) && (L.i8 || lu_uses_pairs(g, L))) {
    g.sym = 1;
    if (sym_used) *sym_used = true;
  }
  run_band_lu(c, g, tiles, Tmax, status, L);
  return L.i8 != nullptr ? L.steps : 0;
}

// Right-looking tiled LU with look-ahead depth 1 over two streams:
//   crit (high priority): [wait rest(K-1)] next(K) -> diag(K+1) -> panel(K+1)
//   main               : [wait panel(K)]  rest(K)
// next(K) applies step K to pivot row/column K+1 only, so diag/panel of step K+1
// overlap the bulk trailing update rest(K) (I, J >= K+2) instead of idling the GPU.
bool lu_uses_pairs(const BandGeom& g, const LuKernels& L) {
  return L.pairs && g.wl >= 3 && g.wu >= 3;
}

void run_band_lu(Ctx* c, const BandGeom& g, void* tiles, int Tmax, int* status,
                 const LuKernels& L) {
  if (Tmax <= 0) return;
  cudaStream_t sm = c->stream, sc = c->stream_hi;
  cudaEvent_t ev_start = c->take_event(), ev_panel = c->take_event(), ev_panel2 = c->take_event(),
              ev_rest = c->take_event();
  LRS_CUDA(cudaEventRecord(ev_start, sm));
  LRS_CUDA(cudaStreamWaitEvent(sc, ev_start, 0));
  lu_diag_panel(c, sc, g, tiles, 0, status, L);
  LRS_CUDA(cudaEventRecord(ev_panel, sc));
  auto gemm = [&](cudaStream_t s, int K, int kind, int cls) {
    ProfScope ps_(c, cls, s);
    L.gemm(c, s, g, tiles, K, status, kind);
    LRS_LAUNCHED(c);
  };
  // INT8 path: slice(K) digitises the panels of pair K right after panel(K+1) on the
  // critical stream; the pair buffers alternate (pair K-4's readers -- rest2(K-4) on main,
  // next3(K-4) on crit -- completed before crit reaches slice(K)).
  auto slice = [&](int K) {
    if (!L.i8) return;
    ProfScope ps_(c, K_LU_PANEL, sc);
    if (L.cplx)
      launch_lu_i8_slice_z(c, sc, g, static_cast<const zc*>(tiles), K, L.i8[(K / L.steps) & 1]);
    else
      launch_lu_i8_slice(c, sc, g, static_cast<const double*>(tiles), K, L.steps,
                         L.i8[(K / L.steps) & 1]);
  };
  auto upd2 = [&](cudaStream_t s, int K, int kind, int cls) {
    if (!L.i8) return gemm(s, K, kind, cls);
    ProfScope ps_(c, cls, s);
    if (L.cplx)
      launch_lu_i8_gemm_z(c, s, g, static_cast<zc*>(tiles), K, kind, L.i8[(K / L.steps) & 1]);
    else
      launch_lu_i8_gemm(c, s, g, static_cast<double*>(tiles), K, kind, L.steps,
                        L.i8[(K / L.steps) & 1]);
  };
  if (L.i8 && L.steps == 4) {
    // Steps in quads (K .. K+3) with a rank-512 INT8 bulk update and look-ahead depth 4:
    //   main: [wait slice(K)] rest4(K)                                   (I, J >= K+8)
    //   crit: [wait rest4(K-4)] next4(K) (rows / columns K+4..K+7, INT8) -> for s = K+4..K+7:
    //         diag/panel(s), step s on rows / columns s+1..K+7 (DMMA kind 60 + m)
    //         -> slice(K+4)
    // Every tile takes its updates in step order; main never waits on crit's latency chain.
    // The serial LU of steps K0 .. K0+3 inside the look-ahead.  A full quad runs it as the
    // pair schedule does: step K0 on row / column K0+1 (DMMA), diag / panel(K0+1), the
    // INT8 pair update of rows / columns K0+2, K0+3 with steps K0, K0+1 (the look-ahead pair
    // buffer L.i8[2]), step K0+2 on row / column K0+3 (DMMA), diag / panel(K0+3): a third of
    // the DMMA tile-steps of applying each step to the rest of the quad window (kind 60+m,
    // kept for a partial last quad).  LRS_QUAD_MINI_DMMA=1 selects the all-DMMA form.
    static const bool mini_dmma = std::getenv("LRS_QUAD_MINI_DMMA") &&
                                  std::getenv("LRS_QUAD_MINI_DMMA")[0] == '1';
    auto mini = [&](int K0) {
      const int last = std::min(K0 + 3, Tmax - 1);
      if (!mini_dmma && last == K0 + 3 && g.wl >= 4 && g.wu >= 4) {
        if (K0 > 0) lu_diag_panel(c, sc, g, tiles, K0, status, L);  // step 0: done above
        gemm(sc, K0, 2, K_LU_PANEL);
        lu_diag_panel(c, sc, g, tiles, K0 + 1, status, L);
        {
          ProfScope ps_(c, K_LU_PANEL, sc);
          launch_lu_i8_slice(c, sc, g, static_cast<const double*>(tiles), K0, 2, L.i8[2]);
          launch_lu_i8_gemm(c, sc, g, static_cast<double*>(tiles), K0, 3, 2, L.i8[2]);
        }
        lu_diag_panel(c, sc, g, tiles, K0 + 2, status, L);
        gemm(sc, K0 + 2, 2, K_LU_PANEL);
        lu_diag_panel(c, sc, g, tiles, K0 + 3, status, L);
        return;
      }
      for (int st = K0; st <= last; ++st) {
        if (st > 0) lu_diag_panel(c, sc, g, tiles, st, status, L);  // step 0: done above
        if (last - st > 0 && g.wl > 0 && g.wu > 0) gemm(sc, st, 60 + (last - st), K_LU_PANEL);
      }
    };
    mini(0);
    if (Tmax > 4) slice(0);
    LRS_CUDA(cudaEventRecord(ev_panel, sc));
    bool have_rest = false;
    for (int K = 0; K + 4 < Tmax; K += 4) {
      if (have_rest) LRS_CUDA(cudaStreamWaitEvent(sc, ev_rest, 0));  // rest4(K-4)
      LRS_CUDA(cudaStreamWaitEvent(sm, ev_panel, 0));                  // slice(K)
      upd2(sm, K, 4, K_LU_UPDATE);
      LRS_CUDA(cudaEventRecord(ev_rest, sm));
      have_rest = true;
      upd2(sc, K, 3, K_LU_PANEL);
      mini(K + 4);
      if (K + 8 < Tmax) slice(K + 4);
      LRS_CUDA(cudaEventRecord(ev_panel, sc));
    }
  } else if (lu_uses_pairs(g, L)) {
    // Steps in pairs (K, K+1) with a rank-256 bulk update and look-ahead depth 2:
    //   main: [wait panel(K+1)] rest2(K, K+1)                       (I, J >= K+4)
    //   crit: [wait rest2(K-2, K-1)] next3(K, K+1) (rows/cols K+2, K+3) -> diag/panel(K+2)
    //         -> next(K+2) (row/col K+3) -> diag/panel(K+3)
    // so diag/panel(K+2), (K+3) run under rest2(K, K+1) and main never waits on crit.
    if (Tmax > 1) {
      gemm(sc, 0, 2, K_LU_PANEL);
      lu_diag_panel(c, sc, g, tiles, 1, status, L);
      slice(0);
      LRS_CUDA(cudaEventRecord(ev_panel, sc));
    }
    bool have_rest = false;
    for (int K = 0; K + 1 < Tmax; K += 2) {
      if (have_rest) LRS_CUDA(cudaStreamWaitEvent(sc, ev_rest, 0));  // rest2(K-2, K-1)
      LRS_CUDA(cudaStreamWaitEvent(sm, ev_panel, 0));                  // diag/panel(K+1)
      upd2(sm, K, 4, K_LU_UPDATE);
      LRS_CUDA(cudaEventRecord(ev_rest, sm));
      have_rest = true;
      if (K + 2 < Tmax) {
        upd2(sc, K, 3, K_LU_PANEL);
        lu_diag_panel(c, sc, g, tiles, K + 2, status, L);
        if (K + 3 < Tmax) {
          gemm(sc, K + 2, 2, K_LU_PANEL);
          lu_diag_panel(c, sc, g, tiles, K + 3, status, L);
          slice(K + 2);
        }
        LRS_CUDA(cudaEventRecord(ev_panel, sc));
      }
    }
  } else
  for (int K = 0; K < Tmax; ++K) {
    if (K + 1 < Tmax) {
      if (K >= 1) LRS_CUDA(cudaStreamWaitEvent(sc, ev_rest, 0));
      if (g.wl > 0 && g.wu > 0) {
        // the look-ahead update of row/column K+1 is critical-path work: profiled with
        // the panel, so K_LU_UPDATE times exactly the bulk trailing update lu_gemm<1>
        ProfScope ps_(c, K_LU_PANEL, sc);
        L.gemm(c, sc, g, tiles, K, status, 2);
        LRS_LAUNCHED(c);
      }
      lu_diag_panel(c, sc, g, tiles, K + 1, status, L);
      LRS_CUDA(cudaEventRecord(ev_panel2, sc));
    }
    LRS_CUDA(cudaStreamWaitEvent(sm, ev_panel, 0));
    if (g.wl > 1 && g.wu > 1) {
      ProfScope ps_(c, K_LU_UPDATE, sm);
      L.gemm(c, sm, g, tiles, K, status, 1);
      LRS_LAUNCHED(c);
    }
    LRS_CUDA(cudaEventRecord(ev_rest, sm));
    std::swap(ev_panel, ev_panel2);
  }
  // join: everything issued on the crit stream precedes what follows on main
  LRS_CUDA(cudaEventRecord(ev_panel2, sc));
  LRS_CUDA(cudaStreamWaitEvent(sm, ev_panel2, 0));
  LRS_CUDA(cudaEventRecord(ev_panel, sm));
  LRS_CUDA(cudaEventSynchronize(ev_panel));  // events go back to the pool only once idle
  c->ev_pool.push_back(ev_start);
  c->ev_pool.push_back(ev_panel);
  c->ev_pool.push_back(ev_panel2);
  c->ev_pool.push_back(ev_rest);
}

// ---------------------------------------------------------------------------------------
// FP64 DMMA peak microbenchmark (roofline denominator; MEASURED_PEAKS.json has no FP64)
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  double acc[8][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[i][0], acc[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

double run_dmma_peak(Ctx* c) {
  DevBuf<double> out;
  out.alloc(256);
  const int iters = 20000;
  const int blocks = c->num_sms * 4;
  dmma_peak_kernel<<<blocks, 256, 0, c->stream>>>(out.get(), 200);
  LRS_LAUNCHED(c);
  LRS_CUDA(cudaEventRecord(c->ev0, c->stream));
  dmma_peak_kernel<<<blocks, 256, 0, c->stream>>>(out.get(), iters);
  LRS_LAUNCHED(c);
  LRS_CUDA(cudaEventRecord(c->ev1, c->stream));
  LRS_CUDA(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  LRS_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  const double flops = 2.0 * 256.0 * 8.0 * iters * (double)blocks * 8.0;  // 8 warps, 8 dmma, 256 FMA
  return flops / (ms * 1e-3) / 1e12;
}

}  // namespace lrs
