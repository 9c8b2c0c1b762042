// Dataflow banded triangular solves (K3/K4/K5 of SURVEY.md 2.3): the D-stage
// y_p = A_p^-1 f_p of apply_precond_T / apply_block_jacobi,
// solve_block and solve_block_adjoint.
//
// One CTA per (partition, row tile).  CTAs take tickets in start order, so a
// CTA only ever waits on tiles whose CTAs already started: no deadlock for
// any residency.  Each CTA streams its row panel (wl or wu off-diagonal tiles
// plus the diagonal tile, contiguous in HBM) through a shared-memory ring with
// 1D bulk copies (cp.async.bulk, the TMA engine) *before* its dependencies
// resolve, and only waits on the per-tile ready flag (release / acquire at gpu
// scope, epoch-tagged so flags never need resetting) right before it needs
// x_s.  The diagonal tile holds the explicit inverses of the LU diagonal
// blocks, so the per-tile critical path is a flag round trip plus one
// 128 x 128 product; the factor stream runs at HBM speed behind it.
//
// A chunk is 32 contiguous tile columns (32 KB, one bulk copy).  Multi-RHS
// chunk products are (128 x 32) x (32 x NR) GEMMs (or their transposes) on the
// FP64 tensor cores (DMMA.8x8x4), NR in {8, 16}; one code path for every
// width keeps each column's arithmetic independent of the batch, so
// solve_block on a multi-column RHS equals column-by-column bit-exactly
// (solve_block always takes this path).  Wider blocks (the 2l spike
// columns of the setup) run as independent 16-column groups in the same launch,
// each with its own ready flags: the per-tile critical path is a 16-column product,
// and the groups of one row tile start together so their factor reads share L2.  The Krylov hot path
// (apply with one right-hand side) uses an FP64-FMA variant, one thread per
// row, which keeps less work on the per-tile critical path and streams the
// factor at ~96% of the measured HBM copy bandwidth.
//
// One-RHS L and U sweeps (the Krylov hot path) hand x_t to their dependants through a
// self-validating mailbox instead of x + a ready flag: each double of x_t travels as two
// 8-byte words (epoch << 32 | 32-bit half), stored relaxed and polled relaxed, one word
// per consumer thread.  A consumer's poll IS its data load (one L2 round trip instead of
// flag-acquire then load), and the producer needs no fence before publishing.
//
// Modes: 0  L  forward (unit lower),   1  U  backward,
//        2  U^T forward (adjoint),     3  L^T backward (adjoint).
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lrs {

#ifndef LRS_SOLVE_FMA_ACC
#define LRS_SOLVE_FMA_ACC 4  // partial sums per chunk of the one-RHS FMA sweeps (1: a single chain)
#endif
constexpr int SOLVE_THREADS = 256;
constexpr int CH_COLS = 32;
constexpr int CLD = NB;                  // column stride of a chunk in shared memory
constexpr int CH_SM = CH_COLS * CLD;     // doubles per shared chunk
constexpr int NCH = NB / CH_COLS;        // chunks per tile

// DIAGPK (NR == 1, L and U sweeps; off): the triangle of the diagonal tile the sweep uses
// (strictly lower inv(L) in mode 0, upper inv(U) in mode 1: 8128 / 8256 doubles) is
// copied packed into a resident 64.5 KB region at CTA start (cp.async), next to the full
// 5-stage ring, so no diagonal chunk is fetched after the last dependency resolves.
// Measured on c2 with the mailbox handoff: apply 2.63 ms with it, 2.51 ms without (the
// triangular product's shared-memory reads cost more than the chunk refetch, which the
// ring already overlaps); kept as a switch.  (A resident full 128 KB tile, which forces the
// ring down to 3 stages, was slower still.)
#ifndef LRS_SOLVE_DIAGPK
#define LRS_SOLVE_DIAGPK 0
#endif
constexpr int DPK_ELEMS = NB * (NB + 1) / 2;  // 8256: upper incl. diagonal (lower: 8128)
// Shared-memory plan per (mode, width).  `red` (half sums of the FMA path, the transposed
// accumulator) and `part` (K-quarter partials of the transposed DMMA path) exist only where
// they are used, so the 48-column DMMA sweeps fit: forward 5 x 32 KB ring + 53 KB of x_s,
// adjoint 2-stage ring + x_s + red + part.
template <int MODE, int NR> struct SolveCfg {
  static constexpr bool TRANS = MODE >= 2;
  static constexpr bool DIAGPK = LRS_SOLVE_DIAGPK && NR == 1;
  static constexpr int STAGES = (TRANS && NR > 16) ? 2 : 5;
  static constexpr int XLD = NR == 1 ? 1 : NR + 4;  // padded row stride of xs / red
  static constexpr int PLD = NR + 1;                // K-quarter partials (adjoint DMMA)
  static constexpr int RED = (NR == 1 || TRANS) ? NB * XLD : 0;
  static constexpr int PART = (NR > 1 && TRANS) ? 4 * CH_COLS * PLD : 0;
  static constexpr int DREG = DIAGPK ? DPK_ELEMS : 0;
};
// packed index of diagonal-tile element (r, c) of the triangle the sweep uses
template <int MODE>
__device__ __forceinline__ int dpk_col(int c) {
  return MODE == 0 ? c * NB - c * (c + 1) / 2 - c - 1 : c * (c + 1) / 2;
}

template <int MODE, int NR>
constexpr size_t solve_smem_bytes() {
  using C = SolveCfg<MODE, NR>;
  return sizeof(double) * ((size_t)C::STAGES * CH_SM + C::DREG + (size_t)NB * C::XLD + C::RED +
                           C::PART) +
         16 * (C::STAGES + 1) + 64;
}

#ifdef LRS_SOLVE_TRACE
// development aid: per-CTA globaltimer stamps (start, last-dependency wait begins, last
// dependency ready, diagonal step, diagonal product done, published)
__device__ unsigned long long* g_strace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STRACE(i) \
  if (g_strace && tid == 0) g_strace[(size_t)tk0 * 8 + (i)] = gtimer()
#else
#define STRACE(i)
#endif


// the int slot after the barriers: the CTA's ticket (then the x-prefetch "ready" word)
template <int MODE, int NR>
__device__ __forceinline__ int* solve_ticket_slot(unsigned char* smraw) {
  using Cfg = SolveCfg<MODE, NR>;
  return reinterpret_cast<int*>(smraw + sizeof(double) * ((size_t)Cfg::STAGES * CH_SM + Cfg::DREG +
                                                          (size_t)NB * Cfg::XLD + Cfg::RED +
                                                          Cfg::PART) +
                                8 * (Cfg::STAGES + 1));
}

// One CTA of a sweep: ticket tk0 (taken by the caller).  FUSED_U: the U sweep of the fused
// one-RHS L + U launch -- tile t's right-hand side comes from the L sweep's mailbox words of
// tile t (epoch epoch_l: the values the L sweep also stores into x), so the U CTAs need no
// kernel boundary after the L sweep.
template <int MODE, int NR, bool FUSED_U = false>
__device__ __forceinline__ void band_solve_body(BandGeom g, const double* __restrict__ tiles,
                                                double* x, int64_t ld, int nrhs, unsigned* flags,
                                                unsigned epoch, int p_only, int ngroups,
                                                int64_t flag_stride,
                                                const float* __restrict__ t32,
                                                unsigned long long* mbox, const int tk0,
                                                unsigned epoch_l) {
  using Cfg = SolveCfg<MODE, NR>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int XLD = Cfg::XLD;
  constexpr bool FWD = (MODE == 0 || MODE == 2);
  constexpr bool TRANS = (MODE >= 2);
  constexpr bool MMA = NR >= 8;
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr bool DPK = Cfg::DIAGPK && !TRANS;
  constexpr bool LLM = NR == 1 && !TRANS;  // mailbox handoff (2 words per row of x_t)
  static_assert(!LLM || SOLVE_THREADS == 2 * NB, "one mailbox word per thread");
  double* ring = reinterpret_cast<double*>(smraw);
  double* dreg = ring + (size_t)STAGES * CH_SM;  // resident packed diagonal triangle
  double* xs = dreg + Cfg::DREG;      // [NB][XLD]: x_s, or the diagonal-step input
  double* red = xs + NB * XLD;                 // [NB][XLD]: half sums / transposed accumulator
  double* part = red + Cfg::RED;               // [4][CH_COLS][PLD]: adjoint K-quarter partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(part + Cfg::PART);  // + [STAGES]: diag
  int* s_tk = reinterpret_cast<int*>(bars + STAGES + 1);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  STRACE(0);
  // column group (adjacent tickets: the groups of one row tile start together)
  const int grp = tk0 % ngroups, tk = tk0 / ngroups;
  x += (int64_t)grp * NR * ld;
  nrhs = min(NR, nrhs - grp * NR);
  flags += grp * flag_stride;
  int p, tt;
  if (p_only >= 0) {
    p = p_only;
    tt = tk;
  } else {
    p = tk % g.P;
    tt = tk / g.P;
  }
  const int T = g.T[p];
  if (tt >= T) return;
  const int t = FWD ? tt : T - 1 - tt;
  const int64_t base = g.tbase[p], off = g.off[p], size = g.size[p];
  const int W = g.W, wl = g.wl;
  int s0, ndeps, sstep;
  if (MODE == 0) { s0 = max(0, t - g.wl); ndeps = t - s0; sstep = 1; }
  else if (MODE == 1) { s0 = min(T - 1, t + g.wu); ndeps = s0 - t; sstep = -1; }
  else if (MODE == 2) { s0 = max(0, t - g.wu); ndeps = t - s0; sstep = 1; }
  else { s0 = min(T - 1, t + g.wl); ndeps = s0 - t; sstep = -1; }
  auto tile_ptr = [&](int d) -> const double* {
    if (d == ndeps) return tiles + (base + (int64_t)t * W + wl) * TILE_ELEMS;
    const int s = s0 + d * sstep;
    if (!TRANS) return tiles + (base + (int64_t)t * W + (s - t + wl)) * TILE_ELEMS;
    return tiles + (base + (int64_t)s * W + (t - s + wl)) * TILE_ELEMS;
  };
  const int Q = (ndeps + 1) * NCH;
  const int Qring = DPK ? ndeps * NCH : Q;  // chunks that go through the ring
  // producer: one 32 KB bulk copy per chunk (32 contiguous tile columns); with FP32
  // off-diagonal factors (t32) those chunks are 16 KB
  auto issue = [&](int q, int st) {
    const int d = q / NCH;
    if (t32 && d != ndeps) {
      // the FP32 copy is compact: slot -> its index among the in-block tiles
      const int64_t slot = (tile_ptr(d) - tiles) / TILE_ELEMS;
      const float* src = t32 + (size_t)g.t32_idx[slot] * TILE_ELEMS + (size_t)(q % NCH) * CH_COLS * NB;
      mbar_expect_tx(&bars[st], CH_COLS * NB * sizeof(float));
      bulk_g2s(ring + (size_t)st * CH_SM, src, CH_COLS * NB * sizeof(float), &bars[st]);
      return;
    }
    const double* src = tile_ptr(d) + (size_t)(q % NCH) * CH_COLS * NB;
    mbar_expect_tx(&bars[st], CH_COLS * NB * sizeof(double));
    bulk_g2s(ring + (size_t)st * CH_SM, src, CH_COLS * NB * sizeof(double), &bars[st]);
  };
  if (tid == 0) {
    for (int st = 0; st <= STAGES; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < STAGES && q < Qring; ++q) issue(q, q);
  if (DPK) {
    // warp per column: column c of the triangle is contiguous in the tile (column-major)
    const double* dt = tile_ptr(ndeps);
    for (int c = w; c < NB; c += SOLVE_THREADS / 32) {
      const int r0 = MODE == 0 ? c + 1 : 0, r1 = MODE == 0 ? NB : c + 1;
      double* dst = dreg + dpk_col<MODE>(c);
      for (int r = r0 + lane; r < r1; r += 32) cp_async8(dst + r, dt + (size_t)c * NB + r);
    }
    cp_async_commit();
  }

  const int64_t row0 = (int64_t)t * NB;
  const int gq = lane >> 2, tq = lane & 3;  // DMMA fragment coordinates
  // ---- accumulators -----------------------------------------------------------------
  // FMA path (NR == 1): thread (row = tid & 127, half = tid >> 7) sums half the columns.
  // DMMA non-trans: warp w owns rows 16w..16w+15 (2 m8 tiles) x NR/8 n8 tiles.
  constexpr int NJ = MMA ? NR / 8 : 1;
  double acc[2][NJ][2];
  double acc1 = 0.0;
  const int row = tid & (NB - 1), hh = tid >> 7;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
  if (!TRANS) {
    if (FUSED_U) {
      static_assert(!FUSED_U || (LLM && MODE == 1), "fused U sweep: one-RHS mailbox path");
      const unsigned long long* mb = mbox + (size_t)(g.fbase[p] + t) * (2 * NB) + tid;
      unsigned long long v = ld_relaxed_u64(mb);
      while ((unsigned)(v >> 32) != epoch_l) {
        __nanosleep(16);
        v = ld_relaxed_u64(mb);
      }
      reinterpret_cast<unsigned*>(xs)[tid] = (unsigned)v;
      __syncthreads();
      if (hh == 0 && row0 + row < size && nrhs > 0) acc1 = xs[row];
      __syncthreads();  // xs is rewritten by the first dependency's poll
    } else if (!MMA) {
      if (hh == 0 && row0 + row < size && nrhs > 0) acc1 = x[off + row0 + row];
    } else {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int m = 16 * w + 8 * mi + gq;
        if (row0 + m < size)
#pragma unroll
          for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int n = 8 * nj + 2 * tq + e;
              if (n < nrhs) acc[mi][nj][e] = x[off + row0 + m + n * ld];
            }
      }
    }
  } else {
    for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
      const int r = e % NB, j = e / NB;
      red[r * XLD + j] = (j < nrhs && row0 + r < size) ? x[off + row0 + r + j * ld] : 0.0;
    }
  }

  // multi-RHS sweeps: x_s of the NEXT dependency is loaded into registers while the chunks
  // of the current one run (when its ready flag is already up -- always, except for the last
  // few dependencies), so the 128 x NR load from L2 leaves the per-dependency critical path
  constexpr int XPT = (MMA && !LLM) ? NB * NR / SOLVE_THREADS : 1;
  static_assert(!MMA || (NB * NR) % SOLVE_THREADS == 0, "x prefetch split");
  double xpre[XPT];
  bool have_pre = false;
  int* s_ready = s_tk;  // the ticket slot is free once every thread has read it
  for (int q = 0; q < Q; ++q) {
    const int d = q / NCH, sub = q % NCH, st = q % STAGES;
    const bool diag = (d == ndeps);
    if (sub == 0) {
      if (!diag) {
        const int s = s0 + d * sstep;
        if (d == ndeps - 1) STRACE(1);
        if (!LLM && MMA) {
          if (have_pre) {
#pragma unroll
            for (int i = 0; i < XPT; ++i) {
              const int e = tid + i * SOLVE_THREADS;
              xs[(e % NB) * XLD + e / NB] = xpre[i];
            }
          } else {
            if (tid == 0) {
              const unsigned* f = flags + g.fbase[p] + s;
              while (ld_acquire_u32(f) != epoch) __nanosleep(32);
            }
            __syncthreads();
            const int64_t srow0 = (int64_t)s * NB;
            for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
              const int r = e % NB, j = e / NB;
              xs[r * XLD + j] = (j < nrhs && srow0 + r < size) ? __ldcg(x + off + srow0 + r + j * ld) : 0.0;
            }
          }
          if (tid == 0)
            *s_ready = d + 1 < ndeps && ld_acquire_u32(flags + g.fbase[p] + s + sstep) == epoch;
          __syncthreads();
          have_pre = *s_ready != 0;
          if (have_pre) {
            const int64_t srow0 = (int64_t)(s + sstep) * NB;
#pragma unroll
            for (int i = 0; i < XPT; ++i) {
              const int e = tid + i * SOLVE_THREADS;
              const int r = e % NB, j = e / NB;
              xpre[i] = (j < nrhs && srow0 + r < size) ? __ldcg(x + off + srow0 + r + j * ld) : 0.0;
            }
          }
        } else if (LLM) {
          const unsigned long long* mb = mbox + (size_t)(g.fbase[p] + s) * (2 * NB) + tid;
          unsigned long long v = ld_relaxed_u64(mb);
          while ((unsigned)(v >> 32) != epoch) {
            __nanosleep(16);
            v = ld_relaxed_u64(mb);
          }
          reinterpret_cast<unsigned*>(xs)[tid] = (unsigned)v;
          if (d == ndeps - 1) STRACE(2);
        } else {
          if (tid == 0) {
            const unsigned* f = flags + g.fbase[p] + s;
            while (ld_acquire_u32(f) != epoch) __nanosleep(32);
          }
          __syncthreads();
          const int64_t srow0 = (int64_t)s * NB;
          for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
            const int r = e % NB, j = e / NB;
            xs[r * XLD + j] = (j < nrhs && srow0 + r < size) ? __ldcg(x + off + srow0 + r + j * ld) : 0.0;
          }
        }
      } else {
        // diagonal step: the accumulated right-hand side becomes the product input
        if (!TRANS) {
          if (!MMA) {
            if (hh == 1) red[row] = acc1;
            if (DPK) cp_async_wait<0>();
            __syncthreads();
            if (hh == 0) xs[row] = acc1 + red[row];
            acc1 = 0.0;
          } else {
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
              for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  xs[(16 * w + 8 * mi + gq) * XLD + 8 * nj + 2 * tq + e] = acc[mi][nj][e];
                  acc[mi][nj][e] = 0.0;
                }
          }
        } else {
          __syncthreads();
          for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
            const int r = e % NB, j = e / NB;
            xs[r * XLD + j] = red[r * XLD + j];
            red[r * XLD + j] = 0.0;
          }
        }
      }
      __syncthreads();
    }
    if (diag && sub == 0) STRACE(3);
    if (DPK && diag) {
      // the whole diagonal product from the resident triangle; columns split by parity
      // between the two row halves, two independent chains per thread
      double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
      for (int c = hh; c < NB; c += 4) {
        const int c2 = c + 2;
        const bool u0 = MODE == 0 ? row > c : row <= c, u1 = MODE == 0 ? row > c2 : row <= c2;
        if (u0) a0 = fma(dreg[dpk_col<MODE>(c) + row], xs[c], a0);
        if (u1) a1 = fma(dreg[dpk_col<MODE>(c2) + row], xs[c2], a1);
      }
      acc1 = a0 + a1;
      STRACE(4);
      break;
    }
    mbar_wait(&bars[st], (unsigned)((q / STAGES) & 1));
    const double* ch = ring + (size_t)st * CH_SM;
    const float* chf = reinterpret_cast<const float*>(ch);
    const bool f32 = t32 != nullptr && !diag;
    const int cbase = sub * CH_COLS;
    if (!TRANS && !MMA && f32) {
      // four independent partial sums per chunk: the FP32 chunk carries half the bytes of
      // an FP64 one, and a single 16-step dependent FMA chain per chunk (as the FP64 branch
      // below keeps, for its bitwise guarantees) would bound the sweep below the HBM rate
      double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
#pragma unroll
      for (int c4 = 0; c4 < 16; c4 += 4) {
        const int cc = hh * 16 + c4;
        b0 = fma(-(double)chf[cc * NB + row], xs[cbase + cc], b0);
        b1 = fma(-(double)chf[(cc + 1) * NB + row], xs[cbase + cc + 1], b1);
        b2 = fma(-(double)chf[(cc + 2) * NB + row], xs[cbase + cc + 2], b2);
        b3 = fma(-(double)chf[(cc + 3) * NB + row], xs[cbase + cc + 3], b3);
      }
      acc1 += (b0 + b1) + (b2 + b3);
    } else if (!TRANS && !MMA) {
      // out[row] (+|-)= sum_c Tile[row][c] xs[c], half the chunk columns per thread
#if LRS_SOLVE_FMA_ACC > 1
      // NA partial sums per chunk: a single 16-step dependent FMA chain per chunk held the
      // sweep ~5% under the HBM rate (and more under a power cap: the chain scales with the
      // SM clock).  Fixed order: column cc goes to partial cc mod NA, the partials are summed
      // as a balanced tree and added to the running sum once per chunk.
      constexpr int NA = LRS_SOLVE_FMA_ACC;
      static_assert(NA == 2 || NA == 4 || NA == 8 || NA == 16, "partial sums per chunk");
      double b[NA];
#pragma unroll
      for (int e = 0; e < NA; ++e) b[e] = 0.0;
#pragma unroll
      for (int c4 = 0; c4 < 16; c4 += NA)
#pragma unroll
        for (int e = 0; e < NA; ++e) {
          const int cc = hh * 16 + c4 + e, c = cbase + cc;
          double v = ch[cc * CLD + row];
          if (diag) v = (MODE == 0) ? (row > c ? v : 0.0) : (row <= c ? v : 0.0);
          else v = -v;
          b[e] = fma(v, xs[c], b[e]);
        }
#pragma unroll
      for (int w2 = NA / 2; w2 >= 1; w2 >>= 1)
#pragma unroll
        for (int e = 0; e < w2; ++e) b[e] += b[e + w2];
      acc1 += b[0];
#else
#pragma unroll 4
      for (int cc = hh * 16; cc < hh * 16 + 16; ++cc) {
        const int c = cbase + cc;
        double v = ch[cc * CLD + row];
        if (diag) v = (MODE == 0) ? (row > c ? v : 0.0) : (row <= c ? v : 0.0);
        else v = -v;
        acc1 = fma(v, xs[c], acc1);
      }
#endif
    } else if (!TRANS) {
      // (128 x 32) x (32 x NR) on DMMA: A = chunk (row-major view ch[k*CLD + m]), B = xs rows
#pragma unroll
      for (int k4 = 0; k4 < CH_COLS / 4; ++k4) {
        const int k = 4 * k4 + tq, kg = cbase + k;
        double a[2], b[NJ];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const int m = 16 * w + 8 * mi + gq;
          double v = f32 ? (double)chf[k * NB + m] : ch[k * CLD + m];
          if (diag) v = (MODE == 0) ? (m > kg ? v : 0.0) : (m <= kg ? v : 0.0);
          else v = -v;
          a[mi] = v;
        }
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) b[nj] = xs[kg * XLD + 8 * nj + gq];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < NJ; ++nj) dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
      }
    } else if (!MMA) {
      // transposed, one RHS: out[c] (+|-)= sum_r Tile[r][c] xs[r]; 8 lanes per column
      const int cl = 4 * w + (lane >> 3), rg = lane & 7;
      const int c = cbase + cl;
      double part = 0.0;
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const int r = rg + 8 * i;
        double v = ch[cl * CLD + r];
        if (diag) v = (MODE == 2) ? (r <= c ? v : 0.0) : (r > c ? v : 0.0);
        part = fma(v, xs[r], part);
      }
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      part += __shfl_xor_sync(0xffffffffu, part, 4);
      if (rg == 0) red[c] += diag ? part : -part;
    } else {
      // transposed: out(32 x NR) (+|-)= Tile^T (32 x 128) xs (128 x NR) on DMMA.
      // Warp w takes K-quarter kq = w & 3 (32 tile rows) of half the 4 x NJ output tiles,
      // so each warp runs 4 NJ / 2 independent accumulator chains of 8 DMMAs; the four
      // K-quarter partials are then summed in fixed order (the same for every NR, so
      // multi-column stays bit-identical to column-by-column).
      constexpr int PLD = Cfg::PLD;
      constexpr int TPH = 2 * NJ;  // output tiles per warp
      const int kq = w & 3, th = w >> 2;
      double cacc[TPH][2];
#pragma unroll
      for (int u = 0; u < TPH; ++u) cacc[u][0] = cacc[u][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < CH_COLS / 4; ++k4) {
        const int r = 32 * kq + 4 * k4 + tq;
#pragma unroll
        for (int u = 0; u < TPH; ++u) {
          const int ti = th * TPH + u;
          const int mi = ti & 3, nj = ti >> 2;
          const int mloc = 8 * mi + gq;  // chunk-local output column
          double a = ch[mloc * CLD + r];
          if (diag) a = (MODE == 2) ? (r <= cbase + mloc ? a : 0.0) : (r > cbase + mloc ? a : 0.0);
          dmma_8x8x4(cacc[u][0], cacc[u][1], a, xs[r * XLD + 8 * nj + gq]);
        }
      }
#pragma unroll
      for (int u = 0; u < TPH; ++u) {
        const int ti = th * TPH + u;
        const int mi = ti & 3, nj = ti >> 2;
        // fragment (m = 8 mi + gq, n = 8 nj + 2 tq + e) is owned by exactly this lane
        double* pp = part + (kq * CH_COLS + 8 * mi + gq) * PLD + 8 * nj + 2 * tq;
        pp[0] = cacc[u][0];
        pp[1] = cacc[u][1];
      }
      __syncthreads();
      for (int e = tid; e < CH_COLS * NR; e += SOLVE_THREADS) {
        const int mm = e / NR, nn = e % NR;
        const double v = ((part[mm * PLD + nn] + part[(CH_COLS + mm) * PLD + nn]) +
                          part[(2 * CH_COLS + mm) * PLD + nn]) +
                         part[(3 * CH_COLS + mm) * PLD + nn];
        double* rp = red + (cbase + mm) * XLD + nn;
        *rp = diag ? *rp + v : *rp - v;
      }
    }
    __syncthreads();
    if (tid == 0 && q + STAGES < Qring) issue(q + STAGES, st);
  }
  // ---- write x_t and publish -----------------------------------------------------------
  if (!TRANS && !MMA) {
    if (hh == 1) red[row] = acc1;
    __syncthreads();
    if (hh == 0) {
      double v = 0.0;
      if (row0 + row < size && nrhs > 0) {
        v = acc1 + red[row];
        if (MODE == 0) v += xs[row];  // unit diagonal of inv(L)
      }
      if (LLM) {
        const unsigned long long tag = (unsigned long long)epoch << 32;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
        unsigned long long* mb = mbox + (size_t)(g.fbase[p] + t) * (2 * NB) + 2 * row;
        st_relaxed_u64(mb, tag | (bits & 0xffffffffull));
        st_relaxed_u64(mb + 1, tag | (bits >> 32));
      }
      if (row0 + row < size && nrhs > 0) x[off + row0 + row] = v;
    }
    if (LLM) {
      STRACE(5);
#ifdef LRS_SOLVE_TRACE
      if (g_strace && tid == 0) g_strace[(size_t)tk0 * 8 + 6] = ((unsigned long long)p << 32) | t;
#endif
      return;
    }
  } else if (!TRANS) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int m = 16 * w + 8 * mi + gq;
      if (row0 + m >= size) continue;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = 8 * nj + 2 * tq + e;
          if (n >= nrhs) continue;
          double v = acc[mi][nj][e];
          if (MODE == 0) v += xs[m * XLD + n];
          x[off + row0 + m + n * ld] = v;
        }
    }
  } else {
    for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
      const int r = e % NB, j = e / NB;
      if (j < nrhs && row0 + r < size) {
        double v = red[r * XLD + j];
        if (MODE == 3) v += xs[r * XLD + j];
        x[off + row0 + r + j * ld] = v;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release_u32(flags + g.fbase[p] + t, epoch);
  STRACE(5);
#ifdef LRS_SOLVE_TRACE
  if (g_strace && tid == 0) {
    g_strace[(size_t)tk0 * 8 + 6] = ((unsigned long long)p << 32) | t;
    g_strace[(size_t)tk0 * 8 + 7] = grp;
  }
#endif
}

template <int MODE, int NR>
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    band_solve_kernel(BandGeom g, const double* __restrict__ tiles, double* x, int64_t ld,
                      int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only,
                      int ngroups, int64_t flag_stride, const float* __restrict__ t32,
                      unsigned long long* mbox) {
  extern __shared__ __align__(128) unsigned char smraw[];
  int* s_tk = solve_ticket_slot<MODE, NR>(smraw);
  if (threadIdx.x == 0) *s_tk = atomicAdd(ticket, 1);
  __syncthreads();
  const int tk0 = *s_tk;
  band_solve_body<MODE, NR>(g, tiles, x, ld, nrhs, flags, epoch, p_only, ngroups, flag_stride,
                            t32, mbox, tk0, 0u);
}

// The one-RHS apply's L and U sweeps in ONE launch: tickets [0, ntiles) are the L sweep's
// CTAs, [ntiles, 2 ntiles) the U sweep's.  Every wait targets a CTA with a smaller ticket
// (an L CTA, or an earlier U tile), which has started, so there is no deadlock for any
// residency; the SMs stream the U sweep's factor panels while the L sweep drains instead of
// idling across a kernel boundary.
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    band_solve_lu1_kernel(BandGeom g, const double* __restrict__ tiles, double* x, int64_t ld,
                          int nrhs, unsigned epoch_l, unsigned epoch_u, int* ticket, int ntiles,
                          const float* __restrict__ t32, unsigned long long* mbox) {
  extern __shared__ __align__(128) unsigned char smraw[];
  static_assert(solve_smem_bytes<0, 1>() == solve_smem_bytes<1, 1>(), "one shared-memory plan");
  int* s_tk = solve_ticket_slot<0, 1>(smraw);
  if (threadIdx.x == 0) *s_tk = atomicAdd(ticket, 1);
  __syncthreads();
  const int tk0 = *s_tk;
  if (tk0 < ntiles)
    band_solve_body<0, 1>(g, tiles, x, ld, nrhs, nullptr, epoch_l, -1, 1, 0, t32, mbox, tk0, 0u);
  else
    band_solve_body<1, 1, true>(g, tiles, x, ld, nrhs, nullptr, epoch_u, -1, 1, 0, t32, mbox,
                                tk0 - ntiles, epoch_l);
}

void launch_band_solve_lu1(Ctx* c, const BandGeom& g, const double* tiles, double* x,
                           int64_t ld, unsigned epoch_l, unsigned epoch_u, int* ticket,
                           int ntiles, const float* t32, unsigned long long* mb) {
  if (ntiles == 0) return;
  static bool attr = false;
  constexpr size_t smem = solve_smem_bytes<0, 1>();
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(band_solve_lu1_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  LRS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), c->stream));
  ProfScope ps_(c, K_SOLVE);
  band_solve_lu1_kernel<<<2 * ntiles, SOLVE_THREADS, smem, c->stream>>>(
      g, tiles, x, ld, 1, epoch_l, epoch_u, ticket, ntiles, t32, mb);
  LRS_LAUNCHED(c);
}

template <int MODE, int NR>
static void launch_mode(Ctx* c, const BandGeom& g, const double* tiles, double* x, int64_t ld,
                        int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only,
                        int ntiles, int64_t flag_stride, const float* t32,
                        unsigned long long* mbox) {
  const int ngroups = (nrhs + NR - 1) / NR;
  static bool attr = false;
  const size_t smem = solve_smem_bytes<MODE, NR>();
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(band_solve_kernel<MODE, NR>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ProfScope ps_(c, c->in_setup ? K_SPIKE_SOLVE : (MODE >= 2 ? K_SOLVE_ADJ : K_SOLVE));
#ifdef LRS_SOLVE_TRACE
  static int launches = 0;
  unsigned long long* tb = nullptr;
  // LRS_STRACE_NR selects the width traced (default 1: the Krylov sweeps; 16: the spike
  // solves, traced from their first launch)
  const char* tnr = std::getenv("LRS_STRACE_NR");
  const int want = tnr ? std::atoi(tnr) : 1;
  const bool tr = NR == want && std::getenv("LRS_STRACE") &&
                  (want == 1 ? (MODE <= 1 && ++launches >= 40 && launches < 44) : ++launches <= 4);
  if (tr) {
    LRS_CUDA(cudaStreamSynchronize(c->stream));
    LRS_CUDA(cudaMalloc(&tb, (size_t)ntiles * ngroups * 8 * 8));
    LRS_CUDA(cudaMemset(tb, 0, (size_t)ntiles * ngroups * 8 * 8));
    LRS_CUDA(cudaMemcpyToSymbol(g_strace, &tb, sizeof(tb)));
  }
#endif
  band_solve_kernel<MODE, NR><<<ntiles * ngroups, SOLVE_THREADS, smem, c->stream>>>(
      g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ngroups, flag_stride,
      MODE <= 1 ? t32 : nullptr, mbox);
  LRS_LAUNCHED(c);
#ifdef LRS_SOLVE_TRACE
  if (tr) {
    LRS_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<unsigned long long> h((size_t)ntiles * ngroups * 8);
    LRS_CUDA(cudaMemcpy(h.data(), tb, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long* z = nullptr;
    LRS_CUDA(cudaMemcpyToSymbol(g_strace, &z, sizeof(z)));
    LRS_CUDA(cudaFree(tb));
    FILE* f = std::fopen(std::getenv("LRS_STRACE"), "ab");
    const int hdr[2] = {MODE, ntiles * ngroups};
    std::fwrite(hdr, sizeof(int), 2, f);
    std::fwrite(h.data(), 8, h.size(), f);
    std::fclose(f);
  }
#endif
}

// 17..48 columns (the spike blocks) run as ONE 48-column group: each row tile's factor
// chunks are streamed once for all columns and the chains have 3x fewer CTAs in flight to
// share the SMs with (16-column groups read every tile three times through L2)
#ifndef LRS_SOLVE_NR48
#define LRS_SOLVE_NR48 1
#endif
#ifndef LRS_SOLVE_NR48_TRANS
#define LRS_SOLVE_NR48_TRANS 1
#endif
template <int MODE>
static void launch_nr(Ctx* c, const BandGeom& g, const double* tiles, double* x, int64_t ld,
                      int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only,
                      int ntiles, int64_t fs, const float* t32, unsigned long long* mb) {
  // every width runs the same DMMA code (one n8 tile for <= 8 columns, 16-column groups
  // beyond 16), so each column's arithmetic is independent of the batch: multi-column ==
  // column-by-column bit-exactly
  if (nrhs <= 1 && c->solve_fma1)
    launch_mode<MODE, 1>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb);
  else if (nrhs <= 8)
    launch_mode<MODE, 8>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb);
  else if (nrhs <= 16 || (MODE >= 2 && !LRS_SOLVE_NR48_TRANS) || !LRS_SOLVE_NR48)
    launch_mode<MODE, 16>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb);
  else
    launch_mode<MODE, 48>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb);
}

void launch_band_solve(Ctx* c, const BandGeom& g, const double* tiles, int mode, double* x,
                       int64_t ld, int nrhs, unsigned* flags, unsigned epoch, int* ticket,
                       int p_only, int ntiles, int64_t fs, const float* t32,
                       unsigned long long* mb) {
  if (ntiles == 0 || nrhs == 0) return;
  if (nrhs > SOLVE_MAX_RHS) throw LrsError(LRS_ERR_PARAMETER, "band solve batch > 48 columns");
  LRS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), c->stream));
  switch (mode) {
    case 0: launch_nr<0>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb); break;
    case 1: launch_nr<1>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb); break;
    case 2: launch_nr<2>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb); break;
    default: launch_nr<3>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs, t32, mb); break;
  }
}

__global__ void __launch_bounds__(256) tiles_to_fp32_kernel(const double* __restrict__ t,
                                                            float* __restrict__ t32,
                                                            const int* __restrict__ idx,
                                                            int64_t nslots) {
  for (int64_t s = blockIdx.x; s < nslots; s += gridDim.x) {
    const int ci = idx[s];
    if (ci < 0) continue;
    const double2* src = reinterpret_cast<const double2*>(t + s * TILE_ELEMS);
    float2* dst = reinterpret_cast<float2*>(t32 + (int64_t)ci * TILE_ELEMS);
    for (int e = threadIdx.x; e < TILE_ELEMS / 2; e += 256) {
      const double2 v = src[e];
      dst[e] = make_float2((float)v.x, (float)v.y);
    }
  }
}

void launch_tiles_to_fp32(Ctx* c, const double* tiles, float* t32, const int* idx,
                          int64_t nslots) {
  if (nslots == 0) return;
  ProfScope ps_(c, K_SETUP);
  tiles_to_fp32_kernel<<<c->num_sms * 16, 256, 0, c->stream>>>(tiles, t32, idx, nslots);
  LRS_LAUNCHED(c);
}

}  // namespace lrs
