// Complex128 dataflow banded triangular solves (config 5).  Same ticket / flag /
// bulk-copy pipeline as band_solve.cu; chunks are 16 complex tile columns (32 KB) and
// every chunk product runs on DMMA as four real products per complex one.  Modes 2/3
// apply the conjugate transpose (U^H, L^H): the adjoint a complex randomized SVD needs
// (Z = Q^H T  =>  T^H Q = pad(C)^H A^-H Q).  All widths share one code path, so
// multi-column == column-by-column bit-exactly.
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

constexpr int ZS_THREADS = 256;
constexpr int ZCH_COLS = 16;
constexpr int ZCH_SM = ZCH_COLS * NB;  // complex elements per chunk
constexpr int ZNCH = NB / ZCH_COLS;    // 8 chunks per tile
// Ring depth 3 (per SM a 32 KB chunk is ~0.75 us of HBM and ~0.8 us of DMMA work in the c5
// apply).  The forward sweeps do not hold the adjoint's transposed accumulator and partials,
// so they could keep 5 chunks in flight: measured 1.8% slower on c5 (shift 0 solve 51.4 s vs
// 50.5 s; ncu: DMMA pipe 57%, the sweeps are bound by the DMMA issue, not the stream).
template <int MODE>
constexpr int zstages() { return 3; }

template <int NR>
constexpr int zpart_elems() { return 4 * ZCH_COLS * (NR + 1); }  // adjoint K-quarter partials

template <int MODE, int NR>
constexpr size_t zsolve_smem_bytes() {
  constexpr bool TRANS = MODE >= 2;
  return sizeof(zc) * ((size_t)zstages<MODE>() * ZCH_SM + (TRANS ? 2 : 1) * (size_t)NB * (NR + 4) +
                       (TRANS ? zpart_elems<NR>() : 0)) +
         16 * zstages<MODE>() + 64;
}

#ifndef LRS_ZSOLVE_3M
#define LRS_ZSOLVE_3M 1
#endif
// (base_r + p1 - p2, base_i + p3 - p1 - p2)
__device__ __forceinline__ zc zacc(double br, double bi, double q1, double q2, double q3) {
  return {br + (q1 - q2), bi + (q3 - (q1 + q2))};
}

// TH threads: the forward 16-column sweeps (the c5 apply) run 16 warps -- 8 row groups x 2
// column groups of 8 -- for twice the warps to hide the DMMA latency; the rest 8 warps.
template <int MODE, int NR, int TH = ZS_THREADS>
__global__ void __launch_bounds__(TH, 1)
    band_solve_z_kernel(BandGeom g, const zc* __restrict__ tiles, zc* x, int64_t ld, int nrhs,
                        unsigned* flags, unsigned epoch, int* ticket, int p_only, int ngroups,
                        int64_t flag_stride) {
  constexpr int XLD = NR + 4;
  constexpr bool FWD = (MODE == 0 || MODE == 2);
  constexpr bool TRANS = (MODE >= 2);
  constexpr int NJ = NR / 8;
  constexpr int CG = TRANS ? 1 : TH / 256;  // column groups of warps (forward only)
  constexpr int NJW = NJ / CG;              // n8 tiles per warp
  static_assert(!TRANS || TH == ZS_THREADS, "adjoint sweeps: 8 warps");
  static_assert(NJ % CG == 0 && TH % 256 == 0, "warp split");
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int ZSTAGES = zstages<MODE>();
  zc* ring = reinterpret_cast<zc*>(smraw);
  zc* xs = ring + (size_t)ZSTAGES * ZCH_SM;
  zc* red = xs + NB * XLD;    // adjoint only
  zc* part = red + (TRANS ? NB * XLD : 0);  // [4][ZCH_COLS][NR + 1]: adjoint K-quarter partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(part + (TRANS ? zpart_elems<NR>() : 0));
  int* s_tk = reinterpret_cast<int*>(bars + ZSTAGES);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = TRANS ? w : (w & 7), NJ0 = TRANS ? 0 : (w >> 3) * NJW;  // forward: rows, n8 base
  if (tid == 0) *s_tk = atomicAdd(ticket, 1);
  __syncthreads();
  const int tk0 = *s_tk;
  // 16-column group (as in band_solve.cu)
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
  auto tile_ptr = [&](int d) -> const zc* {
    if (d == ndeps) return tiles + (base + (int64_t)t * W + wl) * TILE_ELEMS;
    const int s = s0 + d * sstep;
    if (!TRANS) return tiles + (base + (int64_t)t * W + (s - t + wl)) * TILE_ELEMS;
    return tiles + (base + (int64_t)s * W + (t - s + wl)) * TILE_ELEMS;
  };
  const int Q = (ndeps + 1) * ZNCH;
  auto issue = [&](int q, int st) {
    const zc* src = tile_ptr(q / ZNCH) + (size_t)(q % ZNCH) * ZCH_SM;
    mbar_expect_tx(&bars[st], ZCH_SM * sizeof(zc));
    bulk_g2s(ring + (size_t)st * ZCH_SM, src, ZCH_SM * sizeof(zc), &bars[st]);
  };
  if (tid == 0) {
    for (int st = 0; st < ZSTAGES; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < ZSTAGES && q < Q; ++q) issue(q, q);
  const int64_t row0 = (int64_t)t * NB;
  const int gq = lane >> 2, tq = lane & 3;
  double accr[2][NJW][2], acci[2][NJW][2];
  // forward products in the 3M form (LRS_ZSOLVE_3M): p1 = sum ar br, p2 = sum ai bi,
  // p3 = sum (ar + ai)(br + bi); re = p1 - p2, im = p3 - p1 - p2 (three DMMAs per complex
  // product instead of four); accr / acci carry the right-hand side
  double p1[2][NJW][2], p2[2][NJW][2], p3[2][NJW][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJW; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) p1[mi][nj][e] = p2[mi][nj][e] = p3[mi][nj][e] = 0.0;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < NJW; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) accr[mi][nj][e] = acci[mi][nj][e] = 0.0;
  if (!TRANS) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int m = 16 * wr + 8 * mi + gq;
      if (row0 + m < size)
#pragma unroll
        for (int nj = 0; nj < NJW; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = 8 * (NJ0 + nj) + 2 * tq + e;
            if (n < nrhs) {
              const zc v = x[off + row0 + m + n * ld];
              accr[mi][nj][e] = v.x;
              acci[mi][nj][e] = v.y;
            }
          }
    }
  } else {
    for (int e = tid; e < NB * NR; e += TH) {
      const int r = e % NB, j = e / NB;
      red[r * XLD + j] = (j < nrhs && row0 + r < size) ? x[off + row0 + r + j * ld] : zc{0.0, 0.0};
    }
  }
  // x_s of the next dependency is loaded into registers while the current one's chunks run
  // (when its flag is already up), as in band_solve_kernel
  constexpr int XPT = NB * NR / TH;
  static_assert((NB * NR) % TH == 0, "x prefetch split");
  zc xpre[XPT];
  bool have_pre = false;
  int* s_ready = s_tk;  // free once every thread has read its ticket
  auto load_x = [&](int sdep, int i) -> zc {
    const int e = tid + i * TH;
    const int r = e % NB, j = e / NB;
    const int64_t srow0 = (int64_t)sdep * NB;
    zc v = {0.0, 0.0};
    if (j < nrhs && srow0 + r < size) {
      const double2 raw = __ldcg(reinterpret_cast<const double2*>(x + off + srow0 + r + j * ld));
      v = {raw.x, raw.y};
    }
    return v;
  };
  for (int q = 0; q < Q; ++q) {
    const int d = q / ZNCH, sub = q % ZNCH, st = q % ZSTAGES;
    const bool diag = (d == ndeps);
    if (sub == 0) {
      if (!diag) {
        const int s = s0 + d * sstep;
        if (have_pre) {
#pragma unroll
          for (int i = 0; i < XPT; ++i) {
            const int e = tid + i * TH;
            xs[(e % NB) * XLD + e / NB] = xpre[i];
          }
        } else {
          if (tid == 0) {
            const unsigned* f = flags + g.fbase[p] + s;
            while (ld_acquire_u32(f) != epoch) __nanosleep(32);
          }
          __syncthreads();
#pragma unroll
          for (int i = 0; i < XPT; ++i) {
            const int e = tid + i * TH;
            xs[(e % NB) * XLD + e / NB] = load_x(s, i);
          }
        }
        if (tid == 0)
          *s_ready = d + 1 < ndeps && ld_acquire_u32(flags + g.fbase[p] + s + sstep) == epoch;
        __syncthreads();
        have_pre = *s_ready != 0;
        if (have_pre)
#pragma unroll
          for (int i = 0; i < XPT; ++i) xpre[i] = load_x(s + sstep, i);
      } else {
        if (!TRANS) {
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < NJW; ++nj)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                xs[(16 * wr + 8 * mi + gq) * XLD + 8 * (NJ0 + nj) + 2 * tq + e] = zacc(
                    accr[mi][nj][e], acci[mi][nj][e], p1[mi][nj][e], p2[mi][nj][e], p3[mi][nj][e]);
                accr[mi][nj][e] = acci[mi][nj][e] = 0.0;
                p1[mi][nj][e] = p2[mi][nj][e] = p3[mi][nj][e] = 0.0;
              }
        } else {
          __syncthreads();
          for (int e = tid; e < NB * NR; e += TH) {
            const int r = e % NB, j = e / NB;
            xs[r * XLD + j] = red[r * XLD + j];
            red[r * XLD + j] = {0.0, 0.0};
          }
        }
      }
      __syncthreads();
    }
    mbar_wait(&bars[st], (unsigned)((q / ZSTAGES) & 1));
    const zc* ch = ring + (size_t)st * ZCH_SM;
    const int cbase = sub * ZCH_COLS;
    if (!TRANS) {
#pragma unroll
      for (int k4 = 0; k4 < ZCH_COLS / 4; ++k4) {
        const int k = 4 * k4 + tq, kg = cbase + k;
        double ar[2], ai[2], br[NJW], bi[NJW];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const int m = 16 * wr + 8 * mi + gq;
          zc v = ch[k * NB + m];
          if (diag) {
            if (!(MODE == 0 ? m > kg : m <= kg)) v = {0.0, 0.0};
          } else {
            v = {-v.x, -v.y};
          }
          ar[mi] = v.x;
          ai[mi] = v.y;
        }
#pragma unroll
        for (int nj = 0; nj < NJW; ++nj) {
          const zc v = xs[kg * XLD + 8 * (NJ0 + nj) + gq];
          br[nj] = v.x;
          bi[nj] = v.y;
        }
        if (LRS_ZSOLVE_3M) {
          double as[2], bs[NJW];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) as[mi] = ar[mi] + ai[mi];
#pragma unroll
          for (int nj = 0; nj < NJW; ++nj) bs[nj] = br[nj] + bi[nj];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < NJW; ++nj) {
              dmma_8x8x4(p1[mi][nj][0], p1[mi][nj][1], ar[mi], br[nj]);
              dmma_8x8x4(p2[mi][nj][0], p2[mi][nj][1], ai[mi], bi[nj]);
              dmma_8x8x4(p3[mi][nj][0], p3[mi][nj][1], as[mi], bs[nj]);
            }
        } else {
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < NJW; ++nj) {
              dmma_8x8x4(accr[mi][nj][0], accr[mi][nj][1], ar[mi], br[nj]);
              dmma_8x8x4(accr[mi][nj][0], accr[mi][nj][1], -ai[mi], bi[nj]);
              dmma_8x8x4(acci[mi][nj][0], acci[mi][nj][1], ar[mi], bi[nj]);
              dmma_8x8x4(acci[mi][nj][0], acci[mi][nj][1], ai[mi], br[nj]);
            }
        }
      }
    } else {
      // out(16 x NR) (+|-)= conj(Tile)^T (16 x 128) xs (128 x NR).  Warp w takes K-quarter
      // kq = w & 3 (32 tile rows) of half the 2 x NJ output tiles (independent chains);
      // the four partials are summed in fixed order (NR independent: bit-exact columns).
      constexpr int PLD = NR + 1;
      const int kq = w & 3, th = w >> 2;
      double cr[NJ][2], ci[NJ][2], c3[LRS_ZSOLVE_3M ? NJ : 1][2];
#pragma unroll
      for (int u = 0; u < NJ; ++u) cr[u][0] = cr[u][1] = ci[u][0] = ci[u][1] = 0.0;
      if (LRS_ZSOLVE_3M)
#pragma unroll
        for (int u = 0; u < (LRS_ZSOLVE_3M ? NJ : 1); ++u) c3[u][0] = c3[u][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const int r = 32 * kq + 4 * k4 + tq;
#pragma unroll
        for (int u = 0; u < NJ; ++u) {
          const int ti = th * NJ + u;
          const int mi = ti & 1, nj = ti >> 1;
          const int mloc = 8 * mi + gq;
          zc a = ch[mloc * NB + r];
          if (diag && !(MODE == 2 ? r <= cbase + mloc : r > cbase + mloc)) a = {0.0, 0.0};
          const double ar = a.x, ai = -a.y;  // conjugate
          const zc b = xs[r * XLD + 8 * nj + gq];
          if (LRS_ZSOLVE_3M) {  // cr = sum ar br, ci = sum ai bi, c3 = sum (ar + ai)(br + bi)
            const int uu = LRS_ZSOLVE_3M ? u : 0;
            dmma_8x8x4(cr[u][0], cr[u][1], ar, b.x);
            dmma_8x8x4(ci[u][0], ci[u][1], ai, b.y);
            dmma_8x8x4(c3[uu][0], c3[uu][1], ar + ai, b.x + b.y);
          } else {
            dmma_8x8x4(cr[u][0], cr[u][1], ar, b.x);
            dmma_8x8x4(ci[u][0], ci[u][1], ar, b.y);
            dmma_8x8x4(cr[u][0], cr[u][1], -ai, b.y);
            dmma_8x8x4(ci[u][0], ci[u][1], ai, b.x);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < NJ; ++u) {
        const int ti = th * NJ + u;
        const int mi = ti & 1, nj = ti >> 1;
        zc* pp = part + (kq * ZCH_COLS + 8 * mi + gq) * PLD + 8 * nj + 2 * tq;
        if (LRS_ZSOLVE_3M) {
          const int uu = LRS_ZSOLVE_3M ? u : 0;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double q1 = cr[u][e], q2 = ci[u][e], q3 = c3[uu][e];
            pp[e] = {q1 - q2, q3 - (q1 + q2)};
          }
        } else {
          pp[0] = {cr[u][0], ci[u][0]};
          pp[1] = {cr[u][1], ci[u][1]};
        }
      }
      __syncthreads();
      for (int e = tid; e < ZCH_COLS * NR; e += TH) {
        const int mm = e / NR, nn = e % NR;
        const zc v = s_add(s_add(s_add(part[mm * PLD + nn], part[(ZCH_COLS + mm) * PLD + nn]),
                                 part[(2 * ZCH_COLS + mm) * PLD + nn]),
                           part[(3 * ZCH_COLS + mm) * PLD + nn]);
        zc* rp = red + (cbase + mm) * XLD + nn;
        *rp = diag ? s_add(*rp, v) : s_sub(*rp, v);
      }
    }
    __syncthreads();
    if (tid == 0 && q + ZSTAGES < Q) issue(q + ZSTAGES, st);
  }
  if (!TRANS) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int m = 16 * wr + 8 * mi + gq;
      if (row0 + m >= size) continue;
#pragma unroll
      for (int nj = 0; nj < NJW; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = 8 * (NJ0 + nj) + 2 * tq + e;
          if (n >= nrhs) continue;
          zc v = zacc(accr[mi][nj][e], acci[mi][nj][e], p1[mi][nj][e], p2[mi][nj][e], p3[mi][nj][e]);
          if (MODE == 0) v = s_add(v, xs[m * XLD + n]);
          x[off + row0 + m + n * ld] = v;
        }
    }
  } else {
    for (int e = tid; e < NB * NR; e += TH) {
      const int r = e % NB, j = e / NB;
      if (j < nrhs && row0 + r < size) {
        zc v = red[r * XLD + j];
        if (MODE == 3) v = s_add(v, xs[r * XLD + j]);
        x[off + row0 + r + j * ld] = v;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release_u32(flags + g.fbase[p] + t, epoch);
}

#ifndef LRS_ZSOLVE_TH16
#define LRS_ZSOLVE_TH16 256  // 512 (16 warps, 2 column groups): c5 shift 0 solve 63.4 s vs 50.5 s
#endif
template <int MODE, int NR>
static void zlaunch_mode(Ctx* c, const BandGeom& g, const zc* tiles, zc* x, int64_t ld, int nrhs,
                         unsigned* flags, unsigned epoch, int* ticket, int p_only, int ntiles,
                         int64_t fs) {
  constexpr int TH = (MODE < 2 && NR == 16) ? LRS_ZSOLVE_TH16 : ZS_THREADS;
  const int ngroups = (nrhs + NR - 1) / NR;
  static bool attr = false;
  const size_t smem = zsolve_smem_bytes<MODE, NR>();
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(band_solve_z_kernel<MODE, NR, TH>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ProfScope ps_(c, c->in_setup ? K_SPIKE_SOLVE : (MODE >= 2 ? K_SOLVE_ADJ : K_SOLVE));
  band_solve_z_kernel<MODE, NR, TH><<<ntiles * ngroups, TH, smem, c->stream>>>(
      g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ngroups, fs);
  LRS_LAUNCHED(c);
}

template <int MODE>
static void zlaunch_nr(Ctx* c, const BandGeom& g, const zc* tiles, zc* x, int64_t ld, int nrhs,
                       unsigned* flags, unsigned epoch, int* ticket, int p_only, int ntiles,
                       int64_t fs) {
  if (nrhs <= 8)
    zlaunch_mode<MODE, 8>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs);
  else
    zlaunch_mode<MODE, 16>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs);
}

void launch_band_solve_z(Ctx* c, const BandGeom& g, const zc* tiles, int mode, zc* x, int64_t ld,
                         int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only,
                         int ntiles, int64_t fs) {
  if (ntiles == 0 || nrhs == 0) return;
  if (nrhs > ZSOLVE_MAX_RHS) throw LrsError(LRS_ERR_PARAMETER, "complex band solve batch > 96");
  LRS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), c->stream));
  switch (mode) {
    case 0: zlaunch_nr<0>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs); break;
    case 1: zlaunch_nr<1>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs); break;
    case 2: zlaunch_nr<2>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs); break;
    default: zlaunch_nr<3>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles, fs); break;
  }
}

}  // namespace lrs
