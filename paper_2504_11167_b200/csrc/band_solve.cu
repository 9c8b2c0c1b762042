// Dataflow banded triangular solves (K3/K4/K5 of SURVEY.md 2.3): the D-stage
// y_p = A_p^-1 f_p of apply_precond_T / apply_block_jacobi,
// solve_block and solve_block_adjoint.
//
// One CTA per (partition, row tile).  CTAs take tickets in start order, so a
// CTA only ever waits on tiles whose CTAs already started: no deadlock for
// any residency.  Each CTA streams its row panel (wl or wu off-diagonal tiles
// plus the diagonal tile, contiguous in HBM) through a shared-memory ring
// with 1D bulk copies (cp.async.bulk, the TMA engine) *before* its
// dependencies resolve, and only waits on the per-tile ready flag (release /
// acquire at gpu scope, epoch-tagged so flags never need resetting) right
// before it needs x_s.  The diagonal tile holds the explicit inverses of the
// LU diagonal blocks, so the per-tile critical path is a flag round trip plus
// one 128 x 128 mat-vec; the factor stream runs at HBM speed behind it.
//
// Modes: 0  L  forward (unit lower),   1  U  backward,
//        2  U^T forward (adjoint),     3  L^T backward (adjoint).
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

constexpr int SOLVE_THREADS = 256;
constexpr int CH_COLS = 32;
constexpr int CH_ELEMS = NB * CH_COLS;  // 32 KB chunk = 32 tile columns
constexpr int NCH = NB / CH_COLS;
constexpr int STAGES = 5;

template <int NR>
constexpr size_t solve_smem_bytes() {
  return sizeof(double) * ((size_t)STAGES * CH_ELEMS + 2 * (size_t)NB * NR) + 64 + 16 * STAGES;
}

template <int MODE, int NR>
__global__ void __launch_bounds__(SOLVE_THREADS, 1)
    band_solve_kernel(BandGeom g, const double* __restrict__ tiles, double* x, int64_t ld,
                      int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);
  double* xs = ring + (size_t)STAGES * CH_ELEMS;  // [NB][NR]
  double* red = xs + NB * NR;                     // [NB][NR]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + NB * NR);
  int* s_tk = reinterpret_cast<int*>(bars + STAGES);

  const int tid = threadIdx.x;
  if (tid == 0) *s_tk = atomicAdd(ticket, 1);
  __syncthreads();
  const int tk = *s_tk;
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
  constexpr bool FWD = (MODE == 0 || MODE == 2);
  constexpr bool TRANS = (MODE >= 2);
  const int t = FWD ? tt : T - 1 - tt;
  const int64_t base = g.tbase[p], off = g.off[p], size = g.size[p];
  const int W = g.W, wl = g.wl;
  // dependency range
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
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
    for (int q = 0; q < STAGES && q < Q; ++q) {
      mbar_expect_tx(&bars[q], CH_ELEMS * sizeof(double));
      bulk_g2s(ring + (size_t)q * CH_ELEMS, tile_ptr(q / NCH) + (q % NCH) * CH_ELEMS,
               CH_ELEMS * sizeof(double), &bars[q]);
    }
  }
  const int row = tid & (NB - 1), hh = tid >> 7;
  const int64_t row0 = (int64_t)t * NB;
  const bool row_valid = row0 + row < size;
  double acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.0;
  if (!TRANS) {
    if (hh == 0 && row_valid) {
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (j < nrhs) acc[j] = x[off + row0 + row + j * ld];
    }
  } else {
    for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
      const int r = e / NR, j = e % NR;
      red[e] = (j < nrhs && row0 + r < size) ? x[off + row0 + r + j * ld] : 0.0;
    }
  }
  __syncthreads();

  const int lane = tid & 31, w = tid >> 5;
  for (int q = 0; q < Q; ++q) {
    const int d = q / NCH, sub = q % NCH, st = q % STAGES;
    if (sub == 0) {
      if (d < ndeps) {
        const int s = s0 + d * sstep;
        if (tid == 0) {
          const unsigned* f = flags + g.fbase[p] + s;
          while (ld_acquire_u32(f) != epoch) __nanosleep(32);
        }
        __syncthreads();
        const int64_t srow0 = (int64_t)s * NB;
        for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
          const int r = e / NR, j = e % NR;
          xs[e] = (j < nrhs && srow0 + r < size) ? __ldcg(x + off + srow0 + r + j * ld) : 0.0;
        }
      } else {
        // diagonal step: the accumulated right-hand side becomes the GEMV input
        if (!TRANS) {
          if (hh == 1) {
#pragma unroll
            for (int j = 0; j < NR; ++j) red[row * NR + j] = acc[j];
          }
          __syncthreads();
          if (hh == 0) {
#pragma unroll
            for (int j = 0; j < NR; ++j) xs[row * NR + j] = acc[j] + red[row * NR + j];
          }
#pragma unroll
          for (int j = 0; j < NR; ++j) acc[j] = 0.0;
        } else {
          for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
            xs[e] = red[e];
            red[e] = 0.0;
          }
        }
      }
      __syncthreads();
    }
    mbar_wait(&bars[st], (unsigned)((q / STAGES) & 1));
    const double* ch = ring + (size_t)st * CH_ELEMS;
    const int cbase = sub * CH_COLS;
    const bool diag = (d == ndeps);
    if (!TRANS) {
#pragma unroll 4
      for (int cc = hh * 16; cc < hh * 16 + 16; ++cc) {
        const int c = cbase + cc;
        double v = ch[cc * NB + row];
        if (diag) {
          if (MODE == 0) v = (row > c) ? v : 0.0;   // strictly lower part of inv(L)
          else v = (row <= c) ? v : 0.0;             // upper part of inv(U)
        } else {
          v = -v;
        }
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[j] = fma(v, xs[c * NR + j], acc[j]);
      }
    } else {
      const int cl = 4 * w + (lane >> 3), rg = lane & 7;
      const int c = cbase + cl;
      double part[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) part[j] = 0.0;
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const int r = rg + 8 * i;
        double v = ch[cl * NB + r];
        if (diag) {
          if (MODE == 2) v = (r <= c) ? v : 0.0;    // inv(U)^T
          else v = (r > c) ? v : 0.0;               // strictly lower of inv(L), transposed
        }
#pragma unroll
        for (int j = 0; j < NR; ++j) part[j] = fma(v, xs[r * NR + j], part[j]);
      }
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        double v = part[j];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        part[j] = v;
      }
      if (rg == 0) {
#pragma unroll
        for (int j = 0; j < NR; ++j) red[c * NR + j] += diag ? part[j] : -part[j];
      }
    }
    __syncthreads();
    if (tid == 0 && q + STAGES < Q) {
      const int qn = q + STAGES;
      mbar_expect_tx(&bars[st], CH_ELEMS * sizeof(double));
      bulk_g2s(ring + (size_t)st * CH_ELEMS, tile_ptr(qn / NCH) + (qn % NCH) * CH_ELEMS,
               CH_ELEMS * sizeof(double), &bars[st]);
    }
  }
  // ---- write x_t and publish -----------------------------------------------------------
  if (!TRANS) {
    if (hh == 1) {
#pragma unroll
      for (int j = 0; j < NR; ++j) red[row * NR + j] = acc[j];
    }
    __syncthreads();
    if (hh == 0 && row_valid) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j >= nrhs) break;
        double v = acc[j] + red[row * NR + j];
        if (MODE == 0) v += xs[row * NR + j];  // unit diagonal of inv(L)
        x[off + row0 + row + j * ld] = v;
      }
    }
  } else {
    for (int e = tid; e < NB * NR; e += SOLVE_THREADS) {
      const int r = e / NR, j = e % NR;
      if (j < nrhs && row0 + r < size) {
        double v = red[e];
        if (MODE == 3) v += xs[e];
        x[off + row0 + r + j * ld] = v;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release_u32(flags + g.fbase[p] + t, epoch);
}

template <int MODE, int NR>
static void launch_mode(Ctx* c, const BandGeom& g, const double* tiles, double* x, int64_t ld,
                        int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only,
                        int ntiles) {
  static bool attr = false;
  const size_t smem = solve_smem_bytes<NR>();
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(band_solve_kernel<MODE, NR>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  ProfScope ps_(c, c->in_setup ? K_SPIKE_SOLVE : (MODE >= 2 ? K_SOLVE_ADJ : K_SOLVE));
  band_solve_kernel<MODE, NR><<<ntiles, SOLVE_THREADS, smem, c->stream>>>(
      g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only);
  LRS_LAUNCHED(c);
}

template <int MODE>
static void launch_nr(Ctx* c, const BandGeom& g, const double* tiles, double* x, int64_t ld,
                      int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only,
                      int ntiles) {
  if (nrhs <= 1) launch_mode<MODE, 1>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles);
  else if (nrhs <= 4) launch_mode<MODE, 4>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles);
  else launch_mode<MODE, 16>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles);
}

void launch_band_solve(Ctx* c, const BandGeom& g, const double* tiles, int mode, double* x,
                       int64_t ld, int nrhs, unsigned* flags, unsigned epoch, int* ticket,
                       int p_only, int ntiles) {
  if (ntiles == 0 || nrhs == 0) return;
  LRS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), c->stream));
  switch (mode) {
    case 0: launch_nr<0>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles); break;
    case 1: launch_nr<1>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles); break;
    case 2: launch_nr<2>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles); break;
    default: launch_nr<3>(c, g, tiles, x, ld, nrhs, flags, epoch, ticket, p_only, ntiles); break;
  }
}

}  // namespace lrs
