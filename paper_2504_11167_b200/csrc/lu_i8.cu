// Integer-sliced FP64 trailing update of the band LU on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, INT8 x INT8 -> INT32 accumulators in TMEM).
//
// The two-step update C -= A B of factorize_block (the rank-256 update
// lu_gemm<3/4> of band_lu.cu computes on DMMA) has A = [L(I,K) L(I,K+1)] (128 x 256) and
// B = [U(K,J); U(K+1,J)] (256 x 128).  B200 runs FP64 at 37 TF/s but INT8 at 4.5 POPS, so the
// product is formed exactly in integers (the Ozaki splitting):
//
//   row i of A:     a_ik = 2^ea_i * sum_{p=1..7} 2^(2-8p) d_p(i,k)
//   column j of B:  b_kj = 2^eb_j * sum_{q=1..7} 2^(2-8q) e_q(k,j)
//   (A B)_ij = 2^(ea_i + eb_j) * sum_{s=2..8} 2^(4-8s) G_s(i,j),   G_s = sum_{p+q=s} D_p E_q
//
// with ea_i the binary exponent of max_k |a_ik| (so |a_ik| 2^-ea_i < 1).  The digits are
// the balanced base-256 expansion of F = round(a_ik 2^(54 - ea_i)) (|F| < 2^54): six low
// digits in [-128, 127] and a top digit in [-65, 65], all INT8.  54 bits represent every
// entry within 2^-1 of its row (column) maximum exactly; balanced digits have random signs,
// so the dropped s >= 9 terms (below 2^-68 of the row x column scale each) and the
// rounding of F average out like FP64's own rounding: both are of the order of the
// k u max|a| max|b| bound of the 256-long FP64 products.  G_s sums <= 7 products of 256
// INT8 pairs: |G_s| <= 7 * 256 * 2^14 < 2^31, exact in INT32.  (The earlier 8 x 7-bit
// sign-magnitude split needed 36 products; this one needs 28.)
//
// lu_i8_slice (once per step pair, on the critical-path stream): exponents and digits of
// the whole A panel (rows I = K+2 .. K+1+wl) and B panel (columns J = K+2 .. K+1+wu),
// written in the UMMA shared-memory operand layout (K-major, no swizzle: 8-row x 16-byte
// core matrices) so one pipeline stage is two contiguous bulk copies.
//
// lu_i8_gemm (kinds 3 / 4 of the pair schedule; the quad schedule, LRS_LU_QUAD=1, runs the
// same kernel with K = 512): a warp-specialised kernel per 128 x 128 output tile.  The MMA
// shape is M=128, N=128, K=32 (N < 128 leaves the INT8 pipe at 2/3 rate: SS-mode operand
// reads); the seven group accumulators do not fit the 4 x 128 TMEM columns, so a tile runs
// two passes over K: pass A forms G_5..G_8 (22 MMAs per K chunk of 32, all 7 + 7 slices),
// pass B G_2..G_4 (6 MMAs, slices 1-3).  The group accumulators take the four TMEM slots as
// a ring (a pass takes the slots after the previous pass's, so pass B starts in the slots
// pass A's drain frees first); two tfull barriers alternate by pass parity.  Warp 0 streams
// the chunks (56 / 24 KB) through a 4-stage TMA ring; warp 1's elected thread issues the
// MMAs, A slice outer so consecutive MMAs reuse it from the operand collector; warps 2-9
// drain each group accumulator into FP64 registers (tcgen05.ld; smallest group first) and
// release it, and after pass B subtract 2^(ea+eb) sum_s 2^(4-8s) G_s from C with L2
// reductions.  Each CTA walks I8_TPC consecutive tiles (same I first, so A slices are shared
// through L2) and retires, leaving SMs for the high-priority diag / panel kernels of the
// look-ahead.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

constexpr int I8_S = 7;                               // digit slices per operand
constexpr int I8_KC = 32;                             // K per MMA and per pipeline chunk
// chunks over K = 128 STEPS (STEPS = 2: the pair update, K = 256; STEPS = 4: K = 512)
__host__ __device__ constexpr int i8_nch(int steps) { return steps * NB / I8_KC; }
constexpr int I8_SL = NB * I8_KC;                     // 4096 B: one A slice of one chunk
constexpr int I8_BLK = I8_S * I8_SL;                  // 28 KB: all A slices of one chunk
// output columns per CTA: 128 (one CTA per SM, all 512 TMEM columns) or 64 (two CTAs per SM
// with 256 columns each, so one CTA's MMAs run while the other drains)
// LRS_I8_ONEPASS=1: 128 x 64 work items with all seven group accumulators resident (7 x 64
// of the 512 TMEM columns, an eighth 64-column slot spare), ONE pass over K -- no slices
// streamed twice, no pass hand-off inside a tile; the slots form a ring of 8, so the next
// item starts in the spare slot and follows the drain of the previous one slot by slot
#ifndef LRS_I8_ONEPASS
#define LRS_I8_ONEPASS 0
#endif
#if LRS_I8_ONEPASS
#undef LRS_I8_TN
#define LRS_I8_TN 64
#undef LRS_I8_NPASS
#define LRS_I8_NPASS 1
#undef LRS_I8_EPC
#define LRS_I8_EPC 32
#ifndef LRS_I8_STAGES
#define LRS_I8_STAGES 5  // 5 x 42 KB
#endif
#endif
#ifndef LRS_I8_TN
#define LRS_I8_TN 128
#endif
constexpr int I8_TN = LRS_I8_TN;
constexpr int I8_NH = NB / I8_TN;                     // column blocks per tile
constexpr int I8_BSL = I8_TN * I8_KC;                 // one B slice of one chunk
constexpr int I8_BBLK = I8_S * I8_BSL;                // all B slices of one chunk
constexpr int I8_STAGE = I8_BLK + I8_BBLK;            // A + B
#ifndef LRS_I8_STAGES
#define LRS_I8_STAGES 4  // 4 x 56 KB + 2 KB barriers fit the 227 KB opt-in limit
#endif
constexpr int I8_STAGES = (I8_TN == 128 || LRS_I8_ONEPASS) ? LRS_I8_STAGES : 2;
constexpr int I8_GROUPS = LRS_I8_ONEPASS ? 8 : 4;     // TMEM accumulator slots (x TN columns)
// Passes over K per tile.  Pass k forms the groups s = top(k), top(k) - 1, .. (ng(k) of them)
// from slices 1..pmax(k).  The group accumulators take the TMEM slots as a ring: a pass
// takes the next ng slots after the previous pass's, so while the epilogue drains one pass
// the next pass already runs in the other slots.  3 passes (G_8,7 | G_6,5 | G_4,3,2) keep the
// tensor pipe busy during the drains at the price of streaming slices 1..5 and 1..3 again;
// 2 passes (G_8..5 | G_4..2) stream less but stall on the drains.  Measured on c2 (ncu launch
// list, 128 launches): 2 passes 96.4 ms, 3 passes 107.8 ms -- the epilogue (drain + C
// reductions, ~21k cycles per tile with 3 passes) becomes the bottleneck; 16 epilogue warps
// of 32 columns instead of 8 of 64 (LRS_I8_EPC=32) do not change that (98.4 / 109.5 ms).
#ifndef LRS_I8_NPASS
#define LRS_I8_NPASS 2  // measured: 3 passes 0.84 ms vs 2 passes 0.75 ms per c2 launch
#endif
constexpr int I8_NP = LRS_I8_NPASS;
static_assert(I8_NP >= 1 && I8_NP <= 3, "pass split");
__host__ __device__ constexpr int i8_top(int k) {
  return I8_NP == 1 ? 8 : I8_NP == 3 ? (k == 0 ? 8 : k == 1 ? 6 : 4) : (k == 0 ? 8 : 4);
}
__host__ __device__ constexpr int i8_ng(int k) {
  return I8_NP == 1 ? 7 : I8_NP == 3 ? (k == 2 ? 3 : 2) : (k == 0 ? 4 : 3);
}
__host__ __device__ constexpr int i8_pmax(int k) { return i8_top(k) - 1 < I8_S ? i8_top(k) - 1 : I8_S; }
constexpr int I8_PRODUCTS = 28;                       // digit-slice products per K chunk
constexpr int I8_TMEM = I8_GROUPS * I8_TN;            // 512 or 256 columns
#ifndef LRS_I8_EPC
#define LRS_I8_EPC 64
#endif
constexpr int I8_EPC = LRS_I8_EPC;                    // columns per epilogue warp (64 or 32)
constexpr int I8_EPI = 4 * I8_TN / I8_EPC;            // epilogue warps
constexpr int I8_THREADS = 32 * (2 + I8_EPI);         // producer, MMA, epilogue warps
#ifndef LRS_I8_TPC
// Round 1 (pairs): 8 tiles, c2 LU median 0.1535 s vs 0.1596 s (4 tiles), 0.161 s (16).  With
// quads a tile takes twice as long, and c2's critical stream waits on the bulk CTAs to retire:
// session 5 (profiles/r02_lu_tpc_sweep.txt) c2 0.166 s and unsteady (8), 0.159 (4), 0.152-0.159
// (2), 0.158 (1), 0.170 (16); c3 0.6835 (8), 0.6826 (4), 0.694 (2); c4 at 0.25 0.259 (any)
#define LRS_I8_TPC 8  // launches of >= 200 tiles per SM; smaller ones take 4 (i8_gemm_launch)
#endif
constexpr int I8_TPC = LRS_I8_TPC;                    // tiles per CTA (bulk)
#ifndef LRS_I8_TPC3
// round 1 (pairs), c2 LU medians: 1 tile 0.156 s, 2: 0.155, 4: 0.155, 8: 0.154 (noise level);
// session 5 (quads), c2: 8 tiles 0.159-0.174 s from run to run, 4: 0.158-0.171, 2: 0.159
// steady, 1: 0.160; c3: 0.6836 (8) / 0.6847 (2)
#define LRS_I8_TPC3 2
#endif
// LRS_I8_LDPIPE=1: the epilogue's TMEM loads are software pipelined against the INT32 -> FP64
// conversion (two 32-column register buffers); 0: load, wait, convert per batch
#ifndef LRS_I8_LDPIPE
#define LRS_I8_LDPIPE 1
#endif
// LRS_I8_CPREFETCH=1: the producer prefetches the tile's C block into L2 when it starts the
// tile's operand loads, ~1.5 tiles before the epilogue's reductions reach it
#ifndef LRS_I8_CPREFETCH
#define LRS_I8_CPREFETCH 1
#endif
#ifndef LRS_I8_SYM_ORDER
#define LRS_I8_SYM_ORDER 0
#endif
// LRS_I8_EXP (timing experiments only, wrong results): 1 skips the epilogue arithmetic,
// 2 also skips the operand copies
#ifndef LRS_I8_EXP
#define LRS_I8_EXP 0
#endif
// LRS_I8_PROBE (development aid): clock64 accounting of the warp roles, printed by a few CTAs
#ifndef LRS_I8_PROBE
#define LRS_I8_PROBE 0
#endif
#ifndef LRS_I8_WARP_ISSUE
#define LRS_I8_WARP_ISSUE 1
#endif
// LRS_I8_EPI64=1: the epilogue sums the group accumulators of a tile as two exact 64-bit
// integers (H_A = sum_{s=5..8} G_s 2^(8(8-s)) < 2^51, H_B = sum_{s=2..4} G_s 2^(8(4-s)) < 2^43:
// one IMAD.WIDE per value while the TMEM slot is held, instead of an FP64 add and FMA) and
// rounds once: 2^-28 (H_A 2^-32 + H_B)
#ifndef LRS_I8_EPI64
#define LRS_I8_EPI64 0
#endif
// LRS_I8_CRMW=1: C is updated by plain loads and stores in batches of LRS_I8_CBATCH columns
// (every C element of a launch belongs to exactly one thread, so no atomic is needed; REDG
// retires ~1.3 cycles per LANE and SM -- ~20k cycles for the 16,384 elements of a tile, as
// long as the tile's MMAs).  0: fire-and-forget L2 reductions.  Same rounding either way.
#ifndef LRS_I8_CRMW
#define LRS_I8_CRMW 1
#endif
#ifndef LRS_I8_CBATCH
#define LRS_I8_CBATCH 16
#endif
#ifndef LRS_I8_PROBE_K
#define LRS_I8_PROBE_K 100  // the bulk launch whose CTAs report
#endif
#if LRS_I8_PROBE
#define PRB(...) __VA_ARGS__
#else
#define PRB(...)
#endif
constexpr size_t I8_SMEM = (size_t)I8_STAGES * I8_STAGE + 2048;
constexpr int I8_CTAS_PER_SM = (I8_TN == 128 || LRS_I8_ONEPASS) ? 1 : 2;
static_assert(I8_SMEM * I8_CTAS_PER_SM <= 227 * 1024, "shared memory per SM");

size_t lu_i8_chunk_bytes(int steps) { return (size_t)i8_nch(steps) * I8_BLK; }

size_t lu_i8_panel_bytes(const BandGeom& g, int steps) {
  return (size_t)g.P * (g.wl + g.wu) * (i8_nch(steps) * I8_BLK + sizeof(int) * NB);
}

// ---- tcgen05 helpers ------------------------------------------------------------------
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);  // SWIZZLE_NONE, v1
}
// D: s32, A / B: signed int8, K-major, M = 128, N = I8_TN
constexpr uint32_t I8_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(I8_TN >> 3) << 17) |
                              ((uint32_t)(NB >> 4) << 24);
// COLL: the A-operand collector -- 0 none, 1 fill (keep A for the next MMA), 2 use + keep,
// 3 last use.  Consecutive MMAs on one A slice then read it from shared memory once.
template <int COLL>
__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
#define LRS_UMMA_I8(Q)                                                                     \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                          \
               "tcgen05.mma.cta_group::1.kind::i8" Q " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), \
               "l"(a), "l"(b), "r"(I8_IDESC), "r"(acc))
  if (COLL == 0) LRS_UMMA_I8("");
  else if (COLL == 1) LRS_UMMA_I8(".collector::a::fill");
  else if (COLL == 2) LRS_UMMA_I8(".collector::a::use");
  else LRS_UMMA_I8(".collector::a::lastuse");
#undef LRS_UMMA_I8
}
// the same, issued by ONE elected lane while the whole MMA warp runs the (warp-uniform)
// issue loop: descriptor arithmetic then stays on the uniform datapath instead of a
// per-MMA ELECT / R2UR.BROADCAST waterfall of a single-thread loop
template <int COLL>
__device__ __forceinline__ void umma_i8_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
#define LRS_UMMA_I8W(Q)                                                                    \
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"                      \
               "elect.sync _|e, 0xffffffff;\n\t"                                            \
               "@e tcgen05.mma.cta_group::1.kind::i8" Q " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), \
               "l"(a), "l"(b), "r"(I8_IDESC), "r"(acc))
  if (COLL == 0) LRS_UMMA_I8W("");
  else if (COLL == 1) LRS_UMMA_I8W(".collector::a::fill");
  else if (COLL == 2) LRS_UMMA_I8W(".collector::a::use");
  else LRS_UMMA_I8W(".collector::a::lastuse");
#undef LRS_UMMA_I8W
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// Ties 32 registers filled by an earlier tcgen05.ld to this point of the volatile-asm order
// (right after tcgen05.wait::ld): their readers depend on these outputs, so the compiler
// cannot schedule them above the wait when other work sits between the load and the wait.
__device__ __forceinline__ void reg_fence32(uint32_t* v) {
#pragma unroll
  for (int q = 0; q < 32; q += 8)
    asm volatile("" : "+r"(v[q]), "+r"(v[q + 1]), "+r"(v[q + 2]), "+r"(v[q + 3]), "+r"(v[q + 4]),
                      "+r"(v[q + 5]), "+r"(v[q + 6]), "+r"(v[q + 7]));
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// bounded wait: a lost arrival traps (a launch error) instead of hanging the device.
// SLEEP > 0 backs off between probes so waiting warps leave the shared-memory pipe to the
// tensor core's operand reads.
template <int SLEEP = 0>
__device__ __forceinline__ void mbar_wait_trap(uint64_t* bar, unsigned parity) {
  uint32_t ok = 0;
  for (long i = 0;; ++i) {
    if (SLEEP && i) __nanosleep(SLEEP);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (i > (SLEEP ? (1l << 24) : (1l << 28))) __trap();
  }
}
// the same for a whole (converged) warp: the loop exits on a warp vote, so control flow and
// everything computed after it stay warp-uniform for the compiler (uniform registers feed
// the tcgen05 descriptors without per-MMA R2UR moves)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, unsigned parity) {
  for (long i = 0;; ++i) {
    uint32_t ok = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (__all_sync(0xffffffffu, ok != 0)) return;
    if (i > (1l << 28)) __trap();
  }
}
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double exp2i(int e) {
  if (e >= -1022 && e <= 1023) return __longlong_as_double((long long)(e + 1023) << 52);
  return ldexp(1.0, e);
}

// the seven balanced base-256 digits of F = round(x 2^(54 - e)) (|x| < 2^e), from the bits:
// G = F + 0x808080808080 carries the balancing, so digit 1 (the top) is G >> 48 and digits
// 2..7 are the bytes 5..0 of G minus 128 (an xor with 0x80 as int8)
__device__ __forceinline__ void digits7_bits(double x, int e, uint32_t* words, int b) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int bex = (int)((bits >> 52) & 0x7ff);
  unsigned long long mant = bits & 0xfffffffffffffull;
  int ex = bex;
  if (bex == 0) ex = 1;
  else mant |= 1ull << 52;
  const int sh = ex - 1021 - e;  // x 2^(54-e) = mant * 2^sh
  unsigned long long F = 0;
  if (mant != 0) {
    if (sh >= 0) F = mant << sh;  // sh <= 1: |x| < 2^e
    else if (sh > -64) F = (mant + (1ull << (-sh - 1))) >> (-sh);  // round half up
  }
  const long long Fs = (bits >> 63) ? -(long long)F : (long long)F;
  const long long G = Fs + 0x808080808080ll;
  words[0] |= (uint32_t)(uint8_t)(int8_t)(G >> 48) << (8 * b);
#pragma unroll
  for (int q = 1; q < I8_S; ++q)
    words[q] |= ((uint32_t)((G >> (8 * (I8_S - 1 - q))) & 255) ^ 0x80u) << (8 * b);
}

// ---------------------------------------------------------------------------------------
// lu_i8_slice: grid (wl + wu, NB / LINES, P), 512 threads.  Blocks x < wl slice LINES rows
// (y) of the A tile row I = K+STEPS+x, the others LINES columns of the B tile column
// J = K+STEPS+(x-wl); tiles outside the band are zeros.  Thread (line = tid % LINES,
// hc = tid / LINES): the 16 K values of K-core hc (chunk hc / 2, half hc % 2), the line's
// maximum over them (then over every K-core in shared memory), then the K-core's seven
// digit slices as one 16-byte core-matrix row each.  Two threads per 32-value chunk (16
// values in registers each) keep ~50 registers per thread, so several CTAs share an SM:
// the one-thread-per-chunk version (32 values in registers) ran two CTAs per SM and
// streamed at 2.2 TB/s (ncu, c3).  LINES = 32 for pairs, 16 for quads (512 threads).
// ---------------------------------------------------------------------------------------
constexpr int I8_SLICE_THREADS = 512;
#ifndef LRS_I8_SLICE_L1
#define LRS_I8_SLICE_L1 1
#endif
__host__ __device__ constexpr int i8_slice_lines(int steps) {
  return I8_SLICE_THREADS / (2 * i8_nch(steps));
}

template <int STEPS>
__global__ void __launch_bounds__(I8_SLICE_THREADS) lu_i8_slice_kernel(BandGeom g,
                                                                       const double* tiles, int K,
                                                                       I8Panel pn) {
  constexpr int NCH = i8_nch(STEPS);
  constexpr int LINES = i8_slice_lines(STEPS);
  constexpr int NHC = 2 * NCH;  // K-cores of 16 values
  __shared__ double mx[NHC][LINES];
  const int p = blockIdx.z, T = g.T[p];
  const int64_t base = g.tbase[p];
  auto tile = [&](int I, int J) -> const double* {
    return tiles + (base + (int64_t)I * g.W + (J - I + g.wl)) * TILE_ELEMS;
  };
  const int tid = threadIdx.x, ln = tid % LINES, hc = tid / LINES;
  const int line = LINES * blockIdx.y + ln;  // A: row i, B: column j of the tile
  const int x = blockIdx.x;
  const bool isA = x < g.wl;
  const int idx = isA ? x : x - g.wl;
  const int IJ = K + STEPS + idx;
  if (IJ >= T) return;
  const int kc = hc >> 1, hh = hc & 1;
  const int d = kc >> 2;  // step K + d
  const double* src;
  if (isA) src = (IJ - (K + d) <= g.wl) ? tile(IJ, K + d) : nullptr;
  else src = (IJ - (K + d) <= g.wu) ? tile(K + d, IJ) : nullptr;
  // the 16 K values k0 .. k0+15 of this line: A reads a column-major tile along its row
  // (stride 128, lanes on consecutive rows: coalesced), B reads a column (contiguous per
  // thread, lanes on different columns: through L1, a 32-byte sector serves 4 values)
  const int k0 = (kc & 3) * I8_KC + 16 * hh;
  double v[16];
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    const int k = k0 + kk;
#if LRS_I8_SLICE_L1
    v[kk] = src ? (isA ? __ldcg(src + (int64_t)k * NB + line) : __ldca(src + (int64_t)line * NB + k))
                : 0.0;
#else
    v[kk] = src ? (isA ? __ldcg(src + (int64_t)k * NB + line) : __ldcg(src + (int64_t)line * NB + k))
                : 0.0;
#endif
  }
  double m = 0.0;
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) m = fmax(m, fabs(v[kk]));
  mx[hc][ln] = m;
  __syncthreads();
  m = mx[0][ln];
#pragma unroll
  for (int c = 1; c < NHC; ++c) m = fmax(m, mx[c][ln]);
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  if (hc == 0) {
    int* ex = isA ? pn.ea + ((int64_t)p * g.wl + idx) * NB : pn.eb + ((int64_t)p * g.wu + idx) * NB;
    ex[line] = e;
  }
  // B: column block h = line / TN, operand row line % TN, in [p][jb][h][chunk][slice]
  const int bl = isA ? line : (line & (I8_TN - 1));
  const int sl = isA ? I8_SL : I8_BSL;
  uint8_t* dst = isA ? pn.A + (((int64_t)p * g.wl + idx) * NCH + kc) * I8_BLK
                     : pn.B + ((((int64_t)p * g.wu + idx) * I8_NH + line / I8_TN) * NCH + kc) *
                                  I8_BBLK;
  const int rows = isA ? NB : I8_TN;
  uint32_t wd[I8_S][4];
#pragma unroll
  for (int q = 0; q < I8_S; ++q) wd[q][0] = wd[q][1] = wd[q][2] = wd[q][3] = 0u;
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    uint32_t tmp[I8_S] = {0, 0, 0, 0, 0, 0, 0};
    digits7_bits(v[kk], e, tmp, kk & 3);
#pragma unroll
    for (int q = 0; q < I8_S; ++q) wd[q][kk >> 2] |= tmp[q];
  }
  const int off = (hh * (rows / 8) + (bl >> 3)) * 128 + (bl & 7) * 16;
#pragma unroll
  for (int q = 0; q < I8_S; ++q)
    *reinterpret_cast<uint4*>(dst + q * sl + off) = make_uint4(wd[q][0], wd[q][1], wd[q][2], wd[q][3]);
}

// the seven digit slices of 16 K values (one K-core row of a core matrix) at dst + q sl + off
__device__ __forceinline__ void i8_store_kcore(const double* v, bool neg, int e, uint8_t* dst,
                                               int sl, int off) {
  uint32_t wd[I8_S][4];
#pragma unroll
  for (int q = 0; q < I8_S; ++q) wd[q][0] = wd[q][1] = wd[q][2] = wd[q][3] = 0u;
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    uint32_t tmp[I8_S] = {0, 0, 0, 0, 0, 0, 0};
    digits7_bits(neg ? -v[kk] : v[kk], e, tmp, kk & 3);
#pragma unroll
    for (int q = 0; q < I8_S; ++q) wd[q][kk >> 2] |= tmp[q];
  }
#pragma unroll
  for (int q = 0; q < I8_S; ++q)
    *reinterpret_cast<uint4*>(dst + q * sl + off) = make_uint4(wd[q][0], wd[q][1], wd[q][2], wd[q][3]);
}

// Complex panels of the realified update (lu_i8_gemm_kernel<.., true>): A' = [Ar Ai] (K' = 2K:
// the real parts' chunks, then the imaginary parts'), B'_re = [Br; -Bi] and B'_im = [Bi; Br]
// (part 0 / 1 of each B tile column).  One exponent per row of A' (the maximum over both
// parts) and per column of B'_re / B'_im (the same set of magnitudes).  Thread layout as
// lu_i8_slice_kernel; each thread loads 16 complex values and writes both parts.
constexpr int I8_ZSLICE_THREADS = 256;  // 32 complex values in registers per thread
template <int STEPS>
__global__ void __launch_bounds__(I8_ZSLICE_THREADS) lu_i8_slice_z_kernel(BandGeom g,
                                                                          const zc* tiles, int K,
                                                                          I8Panel pn) {
  constexpr int NCH = i8_nch(STEPS);
  constexpr int NHC = 2 * NCH;
  constexpr int LINES = I8_ZSLICE_THREADS / NHC;
  __shared__ double mx[NHC][LINES];
  const int p = blockIdx.z, T = g.T[p];
  const int64_t base = g.tbase[p];
  auto tile = [&](int I, int J) -> const zc* {
    return tiles + (base + (int64_t)I * g.W + (J - I + g.wl)) * TILE_ELEMS;
  };
  const int tid = threadIdx.x, ln = tid % LINES, hc = tid / LINES;
  const int line = LINES * blockIdx.y + ln;
  const int x = blockIdx.x;
  const bool isA = x < g.wl;
  const int idx = isA ? x : x - g.wl;
  const int IJ = K + STEPS + idx;
  if (IJ >= T) return;
  const int kc = hc >> 1, hh = hc & 1, d = kc >> 2;
  const zc* src;
  if (isA) src = (IJ - (K + d) <= g.wl) ? tile(IJ, K + d) : nullptr;
  else src = (IJ - (K + d) <= g.wu) ? tile(K + d, IJ) : nullptr;
  const int k0 = (kc & 3) * I8_KC + 16 * hh;
  double vr[16], vi[16];
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    const int k = k0 + kk;
    double2 z = make_double2(0.0, 0.0);
    if (src)
      z = isA ? __ldcg(reinterpret_cast<const double2*>(src + (int64_t)k * NB + line))
              : __ldca(reinterpret_cast<const double2*>(src + (int64_t)line * NB + k));
    vr[kk] = z.x;
    vi[kk] = z.y;
  }
  double m = 0.0;
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) m = fmax(m, fmax(fabs(vr[kk]), fabs(vi[kk])));
  mx[hc][ln] = m;
  __syncthreads();
  m = mx[0][ln];
#pragma unroll
  for (int c = 1; c < NHC; ++c) m = fmax(m, mx[c][ln]);
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  if (hc == 0) {
    int* ex = isA ? pn.ea + ((int64_t)p * g.wl + idx) * NB : pn.eb + ((int64_t)p * g.wu + idx) * NB;
    ex[line] = e;
  }
  const int bl = isA ? line : (line & (I8_TN - 1));
  const int rows = isA ? NB : I8_TN;
  const int off = (hh * (rows / 8) + (bl >> 3)) * 128 + (bl & 7) * 16;
  if (isA) {
    uint8_t* a = pn.A + ((int64_t)p * g.wl + idx) * (2 * NCH) * I8_BLK;
    i8_store_kcore(vr, false, e, a + (int64_t)kc * I8_BLK, I8_SL, off);
    i8_store_kcore(vi, false, e, a + (int64_t)(kc + NCH) * I8_BLK, I8_SL, off);
  } else {
    auto bdst = [&](int part, int kcp) -> uint8_t* {
      return pn.B + (((((int64_t)p * g.wu + idx) * 2 + part) * I8_NH + line / I8_TN) * (2 * NCH) +
                     kcp) * I8_BBLK;
    };
    i8_store_kcore(vr, false, e, bdst(0, kc), I8_BSL, off);         // B'_re = [Br; -Bi]
    i8_store_kcore(vi, true, e, bdst(0, kc + NCH), I8_BSL, off);
    i8_store_kcore(vi, false, e, bdst(1, kc), I8_BSL, off);         // B'_im = [Bi; Br]
    i8_store_kcore(vr, false, e, bdst(1, kc + NCH), I8_BSL, off);
  }
}

// work item t of the kind-3 / kind-4 lists of a STEPS-step update (steps K .. K+D-1, D =
// STEPS) -> (p, ia, jb, column block h); false when outside the blocks.
//   KIND 3 (look-ahead): columns K+D .. K+2D-1 (rows K+D .. K+D-1+wl) and rows
//                        K+D .. K+2D-1 (columns K+2D .. K+D-1+wu)
//   KIND 4 (bulk):       I = K+2D .. K+D-1+wl, J = K+2D .. K+D-1+wu
// Work items per partition.  g.sym (symmetric blocks, wl == wu): only the lower trailing
// tiles are formed -- kind 4 the triangle I >= J of the bulk window, kind 3 the columns
// K+D .. K+2D-1 (the rows of the look-ahead come from the mirrored L panels, band_lu.cu).
template <int KIND, int STEPS>
__host__ __device__ __forceinline__ int i8_per(const BandGeom& g) {
  constexpr int D = STEPS;
  if (KIND == 4) return g.sym ? (g.wl - D) * (g.wl - D + 1) / 2 : (g.wl - D) * (g.wu - D);
  if (g.sym) return D == 2 ? 2 * g.wl - 1 : D * g.wl;
  return D * g.wl + D * (g.wu - D);
}

template <int KIND, int STEPS>
__device__ __forceinline__ bool i8_decode(const BandGeom& g, int K, int t, int& p, int& ia,
                                          int& jb, int& h) {
  constexpr int D = STEPS;
  const int per = i8_per<KIND, STEPS>(g);
  h = t % I8_NH;
  t /= I8_NH;
  p = t / per;
  int r = t % per;
  int I, J;
  if (KIND == 4 && g.sym) {
    // row-major over the lower triangle: r = a (a + 1) / 2 + b, b <= a
    // (LRS_I8_SYM_ORDER=1: column-major -- the mirrored walk, consecutive items share B_J)
    if (LRS_I8_SYM_ORDER == 1) r = per - 1 - r;
    int a = (int)((sqrtf(8.0f * (float)r + 1.0f) - 1.0f) * 0.5f);
    while ((a + 1) * (a + 2) / 2 <= r) ++a;
    while (a * (a + 1) / 2 > r) --a;
    int b = r - a * (a + 1) / 2;
    if (LRS_I8_SYM_ORDER == 1) {
      const int m = g.wl - D, a2 = m - 1 - b;
      b = m - 1 - a;
      a = a2;
    }
    I = K + 2 * D + a;
    J = K + 2 * D + b;
  } else if (KIND == 4) {
    I = K + 2 * D + r / (g.wu - D);
    J = K + 2 * D + r % (g.wu - D);
  } else if (D == 2) {  // pairs: column K+2, column K+3, row K+2, row K+3
    if (r < g.wl) {
      I = K + 2 + r;
      J = K + 2;
    } else if ((r -= g.wl) < g.wl - 1) {
      I = K + 3 + r;
      J = K + 3;
    } else if ((r -= g.wl - 1) < g.wu - 1) {
      I = K + 2;
      J = K + 3 + r;
    } else {
      r -= g.wu - 1;
      I = K + 3;
      J = K + 4 + r;
    }
  } else if (r < D * g.wl) {
    I = K + D + r % g.wl;
    J = K + D + r / g.wl;
  } else {
    r -= D * g.wl;
    I = K + D + r / (g.wu - D);
    J = K + 2 * D + r % (g.wu - D);
  }
  ia = I - K - D;
  jb = J - K - D;
  const int T = g.T[p];
  return I < T && J < T;  // I, J >= K + D: every step K .. K+D-1 exists
}

// MMAs of one K chunk of one pass: A slice p outer (collector), B slice q descending, so the
// first writes of the groups (p = 1) go to the pass's slots in ring order -- the order the
// epilogue releases them.  Before its first write a slot waits for the drain of its
// previous use (uses[slot] counts them).
// used / par: bit masks over the slots -- the slot has been used before / parity of its
// number of uses (its tempty barrier has completed that many phases once drained)
template <int PASS, bool WARP = false>
__device__ __forceinline__ void i8_chunk_mmas(uint32_t tm, uint32_t a0, uint32_t b0, bool first,
                                              uint64_t* tempty, int ptr, uint32_t used,
                                              uint32_t par) {
  constexpr int top = i8_top(PASS), ng = i8_ng(PASS), pmax = i8_pmax(PASS);
#pragma unroll
  for (int pp = 1; pp <= pmax; ++pp) {
    const int qhi = min(I8_S, top - pp), qlo = max(1, top - ng + 1 - pp);
#pragma unroll
    for (int q = I8_S; q >= 1; --q) {
      if (q > qhi || q < qlo) continue;
      const int slot = (ptr + top - pp - q) & (I8_GROUPS - 1);
      if (first && pp == 1 && ((used >> slot) & 1u)) {
        if (WARP) mbar_wait_warp(&tempty[slot], ((par >> slot) & 1u) ^ 1u);
        else mbar_wait_trap(&tempty[slot], ((par >> slot) & 1u) ^ 1u);
        tc_fence_after();
      }
      const uint32_t dd = tm + slot * I8_TN;
      const uint64_t ad = umma_sdesc(a0 + (pp - 1) * I8_SL, NB * 16, 128);
      const uint64_t bd = umma_sdesc(b0 + (q - 1) * I8_BSL, I8_TN * 16, 128);
      const uint32_t ac = (first && pp == 1) ? 0u : 1u;
      if (WARP) {
        if (qhi == qlo) umma_i8_warp<0>(dd, ad, bd, ac);
        else if (q == qhi) umma_i8_warp<1>(dd, ad, bd, ac);
        else if (q == qlo) umma_i8_warp<3>(dd, ad, bd, ac);
        else umma_i8_warp<2>(dd, ad, bd, ac);
      } else {
        if (qhi == qlo) umma_i8<0>(dd, ad, bd, ac);
        else if (q == qhi) umma_i8<1>(dd, ad, bd, ac);
        else if (q == qlo) umma_i8<3>(dd, ad, bd, ac);
        else umma_i8<2>(dd, ad, bd, ac);
      }
    }
  }
}

// CPLX: complex128 tiles, the 4M product realified -- C_re -= [Ar Ai] [Br; -Bi] and
// C_im -= [Ar Ai] [Bi; Br] -- as two real updates with K doubled (work item = tile x part,
// part the lowest index; the A' = [Ar Ai] slices are shared, B'_re / B'_im have their own;
// C is written at stride 2 into the interleaved complex tile).  lu_i8_slice_z_kernel makes
// the panels.
template <int KIND, int STEPS, bool CPLX = false>
__global__ void __launch_bounds__(I8_THREADS, I8_CTAS_PER_SM)
    lu_i8_gemm_kernel(BandGeom g, double* tiles, int K, I8Panel pn, int total, int tpc) {
  constexpr int I8_NCH = i8_nch(STEPS) * (CPLX ? 2 : 1);
  constexpr int CS = CPLX ? 2 : 1;  // doubles per tile element
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* stage = smraw;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + I8_STAGES * I8_STAGE);
  uint64_t* empty = full + I8_STAGES;
  uint64_t* tfull = empty + I8_STAGES;
  // tfull[2]: pass u's accumulators complete, alternating by pass parity -- pass u+2 needs
  // slots pass u's drain frees, so a barrier never completes twice ahead of its waiter
  uint64_t* tempty = tfull + 2;  // [I8_GROUPS]: slot drained by the epilogue
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + I8_GROUPS);
  double* sj = reinterpret_cast<double*>(smraw + I8_STAGES * I8_STAGE + 1024);  // [128]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * tpc, t1 = min(total, t0 + tpc);
  auto ctile = [&](int p, int ia, int jb, int h) -> double* {
    const int I = K + STEPS + ia, J = K + STEPS + jb;
    return tiles + ((g.tbase[p] + (int64_t)I * g.W + (J - I + g.wl)) * TILE_ELEMS +
                    (int64_t)h * I8_TN * NB) * CS;
  };
  // work item t -> (p, ia, jb, h) and the complex part (0: re, 1: im)
  auto decode = [&](int t, int& p, int& ia, int& jb, int& h, int& part) -> bool {
    part = CPLX ? (t & 1) : 0;
    return i8_decode<KIND, STEPS>(g, K, CPLX ? (t >> 1) : t, p, ia, jb, h);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < I8_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    for (int gi = 0; gi < I8_GROUPS; ++gi) mbar_init(&tempty[gi], I8_EPI);
    fence_mbar_init();
  }
  if (w == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tbase)), "n"(I8_TMEM)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tbase;

  if (w == 0) {
    // ---- producer: per tile and pass, slices 1..pmax of every K chunk -----------------
    if (lane == 0) {
      int it = 0;
      for (int t = t0; t < t1; ++t) {
        int p, ia, jb, h, part;
        if (!decode(t, p, ia, jb, h, part)) continue;
        if (LRS_I8_CPREFETCH && part == 0)
          bulk_prefetch_l2(ctile(p, ia, jb, h), sizeof(double) * NB * I8_TN * CS);
        const uint8_t* a = pn.A + ((int64_t)p * g.wl + ia) * I8_NCH * I8_BLK;
        const uint8_t* b =
            pn.B + ((((int64_t)p * g.wu + jb) * CS + part) * I8_NH + h) * I8_NCH * I8_BBLK;
        for (int pass = 0; pass < I8_NP; ++pass) {
          const unsigned abytes = i8_pmax(pass) * I8_SL;
          const unsigned bbytes = i8_pmax(pass) * I8_BSL;
          for (int kc = 0; kc < I8_NCH; ++kc, ++it) {
            const int s = it % I8_STAGES;
            if (it >= I8_STAGES) mbar_wait_trap<64>(&empty[s], ((it / I8_STAGES) & 1) ^ 1);
            if (LRS_I8_EXP >= 2) {
              mbar_arrive1(&full[s]);
              continue;
            }
            mbar_expect_tx(&full[s], abytes + bbytes);
            bulk_g2s(stage + s * I8_STAGE, a + kc * I8_BLK, abytes, &full[s]);
            bulk_g2s(stage + s * I8_STAGE + I8_BLK, b + kc * I8_BBLK, bbytes, &full[s]);
          }
        }
      }
    }
  } else if (w == 1) {
    // ---- MMA issuer: the whole warp runs the loop, one elected lane issues ------------
    if (LRS_I8_WARP_ISSUE || lane == 0) {
      int it = 0, ptr = 0, u = 0;
      uint32_t used = 0u, par = 0u;
      PRB(long long c_full = 0, c_chunk0 = 0; const long long c_start = clock64();)
      for (int t = t0; t < t1; ++t) {
        int p, ia, jb, h, part;
        if (!decode(t, p, ia, jb, h, part)) continue;
#pragma unroll
        for (int pass = 0; pass < I8_NP; ++pass) {
          for (int kc = 0; kc < I8_NCH; ++kc, ++it) {
            const int s = it % I8_STAGES;
            PRB(long long c0 = clock64();)
            constexpr bool WI = LRS_I8_WARP_ISSUE != 0;
            if (WI) mbar_wait_warp(&full[s], (it / I8_STAGES) & 1);
            else mbar_wait_trap(&full[s], (it / I8_STAGES) & 1);
            PRB(c_full += clock64() - c0; c0 = clock64();)
            tc_fence_after();
            const uint32_t a0 = smem_u32(stage + s * I8_STAGE), b0 = a0 + I8_BLK;
            if (pass == 0) i8_chunk_mmas<0, WI>(tm, a0, b0, kc == 0, tempty, ptr, used, par);
            else if (pass == 1) i8_chunk_mmas<1 % I8_NP, WI>(tm, a0, b0, kc == 0, tempty, ptr, used, par);
            else i8_chunk_mmas<2 % I8_NP, WI>(tm, a0, b0, kc == 0, tempty, ptr, used, par);
            PRB(if (kc == 0) c_chunk0 += clock64() - c0;)
            if (WI) umma_commit_warp(&empty[s]);
            else umma_commit(&empty[s]);
          }
          if (LRS_I8_WARP_ISSUE) umma_commit_warp(&tfull[u & 1]);
          else umma_commit(&tfull[u & 1]);
          ++u;
#pragma unroll
          for (int gi = 0; gi < i8_ng(pass); ++gi) {
            const uint32_t bit = 1u << ((ptr + gi) & (I8_GROUPS - 1));
            used |= bit;
            par ^= bit;
          }
          ptr = (ptr + i8_ng(pass)) & (I8_GROUPS - 1);
        }
      }
      PRB(if (KIND == 4 && K == LRS_I8_PROBE_K && (blockIdx.x % 997) == 0 && lane == 0) printf(
              "PROBE mma cta %d tiles %d total %lld full_wait %lld chunk0(tempty) %lld\n",
              blockIdx.x, t1 - t0, clock64() - c_start, c_full, c_chunk0);)
    }
  } else {
    // ---- epilogue: warp w drains TMEM lanes 32 (w % 4).. (rows) and column half
    // (w - 2) / 4 of every slot.  INT32 -> FP64 by the exponent trick (2^52 + 2^31 + x is
    // exact), so a conversion is an xor and an FP64 add instead of an XU I2F.
    const int qd = w & 3, ch = (w - 2) >> 2, i = 32 * qd + lane;
    constexpr double BIAS = 4503601774854144.0;  // 2^52 + 2^31
    int u = 0, ptr = 0;
    PRB(long long c_tf = 0, c_drain = 0, c_red = 0; const long long c_start = clock64();)
    for (int t = t0; t < t1; ++t) {
      int p, ia, jb, h, part;
      if (!decode(t, p, ia, jb, h, part)) continue;
      double* C = ctile(p, ia, jb, h) + (int64_t)ch * I8_EPC * NB * CS + part;
      const double si = exp2i(pn.ea[((int64_t)p * g.wl + ia) * NB + i]);
      if (w == 2) {  // the previous tile's readers of sj passed the closing barrier
        const int* eb = pn.eb + ((int64_t)p * g.wu + jb) * NB + h * I8_TN;
#pragma unroll
        for (int r = 0; r < I8_TN / 32; ++r) sj[lane + 32 * r] = exp2i(eb[lane + 32 * r]);
      }
      const uint32_t trow = tm + ((uint32_t)(32 * qd) << 16) + ch * I8_EPC;
#if LRS_I8_EPI64
      // hA: groups 8..5 as one exact integer; groups 4..2 likewise in hB when the registers
      // allow (32 columns per warp), else in FP64 on top of the converted hA
      constexpr bool B64 = I8_EPC <= 32;
      constexpr long long MAGIC = 0x4338000000000000ll;  // bits of 2^52 + 2^51
      constexpr double MAGICD = 6755399441055744.0;
      long long hA[I8_EPC], hB[B64 ? I8_EPC : 1];
      double acc[B64 ? 1 : I8_EPC];
#else
      double acc[I8_EPC];
#pragma unroll
      for (int j = 0; j < I8_EPC; ++j) acc[j] = 0.0;
#endif
#pragma unroll
      for (int pass = 0; pass < I8_NP; ++pass, ++u) {
        PRB(long long c0 = clock64();)
        mbar_wait_trap<128>(&tfull[u & 1], (u >> 1) & 1);
        PRB(c_tf += clock64() - c0; c0 = clock64();)
        tc_fence_after();
        if (LRS_I8_EXP == 3) {
          __syncwarp();
          if (lane == 0)
            for (int gi = 0; gi < i8_ng(pass); ++gi)
              mbar_arrive1(&tempty[(ptr + gi) & (I8_GROUPS - 1)]);
          ptr = (ptr + i8_ng(pass)) & (I8_GROUPS - 1);
          continue;
        }
        // drain in ring order (the next pass reuses the first slots first), smallest
        // group weight first for the FP64 accumulation
#if LRS_I8_LDPIPE
        // two 32-column register buffers: the TMEM load of batch b + 1 is in flight while
        // batch b converts, and a slot is released as soon as its last load has landed
        // (not after the conversion of the batch before it)
        uint32_t vb[2][32];
        {
          const int slot0 = ptr & (I8_GROUPS - 1);
#pragma unroll
          for (int c8 = 0; c8 < 32; c8 += 8) tmem_ld8(trow + slot0 * I8_TN + c8, vb[0] + c8);
        }
#endif
#pragma unroll
        for (int gi = 0; gi < i8_ng(pass); ++gi) {
          const int slot = (ptr + gi) & (I8_GROUPS - 1);
          const double sc = exp2i(4 - 8 * (i8_top(pass) - gi));
#pragma unroll
          for (int h2 = 0; h2 < I8_EPC / 32; ++h2) {
#if LRS_I8_LDPIPE
            constexpr int NB2 = I8_EPC / 32;
            const int b = gi * NB2 + h2;
            uint32_t* v = vb[b & 1];
            tmem_ld_wait();
            reg_fence32(v);
            if (b + 1 < i8_ng(pass) * NB2) {
              const int slot1 = (ptr + (b + 1) / NB2) & (I8_GROUPS - 1);
#pragma unroll
              for (int c8 = 0; c8 < 32; c8 += 8)
                tmem_ld8(trow + slot1 * I8_TN + ((b + 1) % NB2) * 32 + c8, vb[(b + 1) & 1] + c8);
            }
#else
            uint32_t v[32];
#pragma unroll
            for (int c8 = 0; c8 < 32; c8 += 8) tmem_ld8(trow + slot * I8_TN + h2 * 32 + c8, v + c8);
            tmem_ld_wait();
#endif
            if (h2 == I8_EPC / 32 - 1) {  // the warp's part of the slot is in registers: release it
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive1(&tempty[slot]);
            }
#if LRS_I8_EPI64
            {
              const int sg = i8_top(pass) - gi;  // group s (the loops are fully unrolled)
              const long long wt = 1ll << (8 * ((sg >= 5 ? 8 : 4) - sg));
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int c = h2 * 32 + j;
                const long long gv = (long long)(int)v[j];
                if (sg == 8) hA[c] = gv;
                else if (sg >= 5) hA[c] += gv * wt;
                else if (B64) {
                  if (sg == 4) hB[c] = gv;
                  else hB[c] += gv * wt;
                } else {
                  if (sg == 4)  // |hA| < 2^51: 2^52 + 2^51 + hA is exact
                    acc[c] = (__longlong_as_double(hA[c] + MAGIC) - MAGICD) * exp2i(4 - 64);
                  acc[c] = fma(__hiloint2double(0x43300000, (int)(v[j] ^ 0x80000000u)) - BIAS, sc,
                               acc[c]);
                }
              }
            }
#else
#pragma unroll
            for (int j = 0; j < 32; ++j)
              acc[h2 * 32 + j] = fma(
                  __hiloint2double(0x43300000, (int)(v[j] ^ 0x80000000u)) - BIAS, sc,
                  acc[h2 * 32 + j]);
#endif
          }
        }
        ptr = (ptr + i8_ng(pass)) & (I8_GROUPS - 1);
        PRB(c_drain += clock64() - c0;)
      }
      PRB(long long c1 = clock64();)
      asm volatile("bar.sync 1, %0;" ::"n"(32 * I8_EPI) : "memory");  // sj written
      // C -= 2^(ea+eb) acc as fire-and-forget L2 reductions: no load round trip in the
      // epilogue, and with one contribution per element fl(c + (-r)) == fl(c - r) exactly
      if (!LRS_I8_EXP) {
        // r(j) = the update of C(i, j); C -= r either by load / store batches or by L2 reductions
#if LRS_I8_EPI64
        const double si28 = si * exp2i(-28);
#endif
        auto upd = [&](int j) -> double {
#if LRS_I8_EPI64
          if (B64) {
            const double dA = __longlong_as_double(hA[j] + MAGIC) - MAGICD;
            const double dB = __longlong_as_double(hB[B64 ? j : 0] + MAGIC) - MAGICD;
            const double u = fma(dA, 2.3283064365386963e-10 /* 2^-32 */, dB);  // one rounding
            return u * si28 * sj[ch * I8_EPC + j];
          }
          return acc[B64 ? 0 : j] * si * sj[ch * I8_EPC + j];
#else
          return acc[j] * si * sj[ch * I8_EPC + j];
#endif
        };
#if LRS_I8_CRMW
        constexpr int CB = LRS_I8_CBATCH;
        static_assert(I8_EPC % CB == 0, "C batch");
#pragma unroll
        for (int j0 = 0; j0 < I8_EPC; j0 += CB) {
          double cv[CB];
#pragma unroll
          for (int jj = 0; jj < CB; ++jj) cv[jj] = __ldcg(C + ((int64_t)(j0 + jj) * NB + i) * CS);
#pragma unroll
          for (int jj = 0; jj < CB; ++jj)
            __stcg(C + ((int64_t)(j0 + jj) * NB + i) * CS, cv[jj] - upd(j0 + jj));
        }
#else
#pragma unroll
        for (int j = 0; j < I8_EPC; ++j) red_add_f64(C + ((int64_t)j * NB + i) * CS, -upd(j));
#endif
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * I8_EPI) : "memory");  // sj free for the next tile
      PRB(c_red += clock64() - c1;)
    }
    PRB(if (KIND == 4 && K == LRS_I8_PROBE_K && (blockIdx.x % 997) == 0 && lane == 0 && (w == 2 || w == 9))
            printf("PROBE epi cta %d warp %d total %lld tfull_wait %lld drain %lld red %lld\n",
                   blockIdx.x, w, clock64() - c_start, c_tf, c_drain, c_red);)
  }
  tc_fence_before();
  __syncthreads();
  if (w == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(I8_TMEM)
                 : "memory");
  }
}

// ---- 2-SM bulk update (LRS_I8_2SM=1): tcgen05.mma.cta_group::2, M = 256 ------------------
// A cluster of two CTAs on one SM pair computes tile rows I0 (rank 0) and I0 + 1 (rank 1)
// of tile column J: each CTA stages its own 128 rows of the A slices and HALF of the B
// slices (columns 64 r .. 64 r + 63), the leader's elected thread issues the M = 256, N = 128
// MMAs for both (the pair's tensor cores exchange the B halves), and each CTA's TMEM holds
// its 128 rows x 128 columns -- so per SM a K chunk streams 42 KB instead of 56 KB (pass A)
// and the shared-memory B reads per MMA halve.  Hand-offs: the peer's idle MMA warp relays
// "stage landed" to the leader (fullp), the leader's commits multicast to both CTAs' empty /
// tfull barriers, and both CTAs' epilogue warps arrive on the leader's tempty.  The pass
// structure, digit products, drain order and C reductions are those of lu_i8_gemm_kernel,
// so the factors are bitwise identical.  An odd last row pair runs a dummy rank-1 half
// (rows of I0, product discarded).
#ifndef LRS_I8_2SM_STAGES
#define LRS_I8_2SM_STAGES 5
#endif
constexpr int I8P_BSL = 64 * I8_KC;            // 2 KB: one half B slice of one chunk
constexpr int I8P_BBLK = I8_S * I8P_BSL;       // 14 KB
constexpr int I8P_STAGE = I8_BLK + I8P_BBLK;   // 42 KB
constexpr int I8P_STAGES = LRS_I8_2SM_STAGES;
constexpr size_t I8P_SMEM = (size_t)I8P_STAGES * I8P_STAGE + 2048;
static_assert(I8P_SMEM <= 227 * 1024, "2-SM stages");
constexpr uint32_t I8P_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NB >> 3) << 17) |
                               ((uint32_t)(2 * NB >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// arrive on a barrier of another CTA of the cluster (default .release.cta semantics, as
// CUTLASS's ClusterBarrier::arrive: a .cluster-scope release fences the epilogue's
// outstanding L2 reductions of C before every TMEM slot release -- measured 1.6x slower)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
template <int COLL>
__device__ __forceinline__ void umma_i8_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
#define LRS_UMMA_I8P(Q)                                                                    \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                          \
               "tcgen05.mma.cta_group::2.kind::i8" Q " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), \
               "l"(a), "l"(b), "r"(I8P_IDESC), "r"(acc))
  if (COLL == 0) LRS_UMMA_I8P("");
  else if (COLL == 1) LRS_UMMA_I8P(".collector::a::fill");
  else if (COLL == 2) LRS_UMMA_I8P(".collector::a::use");
  else LRS_UMMA_I8P(".collector::a::lastuse");
#undef LRS_UMMA_I8P
}
// arrive on the barrier at this offset in BOTH CTAs of the pair when the MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// work item t -> (p, ia, jb) of this rank; false outside the blocks.  own = this rank's
// rows exist (else it runs the dummy half on row I0).
template <int STEPS>
__device__ __forceinline__ bool i8p_decode(const BandGeom& g, int K, int t, int rank, int& p,
                                           int& ia, int& jb, bool& own) {
  constexpr int D = STEPS;
  const int R = g.wl - D, Cn = g.wu - D, per = ((R + 1) / 2) * Cn;
  p = t / per;
  const int r = t % per, rp = r / Cn;
  const int J = K + 2 * D + r % Cn, I0 = K + 2 * D + 2 * rp;
  const int T = g.T[p];
  if (I0 >= T || J >= T) return false;
  own = 2 * rp + rank < R && I0 + rank < T;
  ia = (own ? I0 + rank : I0) - K - D;
  jb = J - K - D;
  return true;
}

#if !LRS_I8_ONEPASS
template <int PASS>
__device__ __forceinline__ void i8p_chunk_mmas(uint32_t tm, uint32_t a0, uint32_t b0, bool first,
                                               uint64_t* tempty, int ptr, const int* uses) {
  constexpr int top = i8_top(PASS), ng = i8_ng(PASS), pmax = i8_pmax(PASS);
#pragma unroll
  for (int pp = 1; pp <= pmax; ++pp) {
    const int qhi = min(I8_S, top - pp), qlo = max(1, top - ng + 1 - pp);
#pragma unroll
    for (int q = I8_S; q >= 1; --q) {
      if (q > qhi || q < qlo) continue;
      const int slot = (ptr + top - pp - q) & (I8_GROUPS - 1);
      if (first && pp == 1 && uses[slot] > 0) {
        mbar_wait_trap(&tempty[slot], (uses[slot] - 1) & 1);
        tc_fence_after();
      }
      const uint32_t dd = tm + slot * NB;
      const uint64_t ad = umma_sdesc(a0 + (pp - 1) * I8_SL, NB * 16, 128);
      const uint64_t bd = umma_sdesc(b0 + (q - 1) * I8P_BSL, 64 * 16, 128);
      const uint32_t ac = (first && pp == 1) ? 0u : 1u;
      if (qhi == qlo) umma_i8_2sm<0>(dd, ad, bd, ac);
      else if (q == qhi) umma_i8_2sm<1>(dd, ad, bd, ac);
      else if (q == qlo) umma_i8_2sm<3>(dd, ad, bd, ac);
      else umma_i8_2sm<2>(dd, ad, bd, ac);
    }
  }
}

template <int STEPS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(I8_THREADS, 1)
    lu_i8_gemm2_kernel(BandGeom g, double* tiles, int K, I8Panel pn, int total, int tpc) {
  static_assert(I8_TN == 128 && I8_NP == 2, "2-SM update: 128-column tiles, two passes");
  constexpr int NCH = i8_nch(STEPS);
  constexpr int ST = I8P_STAGES;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* stage = smraw;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + ST * I8P_STAGE);
  uint64_t* fullp = full + ST;    // leader: the peer's copy of the stage landed
  uint64_t* empty = fullp + ST;   // the pair's MMAs finished reading the stage
  uint64_t* tfull = empty + ST;   // [2]
  uint64_t* tempty = tfull + 2;   // [I8_GROUPS] leader: both CTAs drained the slot
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + I8_GROUPS);
  double* sj = reinterpret_cast<double*>(smraw + ST * I8P_STAGE + 1024);  // [128]
  const int rank = (int)cluster_rank();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = (blockIdx.x >> 1) * tpc, t1 = min(total, t0 + tpc);
  auto ctile = [&](int p, int ia, int jb) -> double* {
    const int I = K + STEPS + ia, J = K + STEPS + jb;
    return tiles + (g.tbase[p] + (int64_t)I * g.W + (J - I + g.wl)) * TILE_ELEMS;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&fullp[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    for (int gi = 0; gi < I8_GROUPS; ++gi) mbar_init(&tempty[gi], 2 * I8_EPI);
    fence_mbar_init();
  }
  if (w == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tbase)), "n"(I8_TMEM)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tm = *tbase;

  if (w == 0) {
    // ---- producer (both CTAs): own A rows, own half of the B slices ---------------------
    if (lane == 0) {
      int it = 0;
      for (int t = t0; t < t1; ++t) {
        int p, ia, jb;
        bool own;
        if (!i8p_decode<STEPS>(g, K, t, rank, p, ia, jb, own)) continue;
        if (own) bulk_prefetch_l2(ctile(p, ia, jb), sizeof(double) * NB * NB);
        const uint8_t* a = pn.A + ((int64_t)p * g.wl + ia) * NCH * I8_BLK;
        const uint8_t* b = pn.B + ((int64_t)p * g.wu + jb) * NCH * I8_BBLK + (8 * rank) * 128;
        for (int pass = 0; pass < I8_NP; ++pass) {
          const int pm = i8_pmax(pass);
          for (int kc = 0; kc < NCH; ++kc, ++it) {
            const int s = it % ST;
            if (it >= ST) mbar_wait_trap<64>(&empty[s], ((it / ST) & 1) ^ 1);
            uint8_t* dst = stage + s * I8P_STAGE;
            mbar_expect_tx(&full[s], pm * (I8_SL + I8P_BSL));
            bulk_g2s(dst, a + kc * I8_BLK, pm * I8_SL, &full[s]);
            for (int q = 0; q < pm; ++q)
#pragma unroll
              for (int kcore = 0; kcore < 2; ++kcore)
                bulk_g2s(dst + I8_BLK + q * I8P_BSL + kcore * 1024,
                         b + kc * I8_BBLK + q * I8_BSL + kcore * (NB / 8) * 128, 1024, &full[s]);
          }
        }
      }
      // drain: every commit into this CTA's empty barriers has landed before it exits
      for (int k = (it > ST ? it - ST : 0); k < it; ++k)
        mbar_wait_trap<64>(&empty[k % ST], (k / ST) & 1);
    }
  } else if (w == 1) {
    if (lane == 0 && rank == 1) {
      // ---- relay (peer): "my copy of the stage landed" -> the leader's fullp ----------
      const uint32_t rem0 = mapa_rank(smem_u32(fullp), 0);
      int it = 0;
      for (int t = t0; t < t1; ++t) {
        int p, ia, jb;
        bool own;
        if (!i8p_decode<STEPS>(g, K, t, rank, p, ia, jb, own)) continue;
        for (int pass = 0; pass < I8_NP; ++pass)
          for (int kc = 0; kc < NCH; ++kc, ++it) {
            const int s = it % ST;
            mbar_wait_trap<32>(&full[s], (it / ST) & 1);
            mbar_arrive_remote(rem0 + s * 8);
          }
      }
    } else if (lane == 0) {
      // ---- MMA issuer (leader) ---------------------------------------------------------
      int it = 0, ptr = 0, u = 0;
      int uses[I8_GROUPS] = {0, 0, 0, 0};
      PRB(long long c_full = 0, c_fullp = 0, c_chunk0 = 0; const long long c_start = clock64();)
      for (int t = t0; t < t1; ++t) {
        int p, ia, jb;
        bool own;
        if (!i8p_decode<STEPS>(g, K, t, rank, p, ia, jb, own)) continue;
#pragma unroll
        for (int pass = 0; pass < I8_NP; ++pass) {
          for (int kc = 0; kc < NCH; ++kc, ++it) {
            const int s = it % ST;
            PRB(long long c0 = clock64();)
            mbar_wait_trap(&full[s], (it / ST) & 1);
            PRB(c_full += clock64() - c0; c0 = clock64();)
            mbar_wait_trap(&fullp[s], (it / ST) & 1);
            PRB(c_fullp += clock64() - c0; c0 = clock64();)
            tc_fence_after();
            const uint32_t a0 = smem_u32(stage + s * I8P_STAGE), b0 = a0 + I8_BLK;
            if (pass == 0) i8p_chunk_mmas<0>(tm, a0, b0, kc == 0, tempty, ptr, uses);
            else i8p_chunk_mmas<1>(tm, a0, b0, kc == 0, tempty, ptr, uses);
            PRB(if (kc == 0) c_chunk0 += clock64() - c0;)
            umma_commit_pair(&empty[s]);
          }
          umma_commit_pair(&tfull[u & 1]);
          ++u;
#pragma unroll
          for (int gi = 0; gi < i8_ng(pass); ++gi) ++uses[(ptr + gi) & (I8_GROUPS - 1)];
          ptr = (ptr + i8_ng(pass)) & (I8_GROUPS - 1);
        }
      }
      PRB(if (K == LRS_I8_PROBE_K && ((blockIdx.x >> 1) % 499) == 0) printf(
              "PROBE2 mma cl %d items %d total %lld full_wait %lld fullp_wait %lld "
              "chunk0(tempty) %lld\n",
              blockIdx.x >> 1, t1 - t0, clock64() - c_start, c_full, c_fullp, c_chunk0);)
    }
  } else {
    // ---- epilogue (both CTAs): drain own TMEM rows, release to the leader, C update ----
    const int qd = w & 3, ch = (w - 2) >> 2, i = 32 * qd + lane;
    constexpr double BIAS = 4503601774854144.0;  // 2^52 + 2^31
    int u = 0, ptr = 0;
    for (int t = t0; t < t1; ++t) {
      int p, ia, jb;
      bool own;
      if (!i8p_decode<STEPS>(g, K, t, rank, p, ia, jb, own)) continue;
      double* C = ctile(p, ia, jb) + (int64_t)ch * I8_EPC * NB;
      const double si = exp2i(pn.ea[((int64_t)p * g.wl + ia) * NB + i]);
      if (w == 2) {
        const int* eb = pn.eb + ((int64_t)p * g.wu + jb) * NB;
#pragma unroll
        for (int r = 0; r < NB / 32; ++r) sj[lane + 32 * r] = exp2i(eb[lane + 32 * r]);
      }
      const uint32_t trow = tm + ((uint32_t)(32 * qd) << 16) + ch * I8_EPC;
      double acc[I8_EPC];
#pragma unroll
      for (int j = 0; j < I8_EPC; ++j) acc[j] = 0.0;
#pragma unroll
      for (int pass = 0; pass < I8_NP; ++pass, ++u) {
        mbar_wait_trap<128>(&tfull[u & 1], (u >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int gi = 0; gi < i8_ng(pass); ++gi) {
          const int slot = (ptr + gi) & (I8_GROUPS - 1);
          const double sc = exp2i(4 - 8 * (i8_top(pass) - gi));
#pragma unroll
          for (int h2 = 0; h2 < I8_EPC / 32; ++h2) {
            uint32_t v[32];
#pragma unroll
            for (int c8 = 0; c8 < 32; c8 += 8) tmem_ld8(trow + slot * NB + h2 * 32 + c8, v + c8);
            tmem_ld_wait();
            if (h2 == I8_EPC / 32 - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if (rank == 0) mbar_arrive1(&tempty[slot]);
                else mbar_arrive_remote(mapa_rank(smem_u32(&tempty[slot]), 0));
              }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j)
              acc[h2 * 32 + j] = fma(
                  __hiloint2double(0x43300000, (int)(v[j] ^ 0x80000000u)) - BIAS, sc,
                  acc[h2 * 32 + j]);
          }
        }
        ptr = (ptr + i8_ng(pass)) & (I8_GROUPS - 1);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * I8_EPI) : "memory");  // sj written
      if (own) {
#pragma unroll
        for (int j = 0; j < I8_EPC; ++j)
          red_add_f64(C + (int64_t)j * NB + i, -(acc[j] * si * sj[ch * I8_EPC + j]));
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * I8_EPI) : "memory");  // sj free
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its peer can still signal its barriers
  if (w == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(I8_TMEM)
                 : "memory");
  }
}

#endif  // !LRS_I8_ONEPASS

// ---- INT8 peak (roofline denominator): every SM issues M=128, N=256, K=32 MMAs from
// resident operands into 2 accumulators (the best-rate shape), 8 K-steps each
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  constexpr int N = 256, KK = 256;
  constexpr uint32_t ID = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                          ((uint32_t)(NB >> 4) << 24);
  const int w = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < (NB + N) * KK; e += blockDim.x) sm[e] = (uint8_t)((e * 7) & 63);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tb))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tb;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sm), b0 = a0 + NB * KK;
    for (int it = 0; it < iters; ++it)
      for (int a = 0; a < 2; ++a)
        for (int k = 0; k < KK / 32; ++k)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + a * N),
              "l"(umma_sdesc(a0 + 2 * k * NB * 16, NB * 16, 128)),
              "l"(umma_sdesc(b0 + 2 * k * N * 16, N * 16, 128)), "r"(ID),
              "r"((uint32_t)(it + k > 0)));
    umma_commit(&bar);
  }
  mbar_wait_trap<64>(&bar, 0);
  tc_fence_after();
  uint32_t v[8];
  tmem_ld8(tm + ((uint32_t)(32 * w) << 16), v);
  tmem_ld_wait();
  if (v[0] == 12345u) out[threadIdx.x] = (int)v[1];
  tc_fence_before();
  __syncthreads();
  if (w == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
}

double run_i8_peak(Ctx* c) {
  constexpr int smem = (NB + 256) * 256;
  LRS_CUDA(cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int* out = nullptr;
  LRS_CUDA(cudaMalloc(&out, 4096));
  cudaEvent_t e0, e1;
  LRS_CUDA(cudaEventCreate(&e0));
  LRS_CUDA(cudaEventCreate(&e1));
  const int iters = 2048;
  i8_peak_kernel<<<c->num_sms, 128, smem, c->stream>>>(8, out);
  LRS_CUDA(cudaEventRecord(e0, c->stream));
  i8_peak_kernel<<<c->num_sms, 128, smem, c->stream>>>(iters, out);
  LRS_CUDA(cudaEventRecord(e1, c->stream));
  LRS_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  LRS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  LRS_CUDA(cudaEventDestroy(e0));
  LRS_CUDA(cudaEventDestroy(e1));
  LRS_CUDA(cudaFree(out));
  const double ops = 2.0 * NB * 256 * 256 * 2.0 * iters * c->num_sms;
  return ops / (ms * 1e-3) / 1e12;
}

void launch_lu_i8_slice(Ctx* c, cudaStream_t s, const BandGeom& g, const double* tiles, int K,
                        int steps, const I8Panel& pn) {
  if (steps == 4)
    lu_i8_slice_kernel<4><<<dim3(g.wl + g.wu, NB / i8_slice_lines(4), g.P), I8_SLICE_THREADS, 0,
                            s>>>(g, tiles, K, pn);
  else
    lu_i8_slice_kernel<2><<<dim3(g.wl + g.wu, NB / i8_slice_lines(2), g.P), I8_SLICE_THREADS, 0,
                            s>>>(g, tiles, K, pn);
  LRS_LAUNCHED(c);
}

template <int KIND, int STEPS, bool CPLX = false>
static void i8_gemm_launch(Ctx* c, cudaStream_t s, const BandGeom& g, double* tiles, int K,
                           const I8Panel& pn) {
  static bool attr = false;
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(lu_i8_gemm_kernel<KIND, STEPS, CPLX>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)I8_SMEM));
    attr = true;
  }
  const int per = i8_per<KIND, STEPS>(g);
  const int total = per * g.P * I8_NH * (CPLX ? 2 : 1);
  if (total <= 0) return;
  // the look-ahead launch (kind 3, on the critical stream) takes fewer tiles per CTA
  static const int tpc3 = std::getenv("LRS_I8_TPC3") ? std::atoi(std::getenv("LRS_I8_TPC3"))
                                                      : LRS_I8_TPC3;
  // bulk: LRS_I8_TPC tiles per CTA (environment LRS_I8_TPC_RT overrides it at run time)
  // Small bulk launches (c2: 42 tiles per SM) run under a critical stream that waits for bulk
  // CTAs to retire: they take 4 tiles per CTA, large ones (c3: ~1000 per SM) LRS_I8_TPC = 8.
  static const int tpc_env = std::getenv("LRS_I8_TPC_RT") ? std::atoi(std::getenv("LRS_I8_TPC_RT"))
                                                           : 0;
  const int tpc4 = tpc_env > 0 ? tpc_env : (total < 200 * c->num_sms ? std::min(4, I8_TPC) : I8_TPC);
  const int tpc = KIND == 4 ? std::max(1, tpc4) : std::max(1, tpc3);
  const int grid = (total + tpc - 1) / tpc;
  lu_i8_gemm_kernel<KIND, STEPS, CPLX><<<grid, I8_THREADS, I8_SMEM, s>>>(g, tiles, K, pn, total,
                                                                         tpc);
  LRS_LAUNCHED(c);
}

// complex128 tiles (pairs only): the realified update of lu_i8_gemm_kernel<.., true>
void launch_lu_i8_slice_z(Ctx* c, cudaStream_t s, const BandGeom& g, const zc* tiles, int K,
                          const I8Panel& pn) {
  lu_i8_slice_z_kernel<2><<<dim3(g.wl + g.wu, NB / (I8_ZSLICE_THREADS / (2 * i8_nch(2))), g.P),
                            I8_ZSLICE_THREADS, 0, s>>>(g, tiles, K, pn);
  LRS_LAUNCHED(c);
}
void launch_lu_i8_gemm_z(Ctx* c, cudaStream_t s, const BandGeom& g, zc* tiles, int K, int kind,
                         const I8Panel& pn) {
  double* t = reinterpret_cast<double*>(tiles);
  if (kind == 4) i8_gemm_launch<4, 2, true>(c, s, g, t, K, pn);
  else i8_gemm_launch<3, 2, true>(c, s, g, t, K, pn);
}
// A' and B' panel bytes of the complex pair update (one buffer): A' twice the real A panel,
// B' four times the real B panel (two parts, K doubled)
size_t lu_i8_panel_bytes_z(const BandGeom& g) {
  return (size_t)g.P * (2 * g.wl + 4 * g.wu) * (i8_nch(2) * I8_BLK) +
         sizeof(int) * (size_t)g.P * (g.wl + g.wu) * NB;
}

#if !LRS_I8_ONEPASS
template <int STEPS>
static void i8_gemm2_launch(Ctx* c, cudaStream_t s, const BandGeom& g, double* tiles, int K,
                            const I8Panel& pn) {
  static bool attr = false;
  if (!attr) {
    LRS_CUDA(cudaFuncSetAttribute(lu_i8_gemm2_kernel<STEPS>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)I8P_SMEM));
    attr = true;
  }
  constexpr int D = STEPS;
  const int per = ((g.wl - D + 1) / 2) * (g.wu - D);
  const int total = per * g.P;
  if (total <= 0) return;
  static const int tpc = std::getenv("LRS_I8_2SM_TPC") ? std::atoi(std::getenv("LRS_I8_2SM_TPC"))
                                                        : I8_TPC;
  const int clusters = (total + tpc - 1) / tpc;
  lu_i8_gemm2_kernel<STEPS><<<2 * clusters, I8_THREADS, I8P_SMEM, s>>>(g, tiles, K, pn, total,
                                                                       tpc);
  LRS_LAUNCHED(c);
}

#endif

bool lu_i8_2sm() {
#if LRS_I8_ONEPASS
  return false;
#else
  const char* e = std::getenv("LRS_I8_2SM");
  return e && e[0] == '1';
#endif
}

void launch_lu_i8_gemm(Ctx* c, cudaStream_t s, const BandGeom& g, double* tiles, int K, int kind,
                       int steps, const I8Panel& pn) {
#if !LRS_I8_ONEPASS
  if (kind == 4 && lu_i8_2sm()) {
    if (steps == 4) i8_gemm2_launch<4>(c, s, g, tiles, K, pn);
    else i8_gemm2_launch<2>(c, s, g, tiles, K, pn);
    return;
  }
#endif
  if (steps == 4) {
    if (kind == 4) i8_gemm_launch<4, 4>(c, s, g, tiles, K, pn);
    else i8_gemm_launch<3, 4>(c, s, g, tiles, K, pn);
  } else {
    if (kind == 4) i8_gemm_launch<4, 2>(c, s, g, tiles, K, pn);
    else i8_gemm_launch<3, 2>(c, s, g, tiles, K, pn);
  }
}

}  // namespace lrs
