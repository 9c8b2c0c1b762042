/* Counter-based RNG shared by the input generators, the CPU oracle (through
 * liblrs_gen.so) and the CUDA library's host side (the Gaussian test block
 * Omega of the randomized spike SVD).
 *
 * SPEC.md:312 asks for "a named counter-based or equivalent splittable
 * generator with a 64-bit seed"; SPEC.md:314 derives one stream per
 * (seed, partition index, side).  We use splitmix64 (Steele, Lea, Flood 2014)
 * as both the key mixer and the counter hash, so draw i of stream s is a pure
 * function of (seed, s, i): results do not depend on thread count or order.
 *
 * Header-only, C99, no allocation.  Every consumer of these functions gets
 * bit-identical doubles on the same libm (Box-Muller uses log/sqrt/cos).
 */
#ifndef LRS_RNG_H
#define LRS_RNG_H

#include <math.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Stream ids.  Omega streams are LRS_STREAM_OMEGA + 2*partition + side. */
#define LRS_STREAM_RHS 0x52485331ull    /* "RHS1" */
#define LRS_STREAM_MATRIX 0x4D415431ull /* "MAT1" : matrix values / kappa */
#define LRS_STREAM_PATTERN 0x50415431ull /* "PAT1" : sampled sparsity pattern */
#define LRS_STREAM_OMEGA 0x4F4D0000ull  /* + 2*partition + side (T=0, W=1) */

static inline uint64_t lrs_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline uint64_t lrs_rng_key(uint64_t seed, uint64_t stream) {
  return lrs_splitmix64(seed ^ lrs_splitmix64(stream + 0x632BE59BD9B4E019ull));
}

static inline uint64_t lrs_rng_u64(uint64_t key, uint64_t ctr) {
  return lrs_splitmix64(key ^ lrs_splitmix64(ctr ^ 0xD1B54A32D192ED03ull));
}

/* Uniform double in [0, 1) with 53 random bits. */
static inline double lrs_rng_unit(uint64_t key, uint64_t ctr) {
  return (double)(lrs_rng_u64(key, ctr) >> 11) * 0x1.0p-53;
}

/* Uniform double in [-1, 1). */
static inline double lrs_rng_sym(uint64_t key, uint64_t ctr) {
  return 2.0 * lrs_rng_unit(key, ctr) - 1.0;
}

/* Standard normal, Box-Muller (cosine branch) on draws 2i and 2i+1. */
static inline double lrs_rng_normal(uint64_t key, uint64_t i) {
  const double u1 = 1.0 - lrs_rng_unit(key, 2 * i); /* (0, 1] */
  const double u2 = lrs_rng_unit(key, 2 * i + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
}

/* Uniform integer in [0, m), m > 0 (multiply-shift on the top 32 bits; the
 * bias is < m / 2^32 and irrelevant for pattern sampling). */
static inline uint64_t lrs_rng_below(uint64_t key, uint64_t ctr, uint64_t m) {
  const uint64_t hi = lrs_rng_u64(key, ctr) >> 32;
  return (hi * m) >> 32;
}

#ifdef __cplusplus
}
#endif

#endif /* LRS_RNG_H */
