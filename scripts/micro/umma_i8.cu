// tcgen05.mma kind::i8 (INT8 x INT8 -> INT32 in TMEM) correctness + throughput probe
// (development microbenchmark for the integer-sliced FP64 trailing update).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8 umma_i8.cu
//
// Operands are K-major, no swizzle: core matrices of 8 rows x 16 bytes (128 B contiguous);
// core (row group g, K chunk kc) of an R-row operand sits at (kc * R/8 + g) * 128 bytes, so
// SBO (next 8-row group) = 128 B and LBO (next 16-byte K chunk) = R/8 * 128 B.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)                      // D: s32
         | (1u << 7) | (1u << 10)       // A, B: signed int8
         | ((uint32_t)(N >> 3) << 17)   // N / 8
         | ((uint32_t)(M >> 4) << 24);  // M / 16
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// A-operand collector: 0 none, 1 fill (keep), 2 use (reuse + keep), 3 lastuse (reuse)
template <int COLL>
__device__ __forceinline__ void mma_i8c(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  if (COLL == 0) mma_i8(tmem_d, a, b, idesc, acc);
  else if (COLL == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if (COLL == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, unsigned parity) {
  for (long i = 0; !mbar_try(bar, parity); ++i)
    if (i > (1l << 26)) __trap();
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// copy a row-major [R][K] int8 matrix into the core-matrix layout
__device__ void to_cores(int8_t* dst, const int8_t* src, int R, int K) {
  for (int e = threadIdx.x; e < R * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const int g = r >> 3, kc = k >> 4;
    dst[(kc * (R / 8) + g) * 128 + (r & 7) * 16 + (k & 15)] = src[e];
  }
}

template <int N>
__global__ void __launch_bounds__(128, 1) check_kernel(const int8_t* A, const int8_t* B, int K,
                                                       int* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  int8_t* sa = reinterpret_cast<int8_t*>(sm);
  int8_t* sb = sa + 128 * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5;
  to_cores(sa, A, 128, K);
  to_cores(sb, B, N, K);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)),
                 "n"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t lboA = 128 / 8 * 128, lboB = N / 8 * 128;
    for (int k = 0; k < K / 32; ++k)
      mma_i8(tm, sdesc(smem_u32(sa) + 2 * k * lboA, lboA, 128),
             sdesc(smem_u32(sb) + 2 * k * lboB, lboB, 128), idesc_i8(128, N), k > 0);
    mma_commit(&bar);
  }
  mbar_wait_bounded(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = threadIdx.x;  // warp w reads lanes 32w..32w+31
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    tmem_ld8(tm + ((uint32_t)(32 * w) << 16) + c, v);
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm),
                 "n"(N < 32 ? 32 : N));
}

// throughput: each CTA (one per SM) issues `iters` x (K/32) MMAs of 128 x N x 32 from
// resident shared-memory operands into NACC accumulators (NACC * N TMEM columns)
template <int N, int NACC>
__global__ void __launch_bounds__(128) tput_kernel(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int K = 256;
  int8_t* sa = reinterpret_cast<int8_t*>(sm);
  int8_t* sb = sa + 128 * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < (128 + N) * K; e += blockDim.x) sa[e] = (int8_t)((e * 7) & 63);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr int COLS = NACC * N < 32 ? 32 : NACC * N;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)),
                 "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t lboA = 128 / 8 * 128, lboB = N / 8 * 128;
    for (int it = 0; it < iters; ++it)
      for (int a = 0; a < NACC; ++a)
        for (int k = 0; k < K / 32; ++k)
          mma_i8(tm + a * N, sdesc(smem_u32(sa) + 2 * k * lboA, lboA, 128),
                 sdesc(smem_u32(sb) + 2 * k * lboB, lboB, 128), idesc_i8(128, N), it + k > 0);
    mma_commit(&bar);
  }
  mbar_wait_bounded(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[8];
  tmem_ld8(tm + ((uint32_t)(32 * w) << 16), v);
  if (v[0] == 12345u) out[threadIdx.x] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(COLS));
}

// the Ozaki chunk: 8 A slices (128 x 32) and 8 B slices (64 x 32) in one 48 KB stage, 36
// MMAs (p + q <= 9) into 8 group accumulators; `stages` distinct stages cycled
__global__ void __launch_bounds__(128, 1) slices_kernel(int iters, int stages, int* out, int order) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < stages * 49152; e += blockDim.x) sm[e] = (uint8_t)((e * 7) & 63);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const uint32_t a0 = smem_u32(sm) + (it % stages) * 49152, b0 = a0 + 32768;
      if (order == 0) {
        for (int d = 2; d <= 9; ++d)
          for (int p = 1; p < d; ++p)
            mma_i8(tm + (d - 2) * 64, sdesc(a0 + (p - 1) * 4096, 2048, 128),
                   sdesc(b0 + (d - p - 1) * 2048, 1024, 128), idesc_i8(128, 64), it > 0 || p > 1);
      } else if (order == 1) {
        for (int p = 1; p <= 8; ++p)
          for (int q = 1; q <= 9 - p; ++q)
            mma_i8(tm + (p + q - 2) * 64, sdesc(a0 + (p - 1) * 4096, 2048, 128),
                   sdesc(b0 + (q - 1) * 2048, 1024, 128), idesc_i8(128, 64), it > 0 || p > 1);
      } else {
#pragma unroll
        for (int p = 1; p <= 8; ++p)
#pragma unroll
          for (int q = 1; q <= 9 - p; ++q) {
            const uint64_t ad = sdesc(a0 + (p - 1) * 4096, 2048, 128);
            const uint64_t bd = sdesc(b0 + (q - 1) * 2048, 1024, 128);
            const uint32_t dd = tm + (p + q - 2) * 64, ac = it > 0 || p > 1;
            if (p == 8) mma_i8c<0>(dd, ad, bd, idesc_i8(128, 64), ac);
            else if (q == 1) mma_i8c<1>(dd, ad, bd, idesc_i8(128, 64), ac);
            else if (q == 9 - p) mma_i8c<3>(dd, ad, bd, idesc_i8(128, 64), ac);
            else mma_i8c<2>(dd, ad, bd, idesc_i8(128, 64), ac);
          }
      }
    }
    mma_commit(&bar);
  }
  mbar_wait_bounded(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[8];
  tmem_ld8(tm + ((uint32_t)(32 * w) << 16), v);
  if (v[0] == 12345u) out[threadIdx.x] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static void slices(int sms, int stages, int order) {
  const int smem = stages * 49152;
  CK(cudaFuncSetAttribute(slices_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int* out;
  CK(cudaMalloc(&out, 4096));
  slices_kernel<<<sms, 128, smem>>>(8, stages, out, order);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 2048;
  CK(cudaEventRecord(e0));
  slices_kernel<<<sms, 128, smem>>>(iters, stages, out, order);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double ops = 2.0 * 128 * 64 * 32 * 36.0 * iters * sms;
  std::printf("slices order=%d stages=%d: %.3f ms  %.0f TOPS int8  (%.1f ns per MMA per SM)\n", order, stages, ms,
              ops / ms / 1e9, ms * 1e6 / (36.0 * iters));
  CK(cudaFree(out));
}

// cta_group::2: a cluster of 2 CTAs (one per SM of a TPC) computes a 256 x 64 block; each
// CTA holds its 128 A rows (8 slices x 4 KB) and 32 of the 64 B rows (8 slices x 1 KB); the
// leader issues the slices-pattern MMAs (p outer with the A collector) for both
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int e = threadIdx.x; e < 40960; e += blockDim.x) sm[e] = (uint8_t)((e * 7 + rank) & 63);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  constexpr uint32_t ID = (2u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (16u << 24);
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 32768;
    for (int it = 0; it < iters; ++it)
      for (int p = 1; p <= 8; ++p)
        for (int q = 1; q <= 9 - p; ++q) {
          const uint64_t ad = sdesc(a0 + (p - 1) * 4096, 2048, 128);
          const uint64_t bd = sdesc(b0 + (q - 1) * 1024, 512, 128);
          const uint32_t dd = tm + (p + q - 2) * 64, ac = it > 0 || p > 1;
          if (p == 8 || q == 1 && p == 8)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dd),
                         "l"(ad), "l"(bd), "r"(ID), "r"(ac));
          else if (q == 1)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dd),
                         "l"(ad), "l"(bd), "r"(ID), "r"(ac));
          else if (q == 9 - p)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dd),
                         "l"(ad), "l"(bd), "r"(ID), "r"(ac));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dd),
                         "l"(ad), "l"(bd), "r"(ID), "r"(ac));
        }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((unsigned short)3)
        : "memory");
  }
  mbar_wait_bounded(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[8];
  tmem_ld8(tm + ((uint32_t)(32 * w) << 16), v);
  if (v[0] == 12345u) out[threadIdx.x] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// plain pair throughput: NACC accumulators of N columns, 8 K-steps each, A and B resident
template <int N, int NACC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_tput_kernel(int iters, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  constexpr int K = 256;
  for (int e = threadIdx.x; e < (128 + N / 2) * K; e += blockDim.x) sm[e] = (uint8_t)((e * 7 + rank) & 63);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  constexpr uint32_t ID = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (16u << 24);
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 128 * K;
    const uint32_t lboA = 2048, lboB = (N / 2) / 8 * 128;
    for (int it = 0; it < iters; ++it)
      for (int a = 0; a < NACC; ++a)
        for (int k = 0; k < K / 32; ++k)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + a * N),
                       "l"(sdesc(a0 + 2 * k * lboA, lboA, 128)), "l"(sdesc(b0 + 2 * k * lboB, lboB, 128)),
                       "r"(ID), "r"((uint32_t)(it + k > 0)));
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((unsigned short)3)
        : "memory");
  }
  mbar_wait_bounded(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[8];
  tmem_ld8(tm + ((uint32_t)(32 * w) << 16), v);
  if (v[0] == 12345u) out[threadIdx.x] = v[1];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int NACC>
static void pair_tput(int sms) {
  const int smem = (128 + N / 2) * 256;
  CK(cudaFuncSetAttribute(pair_tput_kernel<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int* out;
  CK(cudaMalloc(&out, 4096));
  const int grid = sms & ~1;
  pair_tput_kernel<N, NACC><<<grid, 128, smem>>>(4, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 4096 / NACC;
  CK(cudaEventRecord(e0));
  pair_tput_kernel<N, NACC><<<grid, 128, smem>>>(iters, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double ops = 2.0 * 256 * N * 256 * (double)iters * NACC * (grid / 2);
  std::printf("pair tput M=256 N=%3d acc=%d: %.3f ms  %.0f TOPS int8\n", N, NACC, ms, ops / ms / 1e9);
  CK(cudaFree(out));
}

static void pair(int sms) {
  const int smem = 40960;
  CK(cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int* out;
  CK(cudaMalloc(&out, 4096));
  const int grid = sms & ~1;
  pair_kernel<<<grid, 128, smem>>>(8, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 2048;
  CK(cudaEventRecord(e0));
  pair_kernel<<<grid, 128, smem>>>(iters, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double ops = 2.0 * 256 * 64 * 32 * 36.0 * iters * (grid / 2);
  std::printf("pair M=256 N=64 slices+collector: %.3f ms  %.0f TOPS int8  (%.1f ns per MMA)\n", ms,
              ops / ms / 1e9, ms * 1e6 / (36.0 * iters));
  CK(cudaFree(out));
}

template <int N>
static bool check(int K) {
  std::vector<int8_t> A(128 * K), B(N * K);
  unsigned s = 12345u + N + K;
  for (auto& x : A) x = (int8_t)((s = s * 1103515245u + 12345u) >> 24);
  for (auto& x : B) x = (int8_t)((s = s * 1103515245u + 12345u) >> 24);
  int8_t *dA, *dB;
  int* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const int smem = (128 + N) * K;
  CK(cudaFuncSetAttribute(check_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  check_kernel<N><<<1, 128, smem>>>(dA, dB, K, dD);
  CK(cudaDeviceSynchronize());
  std::vector<int> D(128 * N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      int ref = 0;
      for (int k = 0; k < K; ++k) ref += (int)A[i * K + k] * (int)B[j * K + k];
      if (ref != D[i * N + j] && bad++ < 5)
        std::printf("  mismatch (%d,%d): got %d want %d\n", i, j, D[i * N + j], ref);
    }
  std::printf("check N=%d K=%d: %s (%ld bad)\n", N, K, bad ? "FAIL" : "ok", bad);
  CK(cudaFree(dA));
  CK(cudaFree(dB));
  CK(cudaFree(dD));
  return bad == 0;
}

template <int N, int NACC>
static void tput(int sms, int per_sm = 1) {
  const int smem = (128 + N) * 256;
  CK(cudaFuncSetAttribute(tput_kernel<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          smem));
  int* out;
  CK(cudaMalloc(&out, 4096));
  const int iters = 4096 / NACC;
  tput_kernel<N, NACC><<<sms, 128, smem>>>(4, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  tput_kernel<N, NACC><<<sms * per_sm, 128, smem>>>(iters, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double ops = 2.0 * 128 * N * 256 * (double)iters * NACC * sms * per_sm;
  std::printf("tput M=128 N=%3d acc=%d ctas/sm=%d: %.3f ms  %.0f TOPS int8\n", N, NACC, per_sm, ms,
              ops / ms / 1e9);
  CK(cudaFree(out));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  bool ok = check<64>(32) && check<64>(256) && check<128>(256) && check<256>(64) &&
            check<32>(128);
  if (!ok) return 1;
  tput<64, 8>(sms);
  tput<128, 4>(sms);
  tput<256, 2>(sms);
  tput<64, 8>(sms);
  tput<32, 8>(sms, 1);
  tput<32, 8>(sms, 2);
  tput<64, 4>(sms, 2);
  slices(sms, 4, 0);
  slices(sms, 4, 1);
  slices(sms, 4, 2);
  pair(sms);
  pair_tput<64, 8>(sms);
  pair_tput<128, 4>(sms);
  pair_tput<256, 2>(sms);
  return 0;
}
