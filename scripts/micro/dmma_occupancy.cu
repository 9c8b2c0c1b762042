// DMMA.8x8x4 throughput vs occupancy and accumulator count (development microbenchmark).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_occ dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC, int NLD>
__global__ void kern(double* out, const double* src, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = src[i % 64];
  __syncthreads();
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    double fa[NLD];
#pragma unroll
    for (int q = 0; q < NLD; ++q) fa[q] = sm[(it * 37 + q * 132 + lane) & 4095];
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i][0], acc[i][1], fa[i % NLD], fa[(i / NLD) % NLD]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int NACC, int NLD>
void run(int threads, int blocks_per_sm, int sms, double* out, const double* src) {
  const int iters = 4000;
  const int blocks = sms * blocks_per_sm;
  kern<NACC, NLD><<<blocks, threads>>>(out, src, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<NACC, NLD><<<blocks, threads>>>(out, src, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 512.0 * NACC * iters * (threads / 32) * (double)blocks;
  printf("nacc %2d nld %2d threads %4d blocks/SM %d warps/SMSP %2d : %.1f TF/s\n", NACC, NLD,
         threads, blocks_per_sm, threads / 32 * blocks_per_sm / 4, flops / ms / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out, *src;
  cudaMalloc(&out, 8192);
  cudaMalloc(&src, 8192);
  cudaMemset(src, 0, 8192);
  run<8, 4>(256, 4, sms, out, src);
  run<32, 12>(256, 1, sms, out, src);
  run<32, 12>(128, 2, sms, out, src);
  run<32, 12>(128, 1, sms, out, src);
  run<32, 12>(256, 2, sms, out, src);
  run<32, 0 + 12>(512, 1, sms, out, src);
  run<16, 8>(256, 2, sms, out, src);
  run<16, 8>(512, 1, sms, out, src);
  run<64, 16>(128, 1, sms, out, src);
  run<64, 16>(256, 1, sms, out, src);
  run<32, 12>(384, 1, sms, out, src);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
