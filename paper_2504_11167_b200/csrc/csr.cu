// Device-side CSR transpose (the CSR of A^T used by the spike range finder's adjoint
// coupling products).  Structural and deterministic: column counts, a
// prefix sum, an atomic scatter, then every transposed row sorted by its (original) row
// index -- the same arrays a sequential counting sort produces.
#include "common.cuh"
#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

__global__ void csr_count_cols_kernel(const int* __restrict__ ci, int64_t nnz, int* cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ci[e] + 1], 1);
}

__global__ void csr_scatter_kernel(const int* __restrict__ rp, const int* __restrict__ ci,
                                   const double* __restrict__ va, int64_t n, int w, int* pos,
                                   int* tci, double* tva) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int q = rp[r]; q < rp[r + 1]; ++q) {
    const int slot = atomicAdd(&pos[ci[q]], 1);
    tci[slot] = (int)r;
    for (int e = 0; e < w; ++e) tva[(int64_t)slot * w + e] = va[(int64_t)q * w + e];
  }
}

__global__ void csr_sort_segments_kernel(const int* __restrict__ trp, int64_t n, int w, int* tci,
                                         double* tva) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int s = trp[c], e = trp[c + 1];
  for (int i = s + 1; i < e; ++i) {  // insertion sort by row index (segments are short)
    const int key = tci[i];
    double v0 = tva[(int64_t)i * w], v1 = w == 2 ? tva[(int64_t)i * w + 1] : 0.0;
    int j = i - 1;
    while (j >= s && tci[j] > key) {
      tci[j + 1] = tci[j];
      for (int q = 0; q < w; ++q) tva[(int64_t)(j + 1) * w + q] = tva[(int64_t)j * w + q];
      --j;
    }
    tci[j + 1] = key;
    tva[(int64_t)(j + 1) * w] = v0;
    if (w == 2) tva[(int64_t)(j + 1) * w + 1] = v1;
  }
}

// inclusive prefix sum of n ints (out may alias in): per-1024 block scans, a scan of the
// block totals in one CTA, and the block offsets added back
constexpr int SCAN_B = 1024;

__global__ void __launch_bounds__(SCAN_B) scan_blocks_kernel(const int* in, int* out, int64_t n,
                                                             int* totals) {
  __shared__ int s[SCAN_B];
  const int64_t i = (int64_t)blockIdx.x * SCAN_B + threadIdx.x;
  s[threadIdx.x] = i < n ? in[i] : 0;
  __syncthreads();
  for (int o = 1; o < SCAN_B; o <<= 1) {
    const int v = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += v;
    __syncthreads();
  }
  if (i < n) out[i] = s[threadIdx.x];
  if (threadIdx.x == SCAN_B - 1) totals[blockIdx.x] = s[SCAN_B - 1];
}

__global__ void __launch_bounds__(SCAN_B) scan_totals_kernel(int* totals, int nb) {
  __shared__ int carry;
  __shared__ int s[SCAN_B];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += SCAN_B) {
    const int i = b0 + threadIdx.x;
    s[threadIdx.x] = i < nb ? totals[i] : 0;
    __syncthreads();
    for (int o = 1; o < SCAN_B; o <<= 1) {
      const int v = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += v;
      __syncthreads();
    }
    if (i < nb) totals[i] = carry + s[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) carry += s[SCAN_B - 1];
    __syncthreads();
  }
}

__global__ void scan_add_kernel(int* out, int64_t n, const int* totals) {
  const int64_t i = (int64_t)blockIdx.x * SCAN_B + threadIdx.x;
  if (blockIdx.x > 0 && i < n) out[i] += totals[blockIdx.x - 1];
}

void launch_csr_transpose(Ctx* c, Mat* m) {
  const int64_t n = m->n, nnz = m->nnz;
  const int w = m->scalar == LRS_C128 ? 2 : 1;
  m->trow_ptr.alloc(n + 1);
  m->tcol_idx.alloc(std::max<int64_t>(nnz, 1));
  m->tvals.alloc(std::max<int64_t>(nnz, 1) * w);
  DevBuf<int> cnt, pos;
  cnt.alloc(n + 1);
  pos.alloc(std::max<int64_t>(n, 1));
  LRS_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int) * (n + 1), c->stream));
  ProfScope ps_(c, K_SETUP);
  if (nnz > 0) {
    csr_count_cols_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(m->col_idx.get(), nnz, cnt.get());
    LRS_LAUNCHED(c);
  }
  {
    const int64_t len = n + 1;
    const int nb = (int)((len + SCAN_B - 1) / SCAN_B);
    DevBuf<int> totals;
    totals.alloc(nb);
    scan_blocks_kernel<<<nb, SCAN_B, 0, c->stream>>>(cnt.get(), m->trow_ptr.get(), len, totals.get());
    LRS_LAUNCHED(c);
    scan_totals_kernel<<<1, SCAN_B, 0, c->stream>>>(totals.get(), nb);
    LRS_LAUNCHED(c);
    scan_add_kernel<<<nb, SCAN_B, 0, c->stream>>>(m->trow_ptr.get(), len, totals.get());
    LRS_LAUNCHED(c);
  }
  if (nnz == 0 || n == 0) return;
  LRS_CUDA(cudaMemcpyAsync(pos.get(), m->trow_ptr.get(), sizeof(int) * n, cudaMemcpyDeviceToDevice,
                           c->stream));
  const unsigned blocks = (unsigned)((n + 255) / 256);
  csr_scatter_kernel<<<blocks, 256, 0, c->stream>>>(m->row_ptr.get(), m->col_idx.get(),
                                                     m->vals.get(), n, w, pos.get(),
                                                     m->tcol_idx.get(), m->tvals.get());
  LRS_LAUNCHED(c);
  csr_sort_segments_kernel<<<blocks, 256, 0, c->stream>>>(m->trow_ptr.get(), n, w,
                                                           m->tcol_idx.get(), m->tvals.get());
  LRS_LAUNCHED(c);
}

// int64 column indices (the reference's index_t, matrix.hpp:11) -> the device's int32
__global__ void narrow_i64_kernel(const long long* __restrict__ src, int* __restrict__ dst,
                                  int64_t cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = (int)src[e];
}
void launch_narrow_i64(Ctx* c, const int64_t* src, int* dst, int64_t cnt) {
  if (cnt <= 0) return;
  narrow_i64_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(
      reinterpret_cast<const long long*>(src), dst, cnt);
  LRS_LAUNCHED(c);
}

// A == A^T bitwise (plain transpose; w doubles per value): the transposed CSR (rows sorted by
// column) equals the CSR itself
__global__ void csr_equal_kernel(const int* __restrict__ rp, const int* __restrict__ trp,
                                 int64_t n1, const int* __restrict__ ci,
                                 const int* __restrict__ tci, const long long* __restrict__ va,
                                 const long long* __restrict__ tva, int64_t nnz, int w,
                                 int* differ) {
  bool bad = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    bad |= ci[e] != tci[e];
    for (int q = 0; q < w; ++q) bad |= va[e * w + q] != tva[e * w + q];
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n1;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= rp[i] != trp[i];
  if (bad) *differ = 1;
}

bool mat_is_symmetric(Ctx* c, Mat* m) {
  if (m->symmetric >= 0) return m->symmetric == 1;
  if (m->nnz == 0 || m->n == 0) return (m->symmetric = 0) == 1;
  DevBuf<int> differ;
  differ.alloc(1);
  LRS_CUDA(cudaMemsetAsync(differ.get(), 0, sizeof(int), c->stream));
  {
    ProfScope ps_(c, K_SETUP);
    csr_equal_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(
        m->row_ptr.get(), m->trow_ptr.get(), m->n + 1, m->col_idx.get(), m->tcol_idx.get(),
        reinterpret_cast<const long long*>(m->vals.get()),
        reinterpret_cast<const long long*>(m->tvals.get()), m->nnz,
        m->scalar == LRS_C128 ? 2 : 1, differ.get());
    LRS_LAUNCHED(c);
  }
  int h = 1;
  LRS_CUDA(cudaMemcpyAsync(&h, differ.get(), sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  LRS_CUDA(cudaStreamSynchronize(c->stream));
  m->symmetric = h ? 0 : 1;
  return m->symmetric == 1;
}

}  // namespace lrs
