// Internal types of liblrspike_cuda.so.  Not part of the public boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lrspike_capi.h"

namespace lrs {

constexpr int NB = 128;                    // band-factor tile size (rows = cols)
constexpr int64_t TILE_ELEMS = (int64_t)NB * NB;
constexpr int MAX_RHS = 16;                // columns per Krylov batch
constexpr int SOLVE_MAX_RHS = 48;          // columns per band-solve launch (DMMA path)
constexpr int SOLVE_GROUPS = 6;            // 16-column groups per launch (ready-flag sets):
                                           // 48 / 16 real, 96 / 16 complex (2 l <= 96)
constexpr double COND_LIMIT = 1e12;        // interface condition limit (oracle: COND_LIMIT)

// Error carried from deep inside the implementation to the C-ABI wrapper.
struct LrsError : std::runtime_error {
  lrs_status status;
  int64_t line = -1, row = -1, col = -1, column = -1, iface = -1;
  double cond = 0.0;
  LrsError(lrs_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define LRS_CUDA(call)                                                   \
  do {                                                                   \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) ::lrs::throw_cuda(e_, #call, __FILE__, __LINE__); \
  } while (0)

#define LRS_LAUNCHED(ctx)                                                  \
  do {                                                                     \
    (ctx)->launches++;                                                     \
    cudaError_t e_ = cudaGetLastError();                                   \
    if (e_ != cudaSuccess) ::lrs::throw_cuda(e_, "kernel launch", __FILE__, __LINE__); \
  } while (0)

// ---- stream-ordered caching device allocator (pool.cu) ---------------------------------
// Blocks freed on a stream are cached per stream and handed out again only to
// allocations on the same stream (stream order makes the reuse safe), so repeated
// factorize/solve calls do not pay cudaMalloc/cudaFree (which also synchronize the
// device).  The stream key comes from the C-ABI call in progress (set by guard()).
void* pool_alloc(cudaStream_t s, size_t bytes, size_t* rounded);
void pool_release(cudaStream_t s, void* p, size_t bytes);
void pool_stream_open(cudaStream_t s);
void pool_stream_retire(cudaStream_t s);
size_t pool_cached_bytes();
cudaStream_t& current_pool_stream();  // thread-local

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t bytes = 0;
  cudaStream_t key = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) pool_release(key, p, bytes);
    p = nullptr;
    n = 0;
    bytes = 0;
  }
  void alloc(size_t count) {
    reset();
    if (count == 0) return;
    key = current_pool_stream();
    p = static_cast<T*>(pool_alloc(key, count * sizeof(T), &bytes));
    n = count;
  }
  T* get() const { return p; }
};

// Kernel classes for the optional per-class CUDA-event timing (lrs_ctx_set_profiling).
enum KClass {
  K_LU_DIAG = 0, K_LU_PANEL, K_LU_UPDATE, K_SOLVE, K_SOLVE_ADJ, K_SPMV, K_IFACE, K_RECOVERY,
  K_KRYLOV, K_SETUP, K_SPIKE_SOLVE, K_NCLASS
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream_hi = nullptr;  // high-priority side stream (LU look-ahead critical path)
  bool own_stream = false;
  // live lrs_mat / lrs_fact handles created on this context: lrs_ctx_destroy defers the
  // teardown (stream, pool, staging) until the last of them is destroyed
  int64_t children = 0;
  bool closing = false;
  int64_t launches = 0;
  lrs_error_info last{};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int num_sms = 148;
  bool in_setup = false;  // band solves issued by the spike construction (profiling class)
  bool solve_fma1 = true;  // one-RHS band solves use the FMA kernel (false: DMMA, solve_block)
  // pinned staging ring for small host->device uploads (job tables, Krylov scalars):
  // a pageable cudaMemcpyAsync would first wait for the stream to drain.
  char* stage = nullptr;
  size_t stage_cap = 0, stage_pos = 0;
  void stage_h2d(void* dst, const void* src, size_t bytes);  // pool.cu
  // pinned landing buffer of the Krylov dot products (allocated once: cudaMallocHost /
  // cudaFreeHost per solve cost milliseconds and synchronize the device)
  static constexpr size_t DOTS_HOST_BYTES = sizeof(double) * 64 * MAX_RHS * 2 * 3;  // 3 slots
  double* dots_host = nullptr;
  // spike test matrices Omega: page-locked staging (grown on demand, reused across
  // factorizations) and the copy stream a host thread uploads them on while the band LU runs
  double* omega_host = nullptr;
  size_t omega_host_cap = 0;
  cudaStream_t stream_copy = nullptr;
  cudaEvent_t ev_omega = nullptr;
  // profiling: (class, start, end) event triples, summed on demand
  bool prof = false;
  uint32_t prof_mask = ~0u;  // classes timed while profiling (bit k: class k)
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> prof_class;
  std::vector<cudaEvent_t> prof_ev;  // 2 per record
  double prof_ms[K_NCLASS] = {0};
  int64_t prof_cnt[K_NCLASS] = {0};
  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void collect() {
    if (prof_class.empty()) return;
    cudaStreamSynchronize(stream);
    for (size_t i = 0; i < prof_class.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prof_ev[2 * i], prof_ev[2 * i + 1]);
      prof_ms[prof_class[i]] += ms;
      prof_cnt[prof_class[i]] += 1;
      ev_pool.push_back(prof_ev[2 * i]);
      ev_pool.push_back(prof_ev[2 * i + 1]);
    }
    prof_class.clear();
    prof_ev.clear();
  }
};

// RAII event pair around one launch (no-op unless profiling is on).
struct ProfScope {
  Ctx* c;
  int cls;
  cudaStream_t s;
  cudaEvent_t b = nullptr;
  ProfScope(Ctx* ctx, int k, cudaStream_t st = nullptr) : c(ctx), cls(k), s(st ? st : ctx->stream) {
    if (c->prof && ((c->prof_mask >> cls) & 1u)) {
      b = c->take_event();
      cudaEventRecord(b, s);
    }
  }
  ~ProfScope() {
    if (b) {
      cudaEvent_t e = c->take_event();
      cudaEventRecord(e, s);
      c->prof_class.push_back(cls);
      c->prof_ev.push_back(b);
      c->prof_ev.push_back(e);
      if (c->prof_class.size() > (size_t(1) << 22)) c->collect();
    }
  }
};

struct Mat {
  Ctx* ctx = nullptr;
  int64_t n = 0, nnz = 0;
  int32_t scalar = LRS_F64;
  int64_t ku = 0, kl = 0, k = 0;
  double diag_weight = 0.0, band_density = 0.0;
  DevBuf<int> row_ptr, col_idx;      // CSR of A (int32 on device; n, nnz < 2^31)
  DevBuf<double> vals;
  DevBuf<int> trow_ptr, tcol_idx;    // CSR of A^T (spike adjoint couplings)
  DevBuf<double> tvals;
  int symmetric = -1;                // A == A^T bitwise: -1 not checked yet, 0, 1
};

struct Fact;  // defined in fact.h

// ------------------------------------------------------------------------------------
// kernel launchers (implemented in the .cu files)
// ------------------------------------------------------------------------------------

// spmv.cu
// rows [row_lo, row_hi) of y (+)= A x; mode: 0 y = A x, 1 y += A x, 2 y = b - A x.
// x, y, b are full-length (global row indexing).
void launch_spmv(Ctx* c, const Mat* m, const double* x, int64_t ldx, double* y, int64_t ldy,
                 int nrhs, int mode, const double* b, int64_t ldb, int64_t row_lo = 0,
                 int64_t row_hi = -1);

}  // namespace lrs
