// The extern "C" boundary (include/lrspike_capi.h).  Every entry point maps the
// internal LrsError to an lrs_status and records the payload the reference's
// exception classes carry (proj/core/include/lrspike/errors.hpp:11-94).
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstring>
#include <memory>
#include <new>
#include <thread>
#include <vector>

#include "fact.h"
#include "kernels.h"
#include "lrs_internal.h"

struct lrs_ctx : lrs::Ctx {};
struct lrs_mat : lrs::Mat {};
struct lrs_fact : lrs::Fact {};

namespace lrs {

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  const lrs_status s = (e == cudaErrorMemoryAllocation) ? LRS_ERR_OOM : LRS_ERR_CUDA;
  throw LrsError(s, std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" +
                        std::to_string(line) + ")");
}

static thread_local lrs_error_info g_last{};

static void record(Ctx* c, const LrsError& e) {
  lrs_error_info info{};
  info.status = e.status;
  std::snprintf(info.message, sizeof(info.message), "%s", e.what());
  info.line = e.line;
  info.row = e.row;
  info.col = e.col;
  info.column = e.column;
  info.interface_index = e.iface;
  info.cond_estimate = e.cond;
  g_last = info;
  if (c) c->last = info;
}

// Restores the thread's pool stream key on scope exit.
struct PoolScope {
  cudaStream_t prev;
  explicit PoolScope(Ctx* c) : prev(current_pool_stream()) {
    current_pool_stream() = c ? c->stream : nullptr;
  }
  ~PoolScope() { current_pool_stream() = prev; }
};

template <class F>
static lrs_status guard(Ctx* c, F&& fn) {
  PoolScope ps(c);
  try {
    fn();
    return LRS_OK;
  } catch (const LrsError& e) {
    record(c, e);
    return e.status;
  } catch (const std::bad_alloc&) {
    LrsError e(LRS_ERR_OOM, "host allocation failed");
    record(c, e);
    return LRS_ERR_OOM;
  } catch (const std::exception& ex) {
    LrsError e(LRS_ERR_CUDA, ex.what());
    record(c, e);
    return LRS_ERR_CUDA;
  }
}

// Host staging of a user buffer: returns a device pointer (uploading HOST data).
// w = doubles per scalar (1: float64, 2: interleaved complex128).
static void* dev_in(Ctx* c, const void* src, int64_t ld, int64_t rows, int64_t cols, int32_t mem,
                    DevBuf<double>& own, int64_t* ld_out, int w) {
  if (mem == LRS_MEM_DEVICE) {
    *ld_out = ld;
    return const_cast<void*>(src);
  }
  const size_t es = sizeof(double) * w;
  own.alloc((size_t)std::max<int64_t>(1, rows * cols) * w);
  if (rows * cols > 0)
    LRS_CUDA(cudaMemcpy2DAsync(own.get(), es * rows, src, es * ld, es * rows, cols,
                               cudaMemcpyHostToDevice, c->stream));
  *ld_out = rows;
  return own.get();
}

static void dev_out_finish(Ctx* c, void* dst, int64_t ld, const void* dev, int64_t rows,
                           int64_t cols, int32_t mem, int w) {
  if (mem == LRS_MEM_DEVICE) return;
  const size_t es = sizeof(double) * w;
  if (rows * cols > 0)
    LRS_CUDA(cudaMemcpy2DAsync(dst, es * ld, dev, es * rows, es * rows, cols,
                               cudaMemcpyDeviceToHost, c->stream));
  LRS_CUDA(cudaStreamSynchronize(c->stream));
}

static void check_mem(int32_t mem) {
  if (mem != LRS_MEM_HOST && mem != LRS_MEM_DEVICE)
    throw LrsError(LRS_ERR_PARAMETER, "mem must be LRS_MEM_HOST or LRS_MEM_DEVICE");
}

}  // namespace lrs

using namespace lrs;

extern "C" {

const char* lrs_status_string(lrs_status s) {
  switch (s) {
    case LRS_OK: return "ok";
    case LRS_ERR_PARSE: return "ParseError";
    case LRS_ERR_UNSUPPORTED_FIELD: return "UnsupportedFieldError";
    case LRS_ERR_DIMENSION: return "DimensionError";
    case LRS_ERR_SINGULAR_SCALING: return "SingularScalingError";
    case LRS_ERR_LAYOUT: return "LayoutError";
    case LRS_ERR_NOT_BLOCK_TRIDIAGONAL: return "NotBlockTridiagonalError";
    case LRS_ERR_SINGULAR_BLOCK: return "SingularBlockError";
    case LRS_ERR_PARAMETER: return "ParameterError";
    case LRS_ERR_ILL_CONDITIONED_INTERFACE: return "IllConditionedInterfaceError";
    case LRS_ERR_BREAKDOWN: return "BreakdownError";
    case LRS_ERR_CUDA: return "CudaError";
    case LRS_ERR_OOM: return "OutOfMemory";
    case LRS_ERR_NCCL: return "NcclError";
    case LRS_ERR_NOT_IMPLEMENTED: return "NotImplemented";
    case LRS_ERR_PRECOND_FAILURE: return "PreconditionerFailureError";
  }
  return "unknown";
}

lrs_status lrs_ctx_create(int device, void* stream, lrs_ctx** out) {
  if (!out) return LRS_ERR_PARAMETER;
  *out = nullptr;
  std::unique_ptr<lrs_ctx> c(new (std::nothrow) lrs_ctx());
  if (!c) return LRS_ERR_OOM;
  lrs_status s = guard(nullptr, [&] {
    int count = 0;
    LRS_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw LrsError(LRS_ERR_PARAMETER, "no such CUDA device");
    LRS_CUDA(cudaSetDevice(device));
    c->device = device;
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
      c->own_stream = false;
    } else {
      LRS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    LRS_CUDA(cudaEventCreate(&c->ev0));
    LRS_CUDA(cudaEventCreate(&c->ev1));
    LRS_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    int lo_prio = 0, hi_prio = 0;
    LRS_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    LRS_CUDA(cudaStreamCreateWithPriority(&c->stream_hi, cudaStreamNonBlocking, hi_prio));
    LRS_CUDA(cudaStreamCreateWithFlags(&c->stream_copy, cudaStreamNonBlocking));
    LRS_CUDA(cudaEventCreateWithFlags(&c->ev_omega, cudaEventDisableTiming));
    pool_stream_open(c->stream);
    c->stage_cap = size_t(8) << 20;
    LRS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->stage), c->stage_cap));
    LRS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->dots_host), Ctx::DOTS_HOST_BYTES));
  });
  if (s == LRS_OK) *out = c.release();
  return s;
}

static void ctx_teardown(Ctx* c) {
  cudaStreamSynchronize(c->stream);
  c->collect();
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  pool_stream_retire(c->stream);
  if (c->stage) cudaFreeHost(c->stage);
  if (c->dots_host) cudaFreeHost(c->dots_host);
  if (c->stream_copy) {
    cudaStreamSynchronize(c->stream_copy);
    cudaStreamDestroy(c->stream_copy);
  }
  if (c->omega_host) cudaFreeHost(c->omega_host);
  if (c->ev_omega) cudaEventDestroy(c->ev_omega);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->stream_hi) cudaStreamDestroy(c->stream_hi);
  delete static_cast<lrs_ctx*>(c);
}

// a matrix or factorization handle was destroyed: finish a deferred lrs_ctx_destroy
static void ctx_release(Ctx* c) {
  if (c && --c->children == 0 && c->closing) ctx_teardown(c);
}

void lrs_ctx_destroy(lrs_ctx* c) {
  if (!c || c->closing) return;
  if (c->children > 0) {  // handles still alive: tear down with the last of them
    cudaStreamSynchronize(c->stream);
    c->closing = true;
    return;
  }
  ctx_teardown(c);
}

void* lrs_ctx_stream(lrs_ctx* c) { return c ? (void*)c->stream : nullptr; }

int64_t lrs_ctx_launch_count(lrs_ctx* c) { return c ? c->launches : 0; }

lrs_status lrs_ctx_synchronize(lrs_ctx* c) {
  if (!c) return LRS_ERR_PARAMETER;
  return guard(c, [&] { LRS_CUDA(cudaStreamSynchronize(c->stream)); });
}

lrs_status lrs_ctx_set_profiling(lrs_ctx* c, int32_t on) {
  if (!c) return LRS_ERR_PARAMETER;
  return guard(c, [&] {
    c->collect();
    c->prof = on != 0;
    c->prof_mask = on == 1 ? ~0u : ((uint32_t)on >> 1);
  });
}

lrs_status lrs_ctx_kernel_times(lrs_ctx* c, double* ms, int64_t* counts, int32_t reset) {
  if (!c) return LRS_ERR_PARAMETER;
  return guard(c, [&] {
    c->collect();
    for (int k = 0; k < K_NCLASS; ++k) {
      if (ms) ms[k] = c->prof_ms[k];
      if (counts) counts[k] = c->prof_cnt[k];
      if (reset) {
        c->prof_ms[k] = 0.0;
        c->prof_cnt[k] = 0;
      }
    }
  });
}

lrs_status lrs_last_error(lrs_ctx* c, lrs_error_info* info) {
  if (!info) return LRS_ERR_PARAMETER;
  *info = c ? c->last : g_last;
  return LRS_OK;
}

// CsrMatrix upload + validate (matrix.cpp:21-37) + band_metrics (matrix.cpp:138-158).
lrs_status lrs_mat_upload_csr(lrs_ctx* c, int64_t n, int64_t nnz, const int64_t* row_ptr,
                              const int64_t* col_idx, const void* values, int32_t scalar,
                              int32_t mem, lrs_mat** out) {
  if (!c || !out) return LRS_ERR_PARAMETER;
  *out = nullptr;
  std::unique_ptr<lrs_mat> m(new (std::nothrow) lrs_mat());
  if (!m) return LRS_ERR_OOM;
  lrs_status s = guard(c, [&] {
    check_mem(mem);
    if (scalar != LRS_F64 && scalar != LRS_C128)
      throw LrsError(LRS_ERR_PARAMETER, "scalar must be LRS_F64 or LRS_C128");
    if (n < 0 || nnz < 0) throw LrsError(LRS_ERR_DIMENSION, "negative dimension");
    if (n >= (1ll << 31) || nnz >= (1ll << 31))
      throw LrsError(LRS_ERR_DIMENSION, "n and nnz must be < 2^31 on the device");
    const int w = scalar == LRS_C128 ? 2 : 1;  // complex values are interleaved (re, im)
    // host views of the arrays (DEVICE inputs are copied down once for validate())
    std::vector<int64_t> rp_h, ci_h;
    std::vector<double> va_h;
    const int64_t* rp = row_ptr;
    const int64_t* ci = col_idx;
    const double* va = static_cast<const double*>(values);
    if (mem == LRS_MEM_DEVICE) {
      rp_h.resize(n + 1);
      ci_h.resize(nnz);
      va_h.resize((size_t)nnz * w);
      LRS_CUDA(cudaMemcpy(rp_h.data(), row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
      if (nnz) {
        LRS_CUDA(cudaMemcpy(ci_h.data(), col_idx, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost));
        LRS_CUDA(cudaMemcpy(va_h.data(), values, sizeof(double) * nnz * w, cudaMemcpyDeviceToHost));
      }
      rp = rp_h.data();
      ci = ci_h.data();
      va = va_h.data();
    }
    const bool trace = std::getenv("LRS_UPLOAD_TRACE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t_begin = now();
    // The device arrays first: the values and the column indices (int64 -> a device
    // temporary, narrowed to int32 by a kernel) travel while the host threads validate.
    // A failed validation synchronizes the stream before the buffers unwind.
    m->row_ptr.alloc(n + 1);
    m->col_idx.alloc(std::max<int64_t>(nnz, 1));
    m->vals.alloc(std::max<int64_t>(nnz, 1) * w);
    DevBuf<int64_t> ci64;
    struct SyncOnError {
      cudaStream_t s;
      bool armed = true;
      ~SyncOnError() { if (armed) cudaStreamSynchronize(s); }
    } sync_guard{c->stream};
    if (nnz) {
      if (mem == LRS_MEM_DEVICE) {
        LRS_CUDA(cudaMemcpyAsync(m->vals.get(), values, sizeof(double) * nnz * w,
                                 cudaMemcpyDeviceToDevice, c->stream));
        launch_narrow_i64(c, col_idx, m->col_idx.get(), nnz);
      } else {
        ci64.alloc(nnz);
        LRS_CUDA(cudaMemcpyAsync(ci64.get(), ci, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice,
                                 c->stream));
        launch_narrow_i64(c, ci64.get(), m->col_idx.get(), nnz);
        LRS_CUDA(cudaMemcpyAsync(m->vals.get(), va, sizeof(double) * nnz * w,
                                 cudaMemcpyHostToDevice, c->stream));
      }
    }
    const auto t_issued = now();
    auto absv = [&](int64_t p) {
      return w == 1 ? std::fabs(va[p]) : std::hypot(va[2 * p], va[2 * p + 1]);
    };
    // validate() -- matrix.cpp:21-37 -- and band_metrics, over fixed row chunks on host
    // threads; the chunk partials combine in chunk order (independent of the thread count)
    if (rp[0] != 0) throw LrsError(LRS_ERR_DIMENSION, "row_ptr[0] must be 0");
    if (rp[n] != nnz) throw LrsError(LRS_ERR_DIMENSION, "row_ptr[n_rows] must equal nnz");
    const int64_t CH = 65536, nch = (n + CH - 1) / CH;
    struct Part {
      int64_t ku = 0, kl = 0, bad_row = -1;
      int bad = 0;
      double dsum = 0.0, tsum = 0.0;
    };
    std::vector<Part> parts((size_t)nch);
    std::vector<int> rp32(n + 1);
    auto work = [&](int64_t c0, int64_t c1) {
      for (int64_t ch = c0; ch < c1; ++ch) {
        Part& pt = parts[ch];
        for (int64_t i = ch * CH; i < std::min(n, (ch + 1) * CH) && pt.bad == 0; ++i) {
          rp32[i] = (int)rp[i];
          if (rp[i] > rp[i + 1]) { pt.bad = 1; pt.bad_row = i; break; }
          for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int64_t j = ci[p];
            if (j < 0 || j >= n) { pt.bad = 2; pt.bad_row = i; break; }
            if (p > rp[i] && j <= ci[p - 1]) { pt.bad = 3; pt.bad_row = i; break; }
            if (j > i) pt.ku = std::max(pt.ku, j - i);
            if (j < i) pt.kl = std::max(pt.kl, i - j);
            const double a = absv(p);
            pt.tsum += a;
            if (i == j) pt.dsum += a;
          }
        }
      }
    };
    {
      const unsigned nt = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>({nch, 16, (int64_t)std::max(1u, std::thread::hardware_concurrency())}));
      std::vector<std::thread> th;
      for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, nch * t / nt, nch * (t + 1) / nt);
      work(0, nch / nt);
      for (auto& t : th) t.join();
    }
    rp32[n] = (int)rp[n];
    const auto t_valid = now();
    int64_t ku = 0, kl = 0;
    double dsum = 0.0, tsum = 0.0;
    for (const Part& pt : parts) {
      if (pt.bad == 1) throw LrsError(LRS_ERR_DIMENSION, "row_ptr must be non-decreasing");
      if (pt.bad == 2) throw LrsError(LRS_ERR_DIMENSION, "column index out of range");
      if (pt.bad == 3)
        throw LrsError(LRS_ERR_DIMENSION, "column indices must be strictly increasing within a row");
      ku = std::max(ku, pt.ku);
      kl = std::max(kl, pt.kl);
      dsum += pt.dsum;
      tsum += pt.tsum;
    }
    m->ctx = c;
    m->n = n;
    m->nnz = nnz;
    m->scalar = scalar;
    m->ku = ku;
    m->kl = kl;
    m->k = std::max(ku, kl);
    m->diag_weight = tsum > 0 ? dsum / tsum : 0.0;
    const double cells = (double)(ku + kl + 1) * (double)n;
    m->band_density = cells > 0 ? (double)nnz / cells : 0.0;
    // device CSR with int32 indices (col_idx / values are already on their way); the
    // transpose is built on the device (csr.cu)
    LRS_CUDA(cudaMemcpyAsync(m->row_ptr.get(), rp32.data(), sizeof(int) * (n + 1),
                             cudaMemcpyHostToDevice, c->stream));
    launch_csr_transpose(c, m.get());
    const auto t_launched = now();
    LRS_CUDA(cudaStreamSynchronize(c->stream));
    sync_guard.armed = false;
    if (trace)
      std::fprintf(stderr, "lrs upload: alloc + copy issue %.1f ms, validate %.1f ms, transpose "
                   "issue %.1f ms, wait %.1f ms\n", ms(t_begin, t_issued), ms(t_issued, t_valid),
                   ms(t_valid, t_launched), ms(t_launched, now()));
  });
  if (s == LRS_OK) {
    *out = m.release();
    ++c->children;
  }
  return s;
}

void lrs_mat_destroy(lrs_mat* m) {
  if (!m) return;
  Ctx* c = m->ctx;
  delete m;
  ctx_release(c);
}

lrs_status lrs_mat_band_metrics(lrs_mat* m, int64_t* ku, int64_t* kl, int64_t* k,
                                double* diag_weight, double* band_density) {
  if (!m) return LRS_ERR_PARAMETER;
  if (ku) *ku = m->ku;
  if (kl) *kl = m->kl;
  if (k) *k = m->k;
  if (diag_weight) *diag_weight = m->diag_weight;
  if (band_density) *band_density = m->band_density;
  return LRS_OK;
}

lrs_status lrs_spmv(lrs_mat* m, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t n_rhs,
                    int32_t accumulate, int32_t mem) {
  if (!m) return LRS_ERR_PARAMETER;
  Ctx* c = m->ctx;
  return guard(c, [&] {
    check_mem(mem);
    if (n_rhs < 0 || ldx < m->n || ldy < m->n)
      throw LrsError(LRS_ERR_DIMENSION, "spmv: A.n_cols must equal x.n_rows");
    const int w = m->scalar == LRS_C128 ? 2 : 1;
    DevBuf<double> xo, yo;
    int64_t lx, ly;
    void* xd = dev_in(c, x, ldx, m->n, n_rhs, mem, xo, &lx, w);
    void* yd = dev_in(c, y, ldy, m->n, n_rhs, mem, yo, &ly, w);
    if (w == 2)
      launch_spmv_z(c, m, static_cast<const zc*>(xd), lx, static_cast<zc*>(yd), ly, (int)n_rhs,
                    accumulate ? 1 : 0, nullptr, 0);
    else
      launch_spmv(c, m, static_cast<const double*>(xd), lx, static_cast<double*>(yd), ly,
                  (int)n_rhs, accumulate ? 1 : 0, nullptr, 0);
    dev_out_finish(c, y, ldy, yd, m->n, n_rhs, mem, w);
  });
}

lrs_status lrs_make_layout(int64_t n, int64_t p, int64_t k, int64_t* sizes_out) {
  return guard(nullptr, [&] {
    if (p < 1 || k < 0) throw LrsError(LRS_ERR_PARAMETER, "make_layout: p >= 1 and k >= 0");
    for (int64_t i = 0; i < p; ++i) {
      const int64_t s = n / p + (i < n % p ? 1 : 0);
      if (s <= k)
        throw LrsError(LRS_ERR_LAYOUT,
                       "layout infeasible: need n >= p*(k+1) = " + std::to_string(p * (k + 1)));
      if (sizes_out) sizes_out[i] = s;
    }
  });
}

lrs_status lrs_factorize(lrs_ctx* c, lrs_mat* a, const lrs_solver_cfg* cfg, lrs_fact** out) {
  if (!c || !a || !cfg || !out) return LRS_ERR_PARAMETER;
  *out = nullptr;
  return guard(c, [&] {
    LRS_CUDA(cudaSetDevice(c->device));
    Fact* f = factorize(c, a, *cfg, nullptr);
    *out = static_cast<lrs_fact*>(f);
    ++c->children;
  });
}

lrs_status lrs_factorize_dist(lrs_ctx* c, lrs_mat* a, const lrs_solver_cfg* cfg,
                              const lrs_comm* comm, lrs_fact** out) {
  if (!c || !a || !cfg || !comm || !out) return LRS_ERR_PARAMETER;
  *out = nullptr;
  return guard(c, [&] {
    LRS_CUDA(cudaSetDevice(c->device));
    Fact* f = factorize(c, a, *cfg, comm);
    *out = static_cast<lrs_fact*>(f);
    ++c->children;
  });
}

lrs_status lrs_shard_plan(int64_t n, int64_t p, int32_t size, int32_t rank, int64_t* p_lo,
                          int64_t* p_hi, int64_t* row_lo, int64_t* row_hi) {
  return guard(nullptr, [&] {
    if (p < 1 || size < 1 || rank < 0 || rank >= size || p < size || n < p)
      throw LrsError(LRS_ERR_PARAMETER, "shard plan needs p >= size >= 1, 0 <= rank < size");
    int64_t a, b;
    shard_plan(p, size, rank, &a, &b);
    auto off = [&](int64_t i) { return i * (n / p) + std::min<int64_t>(i, n % p); };
    if (p_lo) *p_lo = a;
    if (p_hi) *p_hi = b;
    if (row_lo) *row_lo = off(a);
    if (row_hi) *row_hi = off(b);
  });
}

void lrs_fact_destroy(lrs_fact* f) {
  if (!f) return;
  Ctx* c = f->ctx;
  cudaStreamSynchronize(c->stream);
  delete static_cast<Fact*>(f);
  ctx_release(c);
}

lrs_status lrs_fact_get_info(lrs_fact* f, lrs_fact_info* info) {
  if (!f || !info) return LRS_ERR_PARAMETER;
  *info = f->info;
  return LRS_OK;
}

lrs_status lrs_fact_get_layout(lrs_fact* f, int64_t* sizes, int64_t* offsets) {
  if (!f) return LRS_ERR_PARAMETER;
  for (int i = 0; i < f->Pg; ++i) {  // the global layout (all partitions)
    if (sizes) sizes[i] = f->goff[i + 1] - f->goff[i];
    if (offsets) offsets[i] = f->goff[i];
  }
  return LRS_OK;
}

lrs_status lrs_fact_get_spike(lrs_fact* f, int64_t i, int32_t side, double* u, double* sigma,
                              double* v) {
  if (!f) return LRS_ERR_PARAMETER;
  return guard(f->ctx, [&] {
    if (f->r == 0) throw LrsError(LRS_ERR_PARAMETER, "factorization has no low-rank spikes");
    if (i < f->p0 || i >= f->p0 + f->P || (side == LRS_SIDE_T && i == f->Pg - 1) ||
        (side == LRS_SIDE_W && i == 0) || (side != LRS_SIDE_T && side != LRS_SIDE_W))
      throw LrsError(LRS_ERR_PARAMETER, "no such spike on this GPU");
    const int r = f->r, w = f->sw;
    const size_t es = sizeof(double) * w;
    const int64_t n = f->n, k = f->k, ni = f->size[i - f->p0];
    const double* ub = side == LRS_SIDE_T ? f->uT.get() : f->uW.get();
    const double* vb = side == LRS_SIDE_T ? f->vtT.get() : f->vtW.get();
    const double* sb = side == LRS_SIDE_T ? f->sT.get() : f->sW.get();
    if (u)
      LRS_CUDA(cudaMemcpy2D(u, es * ni, ub + f->goff[i] * w, es * n, es * ni, r,
                            cudaMemcpyDeviceToHost));
    if (sigma) LRS_CUDA(cudaMemcpy(sigma, sb + (size_t)i * r, sizeof(double) * r, cudaMemcpyDeviceToHost));
    if (v) {  // stored as v^T (k x r); return v (r x k, ld r)
      std::vector<double> vt((size_t)k * r * w);
      LRS_CUDA(cudaMemcpy(vt.data(), vb + (size_t)i * k * r * w, es * k * r,
                          cudaMemcpyDeviceToHost));
      for (int a = 0; a < r; ++a)
        for (int64_t row = 0; row < k; ++row)
          for (int e = 0; e < w; ++e) v[(a + row * r) * w + e] = vt[(row + (size_t)a * k) * w + e];
    }
  });
}

lrs_status lrs_fact_get_tiles(lrs_fact* f, int64_t i, double* host_out, int64_t capacity,
                              int64_t* needed) {
  if (!f) return LRS_ERR_PARAMETER;
  return guard(f->ctx, [&] {
    if (i < f->p0 || i >= f->p0 + f->P)
      throw LrsError(LRS_ERR_PARAMETER, "partition not on this GPU");
    const int li = (int)(i - f->p0);
    const int64_t cnt = (int64_t)f->T[li] * f->W * TILE_ELEMS * f->sw;  // doubles
    if (needed) *needed = cnt;
    if (host_out) {
      if (capacity < cnt) throw LrsError(LRS_ERR_DIMENSION, "tile buffer too small");
      LRS_CUDA(cudaStreamSynchronize(f->ctx->stream));
      LRS_CUDA(cudaMemcpy(host_out, f->tiles.get() + f->tbase[li] * TILE_ELEMS * f->sw,
                          sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    }
  });
}

lrs_status lrs_fact_get_ledger(lrs_fact* f, int64_t messages[3], int64_t scalars[3]) {
  if (!f) return LRS_ERR_PARAMETER;
  for (int s = 0; s < 3; ++s) {
    if (messages) messages[s] = f->ledger_msgs[s];
    if (scalars) scalars[s] = f->ledger_sc[s];
  }
  return LRS_OK;
}

lrs_status lrs_solve_block(lrs_fact* f, int64_t i, const void* rhs, int64_t ld_rhs, void* x,
                           int64_t ld_x, int64_t n_rhs, int32_t adjoint, int32_t mem) {
  if (!f) return LRS_ERR_PARAMETER;
  Ctx* c = f->ctx;
  return guard(c, [&] {
    check_mem(mem);
    if (i < f->p0 || i >= f->p0 + f->P)
      throw LrsError(LRS_ERR_PARAMETER, "partition not on this GPU");
    const int li = (int)(i - f->p0);
    const int64_t ni = f->size[li];
    if (ld_rhs < ni || ld_x < ni || n_rhs < 0)
      throw LrsError(LRS_ERR_DIMENSION, "solve_block: RHS rows must equal the block size");
    // work in a global-row-layout buffer so the partition offset addressing of the
    // dataflow kernel applies unchanged
    const int w = f->sw;
    const size_t es = sizeof(double) * w;
    DevBuf<double> work;
    work.alloc((size_t)std::max<int64_t>(1, f->n * n_rhs) * w);
    double* wp = work.get() + f->off[li] * w;
    const cudaMemcpyKind k_in = mem == LRS_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    if (n_rhs > 0)
      LRS_CUDA(cudaMemcpy2DAsync(wp, es * f->n, rhs, es * ld_rhs, es * ni, n_rhs, k_in, c->stream));
    // solve_block always takes the batch-width-independent DMMA path
    struct FmaOff {
      Ctx* c;
      bool prev;
      ~FmaOff() { c->solve_fma1 = prev; }
    } fo{c, c->solve_fma1};
    c->solve_fma1 = false;
    dstage(f, work.get(), f->n, (int)n_rhs, adjoint != 0, li);
    const cudaMemcpyKind k_out = mem == LRS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (n_rhs > 0)
      LRS_CUDA(cudaMemcpy2DAsync(x, es * ld_x, wp, es * f->n, es * ni, n_rhs, k_out, c->stream));
    LRS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

static lrs_status apply_common(lrs_fact* f, const void* in, int64_t ld_in, void* out,
                               int64_t ld_out, int64_t n_rhs, int32_t mem, int mode) {
  if (!f) return LRS_ERR_PARAMETER;
  Ctx* c = f->ctx;
  return guard(c, [&] {
    check_mem(mem);
    if (ld_in < f->n || ld_out < f->n || n_rhs < 0)
      throw LrsError(LRS_ERR_DIMENSION, "apply: vector rows must equal n");
    if (mem == LRS_MEM_DEVICE) {
      apply_precond(f, in, ld_in, out, ld_out, (int)n_rhs, mode);
      return;
    }
    DevBuf<double> io;
    int64_t ld;
    void* d = dev_in(c, in, ld_in, f->n, n_rhs, mem, io, &ld, f->sw);
    apply_precond(f, d, ld, d, ld, (int)n_rhs, mode);
    dev_out_finish(c, out, ld_out, d, f->n, n_rhs, mem, f->sw);
  });
}

lrs_status lrs_apply_precond(lrs_fact* f, const void* in, int64_t ld_in, void* out, int64_t ld_out,
                             int64_t n_rhs, int32_t mem) {
  return apply_common(f, in, ld_in, out, ld_out, n_rhs, mem, APPLY_VARIANT);
}

lrs_status lrs_apply_block_jacobi(lrs_fact* f, const void* in, int64_t ld_in, void* out,
                                  int64_t ld_out, int64_t n_rhs, int32_t mem) {
  return apply_common(f, in, ld_in, out, ld_out, n_rhs, mem, APPLY_BJ);
}

lrs_status lrs_apply_precond_T(lrs_fact* f, const void* in, int64_t ld_in, void* out,
                               int64_t ld_out, int64_t n_rhs, int32_t mem) {
  return apply_common(f, in, ld_in, out, ld_out, n_rhs, mem, APPLY_T);
}

lrs_status lrs_solve(lrs_fact* f, lrs_mat* a, const void* b, int64_t ldb, void* x, int64_t ldx,
                     int64_t n_rhs, const lrs_iter_cfg* cfg, lrs_report* report, int32_t mem) {
  if (!f || !a || !cfg) return LRS_ERR_PARAMETER;
  Ctx* c = f->ctx;
  lrs_report local{};
  lrs_report* rep = report ? report : &local;
  return guard(c, [&] {
    check_mem(mem);
    if (ldb < f->n || ldx < f->n || n_rhs < 0)
      throw LrsError(LRS_ERR_DIMENSION, "solve: vector rows must equal n");
    lrs_iter_cfg cc = *cfg;
    if (cc.breakdown_eps <= 0) cc.breakdown_eps = 1e-30;
    if (cc.restart <= 0) cc.restart = 30;
    if (mem == LRS_MEM_DEVICE) {
      solve(f, a, b, ldb, x, ldx, (int)n_rhs, cc, rep);
      return;
    }
    const int w = f->sw;
    DevBuf<double> bo, xo, x0o;
    int64_t lb, lx0 = f->n;
    const void* bd = dev_in(c, b, ldb, f->n, n_rhs, mem, bo, &lb, w);
    if (cc.x0) cc.x0 = dev_in(c, cc.x0, ldx, f->n, n_rhs, mem, x0o, &lx0, w);
    xo.alloc((size_t)std::max<int64_t>(1, f->n * n_rhs) * w);
    // x0 (if any) is addressed with ldx inside solve(); pass it with ld n
    try {
      solve(f, a, bd, lb, xo.get(), f->n, (int)n_rhs, cc, rep);
    } catch (const LrsError& e) {
      // breakdown keeps the partial result
      if (e.status == LRS_ERR_BREAKDOWN) dev_out_finish(c, x, ldx, xo.get(), f->n, n_rhs, mem, w);
      throw;
    }
    dev_out_finish(c, x, ldx, xo.get(), f->n, n_rhs, mem, w);
  });
}

lrs_status lrs_reduced_apply(lrs_fact* f, int32_t kind, const void* x, int64_t ldx, void* y,
                             int64_t ldy, int64_t n_rhs, int32_t mem) {
  if (!f) return LRS_ERR_PARAMETER;
  Ctx* c = f->ctx;
  return guard(c, [&] {
    check_mem(mem);
    if (kind < 0 || kind > 2) throw LrsError(LRS_ERR_PARAMETER, "unknown reduced operator");
    if (f->dist) throw LrsError(LRS_ERR_NOT_IMPLEMENTED, "lrs_reduced_apply: single GPU only");
    const int64_t m = f->ldr;
    if (ldx < m || ldy < m || n_rhs < 0)
      throw LrsError(LRS_ERR_DIMENSION, "reduced vectors have 2 k p rows");
    const int w = f->sw;
    // device copies with ld = 2 k p (the kernels address full-length compact blocks)
    DevBuf<double> xi, yo;
    xi.alloc((size_t)std::max<int64_t>(1, m * n_rhs) * w);
    yo.alloc((size_t)std::max<int64_t>(1, m * n_rhs) * w);
    const size_t es = sizeof(double) * w;
    const cudaMemcpyKind kin = mem == LRS_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    if (n_rhs > 0) LRS_CUDA(cudaMemcpy2DAsync(xi.get(), es * m, x, es * ldx, es * m, n_rhs, kin, c->stream));
    reduced_op(f, kind, xi.get(), yo.get(), (int)n_rhs);
    const cudaMemcpyKind kout = mem == LRS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (n_rhs > 0) LRS_CUDA(cudaMemcpy2DAsync(y, es * ldy, yo.get(), es * m, es * m, n_rhs, kout, c->stream));
    LRS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

lrs_status lrs_krylov(lrs_ctx* c, int64_t n, int32_t scalar, const lrs_operator* apply_A,
                      const lrs_operator* apply_M, const void* b, int64_t ldb, void* x,
                      int64_t ldx, int64_t n_rhs, const lrs_iter_cfg* cfg, lrs_report* report,
                      int32_t mem) {
  if (!c || !apply_A || !cfg) return LRS_ERR_PARAMETER;
  lrs_report local{};
  lrs_report* rep = report ? report : &local;
  return guard(c, [&] {
    check_mem(mem);
    if (scalar != LRS_F64 && scalar != LRS_C128)
      throw LrsError(LRS_ERR_PARAMETER, "scalar must be LRS_F64 or LRS_C128");
    if (ldb < n || ldx < n || n_rhs < 0) throw LrsError(LRS_ERR_DIMENSION, "krylov: ld >= n");
    lrs_iter_cfg cc = *cfg;
    if (cc.breakdown_eps <= 0) cc.breakdown_eps = 1e-30;
    if (cc.restart <= 0) cc.restart = 30;
    if (mem == LRS_MEM_DEVICE) {
      krylov_ops(c, n, scalar, *apply_A, apply_M, b, ldb, x, ldx, (int)n_rhs, cc, rep);
      return;
    }
    const int w = scalar == LRS_C128 ? 2 : 1;
    DevBuf<double> bo, xo, x0o;
    int64_t lb, lx0 = n;
    const void* bd = dev_in(c, b, ldb, n, n_rhs, mem, bo, &lb, w);
    if (cc.x0) cc.x0 = dev_in(c, cc.x0, ldx, n, n_rhs, mem, x0o, &lx0, w);
    xo.alloc((size_t)std::max<int64_t>(1, n * n_rhs) * w);
    try {
      krylov_ops(c, n, scalar, *apply_A, apply_M, bd, lb, xo.get(), n, (int)n_rhs, cc, rep);
    } catch (const LrsError& e) {
      if (e.status == LRS_ERR_BREAKDOWN) dev_out_finish(c, x, ldx, xo.get(), n, n_rhs, mem, w);
      throw;
    }
    dev_out_finish(c, x, ldx, xo.get(), n, n_rhs, mem, w);
  });
}

// ---- small dense operations and the truncated preconditioner from explicit spikes --------
static int scalar_w(int32_t scalar) {
  if (scalar != LRS_F64 && scalar != LRS_C128)
    throw LrsError(LRS_ERR_PARAMETER, "scalar must be LRS_F64 or LRS_C128");
  return scalar == LRS_C128 ? 2 : 1;
}

lrs_status lrs_dense_qr(lrs_ctx* c, int32_t scalar, int64_t m, int64_t ncols, void* A, int64_t lda,
                        void* R, int32_t mem) {
  if (!c || !A) return LRS_ERR_PARAMETER;
  return guard(c, [&] {
    check_mem(mem);
    const int w = scalar_w(scalar);
    if (ncols < 1 || ncols > 96 || m < ncols || lda < m)
      throw LrsError(LRS_ERR_DIMENSION, "dense_qr: 1 <= ncols <= 96, ncols <= m <= lda");
    LRS_CUDA(cudaSetDevice(c->device));
    DevBuf<double> ao, ro;
    int64_t la;
    void* ad = dev_in(c, A, lda, m, ncols, mem, ao, &la, w);
    void* rd = nullptr;
    if (R) {
      if (mem == LRS_MEM_DEVICE) {
        rd = R;
      } else {
        ro.alloc((size_t)ncols * ncols * w);
        rd = ro.get();
      }
    }
    if (scalar == LRS_C128) {
      DevBuf<QrJobT<zc>> j;
      std::vector<QrJobT<zc>> h{{static_cast<zc*>(ad), m, la, static_cast<zc*>(rd)}};
      j.alloc(1);
      c->stage_h2d(j.get(), h.data(), sizeof(h[0]));
      launch_householder_qr_t<zc>(c, j.get(), 1, (int)ncols, m);
    } else {
      DevBuf<QrJobT<double>> j;
      std::vector<QrJobT<double>> h{{static_cast<double*>(ad), m, la, static_cast<double*>(rd)}};
      j.alloc(1);
      c->stage_h2d(j.get(), h.data(), sizeof(h[0]));
      launch_householder_qr_t<double>(c, j.get(), 1, (int)ncols, m);
    }
    dev_out_finish(c, A, lda, ad, m, ncols, mem, w);
    if (R) dev_out_finish(c, R, ncols, rd, ncols, ncols, mem, w);
    LRS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

lrs_status lrs_dense_svd(lrs_ctx* c, int32_t scalar, int64_t l, void* R, void* U, void* V,
                         double* sigma, int32_t mem) {
  if (!c || !R || !U || !V || !sigma) return LRS_ERR_PARAMETER;
  return guard(c, [&] {
    check_mem(mem);
    const int w = scalar_w(scalar);
    if (l < 1 || l > 96) throw LrsError(LRS_ERR_DIMENSION, "dense_svd: 1 <= l <= 96");
    LRS_CUDA(cudaSetDevice(c->device));
    DevBuf<double> ro, uo, vo, so;
    int64_t lr, lu, lv;
    void* rd = dev_in(c, R, l, l, l, mem, ro, &lr, w);
    void* ud = dev_in(c, U, l, l, l, mem, uo, &lu, w);
    void* vd = dev_in(c, V, l, l, l, mem, vo, &lv, w);
    double* sd = sigma;
    if (mem == LRS_MEM_HOST) {
      so.alloc(l);
      sd = so.get();
    }
    if (scalar == LRS_C128) {
      DevBuf<SvdJobT<zc>> j;
      SvdJobT<zc> h{static_cast<zc*>(rd), static_cast<zc*>(vd), static_cast<zc*>(ud), sd};
      j.alloc(1);
      c->stage_h2d(j.get(), &h, sizeof(h));
      launch_jacobi_svd_t<zc>(c, j.get(), 1, (int)l);
    } else {
      DevBuf<SvdJobT<double>> j;
      SvdJobT<double> h{static_cast<double*>(rd), static_cast<double*>(vd),
                        static_cast<double*>(ud), sd};
      j.alloc(1);
      c->stage_h2d(j.get(), &h, sizeof(h));
      launch_jacobi_svd_t<double>(c, j.get(), 1, (int)l);
    }
    dev_out_finish(c, U, l, ud, l, l, mem, w);
    dev_out_finish(c, V, l, vd, l, l, mem, w);
    if (mem == LRS_MEM_HOST)
      LRS_CUDA(cudaMemcpy(sigma, sd, sizeof(double) * l, cudaMemcpyDeviceToHost));
    LRS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

lrs_status lrs_dense_gemm(lrs_ctx* c, int32_t scalar, int64_t m, int64_t n, int64_t k,
                          const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                          int64_t ldc, int32_t conjC, int32_t mem) {
  if (!c || !A || !B || !C) return LRS_ERR_PARAMETER;
  return guard(c, [&] {
    check_mem(mem);
    const int w = scalar_w(scalar);
    if (m < 0 || n < 1 || k < 1 || n * k > 96 * 64 || lda < m || ldb < k || ldc < m)
      throw LrsError(LRS_ERR_DIMENSION, "dense_gemm: k x n <= 96 x 64 and ld >= rows");
    LRS_CUDA(cudaSetDevice(c->device));
    DevBuf<double> ao, bo, co;
    int64_t la, lb, lc;
    const void* ad = dev_in(c, A, lda, m, k, mem, ao, &la, w);
    const void* bd = dev_in(c, B, ldb, k, n, mem, bo, &lb, w);
    void* cd = dev_in(c, C, ldc, m, n, mem, co, &lc, w);
    if (scalar == LRS_C128) {
      DevBuf<GemmJobT<zc>> j;
      GemmJobT<zc> h{static_cast<const zc*>(ad), la, static_cast<const zc*>(bd), lb,
                     static_cast<zc*>(cd), lc, m, (int)n, (int)k, conjC ? 1 : 0};
      j.alloc(1);
      c->stage_h2d(j.get(), &h, sizeof(h));
      launch_small_gemm_t<zc>(c, j.get(), 1, m, (int)n);
    } else {
      DevBuf<GemmJobT<double>> j;
      GemmJobT<double> h{static_cast<const double*>(ad), la, static_cast<const double*>(bd), lb,
                         static_cast<double*>(cd), lc, m, (int)n, (int)k, conjC ? 1 : 0};
      j.alloc(1);
      c->stage_h2d(j.get(), &h, sizeof(h));
      launch_small_gemm_t<double>(c, j.get(), 1, m, (int)n);
    }
    dev_out_finish(c, C, ldc, cd, m, n, mem, w);
    LRS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

lrs_status lrs_trunc_precond_create(lrs_ctx* c, int32_t scalar, int64_t p, int64_t k, int64_t r,
                                    const void* uT_tips, const void* vT, const double* sT,
                                    const void* uW_tips, const void* vW, const double* sW,
                                    int32_t mem, lrs_fact** out) {
  if (!c || !out || !uT_tips || !vT || !sT || !uW_tips || !vW || !sW) return LRS_ERR_PARAMETER;
  *out = nullptr;
  return guard(c, [&] {
    check_mem(mem);
    const int w = scalar_w(scalar);
    if (p < 2 || k < 1 || r < 1 || r > k || r > 96)
      throw LrsError(LRS_ERR_PARAMETER, "trunc_precond: p >= 2, 1 <= n_svd <= min(k, 96)");
    LRS_CUDA(cudaSetDevice(c->device));
    const int64_t cnt = (p - 1) * k * r;
    DevBuf<double> a, b, d, e, sa, sb;
    int64_t ld;
    const void* uTd = dev_in(c, uT_tips, 2 * cnt, 2 * cnt, 1, mem, a, &ld, w);
    const void* vTd = dev_in(c, vT, cnt, cnt, 1, mem, b, &ld, w);
    const void* uWd = dev_in(c, uW_tips, 2 * cnt, 2 * cnt, 1, mem, d, &ld, w);
    const void* vWd = dev_in(c, vW, cnt, cnt, 1, mem, e, &ld, w);
    const double* sTd = static_cast<const double*>(dev_in(c, sT, (p - 1) * r, (p - 1) * r, 1, mem, sa, &ld, 1));
    const double* sWd = static_cast<const double*>(dev_in(c, sW, (p - 1) * r, (p - 1) * r, 1, mem, sb, &ld, 1));
    Fact* f = make_trunc_precond(c, scalar, p, k, (int)r, uTd, vTd, sTd, uWd, vWd, sWd);
    LRS_CUDA(cudaStreamSynchronize(c->stream));
    *out = static_cast<lrs_fact*>(f);
    ++c->children;
  });
}

lrs_status lrs_bench_dmma_peak(lrs_ctx* c, double* tflops) {
  if (!c || !tflops) return LRS_ERR_PARAMETER;
  return guard(c, [&] { *tflops = run_dmma_peak(c); });
}

lrs_status lrs_bench_i8_peak(lrs_ctx* c, double* tops) {
  if (!c || !tops) return LRS_ERR_PARAMETER;
  return guard(c, [&] { *tops = run_i8_peak(c); });
}

}  // extern "C"
