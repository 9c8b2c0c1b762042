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
constexpr int MAX_RHS = 16;                // columns per Krylov / solve launch batch
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

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    if (count == 0) return;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw LrsError(LRS_ERR_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) +
                                      " bytes failed: " + cudaGetErrorString(e));
    }
    n = count;
  }
  T* get() const { return p; }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t launches = 0;
  lrs_error_info last{};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int num_sms = 148;
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
};

struct Fact;  // defined in fact.h

// ------------------------------------------------------------------------------------
// kernel launchers (implemented in the .cu files)
// ------------------------------------------------------------------------------------

// spmv.cu
void launch_spmv(Ctx* c, const Mat* m, const double* x, int64_t ldx, double* y, int64_t ldy,
                 int nrhs, int mode, const double* b, int64_t ldb);
// mode: 0 y = A x, 1 y += A x, 2 y = b - A x

}  // namespace lrs
