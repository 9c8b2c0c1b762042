// Stream-ordered caching device allocator used by every DevBuf of the library.
//
// A factorization of config 2 owns ~17 GB of band tiles plus a few hundred MB of
// spikes and workspaces; without caching, each factorize/solve cycle paid a
// cudaMalloc + cudaFree of those (the frees also synchronize the whole device and
// stall the launch pipeline).  Freed blocks are kept per stream and reused only
// by later allocations on the same stream, so the usual stream-order argument
// makes reuse race-free.  On cudaMalloc failure every cached block is returned to
// the driver and the allocation is retried once.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <set>

#include "lrs_internal.h"

namespace lrs {

namespace {

struct Pool {
  std::mutex mu;
  std::map<cudaStream_t, std::multimap<size_t, void*>> free_;
  std::set<cudaStream_t> live;
  size_t cached = 0;
};

Pool& pool() {
  static Pool* p = new Pool();  // never destroyed: DevBufs may outlive static teardown order
  return *p;
}

size_t round_bytes(size_t b) {
  const size_t small = 512, large = size_t(2) << 20;
  return b <= (size_t(1) << 20) ? (b + small - 1) / small * small : (b + large - 1) / large * large;
}

void release_all_locked(Pool& P) {
  for (auto& kv : P.free_)
    for (auto& blk : kv.second) cudaFree(blk.second);
  P.free_.clear();
  P.cached = 0;
}

}  // namespace

cudaStream_t& current_pool_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

void pool_stream_open(cudaStream_t s) {
  Pool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  P.live.insert(s);
}

void pool_stream_retire(cudaStream_t s) {
  Pool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  auto it = P.free_.find(s);
  if (it != P.free_.end()) {
    for (auto& blk : it->second) {
      cudaFree(blk.second);
      P.cached -= blk.first;
    }
    P.free_.erase(it);
  }
  P.live.erase(s);
}

size_t pool_cached_bytes() {
  Pool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  return P.cached;
}

void* pool_alloc(cudaStream_t s, size_t bytes, size_t* rounded) {
  Pool& P = pool();
  const size_t rb = round_bytes(bytes);
  *rounded = rb;
  {
    std::lock_guard<std::mutex> g(P.mu);
    if (P.live.count(s)) {
      auto& fl = P.free_[s];
      auto it = fl.lower_bound(rb);
      const size_t slack = rb <= (size_t(1) << 20) ? 0 : std::max(rb / 8, size_t(2) << 20);
      if (it != fl.end() && it->first <= rb + slack) {
        void* p = it->second;
        *rounded = it->first;
        P.cached -= it->first;
        fl.erase(it);
        return p;
      }
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, rb);
  if (e != cudaSuccess) {
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> g(P.mu);
      cudaDeviceSynchronize();
      release_all_locked(P);
    }
    e = cudaMalloc(&p, rb);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw LrsError(LRS_ERR_OOM, "cudaMalloc of " + std::to_string(rb) +
                                      " bytes failed: " + cudaGetErrorString(e));
    }
  }
  return p;
}

void pool_release(cudaStream_t s, void* p, size_t bytes) {
  if (!p) return;
  Pool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  if (!P.live.count(s)) {  // no owning context (or already destroyed): give it back now
    cudaFree(p);
    return;
  }
  P.free_[s].insert({bytes, p});
  P.cached += bytes;
}

void Ctx::stage_h2d(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (!stage || bytes > stage_cap / 4) {
    // large upload: plain (host-synchronous) copy
    LRS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
    LRS_CUDA(cudaStreamSynchronize(stream));
    return;
  }
  const size_t b = (bytes + 255) & ~size_t(255);
  if (stage_pos + b > stage_cap) {
    // wrap: every earlier copy out of the ring must have completed
    LRS_CUDA(cudaStreamSynchronize(stream));
    stage_pos = 0;
  }
  std::memcpy(stage + stage_pos, src, bytes);
  LRS_CUDA(cudaMemcpyAsync(dst, stage + stage_pos, bytes, cudaMemcpyHostToDevice, stream));
  stage_pos += b;
}

}  // namespace lrs
