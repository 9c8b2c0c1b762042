// The in-library NCCL data plane behind lrs_comm ("NVLink 5 /
// NVSwitch equivalent of the communication backend").
//
// One communicator per lrs_ctx (one process per GPU).  Every exchange of a sharded
// factorization is enqueued on the context stream, in stream order with the kernels that
// produce and consume it:
//   neighbors  C1 (rank-r interface messages) / C3 (SpMV halos) / C5 (setup spike tips):
//              ncclSend + ncclRecv of both directions inside ONE ncclGroupStart/End
//   sendrecv   the single-direction form of the same
//   allgather  C4 (the per-partition dot partials, summed afterwards in global partition
//              order on the device, so the iterates do not depend on the GPU count)
// The library therefore never synchronizes the stream before an exchange the device
// consumes (lrs_comm.stream_ordered = 1); the host synchronizes only where it needs a
// Krylov scalar.  libnccl.so.2 is loaded with dlopen on first use (the process may
// already hold torch's copy; the soname makes them one library), so the CUDA library has
// no link-time NCCL dependency for single-GPU users.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "lrs_internal.h"
#include "lrspike_capi.h"

struct lrs_ctx : lrs::Ctx {};  // as in capi.cu

namespace lrs {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  bool ok = false;
  std::string err;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.CommGetAsyncError =
        reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
             api.AllGather && api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw LrsError(LRS_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

struct NcclPlane {
  lrs_comm c{};  // first member: the lrs_comm* handed out is the plane itself
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  int device = 0;
};

int32_t plane_neighbors(void* user, const double* to_next, double* from_prev, const double* to_prev,
                        double* from_next, int64_t count) {
  auto* p = static_cast<NcclPlane*>(user);
  const NcclApi& a = nccl();
  const int r = p->c.rank;
  if (a.GroupStart() != ncclSuccess) return 1;
  ncclResult_t e = ncclSuccess;
  if (to_next && e == ncclSuccess) e = a.Send(to_next, count, ncclFloat64, r + 1, p->comm, p->stream);
  if (from_prev && e == ncclSuccess) e = a.Recv(from_prev, count, ncclFloat64, r - 1, p->comm, p->stream);
  if (to_prev && e == ncclSuccess) e = a.Send(to_prev, count, ncclFloat64, r - 1, p->comm, p->stream);
  if (from_next && e == ncclSuccess) e = a.Recv(from_next, count, ncclFloat64, r + 1, p->comm, p->stream);
  const ncclResult_t g = a.GroupEnd();
  return (e == ncclSuccess && g == ncclSuccess) ? 0 : 1;
}

int32_t plane_sendrecv(void* user, const double* send, int64_t scount, int32_t dest, double* recv,
                       int64_t rcount, int32_t source) {
  auto* p = static_cast<NcclPlane*>(user);
  const NcclApi& a = nccl();
  if (a.GroupStart() != ncclSuccess) return 1;
  ncclResult_t e = ncclSuccess;
  if (dest >= 0 && scount > 0) e = a.Send(send, scount, ncclFloat64, dest, p->comm, p->stream);
  if (source >= 0 && rcount > 0 && e == ncclSuccess)
    e = a.Recv(recv, rcount, ncclFloat64, source, p->comm, p->stream);
  const ncclResult_t g = a.GroupEnd();
  return (e == ncclSuccess && g == ncclSuccess) ? 0 : 1;
}

int32_t plane_allgather(void* user, const double* send, double* recv, int64_t count) {
  auto* p = static_cast<NcclPlane*>(user);
  return nccl().AllGather(send, recv, count, ncclFloat64, p->comm, p->stream) == ncclSuccess ? 0 : 1;
}

}  // namespace
}  // namespace lrs

using namespace lrs;

extern "C" {

lrs_status lrs_comm_nccl_unique_id(void* id128) {
  if (!id128) return LRS_ERR_PARAMETER;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  const NcclApi& a = nccl();
  if (!a.ok) return LRS_ERR_NCCL;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return LRS_ERR_NCCL;
  std::memcpy(id128, &id, sizeof(id));
  return LRS_OK;
}

lrs_status lrs_comm_nccl_create(lrs_ctx* ctx, const void* id128, int32_t rank, int32_t size,
                                lrs_comm** out) {
  if (!ctx || !id128 || !out || size < 1 || rank < 0 || rank >= size) return LRS_ERR_PARAMETER;
  *out = nullptr;
  Ctx* c = static_cast<Ctx*>(ctx);
  try {
    const NcclApi& a = nccl();
    if (!a.ok) throw LrsError(LRS_ERR_NCCL, a.err);
    LRS_CUDA(cudaSetDevice(c->device));
    auto* p = new NcclPlane();
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    const ncclResult_t r = a.CommInitRank(&p->comm, size, id, rank);
    if (r != ncclSuccess) {
      delete p;
      nccl_check(r, "ncclCommInitRank");
    }
    p->stream = c->stream;
    p->device = c->device;
    p->c.rank = rank;
    p->c.size = size;
    p->c.user = p;
    p->c.allgather = plane_allgather;
    p->c.sendrecv = plane_sendrecv;
    p->c.neighbors = plane_neighbors;
    p->c.stream_ordered = 1;
    *out = &p->c;
    return LRS_OK;
  } catch (const LrsError& e) {
    c->last = lrs_error_info{};
    c->last.status = e.status;
    std::strncpy(c->last.message, e.what(), sizeof(c->last.message) - 1);
    return e.status;
  }
}

void lrs_comm_nccl_destroy(lrs_comm* comm) {
  if (!comm) return;
  auto* p = reinterpret_cast<NcclPlane*>(comm);
  if (p->comm) {
    cudaStreamSynchronize(p->stream);
    nccl().CommDestroy(p->comm);
  }
  delete p;
}

}  // extern "C"
