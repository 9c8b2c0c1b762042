// Multi-GPU plumbing of the C++ drop-in API: one process per GPU, partitions sharded
// across the ranks (factorize_dist, solver.hpp).  The library exchanges only what
// SURVEY.md 2.4 lists (C1 rank-r interface messages, C3 SpMV halos, C4 partition-ordered
// dot partials, C5 spike tips at setup) through a Communicator.
//
//   NcclCommunicator  the in-library NCCL data plane (liblrspike_cuda.so links NCCL):
//                     grouped ncclSend / ncclRecv for both neighbour directions and
//                     ncclAllGather, enqueued on the context stream -- the library does
//                     not synchronize the stream before an exchange the device consumes
//   Communicator      any other transport (MPI, gloo, ...): host callbacks on device
//                     buffers, the library synchronizes its stream before each call
#pragma once

#include <array>
#include <cstdint>

#include "lrspike/matrix.hpp"

struct lrs_comm;

namespace lrspike {

class Device;

class Communicator {
 public:
  virtual ~Communicator() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  /// recv[q * count .. (q + 1) * count) = send of rank q (device pointers, doubles).
  virtual void allgather(const double* send, double* recv, index_t count) = 0;
  /// Send `scount` doubles to `dest` and receive `rcount` from `source` (< 0: none).
  virtual void sendrecv(const double* send, index_t scount, int dest, double* recv,
                        index_t rcount, int source) = 0;
  /// The C-ABI view (lrs_comm) the library calls; owned by this object.
  virtual const lrs_comm* c_comm();

 protected:
  std::array<unsigned char, 64> cstore_{};  // lrs_comm storage (see lrspike_api.cpp)
};

/// The NCCL data plane inside liblrspike_cuda.so (lrs_comm_nccl_create).  Every rank
/// passes the same 128-byte ncclUniqueId (made by rank 0 with nccl_unique_id() and
/// broadcast by the launcher, e.g. through a file or torch.distributed).
class NcclCommunicator : public Communicator {
 public:
  static std::array<unsigned char, 128> nccl_unique_id();
  NcclCommunicator(Device& dev, const std::array<unsigned char, 128>& id, int rank, int size);
  ~NcclCommunicator() override;
  NcclCommunicator(const NcclCommunicator&) = delete;
  NcclCommunicator& operator=(const NcclCommunicator&) = delete;
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void allgather(const double* send, double* recv, index_t count) override;
  void sendrecv(const double* send, index_t scount, int dest, double* recv, index_t rcount,
                int source) override;
  const lrs_comm* c_comm() override { return comm_; }

 private:
  lrs_comm* comm_ = nullptr;
  int rank_, size_;
};

}  // namespace lrspike
