// comm.hpp -- NCCL bound at run time (dlopen of libnccl.so.2; reuses the copy
// torch already loaded, if any), so single-GPU users need no NCCL at all.
//
// Multi-GPU scheme of this round: the six periodic cell problems
// are independent solves, so rank r solves the load cases the caller assigns
// it; every solved displacement field is then broadcast from its owner over
// NVLink (ncclBroadcast, grouped) and every rank evaluates C^H, the
// sensitivities and the design update identically -- bitwise equal to the
// 1-GPU result. Per-load solver statistics are combined with one allreduce.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace ihomgpu {

struct NcclUid {
  char internal[128];
};

class Comm {
 public:
  static bool available();                 // libnccl.so.2 loadable
  static NcclUid unique_id();              // rank 0 creates, caller distributes
  Comm(const NcclUid& id, int rank, int nranks, int device);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;

  int rank() const { return rank_; }
  int size() const { return nranks_; }
  // in-place broadcast of n doubles from root
  void broadcast(double* buf, size_t n, int root, cudaStream_t s);
  void group_start();
  void group_end();
  void allreduce_sum(double* buf, size_t n, cudaStream_t s);

 private:
  void* comm_ = nullptr;  // ncclComm_t
  int rank_ = 0, nranks_ = 1;
};

}  // namespace ihomgpu
