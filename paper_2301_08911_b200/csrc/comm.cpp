// comm.cpp -- see comm.hpp.
#include "comm.hpp"

#include <dlfcn.h>

#include <stdexcept>

#include "common.cuh"

namespace ihomgpu {

namespace {

// Minimal NCCL ABI (nccl.h 2.x): the handful of entry points used here.
using ncclResult = int;
using ncclComm = void*;
enum { kNcclFloat64 = 8, kNcclSum = 0 };
struct NcclApi {
  void* h = nullptr;
  ncclResult (*getUniqueId)(NcclUid*) = nullptr;
  ncclResult (*commInitRank)(ncclComm*, int, NcclUid, int) = nullptr;
  ncclResult (*commDestroy)(ncclComm) = nullptr;
  ncclResult (*broadcast)(const void*, void*, size_t, int, int, ncclComm, cudaStream_t) = nullptr;
  ncclResult (*allReduce)(const void*, void*, size_t, int, int, ncclComm, cudaStream_t) = nullptr;
  ncclResult (*groupStart)() = nullptr;
  ncclResult (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a = [] {
    NcclApi x;
    x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // already in the process (torch)?
    if (!x.h) x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) return x;
    auto sym = [&](const char* n) { return dlsym(x.h, n); };
    x.getUniqueId = reinterpret_cast<decltype(x.getUniqueId)>(sym("ncclGetUniqueId"));
    x.commInitRank = reinterpret_cast<decltype(x.commInitRank)>(sym("ncclCommInitRank"));
    x.commDestroy = reinterpret_cast<decltype(x.commDestroy)>(sym("ncclCommDestroy"));
    x.broadcast = reinterpret_cast<decltype(x.broadcast)>(sym("ncclBroadcast"));
    x.allReduce = reinterpret_cast<decltype(x.allReduce)>(sym("ncclAllReduce"));
    x.groupStart = reinterpret_cast<decltype(x.groupStart)>(sym("ncclGroupStart"));
    x.groupEnd = reinterpret_cast<decltype(x.groupEnd)>(sym("ncclGroupEnd"));
    x.getErrorString = reinterpret_cast<decltype(x.getErrorString)>(sym("ncclGetErrorString"));
    x.ok = x.getUniqueId && x.commInitRank && x.commDestroy && x.broadcast && x.allReduce && x.groupStart &&
           x.groupEnd && x.getErrorString;
    return x;
  }();
  return a;
}

void check(ncclResult r, const char* what) {
  if (r != 0) throw CudaError(std::string("NCCL ") + what + ": " + api().getErrorString(r));
}

}  // namespace

bool Comm::available() { return api().ok; }

NcclUid Comm::unique_id() {
  if (!available()) throw std::invalid_argument("libnccl.so.2 not available");
  NcclUid id;
  check(api().getUniqueId(&id), "ncclGetUniqueId");
  return id;
}

Comm::Comm(const NcclUid& id, int rank, int nranks, int device) : rank_(rank), nranks_(nranks) {
  if (!available()) throw std::invalid_argument("libnccl.so.2 not available");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank / world size");
  IHOM_CUDA(cudaSetDevice(device));
  ncclComm c = nullptr;
  check(api().commInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  comm_ = c;
}

Comm::~Comm() {
  if (comm_) api().commDestroy(comm_);
}

void Comm::broadcast(double* buf, size_t n, int root, cudaStream_t s) {
  check(api().broadcast(buf, buf, n, kNcclFloat64, root, comm_, s), "ncclBroadcast");
}

void Comm::group_start() { check(api().groupStart(), "ncclGroupStart"); }
void Comm::group_end() { check(api().groupEnd(), "ncclGroupEnd"); }

void Comm::allreduce_sum(double* buf, size_t n, cudaStream_t s) {
  check(api().allReduce(buf, buf, n, kNcclFloat64, kNcclSum, comm_, s), "ncclAllReduce");
}

}  // namespace ihomgpu
