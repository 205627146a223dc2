// fabric.hpp -- how the z-slabs of one grid reach each other.
//
// A z-slab decomposition puts slab r (global z planes [r t, (r+1) t)) on rank
// r. Kernels read across a slab face directly from the neighbour's buffer (a
// ZLink, common.cuh): peer memory mapped over NVLink between processes, or
// another slab's buffer on the same device when all slabs live in one process
// (the single-GPU test configuration). Synchronisation and reductions are
// stream-ordered device operations, so no rank ever blocks its host on a peer
// except while collectively exchanging buffer addresses at allocation time.
//
//   exchange(local)  collective: every rank's pointer of the same logical
//                    buffer, mapped into this rank (called in the same order
//                    on every rank -- SPMD allocation order);
//   barrier(s)       work enqueued on s after the barrier sees every rank's
//                    work enqueued before its barrier (halo = true: only the
//                    z-neighbour slabs r-1, r+1 -- enough to order halo reads
//                    and writes, which never reach further);
//   check()          throws if a barrier of this rank timed out (a dead or
//                    diverged peer): barriers never spin forever;
//   allreduce(x, n)  n doubles, sum or max, folded in rank order -- the
//                    result is bitwise identical on every rank, so every rank
//                    takes the same convergence / bisection decisions.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace ihomgpu {

constexpr int kMaxRanks = 8;
constexpr int kMailbox = 64;  // doubles per allreduce slot

struct PeerTable {  // a buffer on every rank, by rank (kernel argument)
  const void* p[kMaxRanks];
};

class Fabric {
 public:
  explicit Fabric(int nranks);
  virtual ~Fabric() = default;
  int size() const { return n_; }
  virtual std::vector<void*> exchange(int rank, void* local) = 0;
  virtual void barrier(int rank, cudaStream_t s, bool halo = false) = 0;
  virtual void check(int rank) { (void)rank; }
  void allreduce(int rank, double* x, int n, bool is_max, cudaStream_t s);
  // per-rank mailboxes (2 slots of kMailbox doubles, alternating per allreduce)
  void init_mailboxes(int rank);

 protected:
  int n_;
  struct RankState {
    double* mailbox = nullptr;  // own, device
    PeerTable boxes{};          // every rank's mailbox
    int parity = 0;
  };
  std::vector<RankState> rs_;
};

// All slabs in this process on one device, one host thread per slab.
class LocalFabric : public Fabric {
 public:
  LocalFabric(int nranks, int device);
  ~LocalFabric() override;
  std::vector<void*> exchange(int rank, void* local) override;
  void barrier(int rank, cudaStream_t s, bool halo = false) override;

 private:
  void host_barrier();
  int device_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  long long generation_ = 0;
  std::vector<void*> slots_;
  std::vector<cudaEvent_t> ev_;
};

// One slab per process; buffers exchanged as CUDA IPC handles through a
// host allgather supplied by the caller (torch.distributed, MPI, ...).
// Barriers are device-side flags in peer memory (release/acquire, system scope).
using HostAllgather = void (*)(const void* send, void* recv, std::size_t bytes, void* user);

class IpcFabric : public Fabric {
 public:
  IpcFabric(int rank, int nranks, int device, HostAllgather ag, void* user);
  ~IpcFabric() override;
  std::vector<void*> exchange(int rank, void* local) override;
  void barrier(int rank, cudaStream_t s, bool halo = false) override;
  void check(int rank) override;

 private:
  int rank_, device_;
  HostAllgather ag_;
  void* user_;
  unsigned long long* flag_ = nullptr;  // own arrival counter (device)
  unsigned long long* err_ = nullptr;   // own barrier error word (device): 0, or 1 + the rank waited on
  unsigned long long timeout_ns_ = 0;
  PeerTable flags_{};
  unsigned long long epoch_ = 0;
  std::map<std::pair<int, std::uintptr_t>, void*> opened_;  // (rank, remote base) -> mapped base
};

// z-slab placement: this rank holds global z planes [rank t, (rank+1) t),
// t = n2 / nranks, of a grid whose other slabs are reached through the
// fabric. nranks == 1: one periodic domain (no fabric).
struct Slab {
  Fabric* fab = nullptr;
  int rank = 0;
  int nranks = 1;
  bool on() const { return fab != nullptr && nranks > 1; }
  void sync(cudaStream_t s, bool halo = false) const {
    if (on()) fab->barrier(rank, s, halo);
  }
  void allreduce(double* x, int n, bool is_max, cudaStream_t s) const {
    if (on()) fab->allreduce(rank, x, n, is_max, s);
  }
};

// Kernels (fabric.cu)
// Arrive with `epoch`, then wait for ranks wait_on[0..nwait) to arrive (bounded by timeout_ns; a timeout
// sets *err and later barriers of this rank stop waiting, so the host sees the failure at its next check).
void launch_signal_wait(unsigned long long* own, PeerTable flags, const int* wait_on, int nwait,
                        unsigned long long epoch, unsigned long long* err, unsigned long long timeout_ns,
                        cudaStream_t s);
void launch_mailbox_fold(PeerTable boxes, int nranks, int n, bool is_max, double* out, cudaStream_t s);

}  // namespace ihomgpu
