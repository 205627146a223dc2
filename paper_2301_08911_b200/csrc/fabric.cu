// fabric.cu -- see fabric.hpp.
#include "fabric.hpp"

#include <cuda.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "common.cuh"

namespace ihomgpu {

// ---------------------------------------------------------------- kernels
struct WaitList {
  int r[kMaxRanks];
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Arrive (release at system scope so peers reading this rank's memory over NVLink see everything the stream
// wrote before), then wait for the listed ranks -- bounded: after timeout_ns the wait gives up, records the
// rank it waited on in *err and returns; once *err is set this rank's barriers no longer wait.
__global__ void signal_wait_kernel(unsigned long long* own, PeerTable flags, WaitList wl, int nwait,
                                   unsigned long long epoch, unsigned long long* err, unsigned long long timeout_ns) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(own), "l"(epoch) : "memory");
  if (*err != 0ull) return;
  const unsigned long long t0 = globaltimer_ns();
  for (int i = 0; i < nwait; ++i) {
    const unsigned long long* f = static_cast<const unsigned long long*>(flags.p[wl.r[i]]);
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= epoch) break;
      if (globaltimer_ns() - t0 > timeout_ns) {
        *err = 1ull + (unsigned long long)wl.r[i];
        return;
      }
      __nanosleep(200);
    }
  }
  __threadfence_system();
}

void launch_signal_wait(unsigned long long* own, PeerTable flags, const int* wait_on, int nwait,
                        unsigned long long epoch, unsigned long long* err, unsigned long long timeout_ns,
                        cudaStream_t s) {
  WaitList wl{};
  for (int i = 0; i < nwait; ++i) wl.r[i] = wait_on[i];
  signal_wait_kernel<<<1, 1, 0, s>>>(own, flags, wl, nwait, epoch, err, timeout_ns);
  IHOM_LAUNCH_CHECK();
}

// out[i] = fold over ranks 0..n-1 of box_r[i] (rank order: identical on every rank)
__global__ void mailbox_fold_kernel(PeerTable boxes, int nranks, int n, int is_max, double* out) {
  const int i = threadIdx.x;
  if (i >= n) return;
  double acc = static_cast<const double*>(boxes.p[0])[i];
  for (int r = 1; r < nranks; ++r) {
    const double v = static_cast<const double*>(boxes.p[r])[i];
    acc = is_max ? fmax(acc, v) : acc + v;
  }
  out[i] = acc;
}

void launch_mailbox_fold(PeerTable boxes, int nranks, int n, bool is_max, double* out, cudaStream_t s) {
  mailbox_fold_kernel<<<1, kMailbox, 0, s>>>(boxes, nranks, n, is_max ? 1 : 0, out);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- Fabric
Fabric::Fabric(int nranks) : n_(nranks), rs_(static_cast<size_t>(nranks)) {
  if (nranks < 1 || nranks > kMaxRanks) throw std::invalid_argument("z-slab count must be in [1, 8]");
}

void Fabric::init_mailboxes(int rank) {
  RankState& st = rs_[size_t(rank)];
  IHOM_CUDA(cudaMalloc(&st.mailbox, sizeof(double) * 2 * kMailbox));
  IHOM_CUDA(cudaMemset(st.mailbox, 0, sizeof(double) * 2 * kMailbox));
  const std::vector<void*> all = exchange(rank, st.mailbox);
  for (int r = 0; r < n_; ++r) st.boxes.p[r] = all[size_t(r)];
}

void Fabric::allreduce(int rank, double* x, int n, bool is_max, cudaStream_t s) {
  if (n > kMailbox) throw std::invalid_argument("allreduce: too many values");
  if (n_ == 1) return;
  RankState& st = rs_[size_t(rank)];
  if (!st.mailbox) init_mailboxes(rank);  // collective: the first allreduce is reached by every rank
  const int off = st.parity * kMailbox;
  st.parity ^= 1;
  // slot `off` of every mailbox is not read by anyone before this rank's next
  // barrier (alternating slots: the previous use of this slot was folded by
  // all ranks before they passed the barrier of the allreduce in between).
  IHOM_CUDA(cudaMemcpyAsync(st.mailbox + off, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  barrier(rank, s);
  PeerTable b{};
  for (int r = 0; r < n_; ++r) b.p[r] = static_cast<const double*>(st.boxes.p[r]) + off;
  launch_mailbox_fold(b, n_, n, is_max, x, s);
}

// ---------------------------------------------------------------- LocalFabric
LocalFabric::LocalFabric(int nranks, int device) : Fabric(nranks), device_(device), slots_(static_cast<size_t>(nranks)) {
  IHOM_CUDA(cudaSetDevice(device));
  ev_.resize(size_t(nranks));
  for (auto& e : ev_) IHOM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

LocalFabric::~LocalFabric() {
  for (auto& e : ev_) cudaEventDestroy(e);
  for (auto& st : rs_)
    if (st.mailbox) cudaFree(st.mailbox);
}

void LocalFabric::host_barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  const long long gen = generation_;
  if (++arrived_ == n_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return generation_ != gen; });
  }
}

std::vector<void*> LocalFabric::exchange(int rank, void* local) {
  slots_[size_t(rank)] = local;
  host_barrier();
  std::vector<void*> out = slots_;
  host_barrier();  // nobody overwrites a slot before everyone copied
  return out;
}

void LocalFabric::barrier(int rank, cudaStream_t s, bool halo) {
  (void)halo;  // one process: the host barrier orders every slab anyway
  if (n_ == 1) return;
  IHOM_CUDA(cudaEventRecord(ev_[size_t(rank)], s));
  host_barrier();  // every rank's record is enqueued
  for (int r = 0; r < n_; ++r)
    if (r != rank) IHOM_CUDA(cudaStreamWaitEvent(s, ev_[size_t(r)], 0));
  host_barrier();  // every wait is enqueued before any rank re-records
}

// ---------------------------------------------------------------- IpcFabric
IpcFabric::IpcFabric(int rank, int nranks, int device, HostAllgather ag, void* user)
    : Fabric(nranks), rank_(rank), device_(device), ag_(ag), user_(user) {
  if (!ag) throw std::invalid_argument("IPC fabric needs a host allgather");
  if (rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank");
  IHOM_CUDA(cudaSetDevice(device));
  IHOM_CUDA(cudaMalloc(&flag_, sizeof(unsigned long long)));
  IHOM_CUDA(cudaMemset(flag_, 0, sizeof(unsigned long long)));
  IHOM_CUDA(cudaMalloc(&err_, sizeof(unsigned long long)));
  IHOM_CUDA(cudaMemset(err_, 0, sizeof(unsigned long long)));
  timeout_ns_ = (unsigned long long)knob("FABRIC_TIMEOUT_S", 60) * 1000000000ull;
  const std::vector<void*> f = exchange(rank, flag_);
  for (int r = 0; r < nranks; ++r) flags_.p[r] = f[size_t(r)];
}

IpcFabric::~IpcFabric() {
  for (auto& kv : opened_)
    if (kv.first.first != rank_) cudaIpcCloseMemHandle(kv.second);
  if (flag_) cudaFree(flag_);
  if (err_) cudaFree(err_);
  for (auto& st : rs_)
    if (st.mailbox) cudaFree(st.mailbox);
}

std::vector<void*> IpcFabric::exchange(int rank, void* local) {
  if (rank != rank_) throw std::invalid_argument("IPC fabric: exchange from a foreign rank");
  struct Rec {
    cudaIpcMemHandle_t h;
    std::uintptr_t base;
    std::uint64_t offset;
  };
  // allocation base of `local` (IPC handles name whole allocations); the driver
  // entry point is fetched through the runtime, so no -lcuda link is needed
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<GetRange>(fn);
  }();
  if (!get_range) throw CudaError("cuMemGetAddressRange entry point unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(local)) != CUDA_SUCCESS)
    throw CudaError("cuMemGetAddressRange failed for an exchanged buffer");
  Rec mine{};
  IHOM_CUDA(cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)));
  mine.base = std::uintptr_t(base);
  mine.offset = std::uint64_t(reinterpret_cast<std::uintptr_t>(local) - std::uintptr_t(base));
  std::vector<Rec> all(static_cast<size_t>(n_));
  ag_(&mine, all.data(), sizeof(Rec), user_);
  std::vector<void*> out(static_cast<size_t>(n_));
  for (int r = 0; r < n_; ++r) {
    const Rec& q = all[size_t(r)];
    if (r == rank_) {
      out[size_t(r)] = local;
      continue;
    }
    auto key = std::make_pair(r, q.base);
    auto it = opened_.find(key);
    if (it == opened_.end()) {
      void* p = nullptr;
      IHOM_CUDA(cudaIpcOpenMemHandle(&p, q.h, cudaIpcMemLazyEnablePeerAccess));
      it = opened_.emplace(key, p).first;
    }
    out[size_t(r)] = static_cast<char*>(it->second) + q.offset;
  }
  return out;
}

void IpcFabric::barrier(int rank, cudaStream_t s, bool halo) {
  (void)rank;
  if (n_ == 1) return;
  int wait_on[kMaxRanks], nw = 0;
  if (halo) {  // the z-neighbour slabs (periodic in z)
    const int lo = (rank_ + n_ - 1) % n_, hi = (rank_ + 1) % n_;
    wait_on[nw++] = lo;
    if (hi != lo) wait_on[nw++] = hi;
  } else {
    for (int r = 0; r < n_; ++r)
      if (r != rank_) wait_on[nw++] = r;
  }
  launch_signal_wait(flag_, flags_, wait_on, nw, ++epoch_, err_, timeout_ns_, s);
}

void IpcFabric::check(int rank) {
  (void)rank;
  unsigned long long e = 0;
  IHOM_CUDA(cudaMemcpy(&e, err_, sizeof(e), cudaMemcpyDeviceToHost));
  if (e)
    throw CudaError("z-slab rank " + std::to_string(rank_) + ": barrier timed out after " +
                    std::to_string(timeout_ns_ / 1000000000ull) + " s waiting for rank " + std::to_string(e - 1) +
                    " (dead or diverged peer)");
}

}  // namespace ihomgpu
