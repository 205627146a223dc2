// profiler.cpp -- see profiler.hpp.
#include "profiler.hpp"

#include "common.cuh"

namespace ihomgpu {

void Profiler::reset() {
  resolve();
  totals_.clear();
}

int Profiler::begin(cudaStream_t s) {
  if (used_ + 2 > (int)ev_.size()) {
    for (int k = 0; k < 256; ++k) {
      cudaEvent_t e;
      IHOM_CUDA(cudaEventCreate(&e));
      ev_.push_back(e);
    }
  }
  const int slot = used_;
  used_ += 2;
  IHOM_CUDA(cudaEventRecord(ev_[size_t(slot)], s));
  return slot;
}

void Profiler::end(int slot, cudaStream_t s, const char* family, double bytes) {
  IHOM_CUDA(cudaEventRecord(ev_[size_t(slot + 1)], s));
  pending_.push_back({slot, family, bytes});
  if (used_ >= 8192) resolve();  // bound the pool
}

void Profiler::resolve() {
  for (const auto& p : pending_) {
    IHOM_CUDA(cudaEventSynchronize(ev_[size_t(p.slot + 1)]));
    float ms = 0.0f;
    IHOM_CUDA(cudaEventElapsedTime(&ms, ev_[size_t(p.slot)], ev_[size_t(p.slot + 1)]));
    Entry& e = totals_[p.family];
    e.launches += 1;
    e.ms += ms;
    e.bytes += p.bytes;
  }
  pending_.clear();
  used_ = 0;
}

}  // namespace ihomgpu
