// profiler.hpp -- per-kernel-family device timing with CUDA events recorded on
// the launching stream (the bench's roofline numerator/denominator), plus
// algorithmic byte counts per launch. Disabled by default; when
// disabled a scope costs one branch.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

namespace ihomgpu {

class Profiler {
 public:
  static Profiler& get() {
    static Profiler p;
    return p;
  }
  bool enabled() const { return enabled_; }
  void enable(bool on) { enabled_ = on; }
  void reset();
  // Records a start event; returns a slot (or -1 if disabled).
  int begin(cudaStream_t s);
  void end(int slot, cudaStream_t s, const char* family, double bytes);
  // Resolves pending events (synchronises them) into the per-family totals.
  void resolve();
  struct Entry {
    long long launches = 0;
    double ms = 0.0;
    double bytes = 0.0;
  };
  const std::map<std::string, Entry>& totals() {
    resolve();
    return totals_;
  }

 private:
  struct Pending {
    int slot;
    std::string family;
    double bytes;
  };
  bool enabled_ = false;
  std::vector<cudaEvent_t> ev_;  // pairs
  int used_ = 0;
  std::vector<Pending> pending_;
  std::map<std::string, Entry> totals_;
};

// Scoped launch timing: ProfScope p(stream, "l0_gs", bytes); launch(...);
struct ProfScope {
  int slot;
  cudaStream_t s;
  const char* family;
  double bytes;
  ProfScope(cudaStream_t st, const char* fam, double b) : s(st), family(fam), bytes(b) {
    slot = (fam && Profiler::get().enabled()) ? Profiler::get().begin(st) : -1;  // fam == nullptr: inactive
  }
  ProfScope(ProfScope&& o) noexcept : slot(o.slot), s(o.s), family(o.family), bytes(o.bytes) { o.slot = -1; }
  ProfScope(const ProfScope&) = delete;
  ~ProfScope() {
    if (slot >= 0) Profiler::get().end(slot, s, family, bytes);
  }
};

}  // namespace ihomgpu
