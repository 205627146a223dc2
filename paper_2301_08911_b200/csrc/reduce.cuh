// reduce.cuh -- the deterministic block partition and tree fold shared by every
// reduction (reduce_kernels.cu) and by producers that fold their output's sums
// into the same pass (fem_kernels.cu macro force). Any kernel that uses
// reduce_grid(n) blocks of kRT threads, a grid-stride loop over n and
// block_reduce produces partials bitwise equal to the standalone reduction.
#pragma once

#include "kernels.hpp"

namespace ihomgpu {

constexpr int kRT = 256;

inline int reduce_grid(long long n) {
  long long g = (n + kRT * 8 - 1) / (kRT * 8);
  if (g < 1) g = 1;
  if (g > kReducePartials) g = kReducePartials;
  return int(g);
}

__device__ __forceinline__ double block_reduce(double v, double* sh) {
  const int t = threadIdx.x;
  // warp level, fixed shuffle order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((t & 31) == 0) sh[t >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (t < 32) {
    r = (t < (int)(blockDim.x >> 5)) ? sh[t] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

// Second stage in the grid's last block (ticket: a zeroed counter per workspace, left zeroed): the block
// that finishes last folds the gridDim.x partials of each component exactly as finalize_kernel does
// (same thread stride, same tree), so the result equals the two-launch form bit for bit. No-op when
// ticket is null (the caller launches finalize_kernel instead).
__device__ __forceinline__ void finalize_in_last_block(const double* partials, int ncomp, double* out,
                                                       unsigned* ticket, double* sh) {
  __shared__ int last;
  if (!ticket) return;
  if (threadIdx.x == 0) {
    __threadfence();  // this block's partials are visible before its ticket
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = 0; c < ncomp; ++c) {
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kRT) s += __ldcg(partials + c * kReducePartials + i);
    const double r = block_reduce(s, sh);
    if (threadIdx.x == 0) out[c] = r;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

}  // namespace ihomgpu
