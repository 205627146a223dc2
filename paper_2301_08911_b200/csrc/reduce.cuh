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

}  // namespace ihomgpu
