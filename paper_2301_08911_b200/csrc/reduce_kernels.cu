// reduce_kernels.cu -- deterministic reductions and small vector kernels.
//
// The reference's block_sum (inc/parallel.hpp:38-56) is worker-count
// independent; here the partition is a function of the problem size only
// (fixed grid of <= kReducePartials blocks, grid-stride, fixed tree fold), so
// results are bitwise reproducible run to run on the same device model.
#include "kernels.hpp"
#include "reduce.cuh"

#include <cstdint>
#include <type_traits>

namespace ihomgpu {

template <typename TN>
__global__ void __launch_bounds__(kRT) comp_sums_kernel(const TN* __restrict__ x, long long nv, double* partials,
                                                        unsigned* ticket = nullptr, double* out = nullptr) {
  __shared__ double sh[32];
  double s[3] = {0.0, 0.0, 0.0};
  for (long long i = (long long)blockIdx.x * kRT + threadIdx.x; i < nv; i += (long long)gridDim.x * kRT) {
#pragma unroll
    for (int c = 0; c < 3; ++c) s[c] += double(x[3 * i + c]);
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double r = block_reduce(s[c], sh);
    if (threadIdx.x == 0) partials[c * kReducePartials + blockIdx.x] = r;
  }
  finalize_in_last_block(partials, 3, out, ticket, sh);
}

__global__ void __launch_bounds__(kRT) finalize_kernel(const double* partials, int nparts, int ncomp, double* out) {
  __shared__ double sh[32];
  for (int c = 0; c < ncomp; ++c) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kRT) s += partials[c * kReducePartials + i];
    const double r = block_reduce(s, sh);
    if (threadIdx.x == 0) out[c] = r;
  }
}

void launch_finalize(const double* partials, int nparts, int ncomp, double* out, cudaStream_t s) {
  finalize_kernel<<<1, kRT, 0, s>>>(partials, nparts, ncomp, out);
  IHOM_LAUNCH_CHECK();
}

template <typename TN>
void launch_comp_sums(const TN* x, long long nv, double* partials, double* out, cudaStream_t s, unsigned* ticket) {
  const int g = reduce_grid(nv);
  comp_sums_kernel<TN><<<g, kRT, 0, s>>>(x, nv, partials, ticket, out);
  IHOM_LAUNCH_CHECK();
  if (ticket) return;
  finalize_kernel<<<1, kRT, 0, s>>>(partials, g, 3, out);
  IHOM_LAUNCH_CHECK();
}

template <typename TN>
__global__ void __launch_bounds__(kRT) dot_kernel(const TN* __restrict__ a, const TN* __restrict__ b, long long n,
                                                  double* partials, unsigned* ticket, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kRT + threadIdx.x; i < n; i += (long long)gridDim.x * kRT)
    s += double(a[i]) * double(b[i]);
  const double r = block_reduce(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
  finalize_in_last_block(partials, 1, out, ticket, sh);
}

template <typename TN>
void launch_dot(const TN* a, const TN* b, long long n, double* partials, double* out, cudaStream_t s,
                unsigned* ticket) {
  const int g = reduce_grid(n);
  dot_kernel<TN><<<g, kRT, 0, s>>>(a, b, n, partials, ticket, out);
  IHOM_LAUNCH_CHECK();
  if (ticket) return;
  finalize_kernel<<<1, kRT, 0, s>>>(partials, g, 1, out);
  IHOM_LAUNCH_CHECK();
}

template <typename TN>
__global__ void sub_means_kernel(TN* x, long long nv, const double* sums, long long count) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const double inv = 1.0 / double(count);
#pragma unroll
  for (int c = 0; c < 3; ++c) x[3 * i + c] = TN(fma(-sums[c], inv, double(x[3 * i + c])));
}

// f64 fields: the AoS array as a flat run of 3 nv doubles, two per thread (16-byte accesses); the
// component of flat entry j is j % 3. Same expression per entry (x - sum_c * (1 / count)).
__global__ void sub_means_flat_kernel(double* __restrict__ x, long long n3, const double* __restrict__ sums,
                                      long long count) {
  const long long j = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (j >= n3) return;
  const double inv = 1.0 / double(count);
  const int c = int(j % 3);
  // x - sum_c * inv contracted to one fma, exactly as sub_means_kernel compiles
  if (j + 1 < n3) {
    double2 v = *reinterpret_cast<const double2*>(x + j);
    v.x = fma(-sums[c], inv, v.x);
    v.y = fma(-sums[c == 2 ? 0 : c + 1], inv, v.y);
    *reinterpret_cast<double2*>(x + j) = v;
  } else {
    x[j] = fma(-sums[c], inv, x[j]);
  }
}

__global__ void sub_means_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, long long n3,
                                      const double* __restrict__ sums, long long count) {
  const long long j = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (j >= n3) return;
  const double inv = 1.0 / double(count);
  const int c = int(j % 3);
  if (j + 1 < n3) {
    double2 v = *reinterpret_cast<const double2*>(src + j);
    v.x = fma(-sums[c], inv, v.x);
    v.y = fma(-sums[c == 2 ? 0 : c + 1], inv, v.y);
    *reinterpret_cast<double2*>(dst + j) = v;
  } else {
    dst[j] = fma(-sums[c], inv, src[j]);
  }
}

// x -= mean (per component) and ||x||^2 of the result in one pass: the same per-entry fma as
// sub_means_flat_kernel and the same partition / fold as dot_kernel over the 3 nv entries, so the
// field and the norm are bitwise those of launch_sub_means + launch_dot.
__global__ void __launch_bounds__(kRT) sub_means_norm_kernel(double* __restrict__ x, long long n3,
                                                             const double* __restrict__ sums, long long count,
                                                             double* partials, unsigned* ticket, double* out) {
  __shared__ double sh[32];
  const double inv = 1.0 / double(count);
  const double m[3] = {sums[0], sums[1], sums[2]};
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kRT + threadIdx.x; i < n3; i += (long long)gridDim.x * kRT) {
    const double v = fma(-m[i % 3], inv, x[i]);
    x[i] = v;
    s += v * v;
  }
  const double r = block_reduce(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
  finalize_in_last_block(partials, 1, out, ticket, sh);
}

void launch_sub_means_norm(double* x, long long nv, const double* sums, double* partials, double* out,
                           cudaStream_t s, long long count, unsigned* ticket) {
  const long long n3 = 3 * nv;
  const int g = reduce_grid(n3);
  sub_means_norm_kernel<<<g, kRT, 0, s>>>(x, n3, sums, count > 0 ? count : nv, partials, ticket, out);
  IHOM_LAUNCH_CHECK();
  if (ticket) return;
  finalize_kernel<<<1, kRT, 0, s>>>(partials, g, 1, out);
  IHOM_LAUNCH_CHECK();
}

void launch_sub_means_copy(const double* src, double* dst, long long nv, const double* sums, cudaStream_t s,
                           long long count) {
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    throw std::invalid_argument("sub_means_copy needs 16-byte aligned fields");
  const long long n3 = 3 * nv;
  sub_means_copy_kernel<<<ceil_div((n3 + 1) / 2, 256), 256, 0, s>>>(src, dst, n3, sums, count > 0 ? count : nv);
  IHOM_LAUNCH_CHECK();
}

template <typename TN>
void launch_sub_means(TN* x, long long nv, const double* sums, cudaStream_t s, long long count) {
  if constexpr (std::is_same_v<TN, double>) {
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && knob("SUBMEANS_FLAT", 1)) {
      const long long n3 = 3 * nv;
      sub_means_flat_kernel<<<ceil_div((n3 + 1) / 2, 256), 256, 0, s>>>(x, n3, sums, count > 0 ? count : nv);
      IHOM_LAUNCH_CHECK();
      return;
    }
  }
  sub_means_kernel<TN><<<ceil_div(nv, 256), 256, 0, s>>>(x, nv, sums, count > 0 ? count : nv);
  IHOM_LAUNCH_CHECK();
}

template <typename TN>
__global__ void axpy_kernel(double* u, const TN* __restrict__ e, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[i] += double(e[i]);
}

template <typename TN>
void launch_axpy_update(double* u, const TN* e, long long n, cudaStream_t s) {
  axpy_kernel<TN><<<ceil_div(n, 256), 256, 0, s>>>(u, e, n);
  IHOM_LAUNCH_CHECK();
}

template <typename TI, typename TO>
__global__ void convert_kernel(const TI* __restrict__ x, TO* __restrict__ y, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = TO(x[i]);
}

template <typename TI, typename TO>
void launch_convert(const TI* x, TO* y, long long n, cudaStream_t s) {
  convert_kernel<TI, TO><<<ceil_div(n, 256), 256, 0, s>>>(x, y, n);
  IHOM_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(kRT) sum_kernel_r(const double* __restrict__ a, long long n, double* partials,
                                                    unsigned* ticket, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kRT + threadIdx.x; i < n; i += (long long)gridDim.x * kRT) s += a[i];
  const double r = block_reduce(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
  finalize_in_last_block(partials, 1, out, ticket, sh);
}

void launch_sum(const double* a, long long n, double* partials, double* out, cudaStream_t s, unsigned* ticket) {
  const int g = reduce_grid(n);
  sum_kernel_r<<<g, kRT, 0, s>>>(a, n, partials, ticket, out);
  IHOM_LAUNCH_CHECK();
  if (ticket) return;
  finalize_kernel<<<1, kRT, 0, s>>>(partials, g, 1, out);
  IHOM_LAUNCH_CHECK();
}

// ---- MG-PCG vector kernels (f64 outer vectors, f32 preconditioned residual) ----
__global__ void __launch_bounds__(kRT) dot_df_kernel(const double* __restrict__ a, const float* __restrict__ b,
                                                     long long n, double* partials) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kRT + threadIdx.x; i < n; i += (long long)gridDim.x * kRT)
    s += a[i] * double(b[i]);
  const double r = block_reduce(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

void launch_dot_df(const double* a, const float* b, long long n, double* partials, double* out, cudaStream_t s) {
  const int g = reduce_grid(n);
  dot_df_kernel<<<g, kRT, 0, s>>>(a, b, n, partials);
  IHOM_LAUNCH_CHECK();
  finalize_kernel<<<1, kRT, 0, s>>>(partials, g, 1, out);
  IHOM_LAUNCH_CHECK();
}

// p = z + beta p  (beta read from device memory: no host round trip)
__global__ void pcg_p_kernel(double* __restrict__ p, const float* __restrict__ z, const double* __restrict__ beta,
                             long long n, int first) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  p[i] = first ? double(z[i]) : double(z[i]) + beta[0] * p[i];
}

void launch_pcg_p(double* p, const float* z, const double* beta, long long n, bool first, cudaStream_t s) {
  pcg_p_kernel<<<ceil_div(n, 256), 256, 0, s>>>(p, z, beta, n, first ? 1 : 0);
  IHOM_LAUNCH_CHECK();
}

// u += alpha p; r -= alpha q; r32 = float(r); partials of r^2 (fixed grid, fixed fold)
__global__ void __launch_bounds__(kRT) pcg_ur_kernel(double* __restrict__ u, double* __restrict__ r,
                                                     const double* __restrict__ p, const double* __restrict__ q,
                                                     const double* __restrict__ alpha, float* __restrict__ r32,
                                                     long long n, double* partials) {
  __shared__ double sh[32];
  const double a = alpha[0];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kRT + threadIdx.x; i < n; i += (long long)gridDim.x * kRT) {
    u[i] += a * p[i];
    const double ri = r[i] - a * q[i];
    r[i] = ri;
    r32[i] = float(ri);
    s += ri * ri;
  }
  const double rr = block_reduce(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = rr;
}

void launch_pcg_ur(double* u, double* r, const double* p, const double* q, const double* alpha, float* r32,
                   long long n, double* partials, double* out, cudaStream_t s) {
  const int g = reduce_grid(n);
  pcg_ur_kernel<<<g, kRT, 0, s>>>(u, r, p, q, alpha, r32, n, partials);
  IHOM_LAUNCH_CHECK();
  finalize_kernel<<<1, kRT, 0, s>>>(partials, g, 1, out);
  IHOM_LAUNCH_CHECK();
}

// scalar = num / den on device (alpha, beta)
__global__ void ratio_kernel(const double* num, const double* den, double* out) { out[0] = num[0] / den[0]; }
void launch_ratio(const double* num, const double* den, double* out, cudaStream_t s) {
  ratio_kernel<<<1, 1, 0, s>>>(num, den, out);
  IHOM_LAUNCH_CHECK();
}

template void launch_comp_sums<double>(const double*, long long, double*, double*, cudaStream_t, unsigned*);
template void launch_comp_sums<float>(const float*, long long, double*, double*, cudaStream_t, unsigned*);
template void launch_dot<double>(const double*, const double*, long long, double*, double*, cudaStream_t, unsigned*);
template void launch_dot<float>(const float*, const float*, long long, double*, double*, cudaStream_t, unsigned*);
template void launch_sub_means<double>(double*, long long, const double*, cudaStream_t, long long);
template void launch_sub_means<float>(float*, long long, const double*, cudaStream_t, long long);
template void launch_axpy_update<float>(double*, const float*, long long, cudaStream_t);
template void launch_axpy_update<double>(double*, const double*, long long, cudaStream_t);
template void launch_convert<double, float>(const double*, float*, long long, cudaStream_t);
template void launch_convert<float, double>(const float*, double*, long long, cudaStream_t);

}  // namespace ihomgpu

namespace ihomgpu {

// Nodal fields cross the C ABI in the reference's AoS layout, which is also
// the device layout: a plain device copy.
void copy_nodal(const double* in, double* out, long long nv, cudaStream_t s) {
  if (in != out) IHOM_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * 3 * nv, cudaMemcpyDeviceToDevice, s));
}

}  // namespace ihomgpu

namespace ihomgpu {

// Colour-block location of every vertex, enumerated x-fastest (bit-exact
// check of inc/grid.hpp:73-78 and of the device neighbour arithmetic:
// out27 (optional) receives the 27 neighbour locations of every location).
__global__ void grid_locs_kernel(GridGeo g, long long* __restrict__ out, long long* __restrict__ out27) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.nv) return;
  const int x = int(i % g.n[0]);
  const long long r = i / g.n[0];
  const int y = int(r % g.n[1]), z = int(r / g.n[1]);
  out[i] = vloc(g, x, y, z);
  if (out27) {
    const int color = color_at(g, i);
    int vx, vy, vz;
    block_coords(g, color, (unsigned)(i - g.base[color]), vx, vy, vz);
    Nbhd nb;
    gather27(g, vx, vy, vz, nb);
    for (int n = 0; n < 27; ++n) out27[27 * i + n] = nb.v[n];
  }
}

void launch_grid_locs(const GridGeo& g, long long* out, long long* out27, cudaStream_t s) {
  grid_locs_kernel<<<ceil_div(g.nv, 256), 256, 0, s>>>(g, out, out27);
  IHOM_LAUNCH_CHECK();
}

// First replicated level of a z-slab hierarchy: every slab wrote the planes
// z in [owner * planes, (owner+1) * planes) of its own copy; fetch the others'
// planes from their owners (peer memory). per_vertex: 3 (AoS nodal) or 243
// (blocked stencil rows).
template <typename X>
__global__ void gather_owned_kernel(GridGeo g, PeerTable peers, int planes, int me, int per_vertex, X* dst) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= g.nv) return;
  const int color = color_at(g, loc);
  int x, y, z;
  block_coords(g, color, (unsigned)(loc - g.base[color]), x, y, z);
  const int owner = z / planes;
  if (owner == me) return;
  const X* src = static_cast<const X*>(peers.p[owner]);
  if (per_vertex == 3) {
#pragma unroll
    for (int c = 0; c < 3; ++c) dst[3 * loc + c] = src[3 * loc + c];
  } else {
    for (int k = 0; k < 243; ++k) dst[st_index(k, (unsigned)loc)] = src[st_index(k, (unsigned)loc)];
  }
}

template <typename X>
void launch_gather_owned(const GridGeo& g, PeerTable peers, int planes, int me, int per_vertex, X* dst,
                         cudaStream_t s) {
  gather_owned_kernel<X><<<ceil_div(g.nv, 128), 128, 0, s>>>(g, peers, planes, me, per_vertex, dst);
  IHOM_LAUNCH_CHECK();
}
template void launch_gather_owned<double>(const GridGeo&, PeerTable, int, int, int, double*, cudaStream_t);
template void launch_gather_owned<float>(const GridGeo&, PeerTable, int, int, int, float*, cudaStream_t);

__global__ void int_to_double_kernel(const int* in, double* out) { *out = double(*in); }
void launch_int_to_double(const int* in, double* out, cudaStream_t s) {
  int_to_double_kernel<<<1, 1, 0, s>>>(in, out);
  IHOM_LAUNCH_CHECK();
}

}  // namespace ihomgpu
