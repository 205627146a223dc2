// fem_kernels.cu -- level-0 matrix-free kernels (src/fem.cpp:98-156) and the
// SIMP coefficient kernel (src/multigrid.cpp:263-279).
//
// One thread per vertex. The 27 neighbour locations and 8 incident elements
// are recomputed arithmetically from the colour-block coordinates
// (src/fem.cpp:37-68); nothing topological is stored. Coefficients of one
// neighbour are merged in the arithmetic type TA from the 8 element
// coefficients (converted once per vertex) and applied to the nodal data:
// with TA = double this avoids the per-coefficient f32->f64 conversion
// (F2F, ~16/clk/SM on B200, measured) the reference's float merge would need.
#include "kernels.hpp"
#include "ku_gen.cuh"

namespace ihomgpu {

__constant__ double c_blk_d[8][8][9];
__constant__ float c_blk_f[8][8][9];
__constant__ double c_fmacro[8][6][3];
// kappa classes of the factored stencil (ku_gen.cuh): kappa_k = lam' alpha_k + mu' beta_k
__constant__ double c_kap_d[kKappaClasses];
__constant__ float c_kap_f[kKappaClasses];

void upload_fem_tables(const StiffnessTables& t, const K0Matrix& k, cudaStream_t s) {
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_blk_d, t.blk, sizeof(t.blk), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_blk_f, t.blk_f, sizeof(t.blk_f), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_fmacro, t.fmacro, sizeof(t.fmacro), 0, cudaMemcpyHostToDevice, s));
  // lam' and mu' recovered from K0 itself: K0[0][0] = 8 lam' + 32 mu', K0[0][1] = 3 lam' + 3 mu'
  // (the 14-value structure, tests/test_material.cpp:50-68); verified against every kappa class below.
  const double a = k.k[0][0], b = k.k[0][1];
  const double mu = (a - 8.0 * b / 3.0) / 24.0, lam = b / 3.0 - mu;
  static double kd[kKappaClasses];
  static float kf[kKappaClasses];
  for (int c = 0; c < kKappaClasses; ++c) {
    kd[c] = lam * kKappaAlpha[c] + mu * kKappaBeta[c];
    kf[c] = float(kd[c]);
  }
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_kap_d, kd, sizeof(kd), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_kap_f, kf, sizeof(kf), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaStreamSynchronize(s));
}

template <typename TA>
__device__ __forceinline__ const TA* kappa();
template <>
__device__ __forceinline__ const double* kappa<double>() {
  return c_kap_d;
}
template <>
__device__ __forceinline__ const float* kappa<float>() {
  return c_kap_f;
}

template <typename TA>
__device__ __forceinline__ TA blkv(int ke, int j, int e);
template <>
__device__ __forceinline__ double blkv<double>(int ke, int j, int e) {
  return c_blk_d[ke][j][e];
}
template <>
__device__ __forceinline__ float blkv<float>(int ke, int j, int e) {
  return c_blk_f[ke][j][e];
}

// Merged 3x3 block of neighbour n from the 8 incident coefficients
// (inc/fem.hpp:93-99): pairs (ke, j) with pair_ngb(ke, j) == n, in the
// reference's group order (ke outer, j inner). Fully unrolled; the group
// membership test folds at compile time.
template <typename TA, int N>
__device__ __forceinline__ void merged_block(const TA q[8], TA c[9]) {
#pragma unroll
  for (int e = 0; e < 9; ++e) c[e] = TA(0);
#pragma unroll
  for (int ke = 0; ke < 8; ++ke)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (pair_ngb(ke, j) == N) {
#pragma unroll
        for (int e = 0; e < 9; ++e) c[e] = fma(q[ke], blkv<TA>(ke, j, e), c[e]);
      }
}

template <typename TA, typename TN, int N>
__device__ __forceinline__ void accum_block(const TA q[8], const Nbhd& nb, const TN* __restrict__ ux,
                                            const TN* __restrict__ uy, const TN* __restrict__ uz, TA y[3]) {
  TA c[9];
  merged_block<TA, N>(q, c);
  const TA a = TA(ux[nb.v[N]]), b = TA(uy[nb.v[N]]), d = TA(uz[nb.v[N]]);
  y[0] = fma(c[0], a, fma(c[1], b, fma(c[2], d, y[0])));
  y[1] = fma(c[3], a, fma(c[4], b, fma(c[5], d, y[1])));
  y[2] = fma(c[6], a, fma(c[7], b, fma(c[8], d, y[2])));
}

// Off-diagonal part M u over the 26 neighbours (n != 13).
template <typename TA, typename TN, int N = 0>
__device__ __forceinline__ void accum_offdiag(const TA q[8], const Nbhd& nb, const TN* __restrict__ ux,
                                              const TN* __restrict__ uy, const TN* __restrict__ uz, TA y[3]) {
  if constexpr (N < 27) {
    if constexpr (N != 13) accum_block<TA, TN, N>(q, nb, ux, uy, uz, y);
    accum_offdiag<TA, TN, N + 1>(q, nb, ux, uy, uz, y);
  }
}

template <typename TC, typename TA>
__device__ __forceinline__ void load_q(const TC* __restrict__ coeff, const Nbhd& nb, TA q[8]) {
#pragma unroll
  for (int ke = 0; ke < 8; ++ke) q[ke] = TA(coeff[nb.e[ke]]);
}

// ---------------------------------------------------------------- coeff
template <typename TC>
__global__ void coeff_kernel(const double* __restrict__ rho, TC* __restrict__ coeff, long long m, double p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) coeff[i] = TC(pow(double(TC(rho[i])), p));  // src/multigrid.cpp:270
}

template <typename TC>
void launch_coeff(const double* rho, TC* coeff, long long m, double penal, cudaStream_t s) {
  coeff_kernel<TC><<<ceil_div(m, 256), 256, 0, s>>>(rho, coeff, m, penal);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- apply / residual
template <typename TC, typename TN, typename TA>
__global__ void __launch_bounds__(128) l0_apply_kernel(GridGeo g, const TC* __restrict__ coeff,
                                                       const TN* __restrict__ u, const TN* __restrict__ f,
                                                       TN* __restrict__ y) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= g.nv) return;
  const int color = color_at(g, loc);
  int x, yy, z;
  block_coords(g, color, (unsigned)(loc - g.base[color]), x, yy, z);
  Nbhd nb;
  gather27(g, x, yy, z, nb);
  TA q[8];
  load_q(coeff, nb, q);
  const long long nv = g.nv;
  auto U = [&](int n, int c) { return TA(__ldg(u + c * nv + nb.v[n])); };
  TA acc[3];
  ku_vertex<TA>(q, kappa<TA>(), U, acc);  // factored K0 (ku_gen.cuh), inc/fem.hpp:86-105 semantics
  if (f) {
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c * nv + loc] = TN(TA(f[c * nv + loc]) - acc[c]);
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c * nv + loc] = TN(acc[c]);
  }
}

template <typename TC, typename TN, typename TA>
void launch_l0_apply(const GridGeo& g, const TC* coeff, const TN* u, const TN* f, TN* y, cudaStream_t s) {
  l0_apply_kernel<TC, TN, TA><<<ceil_div(g.nv, 128), 128, 0, s>>>(g, coeff, u, f, y);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- Gauss-Seidel colour pass
template <typename TC, typename TN, typename TA>
__global__ void __launch_bounds__(128) l0_gs_kernel(GridGeo g, const TC* __restrict__ coeff,
                                                    const TN* __restrict__ f, const TN* __restrict__ ur, TN* uw,
                                                    int color) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.size[color]) return;
  int x, yy, z;
  block_coords(g, color, (unsigned)i, x, yy, z);
  Nbhd nb;
  gather27(g, x, yy, z, nb);
  TA q[8];
  load_q(coeff, nb, q);
  const long long nv = g.nv;
  auto U = [&](int n, int c) { return TA(__ldg(ur + c * nv + nb.v[n])); };
  TA m[3], sblk[9];
  ku_vertex_split<TA>(q, kappa<TA>(), U, m, sblk);  // S (n = 13) and M u (n != 13), inc/fem.hpp:109-133
  const long long loc = g.base[color] + i;
  double S[9], rhs[3], out[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) S[e] = double(sblk[e]);
#pragma unroll
  for (int c = 0; c < 3; ++c) rhs[c] = double(f[c * nv + loc]) - double(m[c]);
  solve3(S, rhs, out);  // src/fem.cpp:131-135
#pragma unroll
  for (int c = 0; c < 3; ++c) uw[c * nv + loc] = TN(out[c]);
}

template <typename TC, typename TN, typename TA>
void launch_l0_gs_color(const GridGeo& g, const TC* coeff, const TN* f, TN* u, int color, cudaStream_t s) {
  l0_gs_kernel<TC, TN, TA><<<ceil_div(g.size[color], 128), 128, 0, s>>>(g, coeff, f, u, u, color);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- macro force
template <typename TC>
__global__ void macro_force_kernel(GridGeo g, const TC* __restrict__ coeff, int load, double* __restrict__ f) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= g.nv) return;
  const int color = color_at(g, loc);
  int x, y, z;
  block_coords(g, color, (unsigned)(loc - g.base[color]), x, y, z);
  Nbhd nb;
  gather27(g, x, y, z, nb);
  double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int ke = 0; ke < 8; ++ke) {  // src/fem.cpp:145-150
    const double q = double(coeff[nb.e[ke]]);
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] += q * c_fmacro[ke][load][c];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) f[c * g.nv + loc] = acc[c];
}

template <typename TC>
void launch_macro_force(const GridGeo& g, const TC* coeff, int load, double* f, cudaStream_t s) {
  macro_force_kernel<TC><<<ceil_div(g.nv, 256), 256, 0, s>>>(g, coeff, load, f);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- instantiations
template void launch_coeff<float>(const double*, float*, long long, double, cudaStream_t);
template void launch_coeff<double>(const double*, double*, long long, double, cudaStream_t);
template void launch_macro_force<float>(const GridGeo&, const float*, int, double*, cudaStream_t);
template void launch_macro_force<double>(const GridGeo&, const double*, int, double*, cudaStream_t);

#define INST_L0(TC, TN, TA)                                                                                    \
  template void launch_l0_apply<TC, TN, TA>(const GridGeo&, const TC*, const TN*, const TN*, TN*, cudaStream_t); \
  template void launch_l0_gs_color<TC, TN, TA>(const GridGeo&, const TC*, const TN*, TN*, int, cudaStream_t);
INST_L0(float, double, double)   // mixed, f64 nodal (parity)
INST_L0(double, double, double)  // all-double
INST_L0(float, float, float)     // mixed inner correction cycle
#undef INST_L0

}  // namespace ihomgpu
