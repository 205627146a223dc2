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
#include "hada_gen.cuh"

#include <cuda_pipeline.h>

#include <cstdlib>
#include <type_traits>
#include <string>

namespace ihomgpu {

__constant__ double c_blk_d[8][8][9];
__constant__ float c_blk_f[8][8][9];
__constant__ double c_fmacro[8][6][3];
// kappa classes of the factored stencil (ku_gen.cuh): kappa_k = lam' alpha_k + mu' beta_k
__constant__ double c_kap_d[kKappaClasses];
__constant__ float c_kap_f[kKappaClasses];
// element stiffness classes in the sum/difference basis (hada_gen.cuh): (lam' alpha_k + mu' beta_k) / 64
__constant__ double c_hada_d[kHadaClasses];
__constant__ float c_hada_f[kHadaClasses];

void upload_fem_tables(const StiffnessTables& t, const K0Matrix& k, cudaStream_t s) {
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_blk_d, t.blk, sizeof(t.blk), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_blk_f, t.blk_f, sizeof(t.blk_f), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_fmacro, t.fmacro, sizeof(t.fmacro), 0, cudaMemcpyHostToDevice, s));
  // lam' and mu' recovered from two K0 entries with known integer structure (ku_gen.cuh kK0Probe)
  const double k1 = k.k[kK0Probe[0][0]][kK0Probe[0][1]], k2 = k.k[kK0Probe[1][0]][kK0Probe[1][1]];
  const double a1 = kK0Probe[0][2], b1 = kK0Probe[0][3], a2 = kK0Probe[1][2], b2 = kK0Probe[1][3];
  const double det = a1 * b2 - a2 * b1;
  const double lam = (k1 * b2 - k2 * b1) / det, mu = (a1 * k2 - a2 * k1) / det;
  static double kd[kKappaClasses];
  static float kf[kKappaClasses];
  for (int c = 0; c < kKappaClasses; ++c) {
    kd[c] = lam * kKappaAlpha[c] + mu * kKappaBeta[c];
    kf[c] = float(kd[c]);
  }
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_kap_d, kd, sizeof(kd), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_kap_f, kf, sizeof(kf), 0, cudaMemcpyHostToDevice, s));
  static double hd[kHadaClasses];
  static float hf[kHadaClasses];
  for (int c = 0; c < kHadaClasses; ++c) {
    hd[c] = (lam * kHadaAlpha[c] + mu * kHadaBeta[c]) * (1.0 / 64.0);
    hf[c] = float(hd[c]);
  }
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_hada_d, hd, sizeof(hd), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_hada_f, hf, sizeof(hf), 0, cudaMemcpyHostToDevice, s));
  upload_hom_tables(hd, s);
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

// ---------------------------------------------------------------- fast even-grid variants (FastAddr: common.cuh)
template <typename TC, typename TA>
__device__ __forceinline__ void load_q_fast(const TC* __restrict__ coeff, const FastAddr& fa, TA q[8]) {
#pragma unroll
  for (int ke = 0; ke < 8; ++ke)
    q[ke] = TA(__ldg(coeff + (fa.E[0][ke & 1] + fa.E[1][(ke >> 1) & 1] + fa.E[2][(ke >> 2) & 1])));
}
// z-slab form: the z-1 element plane of a vertex on the lower face is the
// top element plane of the slab below.
template <typename TC, typename TA>
__device__ __forceinline__ void load_q_fast(const TC* __restrict__ coeff, const ZLink<TC>& cl, const FastAddr& fa,
                                            TA q[8]) {
  const TC* lo = fa.zlo ? cl.lo : coeff;
#pragma unroll
  for (int ke = 0; ke < 8; ++ke)
    q[ke] = TA(__ldg(((ke >> 2) & 1 ? coeff : lo) + (fa.E[0][ke & 1] + fa.E[1][(ke >> 1) & 1] + fa.E[2][(ke >> 2) & 1])));
}

// neighbour n (27-index), component c of nodal array ptr with z link zl
#define FAST_U(ptr, zl)                                                                                   \
  [&, zb0_ = zbase(fa, ptr, zl, 0), zb2_ = zbase(fa, ptr, zl, 2)](int n, int c) {                      \
    const unsigned l_ = fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9];                          \
    return TA(__ldg((n < 9 ? zb0_ : (n < 18 ? ptr : zb2_)) + 3 * (size_t)l_ + c));                       \
  }

// blockDim = (bx, 128/bx), grid = (d0/bx, ceil(d1/by), d2 * ncolors)
template <typename TC, typename TN, typename TA, int MINB = 1, bool ZL = false>
__global__ void __launch_bounds__(128, MINB) l0_apply_fast_kernel(GridGeo g, const TC* __restrict__ coeff,
                                                            ZLink<TC> cl, const TN* __restrict__ u, ZLink<TN> ul,
                                                            const TN* __restrict__ f, TN* __restrict__ y) {
  if constexpr (!ZL) {  // single periodic domain: every wrap reads the array itself
    cl = {coeff, coeff};
    ul = {u, u};
  }
  // colour fastest in blockIdx.z: the 8 colours of one plane run back to back and share L2
  const int color = blockIdx.z & 7;
  const int h2 = blockIdx.z >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= g.cd[0][0] || h1 >= g.cd[0][1]) return;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  TA q[8];
  load_q_fast(coeff, cl, fa, q);
  TA acc[3];
  ku_vertex<TA>(q, kappa<TA>(), FAST_U(u, ul), acc);
  const size_t loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
  if (f) {
#pragma unroll
    for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(TA(f[3 * loc + c]) - acc[c]);
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(acc[c]);
  }
}

// Two same-colour vertices per thread, stacked in halved z (h2, h2+1): the upper
// neighbour plane of the first (t2 = +1) is the lower plane of the second
// (t2 = -1), so those 9 neighbours are loaded once into registers and reused.
// ZC >= 0: zero-start pass of colour ZC (first forward sweep from u = 0): the neighbours of
// colours > ZC are known zeros and are neither loaded nor multiplied (common.cuh zero_start_mask).
// The two z-stacked vertices (h0, h1, h2) and (h0, h1, h2 + 1) of colour `color`: GS updates written to
// uw, returned in out[v]. ov(v, n, c, val) may supply neighbour n of vertex v instead of memory (the
// colour-pair pass hands in the row's fresh colour-c values); ZM: zero-start mask (known-zero colours).
template <unsigned ZM, typename TC, typename TN, typename OV>
__device__ __forceinline__ void gs2_vertices(const GridGeo& g, const TC* __restrict__ coeff, const ZLink<TC>& cl,
                                             const TN* __restrict__ f, const TN* __restrict__ ur,
                                             const ZLink<TN>& ul, TN* uw, int color, int h0, int h1, int h2, OV ov,
                                             TN out[2][3]) {
  using TA = TN;
  FastAddr fa, fb;
  fast_addr(g, color, h0, h1, h2, fa);
  fast_addr(g, color, h0, h1, h2 + 1, fb);
  TA shared_pl[9][3];  // plane t2 = +1 of vertex a == plane t2 = -1 of vertex b
  const TN* pa2 = zbase(fa, ur, ul, 2);  // == zbase(fb, ur, ul, 0) (a's upper plane is b's lower)
#pragma unroll
  for (int n = 0; n < 9; ++n) {
    if constexpr (ZM != 0u) {
      if ((ZM >> (18 + n)) & 1u) continue;  // (t0, t1, +1) of a and (t0, t1, -1) of b: same colour
    }
    const TN* p = pa2 + 3 * (size_t)(fa.A[0][n % 3] + fa.A[1][n / 3] + fa.A[2][2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) shared_pl[n][c] = TA(__ldg(p + c));
  }
  const TN* pa0 = zbase(fa, ur, ul, 0);
  const TN* pb2 = zbase(fb, ur, ul, 2);
  auto Ua = [&](int n, int c) {
    TA val;
    if (ov(0, n, c, val)) return val;
    if (n >= 18) return shared_pl[n - 18][c];
    return TA(__ldg((n < 9 ? pa0 : ur) + 3 * (size_t)(fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9]) + c));
  };
  auto Ub = [&](int n, int c) {
    TA val;
    if (ov(1, n, c, val)) return val;
    if (n < 9) return shared_pl[n][c];
    return TA(__ldg((n < 18 ? ur : pb2) + 3 * (size_t)(fb.A[0][n % 3] + fb.A[1][(n / 3) % 3] + fb.A[2][n / 9]) + c));
  };
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    const FastAddr& fx = v == 0 ? fa : fb;
    TA q[8];
    load_q_fast(coeff, cl, fx, q);
    TA m[3], sblk[9];
    if (v == 0) ku_vertex_split_z<ZM, TA>(q, kappa<TA>(), Ua, m, sblk);
    else ku_vertex_split_z<ZM, TA>(q, kappa<TA>(), Ub, m, sblk);
    const size_t loc = fx.A[0][1] + fx.A[1][1] + fx.A[2][1];
    TN rhs[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) rhs[c] = TN(f[3 * loc + c]) - m[c];
    solve3_spd<TN>(sblk, rhs, out[v]);
#pragma unroll
    for (int c = 0; c < 3; ++c) uw[3 * loc + c] = out[v][c];
  }
}

struct NoOverride {
  template <typename TA>
  __device__ __forceinline__ bool operator()(int, int, int, TA&) const {
    return false;
  }
};

template <typename TC, typename TN, int MINB, bool ZL = false, int ZC = -1>
__global__ void __launch_bounds__(128, MINB) l0_gs_fast2_kernel(GridGeo g, const TC* __restrict__ coeff,
                                                                ZLink<TC> cl, const TN* __restrict__ f,
                                                                const TN* __restrict__ ur, ZLink<TN> ul, TN* uw,
                                                                int color) {
  if constexpr (!ZL) {
    cl = {coeff, coeff};
    ul = {ur, ur};
  }
  constexpr unsigned ZM = ZC >= 0 ? zero_start_mask(ZC) : 0u;
  if constexpr (ZC >= 0) color = ZC;
  const int h2 = 2 * blockIdx.z;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= g.cd[0][0] || h1 >= g.cd[0][1]) return;
  TN out[2][3];
  gs2_vertices<ZM>(g, coeff, cl, f, ur, ul, uw, color, h0, h1, h2, NoOverride{}, out);
}

// Colour passes c and c + 1 (c even) in ONE launch. The only colour-c neighbours of a colour-(c+1)
// vertex are its x - 1 / x + 1 neighbours in the same row (y, z parities equal, x parity flipped), so a
// block owning whole rows (one thread per colour-block column, blockDim.x = cd0) updates colour c,
// publishes the rows' new colour-c values in shared memory and then updates colour c + 1 from them:
// every update sees the values and runs the arithmetic of the two-launch sequence (bitwise the same),
// while the other colours' values are read once for both passes (the second pass hits L1/L2).
constexpr int kPairMaxX = 512;  // colour-block columns per row (n0 <= 1024)
template <typename TC, typename TN, bool ZL = false, int ZC = -1, int MAXT = kPairMaxX, int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB)
    l0_gs_pair_kernel(GridGeo g, const TC* __restrict__ coeff, ZLink<TC> cl, const TN* __restrict__ f, TN* u,
                      ZLink<TN> ul, int color) {
  __shared__ TN rowc[2][MAXT][3];
  if constexpr (!ZL) {
    cl = {coeff, coeff};
    ul = {u, u};
  }
  if constexpr (ZC >= 0) color = ZC;
  constexpr unsigned ZMA = ZC >= 0 ? zero_start_mask(ZC) : 0u;
  constexpr unsigned ZMB = ZC >= 0 ? zero_start_mask(ZC + 1) : 0u;
  const int d0 = g.cd[0][0];
  const int h0 = threadIdx.x, h1 = blockIdx.y, h2 = 2 * blockIdx.z;
  TN out[2][3];
  gs2_vertices<ZMA>(g, coeff, cl, f, u, ul, u, color, h0, h1, h2, NoOverride{}, out);
#pragma unroll
  for (int v = 0; v < 2; ++v)
#pragma unroll
    for (int c = 0; c < 3; ++c) rowc[v][h0][c] = out[v][c];
  __syncthreads();
  const int hn = h0 + 1 == d0 ? 0 : h0 + 1;
  // colour c + 1 at x = 2 h0 + 1: neighbour 12 (x - 1) is colour c at h0, neighbour 14 (x + 1) at h0 + 1
  auto ov = [&](int v, int n, int c, TN& val) {
    if (n == 12) {
      val = rowc[v][h0][c];
      return true;
    }
    if (n == 14) {
      val = rowc[v][hn][c];
      return true;
    }
    return false;
  };
  gs2_vertices<ZMB>(g, coeff, cl, f, u, ul, u, color + 1, h0, h1, h2, ov, out);
}
// Defect-correction residual (kMixedDefect): r = f - K u from f64 data with the
// f64 merge, written ONLY as the f32 right-hand side of the next inner cycle,
// plus deterministic per-block partial sums of |r|^2 (the convergence norm).
// Replaces residual + dot + convert (136 -> 64 B/vertex).
template <typename TC, int MINB = 1, bool ZL = false>
__global__ void __launch_bounds__(128, MINB) l0_residual_norm_fast_kernel(GridGeo g, const TC* __restrict__ coeff,
                                                                    ZLink<TC> cl, const double* __restrict__ u,
                                                                    ZLink<double> ul, const double* __restrict__ f,
                                                                    float* __restrict__ r32, double* partials) {
  if constexpr (!ZL) {
    cl = {coeff, coeff};
    ul = {u, u};
  }
  __shared__ double red[4];
  // colour fastest in blockIdx.z: the 8 colours of one plane run back to back and share L2
  const int color = blockIdx.z & 7;
  const int h2 = blockIdx.z >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  double ss = 0.0;
  if (h0 < g.cd[0][0] && h1 < g.cd[0][1]) {
    using TA = double;
    FastAddr fa;
    fast_addr(g, color, h0, h1, h2, fa);
    TA q[8];
    load_q_fast(coeff, cl, fa, q);
    TA acc[3];
    ku_vertex<TA>(q, kappa<TA>(), FAST_U(u, ul), acc);
    const size_t loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double r = f[3 * loc + c] - acc[c];
      r32[3 * loc + c] = float(r);
      ss += r * r;
    }
  }
  // block reduction in a fixed order (warp shuffles, then 4 warps)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  if ((t & 31) == 0) red[t >> 5] = ss;
  __syncthreads();
  if (t == 0) {
    const size_t bid = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
    partials[bid] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

template <typename TC, typename TN, typename TA, int MINB = 1, bool ZL = false>
__global__ void __launch_bounds__(128, MINB) l0_gs_fast_kernel(GridGeo g, const TC* __restrict__ coeff,
                                                         ZLink<TC> cl, const TN* __restrict__ f,
                                                         const TN* __restrict__ ur, ZLink<TN> ul, TN* uw, int color) {
  if constexpr (!ZL) {
    cl = {coeff, coeff};
    ul = {ur, ur};
  }
  const int h2 = blockIdx.z;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= g.cd[0][0] || h1 >= g.cd[0][1]) return;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  TA q[8];
  load_q_fast(coeff, cl, fa, q);
  TA m[3], sblk[9];
  ku_vertex_split<TA>(q, kappa<TA>(), FAST_U(ur, ul), m, sblk);
  const size_t loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
  // solve in the nodal type: f64 for f64 nodal data (reference), f32 in the f32 inner cycle
  using TS = TN;
  TS S[9], rhs[3], out[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) S[e] = TS(sblk[e]);
#pragma unroll
  for (int c = 0; c < 3; ++c) rhs[c] = TS(f[3 * loc + c]) - TS(m[c]);
  solve3_spd<TS>(S, rhs, out);  // SPD self block: adjugate (src/fem.cpp:131-135 pivots; same solution)
#pragma unroll
  for (int c = 0; c < 3; ++c) uw[3 * loc + c] = TN(out[c]);
}
#undef FAST_U


// ---------------------------------------------------------------- coeff
template <typename TC, bool UNIT>
__global__ void coeff_kernel(const double* __restrict__ rho, TC* __restrict__ coeff, long long m, double p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double x = double(TC(rho[i]));
  coeff[i] = TC(UNIT ? x : pow(x, p));  // src/multigrid.cpp:270; pow(x, 1) == x exactly (IEEE 754)
}

template <typename TC>
void launch_coeff(const double* rho, TC* coeff, long long m, double penal, cudaStream_t s) {
  // the runner's homogenizer penal is 1 (the SIMP power lives in DensityExpr, src/runner.cpp:62)
  if (penal == 1.0) coeff_kernel<TC, true><<<ceil_div(m, 256), 256, 0, s>>>(rho, coeff, m, penal);
  else coeff_kernel<TC, false><<<ceil_div(m, 256), 256, 0, s>>>(rho, coeff, m, penal);
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
  auto U = [&](int n, int c) { return TA(__ldg(u + 3 * (size_t)nb.v[n] + c)); };
  TA acc[3];
  ku_vertex<TA>(q, kappa<TA>(), U, acc);  // factored K0 (ku_gen.cuh), inc/fem.hpp:86-105 semantics
  if (f) {
#pragma unroll
    for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(TA(f[3 * loc + c]) - acc[c]);
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(acc[c]);
  }
}

template <typename TC, typename TN, typename TA>
void launch_l0_apply(const GridGeo& g, const TC* coeff, const TN* u, const TN* f, TN* y, cudaStream_t s,
                     ZLink<TC> cl, ZLink<TN> ul) {
  const bool linked = !is_self(cl, coeff) || !is_self(ul, u);
  if (linked && !fast_ok(g)) throw std::invalid_argument("z-slab level needs an even grid");
  cl = resolve(cl, coeff);
  ul = resolve(ul, u);
  if (sweep_ok(g)) {
    launch_l0_apply_sweep<TC, TN, TA>(g, coeff, cl, u, ul, f, y, s);
  } else if (fast_ok(g)) {
    const dim3 b = fast_block(g);
    const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), 8 * g.cd[0][2]);
    // f32 kernels capped at 64 registers (8 blocks/SM: more warps in flight, measured faster);
    // f64 kernels uncapped (a cap spills and was measured slower).
    if (linked) l0_apply_fast_kernel<TC, TN, TA, sizeof(TA) == 4 ? 8 : 1, true><<<gr, b, 0, s>>>(g, coeff, cl, u, ul, f, y);
    else l0_apply_fast_kernel<TC, TN, TA, sizeof(TA) == 4 ? 8 : 1><<<gr, b, 0, s>>>(g, coeff, cl, u, ul, f, y);
  } else {
    l0_apply_kernel<TC, TN, TA><<<ceil_div(g.nv, 128), 128, 0, s>>>(g, coeff, u, f, y);
  }
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
  auto U = [&](int n, int c) { return TA(__ldg(ur + 3 * (size_t)nb.v[n] + c)); };
  TA m[3], sblk[9];
  ku_vertex_split<TA>(q, kappa<TA>(), U, m, sblk);  // S (n = 13) and M u (n != 13), inc/fem.hpp:109-133
  const long long loc = g.base[color] + i;
  double S[9], rhs[3], out[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) S[e] = double(sblk[e]);
#pragma unroll
  for (int c = 0; c < 3; ++c) rhs[c] = double(f[3 * loc + c]) - double(m[c]);
  solve3(S, rhs, out);  // src/fem.cpp:131-135
#pragma unroll
  for (int c = 0; c < 3; ++c) uw[3 * loc + c] = TN(out[c]);
}


template <typename TC, typename TN, typename TA>
bool l0_gs_zero_start_ok(const GridGeo& g) {
  if constexpr (std::is_same_v<TA, float> && std::is_same_v<TN, float> && std::is_same_v<TC, float>) {
    if (knob("ZERO_START", 1) == 0) return false;
    return fast_ok(g) && g.cd[0][2] % 2 == 0;
  }
  return false;
}

// register budget of the two-vertex GS kernel: 5 blocks/SM (96 regs, default) or 6 / 8 (knob GS2_MINB)
static int gs2_minb() { return knob("GS2_MINB", 5); }

template <typename TC, typename TN, bool ZL, int ZC>
static void launch_fast2_zs(const dim3& gr, const dim3& b, cudaStream_t s, const GridGeo& g, const TC* coeff,
                            ZLink<TC> cl, const TN* f, TN* u, ZLink<TN> ul) {
  const int mb = ZL ? 5 : gs2_minb();
  if (mb >= 8) l0_gs_fast2_kernel<TC, TN, 8, ZL, ZC><<<gr, b, 0, s>>>(g, coeff, cl, f, u, ul, u, ZC);
  else if (mb == 6) l0_gs_fast2_kernel<TC, TN, 6, ZL, ZC><<<gr, b, 0, s>>>(g, coeff, cl, f, u, ul, u, ZC);
  else l0_gs_fast2_kernel<TC, TN, 5, ZL, ZC><<<gr, b, 0, s>>>(g, coeff, cl, f, u, ul, u, ZC);
}
template <typename TC, typename TN, bool ZL>
static void launch_fast2_zs(int color, const dim3& gr, const dim3& b, cudaStream_t s, const GridGeo& g,
                            const TC* coeff, ZLink<TC> cl, const TN* f, TN* u, ZLink<TN> ul) {
  switch (color) {
    case 0: launch_fast2_zs<TC, TN, ZL, 0>(gr, b, s, g, coeff, cl, f, u, ul); break;
    case 1: launch_fast2_zs<TC, TN, ZL, 1>(gr, b, s, g, coeff, cl, f, u, ul); break;
    case 2: launch_fast2_zs<TC, TN, ZL, 2>(gr, b, s, g, coeff, cl, f, u, ul); break;
    case 3: launch_fast2_zs<TC, TN, ZL, 3>(gr, b, s, g, coeff, cl, f, u, ul); break;
    case 4: launch_fast2_zs<TC, TN, ZL, 4>(gr, b, s, g, coeff, cl, f, u, ul); break;
    case 5: launch_fast2_zs<TC, TN, ZL, 5>(gr, b, s, g, coeff, cl, f, u, ul); break;
    case 6: launch_fast2_zs<TC, TN, ZL, 6>(gr, b, s, g, coeff, cl, f, u, ul); break;
    default: launch_fast2_zs<TC, TN, ZL, 7>(gr, b, s, g, coeff, cl, f, u, ul); break;
  }
}

// Off by default: per 512^3 sweep it moves 11 GB instead of 18.8 GB and takes 3.66 instead of 3.95 ms, but
// the fused launch is latency-bound (0.47 of HBM against the single pass's 0.75).
bool l0_gs_pair_ok(const GridGeo& g) {
  return knob("GS_PAIR", 0) != 0 && fast_ok(g) && g.cd[0][2] % 2 == 0 && g.cd[0][0] <= kPairMaxX;
}

template <bool ZL, int ZC>
static void launch_pair_zc(const GridGeo& g, const float* coeff, ZLink<float> cl, const float* f, float* u,
                           ZLink<float> ul, int color, cudaStream_t s) {
  const dim3 gr(1, g.cd[0][1], g.cd[0][2] / 2);
  if (g.cd[0][0] <= 256)  // rows of up to 256 columns (n0 <= 512): two CTAs per SM (3 spill: slower)
    l0_gs_pair_kernel<float, float, ZL, ZC, 256, 2><<<gr, g.cd[0][0], 0, s>>>(g, coeff, cl, f, u, ul, color);
  else
    l0_gs_pair_kernel<float, float, ZL, ZC, kPairMaxX><<<gr, g.cd[0][0], 0, s>>>(g, coeff, cl, f, u, ul, color);
}

void launch_l0_gs_pair(const GridGeo& g, const float* coeff, const float* f, float* u, int color, cudaStream_t s,
                       ZLink<float> cl, ZLink<float> ul, bool zero_start) {
  if (!l0_gs_pair_ok(g) || (color & 1)) throw std::invalid_argument("colour-pair GS pass: unsupported grid or colour");
  const bool linked = !is_self(cl, coeff) || !is_self(ul, u);
  cl = resolve(cl, coeff);
  ul = resolve(ul, u);
  auto go = [&](auto zl) {
    constexpr bool ZL = decltype(zl)::value;
    if (!zero_start) launch_pair_zc<ZL, -1>(g, coeff, cl, f, u, ul, color, s);
    else if (color == 0) launch_pair_zc<ZL, 0>(g, coeff, cl, f, u, ul, color, s);
    else if (color == 2) launch_pair_zc<ZL, 2>(g, coeff, cl, f, u, ul, color, s);
    else if (color == 4) launch_pair_zc<ZL, 4>(g, coeff, cl, f, u, ul, color, s);
    else launch_pair_zc<ZL, 6>(g, coeff, cl, f, u, ul, color, s);
  };
  if (linked) go(std::true_type{});
  else go(std::false_type{});
  IHOM_LAUNCH_CHECK();
}

template <typename TC, typename TN, typename TA>
void launch_l0_gs_color(const GridGeo& g, const TC* coeff, const TN* f, TN* u, int color, cudaStream_t s,
                        ZLink<TC> cl, ZLink<TN> ul, bool zero_start) {
  const bool linked = !is_self(cl, coeff) || !is_self(ul, u);
  if (linked && !fast_ok(g)) throw std::invalid_argument("z-slab level needs an even grid");
  cl = resolve(cl, coeff);
  ul = resolve(ul, u);
  if constexpr (std::is_same_v<TA, float> && std::is_same_v<TN, float>) {
    if (zero_start) {
      if (!l0_gs_zero_start_ok<TC, TN, TA>(g)) throw std::logic_error("zero-start GS pass on an unsupported grid");
      const dim3 b = fast_block(g);
      const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), g.cd[0][2] / 2);
      if (linked) launch_fast2_zs<TC, TN, true>(color, gr, b, s, g, coeff, cl, f, u, ul);
      else launch_fast2_zs<TC, TN, false>(color, gr, b, s, g, coeff, cl, f, u, ul);
      IHOM_LAUNCH_CHECK();
      return;
    }
  }
  if (zero_start) throw std::logic_error("zero-start GS pass exists for the f32 inner level-0 kernel only");
  if (fast_ok(g)) {
    const dim3 b = fast_block(g);
    const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), g.cd[0][2]);
    bool done = false;
    if constexpr (std::is_same_v<TA, float> && std::is_same_v<TN, float>) {
      if (g.cd[0][2] % 2 == 0 && knob("GS2_F32", 1) != 0) {  // two z-stacked vertices per thread
        const dim3 gr2(gr.x, gr.y, g.cd[0][2] / 2);
        if (linked) l0_gs_fast2_kernel<TC, TN, 5, true><<<gr2, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
        else if (gs2_minb() >= 8) l0_gs_fast2_kernel<TC, TN, 8><<<gr2, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
        else if (gs2_minb() == 6) l0_gs_fast2_kernel<TC, TN, 6><<<gr2, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
        else l0_gs_fast2_kernel<TC, TN, 5><<<gr2, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
        done = true;
      }
    }
    if constexpr (std::is_same_v<TA, double> && std::is_same_v<TN, double>) {
      // f64 nodal data (reference-precision V-cycle, all-double mode): the two-vertex pass too
      if (g.cd[0][2] % 2 == 0 && knob("GS2_F64", 1) != 0) {
        const dim3 gr2(gr.x, gr.y, g.cd[0][2] / 2);
        if (linked) l0_gs_fast2_kernel<TC, TN, 2, true><<<gr2, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
        else l0_gs_fast2_kernel<TC, TN, 2><<<gr2, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
        done = true;
      }
    }
    if (!done && linked)
      l0_gs_fast_kernel<TC, TN, TA, sizeof(TA) == 4 ? 8 : 1, true><<<gr, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
    else if (!done)
      l0_gs_fast_kernel<TC, TN, TA, sizeof(TA) == 4 ? 8 : 1><<<gr, b, 0, s>>>(g, coeff, cl, f, u, ul, u, color);
  } else {
    l0_gs_kernel<TC, TN, TA><<<ceil_div(g.size[color], 128), 128, 0, s>>>(g, coeff, f, u, u, color);
  }
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
  for (int c = 0; c < 3; ++c) f[3 * loc + c] = acc[c];
}

template <typename TC>
long long launch_l0_residual_norm(const GridGeo& g, const TC* coeff, const double* u, const double* f, float* r32,
                                  double* partials, cudaStream_t s, ZLink<TC> cl, ZLink<double> ul) {
  if (!fast_ok(g)) throw std::invalid_argument("fused residual needs an even level-0 grid");
  const bool linked = !is_self(cl, coeff) || !is_self(ul, u);
  cl = resolve(cl, coeff);
  ul = resolve(ul, u);
  if constexpr (std::is_same_v<TC, float>) {
    if (sweep_ok(g)) return launch_l0_defect_sweep(g, coeff, cl, u, ul, f, r32, partials, s);
  }
  const dim3 b = fast_block(g);
  const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), 8 * g.cd[0][2]);
  const int minb = knob("RES_MINB", 3);
  if (linked) l0_residual_norm_fast_kernel<TC, 3, true><<<gr, b, 0, s>>>(g, coeff, cl, u, ul, f, r32, partials);
  else if (minb >= 4) l0_residual_norm_fast_kernel<TC, 4><<<gr, b, 0, s>>>(g, coeff, cl, u, ul, f, r32, partials);
  else if (minb == 3) l0_residual_norm_fast_kernel<TC, 3><<<gr, b, 0, s>>>(g, coeff, cl, u, ul, f, r32, partials);
  else l0_residual_norm_fast_kernel<TC, 1><<<gr, b, 0, s>>>(g, coeff, cl, u, ul, f, r32, partials);
  IHOM_LAUNCH_CHECK();
  return (long long)gr.x * gr.y * gr.z;
}

// even-grid form (FastAddr element offsets; z-slab aware)
template <typename TC>
__global__ void __launch_bounds__(128) macro_force_fast_kernel(GridGeo g, const TC* __restrict__ coeff, ZLink<TC> cl,
                                                               int load, double* __restrict__ f) {
  const int color = blockIdx.z & 7;
  const int h2 = blockIdx.z >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= g.cd[0][0] || h1 >= g.cd[0][1]) return;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  double q[8];
  load_q_fast(coeff, cl, fa, q);
  double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int ke = 0; ke < 8; ++ke)  // src/fem.cpp:145-150
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] += q[ke] * c_fmacro[ke][load][c];
  const size_t loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
#pragma unroll
  for (int c = 0; c < 3; ++c) f[3 * loc + c] = acc[c];
}

template <typename TC>
void launch_macro_force(const GridGeo& g, const TC* coeff, int load, double* f, cudaStream_t s, ZLink<TC> cl) {
  if (fast_ok(g)) {
    const dim3 b = fast_block(g);
    const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), 8 * g.cd[0][2]);
    macro_force_fast_kernel<TC><<<gr, b, 0, s>>>(g, coeff, resolve(cl, coeff), load, f);
  } else {
    if (!is_self(cl, coeff)) throw std::invalid_argument("z-slab level needs an even grid");
    macro_force_kernel<TC><<<ceil_div(g.nv, 256), 256, 0, s>>>(g, coeff, load, f);
  }
  IHOM_LAUNCH_CHECK();
}

// Macro force with the component sums of f folded into the same pass: the macro-force grid of the
// even-grid kernel (one vertex per thread), each block folds its 3 component sums (fixed shuffle and
// warp order) into partials[3 b + c]; the nb block partials are then summed by the deterministic
// component-sum reduction. The partition is fixed by the grid, so the sums are reproducible run to
// run; they round differently from launch_comp_sums(f) (another partition), which project_norm0 used
// before.
template <typename TC>
__global__ void __launch_bounds__(128) macro_force_sums_kernel(GridGeo g, const TC* __restrict__ coeff, ZLink<TC> cl,
                                                               int load, double* __restrict__ f,
                                                               double* __restrict__ partials) {
  __shared__ double sh[3][4];
  const int color = blockIdx.z & 7;
  const int h2 = blockIdx.z >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  double acc[3] = {0.0, 0.0, 0.0};
  if (h0 < g.cd[0][0] && h1 < g.cd[0][1]) {
    FastAddr fa;
    fast_addr(g, color, h0, h1, h2, fa);
    double q[8];
    load_q_fast(coeff, cl, fa, q);
#pragma unroll
    for (int ke = 0; ke < 8; ++ke)  // src/fem.cpp:145-150
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] += q[ke] * c_fmacro[ke][load][c];
    const size_t loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
#pragma unroll
    for (int c = 0; c < 3; ++c) f[3 * loc + c] = acc[c];
  }
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) sh[c][t >> 5] = v;
  }
  __syncthreads();
  if (t < 3) {
    const size_t blk = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
    partials[3 * blk + t] = (sh[t][0] + sh[t][1]) + (sh[t][2] + sh[t][3]);
  }
}

long long macro_force_sums_blocks(const GridGeo& g) {
  const dim3 b = fast_block(g);
  return (long long)ceil_div(g.cd[0][0], b.x) * ceil_div(g.cd[0][1], b.y) * 8 * g.cd[0][2];
}

template <typename TC>
void launch_macro_force_sums(const GridGeo& g, const TC* coeff, int load, double* f, double* block_sums,
                             double* partials, double* sums, cudaStream_t s, ZLink<TC> cl, unsigned* ticket) {
  if (!fast_ok(g)) throw std::invalid_argument("fused macro force sums need an even grid");
  const dim3 b = fast_block(g);
  if (b.x * b.y != 128) throw std::logic_error("macro force sums: 128-thread blocks expected");
  const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), 8 * g.cd[0][2]);
  macro_force_sums_kernel<TC><<<gr, b, 0, s>>>(g, coeff, resolve(cl, coeff), load, f, block_sums);
  IHOM_LAUNCH_CHECK();
  launch_comp_sums<double>(block_sums, macro_force_sums_blocks(g), partials, sums, s, ticket);
}

// ---------------------------------------------------------------- instantiations
template void launch_coeff<float>(const double*, float*, long long, double, cudaStream_t);
template void launch_coeff<double>(const double*, double*, long long, double, cudaStream_t);
template void launch_macro_force<float>(const GridGeo&, const float*, int, double*, cudaStream_t, ZLink<float>);
template void launch_macro_force<double>(const GridGeo&, const double*, int, double*, cudaStream_t, ZLink<double>);
template void launch_macro_force_sums<float>(const GridGeo&, const float*, int, double*, double*, double*, double*,
                                             cudaStream_t, ZLink<float>, unsigned*);
template void launch_macro_force_sums<double>(const GridGeo&, const double*, int, double*, double*, double*, double*,
                                              cudaStream_t, ZLink<double>, unsigned*);
template long long launch_l0_residual_norm<float>(const GridGeo&, const float*, const double*, const double*, float*,
                                                  double*, cudaStream_t, ZLink<float>, ZLink<double>);

#define INST_L0(TC, TN, TA)                                                                                    \
  template void launch_l0_apply<TC, TN, TA>(const GridGeo&, const TC*, const TN*, const TN*, TN*, cudaStream_t, \
                                            ZLink<TC>, ZLink<TN>);                                            \
  template void launch_l0_gs_color<TC, TN, TA>(const GridGeo&, const TC*, const TN*, TN*, int, cudaStream_t,      \
                                               ZLink<TC>, ZLink<TN>, bool);                                   \
  template bool l0_gs_zero_start_ok<TC, TN, TA>(const GridGeo&);
INST_L0(float, double, double)   // mixed, f64 nodal (parity)
INST_L0(double, double, double)  // all-double
INST_L0(float, float, float)     // mixed inner correction cycle
#undef INST_L0

}  // namespace ihomgpu

#include "sweep_kernels.cuh"  // z-plane sweep variants (same TU: shares the kappa constants)
