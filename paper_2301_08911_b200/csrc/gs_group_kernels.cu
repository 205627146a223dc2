// gs_group_kernels.cu -- level-0 f32 Gauss-Seidel colour pass for a lockstep GROUP of right-hand sides.
//
// The six cell problems share the element coefficients, so everything a GS vertex update derives from
// them -- the 8 incident coefficients, the 52 "Hadamard" forms of the factored stencil (ku_gen.cuh),
// each merged 3x3 coefficient kappa * F and the self block S -- is computed once per vertex and
// applied to NR right-hand sides (ku_vertex_split_g): per RHS only the 26 neighbour loads, the 234
// FMAs and the 3x3 solve remain. The single-RHS pass (l0_gs_fast2_kernel, fem_kernels.cu) spends
// ~730 instructions per vertex, about a third of them on that shared work.
//
// Same operator and colour order as the single-RHS pass; kappa multiplies each coefficient instead
// of the ten per-class partial sums, so rounding differs (tolerance-level variant, knob L0_GROUP,
// tests/test_kernel_variants.py). Lanes beyond the active RHS count repeat lane 0 (same inputs, same
// values written: harmless).
//
// Measured (512^3 bench, groups of six): 2.34 ms per grouped colour pass for ~5 active RHSs, i.e.
// 0.47 ms per RHS -- the same as the single-RHS pass (0.46): the pass is bound by the latency of the
// per-RHS neighbour loads (one vertex per thread, 26 x NR independent load streams), not by the
// coefficient-side instructions it removes. Iteration 0.523 -> 0.518 s, but at a lower per-byte
// efficiency; off by default (L0_GROUP=1 enables it).
#include <type_traits>

#include "kernels.hpp"
#include "ku_gen.cuh"

namespace ihomgpu {

__constant__ float c_kap_g[kKappaClasses];

void upload_gs_group_tables(const float kf[], cudaStream_t s) {
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_kap_g, kf, sizeof(float) * kKappaClasses, 0, cudaMemcpyHostToDevice, s));
}

template <int NR>
struct LanesN {  // one float per RHS of the group
  float v[NR];
  __device__ LanesN() {}
  __device__ explicit LanesN(float x) {
#pragma unroll
    for (int k = 0; k < NR; ++k) v[k] = x;
  }
};
template <int NR>
__device__ __forceinline__ LanesN<NR> vfma(float c, const LanesN<NR>& u, const LanesN<NR>& a) {
  LanesN<NR> r;
#pragma unroll
  for (int k = 0; k < NR; ++k) r.v[k] = fmaf(c, u.v[k], a.v[k]);
  return r;
}

struct GsGroupIO {
  float* u[kMaxRhsGroup];
  ZLink<float> ul[kMaxRhsGroup];
  const float* f[kMaxRhsGroup];
};

// one vertex of colour `color` per thread; grid = (cd0 / 32, cd1 / 4, cd2), block = (32, 4)
template <int NR, bool ZL, int ZC>
__global__ void __launch_bounds__(128) l0_gs_group_kernel(GridGeo g, const float* __restrict__ coeff, ZLink<float> cl,
                                                          GsGroupIO io, int color) {
  if constexpr (!ZL) cl = {coeff, coeff};
  constexpr unsigned ZM = ZC >= 0 ? zero_start_mask(ZC) : 0u;
  if constexpr (ZC >= 0) color = ZC;
  const int h2 = blockIdx.z;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= g.cd[0][0] || h1 >= g.cd[0][1]) return;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  float q[8];
#pragma unroll
  for (int ke = 0; ke < 8; ++ke) {
    const float* src = (ke >> 2) & 1 ? coeff : (fa.zlo ? cl.lo : coeff);
    q[ke] = __ldg(src + (fa.E[0][ke & 1] + fa.E[1][(ke >> 1) & 1] + fa.E[2][(ke >> 2) & 1]));
  }
  const float* lo[NR];
  const float* hi[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const ZLink<float> ul = ZL ? io.ul[k] : ZLink<float>{io.u[k], io.u[k]};
    lo[k] = zbase(fa, io.u[k], ul, 0);
    hi[k] = zbase(fa, io.u[k], ul, 2);
  }
  auto U = [&](int n, int c) -> LanesN<NR> {
    const unsigned l = fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9];
    LanesN<NR> r;
#pragma unroll
    for (int k = 0; k < NR; ++k) r.v[k] = __ldg((n < 9 ? lo[k] : (n < 18 ? io.u[k] : hi[k])) + 3 * (size_t)l + c);
    return r;
  };
  LanesN<NR> m[3];
  float S[9];
  ku_vertex_split_g<ZM, float, LanesN<NR>>(q, c_kap_g, U, m, S);
  const size_t loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    float rhs[3], out[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) rhs[c] = io.f[k][3 * loc + c] - m[c].v[k];
    solve3<float>(S, rhs, out);
#pragma unroll
    for (int c = 0; c < 3; ++c) io.u[k][3 * loc + c] = out[c];
  }
}

bool l0_gs_group_ok(const GridGeo& g) {
  return knob("L0_GROUP", 0) != 0 && fast_ok(g) && g.cd[0][0] % 32 == 0 && g.cd[0][1] % 4 == 0;
}

template <int NR, bool ZL>
static void launch_nr(const GridGeo& g, const float* coeff, ZLink<float> cl, const GsGroupIO& io, int color,
                      bool zero_start, cudaStream_t s) {
  const dim3 b(32, 4), gr(g.cd[0][0] / 32, g.cd[0][1] / 4, g.cd[0][2]);
  if (!zero_start) {
    l0_gs_group_kernel<NR, ZL, -1><<<gr, b, 0, s>>>(g, coeff, cl, io, color);
    return;
  }
  switch (color) {
    case 0: l0_gs_group_kernel<NR, ZL, 0><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
    case 1: l0_gs_group_kernel<NR, ZL, 1><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
    case 2: l0_gs_group_kernel<NR, ZL, 2><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
    case 3: l0_gs_group_kernel<NR, ZL, 3><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
    case 4: l0_gs_group_kernel<NR, ZL, 4><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
    case 5: l0_gs_group_kernel<NR, ZL, 5><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
    case 6: l0_gs_group_kernel<NR, ZL, 6><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
    default: l0_gs_group_kernel<NR, ZL, 7><<<gr, b, 0, s>>>(g, coeff, cl, io, color); break;
  }
}

void launch_l0_gs_group(const GridGeo& g, const float* coeff, ZLink<float> cl, int nr, const float* const* f,
                        float* const* u, const ZLink<float>* ul, int color, bool zero_start, cudaStream_t s) {
  if (nr < 1 || nr > kMaxRhsGroup) throw std::invalid_argument("right-hand-side group size must be in [1, 6]");
  const int NR = nr <= 2 ? 2 : (nr <= 3 ? 3 : 6);
  GsGroupIO io{};
  bool linked = !is_self(cl, coeff);
  for (int k = 0; k < NR; ++k) {
    const int j = k < nr ? k : 0;  // padding lanes repeat lane 0
    io.u[k] = u[j];
    io.f[k] = f[j];
    io.ul[k] = resolve(ul[j], u[j]);
    linked = linked || !is_self(ul[j], u[j]);
  }
  cl = resolve(cl, coeff);
  if (NR == 2) linked ? launch_nr<2, true>(g, coeff, cl, io, color, zero_start, s)
                      : launch_nr<2, false>(g, coeff, cl, io, color, zero_start, s);
  else if (NR == 3) linked ? launch_nr<3, true>(g, coeff, cl, io, color, zero_start, s)
                           : launch_nr<3, false>(g, coeff, cl, io, color, zero_start, s);
  else linked ? launch_nr<6, true>(g, coeff, cl, io, color, zero_start, s)
              : launch_nr<6, false>(g, coeff, cl, io, color, zero_start, s);
  IHOM_LAUNCH_CHECK();
}

}  // namespace ihomgpu
