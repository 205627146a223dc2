// mg_kernels.cu -- multigrid transfer, coarse stencil kernels, Galerkin
// assembly and the coarsest dense solve (src/multigrid.cpp:12-79, 102-239,
// 281-333, 426-451).
#include "kernels.hpp"
#include "gal_gen.cuh"

#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include <mutex>

namespace ihomgpu {

// ---------------------------------------------------------------- transfer
// transfer_weight_1d, src/multigrid.cpp:12-15
__host__ __device__ constexpr double tw1(int c) { return (c < 0 ? -c : c) >= 2 ? 0.0 : (2.0 - (c < 0 ? -c : c)) / 2.0; }

__device__ __forceinline__ int wrapi(int c, int n) {
  c %= n;
  return c < 0 ? c + n : c;
}

// f_c = I^T r_f over the 27 fine vertices around 2*vc (src/multigrid.cpp:19-41).
static bool transfer_f32() { return knob("TRANSFER_F32", 1) != 0; }

template <typename TN>
__global__ void restrict_kernel(GridGeo gf, GridGeo gc, const TN* __restrict__ rf, TN* __restrict__ fc) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= gc.nv) return;
  const int color = color_at(gc, loc);
  int x, y, z;
  block_coords(gc, color, (unsigned)(loc - gc.base[color]), x, y, z);
  double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const double w = tw1(dx) * tw1(dy) * tw1(dz);
        const unsigned fl = vloc(gf, wrapi(2 * x + dx, gf.n[0]), wrapi(2 * y + dy, gf.n[1]), wrapi(2 * z + dz, gf.n[2]));
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += w * double(rf[3 * (size_t)fl + c]);
      }
#pragma unroll
  for (int c = 0; c < 3; ++c) fc[3 * loc + c] = TN(acc[c]);
}

// Fast even-grid transfers. Restriction: coarse vertex vc is the fine colour-0
// vertex with halved coordinates vc, so its 27 fine neighbours are FastAddr of
// (fine grid, colour 0, h = vc). Prolongation: per axis 1 (even) or 2 (odd)
// coarse parents; colour-specialised so the loop bounds are compile-time.
// z-slab forms: rf's lower face links to the slab below (rl); the coarse
// output is either this slab's coarse level (gout == gc, zoff 0) or the
// replicated global coarse level (gout global, zoff = this slab's first coarse
// plane in halved coordinates) -- only the slab's own planes are written.
// TA: arithmetic type; float (knob TRANSFER_F32, f32 fields only) keeps the inner cycle's transfers in
// f32 (the weights are powers of two: exact products) instead of converting every value to f64.
// Up to kMaxRhsGroup (source, link, destination) triples of one transfer, one per RHS lane of a lockstep
// group: blockIdx.z = lane * nz + (colour + 8 h2), same per-lane arithmetic as one launch per lane.
template <typename TN>
struct XferN {
  const TN* src[kMaxRhsGroup];
  ZLink<TN> sl[kMaxRhsGroup];
  TN* dst[kMaxRhsGroup];
};

// coarse vertex (colour, h0, h1, h2) of the restriction of one lane (shared by the grouped kernel and the
// bottom-cycle kernel: the same arithmetic whatever thread computes it)
template <typename TN, typename TA>
__device__ __forceinline__ void restrict_vertex(const GridGeo& gf, const TN* __restrict__ rf, const ZLink<TN>& rl,
                                                TN* __restrict__ fc, int color, int h0, int h1, int h2,
                                                const GridGeo& gout, int zoff) {
  const int cx = 2 * h0 + (color & 1), cy = 2 * h1 + ((color >> 1) & 1), cz = 2 * h2 + ((color >> 2) & 1);
  FastAddr fa;
  fast_addr(gf, 0, cx, cy, cz, fa);
  const TN* rb = zbase(fa, rf, rl, 0);  // fine colour 0: only the z-1 plane can wrap
  TA acc[3] = {TA(0), TA(0), TA(0)};
#pragma unroll
  for (int n = 0; n < 27; ++n) {
    const int dx = n % 3 - 1, dy = (n / 3) % 3 - 1, dz = n / 9 - 1;
    const TA w = TA(tw1(dx) * tw1(dy) * tw1(dz));
    const TN* r = (n < 9 ? rb : rf) + 3 * (size_t)(fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9]);
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] += w * TA(__ldg(r + c));
  }
  const size_t loc =
      (size_t)color * gout.size[0] + h0 + (size_t)gout.cd[0][0] * (h1 + (size_t)gout.cd[0][1] * (h2 + zoff));
#pragma unroll
  for (int c = 0; c < 3; ++c) fc[3 * loc + c] = TN(acc[c]);
}

template <typename TN, typename TA = double>
__global__ void __launch_bounds__(128) restrict_fast_kernel(GridGeo gf, GridGeo gc, XferN<TN> io, int nz, GridGeo gout,
                                                            int zoff) {
  const int lane = blockIdx.z / nz, zz = blockIdx.z % nz;
  const int color = zz & 7;  // colour fastest (L2 reuse across colours of a plane)
  const int h2 = zz >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= gc.cd[0][0] || h1 >= gc.cd[0][1]) return;
  restrict_vertex<TN, TA>(gf, io.src[lane], io.sl[lane], io.dst[lane], color, h0, h1, h2, gout, zoff);
}

// Coarse parents of a fine vertex at halved (h0, h1, h2): coarse coordinates
// h_k and h_k + 1 (wrapped). z-slab: the coarse level is this slab's (zoff 0;
// the wrapped z parent is the first plane of the slab above, cl.hi) or the
// replicated global level (zoff = the slab's first coarse plane).
template <typename TN, int O0, int O1, int O2, typename TA = double>
__device__ __forceinline__ void prolong_vertex(const GridGeo& gc, int h0, int h1, int h2, const TN* __restrict__ uc,
                                               const ZLink<TN>& cl, int zoff, TA acc[3]) {
  const int o[3] = {O0, O1, O2};
  const int h[3] = {h0, h1, h2 + zoff};
  const unsigned Bc = (unsigned)gc.size[0];
  const unsigned sc[3] = {1u, (unsigned)gc.cd[0][0], (unsigned)gc.cd[0][0] * (unsigned)gc.cd[0][1]};
  unsigned P[3][2];
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // coarse coordinate c -> ((c & 1) << k) Bc + sc_k (c >> 1)
    const int c0 = h[k];
    const int c1 = (h[k] + 1 == gc.n[k]) ? 0 : h[k] + 1;
    P[k][0] = (((unsigned)c0 & 1u) << k) * Bc + sc[k] * (unsigned)(c0 >> 1);
    P[k][1] = (((unsigned)c1 & 1u) << k) * Bc + sc[k] * (unsigned)(c1 >> 1);
  }
  const TA w = TA((O0 ? 0.5 : 1.0) * (O1 ? 0.5 : 1.0) * (O2 ? 0.5 : 1.0));
  const TN* ub[2] = {uc, h[2] + 1 == gc.n[2] ? cl.hi : uc};
#pragma unroll
  for (int a = 0; a < 1 + O0; ++a)
#pragma unroll
    for (int b = 0; b < 1 + O1; ++b)
#pragma unroll
      for (int c = 0; c < 1 + O2; ++c) {
        const TN* u = ub[c] + 3 * (size_t)(P[0][a] + P[1][b] + P[2][c]);
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[d] += w * TA(__ldg(u + d));
      }
  (void)o;
}

// fine vertex (colour, h0, h1, h2) of the prolongation-add of one lane
template <typename TN, typename TA>
__device__ __forceinline__ void prolong_add_vertex(const GridGeo& gc, const GridGeo& gf, const TN* __restrict__ uc,
                                                   const ZLink<TN>& cl, TN* __restrict__ uf, int color, int h0,
                                                   int h1, int h2, int zoff) {
  TA acc[3] = {TA(0), TA(0), TA(0)};
  switch (color) {  // uniform per block
    case 0: prolong_vertex<TN, 0, 0, 0, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
    case 1: prolong_vertex<TN, 1, 0, 0, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
    case 2: prolong_vertex<TN, 0, 1, 0, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
    case 3: prolong_vertex<TN, 1, 1, 0, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
    case 4: prolong_vertex<TN, 0, 0, 1, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
    case 5: prolong_vertex<TN, 1, 0, 1, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
    case 6: prolong_vertex<TN, 0, 1, 1, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
    default: prolong_vertex<TN, 1, 1, 1, TA>(gc, h0, h1, h2, uc, cl, zoff, acc); break;
  }
  const size_t loc = (size_t)color * gf.size[0] + h0 + (size_t)gf.cd[0][0] * (h1 + (size_t)gf.cd[0][1] * h2);
#pragma unroll
  for (int d = 0; d < 3; ++d) uf[3 * loc + d] = TN(TA(uf[3 * loc + d]) + acc[d]);
}

template <typename TN, typename TA = double>
__global__ void __launch_bounds__(128) prolong_fast_kernel(GridGeo gc, GridGeo gf, XferN<TN> io, int nz, int zoff) {
  const int lane = blockIdx.z / nz, zz = blockIdx.z % nz;
  const int color = zz & 7;  // colour fastest (L2 reuse across colours of a plane)
  const int h2 = zz >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= gf.cd[0][0] || h1 >= gf.cd[0][1]) return;
  prolong_add_vertex<TN, TA>(gc, gf, io.src[lane], io.sl[lane], io.dst[lane], color, h0, h1, h2, zoff);
}

template <typename TN>
void launch_restrict(const GridGeo& gf, const GridGeo& gc, const TN* rf, TN* fc, cudaStream_t s, ZLink<TN> rl,
                     const GridGeo* gout, int zoff) {
  const bool slab = !is_self(rl, rf) || gout;
  if (fast_ok(gf) && gc.n[0] % 2 == 0 && gc.n[1] % 2 == 0 && gc.n[2] % 2 == 0) {
    const dim3 b = fast_block(gc);
    const dim3 gr(ceil_div(gc.cd[0][0], b.x), ceil_div(gc.cd[0][1], b.y), 8 * gc.cd[0][2]);
    XferN<TN> io{};
    io.src[0] = rf;
    io.sl[0] = resolve(rl, rf);
    io.dst[0] = fc;
    if (std::is_same_v<TN, float> && transfer_f32())
      restrict_fast_kernel<TN, float><<<gr, b, 0, s>>>(gf, gc, io, int(gr.z), gout ? *gout : gc, gout ? zoff : 0);
    else
      restrict_fast_kernel<TN><<<gr, b, 0, s>>>(gf, gc, io, int(gr.z), gout ? *gout : gc, gout ? zoff : 0);
    IHOM_LAUNCH_CHECK();
    return;
  }
  if (slab) throw std::invalid_argument("z-slab restriction needs even fine and coarse grids");
  restrict_kernel<TN><<<ceil_div(gc.nv, 128), 128, 0, s>>>(gf, gc, rf, fc);
  IHOM_LAUNCH_CHECK();
}

// u_f += I u_c (src/multigrid.cpp:43-79).
template <typename TN>
__global__ void prolong_kernel(GridGeo gc, GridGeo gf, const TN* __restrict__ uc, TN* __restrict__ uf) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= gf.nv) return;
  const int color = color_at(gf, loc);
  int v[3];
  block_coords(gf, color, (unsigned)(loc - gf.base[color]), v[0], v[1], v[2]);
  int base[3], cnt[3];
  double w1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if ((v[k] & 1) == 0) {
      base[k] = v[k] / 2;
      cnt[k] = 1;
      w1[k] = 1.0;
    } else {
      base[k] = (v[k] - 1) / 2;
      cnt[k] = 2;
      w1[k] = 0.5;
    }
  }
  const double w = w1[0] * w1[1] * w1[2];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < cnt[0]; ++a)
    for (int b = 0; b < cnt[1]; ++b)
      for (int c = 0; c < cnt[2]; ++c) {
        const unsigned cl = vloc(gc, wrapi(base[0] + a, gc.n[0]), wrapi(base[1] + b, gc.n[1]), wrapi(base[2] + c, gc.n[2]));
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[d] += w * double(uc[3 * (size_t)cl + d]);
      }
#pragma unroll
  for (int d = 0; d < 3; ++d) uf[3 * loc + d] = TN(double(uf[3 * loc + d]) + acc[d]);
}

template <typename TN>
void launch_prolong_add(const GridGeo& gc, const GridGeo& gf, const TN* uc, TN* uf, cudaStream_t s, ZLink<TN> cl,
                        int zoff) {
  const bool slab = !is_self(cl, uc) || zoff != 0;
  if (fast_ok(gf) && gc.n[0] % 2 == 0 && gc.n[1] % 2 == 0 && gc.n[2] % 2 == 0) {
    const dim3 b = fast_block(gf);
    const dim3 gr(ceil_div(gf.cd[0][0], b.x), ceil_div(gf.cd[0][1], b.y), 8 * gf.cd[0][2]);
    XferN<TN> io{};
    io.src[0] = uc;
    io.sl[0] = resolve(cl, uc);
    io.dst[0] = uf;
    if (std::is_same_v<TN, float> && transfer_f32())
      prolong_fast_kernel<TN, float><<<gr, b, 0, s>>>(gc, gf, io, int(gr.z), zoff);
    else
      prolong_fast_kernel<TN><<<gr, b, 0, s>>>(gc, gf, io, int(gr.z), zoff);
    IHOM_LAUNCH_CHECK();
    return;
  }
  if (slab) throw std::invalid_argument("z-slab prolongation needs even fine and coarse grids");
  prolong_kernel<TN><<<ceil_div(gf.nv, 128), 128, 0, s>>>(gc, gf, uc, uf);
  IHOM_LAUNCH_CHECK();
}

bool transfer_group_ok(const GridGeo& gf, const GridGeo& gc) {
  return fast_ok(gf) && gc.n[0] % 2 == 0 && gc.n[1] % 2 == 0 && gc.n[2] % 2 == 0 && transfer_f32();
}

void launch_restrict_group(const GridGeo& gf, const GridGeo& gc, int nl, const float* const* rf,
                           const ZLink<float>* rl, float* const* fc, cudaStream_t s) {
  if (nl < 1 || nl > kMaxRhsGroup || !transfer_group_ok(gf, gc)) throw std::invalid_argument("grouped restriction");
  XferN<float> io{};
  for (int k = 0; k < nl; ++k) io.src[k] = rf[k], io.sl[k] = resolve(rl[k], rf[k]), io.dst[k] = fc[k];
  const dim3 b = fast_block(gc);
  const unsigned nz = 8 * gc.cd[0][2];
  restrict_fast_kernel<float, float><<<dim3(ceil_div(gc.cd[0][0], b.x), ceil_div(gc.cd[0][1], b.y), nz * nl), b, 0,
                                       s>>>(gf, gc, io, int(nz), gc, 0);
  IHOM_LAUNCH_CHECK();
}

void launch_prolong_add_group(const GridGeo& gc, const GridGeo& gf, int nl, const float* const* uc,
                              const ZLink<float>* cl, float* const* uf, cudaStream_t s) {
  if (nl < 1 || nl > kMaxRhsGroup || !transfer_group_ok(gf, gc)) throw std::invalid_argument("grouped prolongation");
  XferN<float> io{};
  for (int k = 0; k < nl; ++k) io.src[k] = uc[k], io.sl[k] = resolve(cl[k], uc[k]), io.dst[k] = uf[k];
  const dim3 b = fast_block(gf);
  const unsigned nz = 8 * gf.cd[0][2];
  prolong_fast_kernel<float, float><<<dim3(ceil_div(gf.cd[0][0], b.x), ceil_div(gf.cd[0][1], b.y), nz * nl), b, 0,
                                      s>>>(gc, gf, io, int(nz), 0);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- stencil apply / GS
// NL = 1, 2, 3 or 6 right-hand sides per launch: the stencil block of a neighbour is read and
// converted once and applied to every RHS, so a group of cell problems solved in lockstep streams the
// coarse stencils (the dominant bytes of levels >= 1) once for all of them. Per RHS the arithmetic is
// the same explicit fma chain for every NL, so a grouped solve is bit-identical to single ones.
template <typename TN>
struct RhsN {      // right-hand side k of a level: input field x (u of a GS pass), f, output y
  const TN* x[kMaxRhsGroup];
  ZLink<TN> xl[kMaxRhsGroup];
  const TN* f[kMaxRhsGroup];
  TN* y[kMaxRhsGroup];
};

template <typename TS>
__device__ __forceinline__ void stencil_block(const TS* __restrict__ bl, double c9[9]) {
#pragma unroll
  for (int e = 0; e < 9; ++e) c9[e] = double(__ldg(bl + 32 * e));
}
template <typename TS>
__device__ __forceinline__ void stencil_block(const TS* __restrict__ bl, float c9[9]) {
#pragma unroll
  for (int e = 0; e < 9; ++e) c9[e] = float(__ldg(bl + 32 * e));
}
__device__ __forceinline__ void block_fma(const float c9[9], float a, float b, float c, float m[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r) m[r] = fmaf(c9[3 * r + 2], c, fmaf(c9[3 * r + 1], b, fmaf(c9[3 * r], a, m[r])));
}
__device__ __forceinline__ void block_fma(const double c9[9], double a, double b, double c, double m[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r) m[r] = fma(c9[3 * r + 2], c, fma(c9[3 * r + 1], b, fma(c9[3 * r], a, m[r])));
}

// y = K x (f == nullptr) or y = f - K x; blocked stencil rows st_index(k, loc) (src/multigrid.cpp:186-205, 412-424).
template <typename TS, typename TN, int NL>
__global__ void __launch_bounds__(128) stencil_apply_kernel(GridGeo g, const TS* __restrict__ st, RhsN<TN> io) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= g.nv) return;
  const int color = color_at(g, loc);
  int vx, vy, vz;
  block_coords(g, color, (unsigned)(loc - g.base[color]), vx, vy, vz);
  Nbhd nb;
  gather27(g, vx, vy, vz, nb);
  double acc[NL][3] = {};
  const TS* row = st + st_index(0, (unsigned)loc);
#pragma unroll 3
  for (int n = 0; n < 27; ++n) {
    double c9[9];
    stencil_block(row + 32 * 9 * n, c9);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const TN* xn = io.x[k] + 3 * (size_t)nb.v[n];
      block_fma(c9, double(xn[0]), double(xn[1]), double(xn[2]), acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < NL; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      io.y[k][3 * loc + c] = io.f[k] ? TN(double(io.f[k][3 * loc + c]) - acc[k][c]) : TN(acc[k][c]);
}

// Fast even-grid variants (FastAddr, common.cuh): one IADD3 per neighbour
// location, AoS components at immediate offsets, blocked stencil rows.
// TACC = float (knob STENCIL_F32, f32 stencils and nodal data only): stencil values and products in
// f32 instead of converted to f64 -- fewer registers (more warps in flight for these latency-bound
// passes) and no F2F, at the f32 rounding level of the inner correction cycle.
template <typename TS, typename TN, bool ZL, int NL, typename TACC = double>
__global__ void __launch_bounds__(128) stencil_apply_fast_kernel(GridGeo g, const TS* __restrict__ st, RhsN<TN> io) {
  // colour fastest in blockIdx.z: the 8 colours of one plane run back to back and share L2
  const int color = blockIdx.z & 7;
  const int h2 = blockIdx.z >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= g.cd[0][0] || h1 >= g.cd[0][1]) return;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  const unsigned loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
  const TS* row = st + st_index(0, loc);
  TACC acc[NL][3] = {};
  const TN* xb[NL][3];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const ZLink<TN> xl = ZL ? io.xl[k] : ZLink<TN>{io.x[k], io.x[k]};
    xb[k][0] = zbase(fa, io.x[k], xl, 0);
    xb[k][1] = io.x[k];
    xb[k][2] = zbase(fa, io.x[k], xl, 2);
  }
#pragma unroll
  for (int n = 0; n < 27; ++n) {
    TACC c9[9];
    stencil_block(row + 32 * 9 * n, c9);
    const size_t off = 3 * (size_t)(fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9]);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const TN* xn = xb[k][n / 9] + off;
      block_fma(c9, TACC(__ldg(xn)), TACC(__ldg(xn + 1)), TACC(__ldg(xn + 2)), acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < NL; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      io.y[k][3 * (size_t)loc + c] = io.f[k] ? TN(TACC(io.f[k][3 * (size_t)loc + c]) - acc[k][c]) : TN(acc[k][c]);
}

// Streamed variant (knob STENCIL_STREAM, f32 stencils / nodal data / products): a warp's 32
// consecutive vertices own one contiguous 31 KB block of the blocked stencil layout, which the warp
// copies into a 3-stage shared-memory ring (three neighbours' 27 rows per stage, 16-byte cp.async,
// two stages in flight) while it computes; only the gathered neighbour values are loaded directly.
// Same per-vertex arithmetic and order as stencil_apply_fast_kernel<..., float>: bit-identical.
constexpr int kStRows = 27;                   // stencil rows per stage (three neighbours)
constexpr int kStStage = kStRows * 32;        // floats per stage
template <bool ZL, int NL>
__global__ void __launch_bounds__(128) stencil_apply_stream_kernel(GridGeo g, const float* __restrict__ st,
                                                                   RhsN<float> io) {
  __shared__ __align__(16) float ring[4][3][kStStage];
  const int color = blockIdx.z & 7;
  const int h2 = blockIdx.z >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h1 >= g.cd[0][1]) return;  // whole warps (cd0 % 32 == 0)
  const int lane = threadIdx.x & 31, w = threadIdx.y;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  const unsigned loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
  const float* chunk = st + st_index(0, loc & ~31u);  // the warp's 243 x 32 block
  float(*rg)[kStStage] = ring[w];
  auto issue = [&](int stage, int slot) {
    const float4* src = reinterpret_cast<const float4*>(chunk + (size_t)stage * kStStage);
    float4* dst = reinterpret_cast<float4*>(rg[slot]);
    for (int i = lane; i < kStStage / 4; i += 32) __pipeline_memcpy_async(dst + i, src + i, 16);
  };
  float acc[NL][3] = {};
  const float* xb[NL][3];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const ZLink<float> xl = ZL ? io.xl[k] : ZLink<float>{io.x[k], io.x[k]};
    xb[k][0] = zbase(fa, io.x[k], xl, 0);
    xb[k][1] = io.x[k];
    xb[k][2] = zbase(fa, io.x[k], xl, 2);
  }
  issue(0, 0);
  __pipeline_commit();
  issue(1, 1);
  __pipeline_commit();
#pragma unroll
  for (int n3 = 0; n3 < 9; ++n3) {
    __pipeline_wait_prior(1);
    __syncwarp();
    const float* sm = rg[n3 % 3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int n = 3 * n3 + j;
      float c9[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) c9[e] = sm[(9 * j + e) * 32 + lane];
      const size_t off = 3 * (size_t)(fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9]);
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        const float* xn = xb[k][n / 9] + off;
        block_fma(c9, __ldg(xn), __ldg(xn + 1), __ldg(xn + 2), acc[k]);
      }
    }
    __syncwarp();
    if (n3 + 2 < 9) issue(n3 + 2, (n3 + 2) % 3);
    __pipeline_commit();
  }
#pragma unroll
  for (int k = 0; k < NL; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      io.y[k][3 * (size_t)loc + c] = io.f[k] ? io.f[k][3 * (size_t)loc + c] - acc[k][c] : acc[k][c];
}

template <typename TS, typename TN>
__device__ __forceinline__ bool gs_solve_store(const double S[9], const double m[3], const TN* f, size_t loc, TN* y,
                                               int* err);

// GS colour pass with the streamed stencil block (plain passes only: a zero-start pass needs a few of
// the 27 blocks, streaming all of them would read more). Same arithmetic and order as
// stencil_gs_fast_kernel<..., float>: bit-identical.
template <bool ZL, int NL>
__global__ void __launch_bounds__(128) stencil_gs_stream_kernel(GridGeo g, const float* __restrict__ st,
                                                                RhsN<float> io, int color, int* err) {
  __shared__ __align__(16) float ring[4][3][kStStage];
  const int h2 = blockIdx.z;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h1 >= g.cd[0][1]) return;  // whole warps (cd0 % 32 == 0)
  const int lane = threadIdx.x & 31, w = threadIdx.y;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  const unsigned loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
  const float* chunk = st + st_index(0, loc & ~31u);
  float(*rg)[kStStage] = ring[w];
  auto issue = [&](int stage, int slot) {
    const float4* src = reinterpret_cast<const float4*>(chunk + (size_t)stage * kStStage);
    float4* dst = reinterpret_cast<float4*>(rg[slot]);
    for (int i = lane; i < kStStage / 4; i += 32) __pipeline_memcpy_async(dst + i, src + i, 16);
  };
  double S[9];
  stencil_block(st + st_index(9 * 13, loc), S);  // self block: same values, read as the fast kernel does
  float m[NL][3] = {};
  const float* ub[NL][3];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const ZLink<float> ul = ZL ? io.xl[k] : ZLink<float>{io.x[k], io.x[k]};
    ub[k][0] = zbase(fa, io.x[k], ul, 0);
    ub[k][1] = io.x[k];
    ub[k][2] = zbase(fa, io.x[k], ul, 2);
  }
  issue(0, 0);
  __pipeline_commit();
  issue(1, 1);
  __pipeline_commit();
#pragma unroll
  for (int n3 = 0; n3 < 9; ++n3) {
    __pipeline_wait_prior(1);
    __syncwarp();
    const float* sm = rg[n3 % 3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int n = 3 * n3 + j;
      if (n == 13) continue;
      float c9[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) c9[e] = sm[(9 * j + e) * 32 + lane];
      const size_t off = 3 * (size_t)(fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9]);
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        const float* un = ub[k][n / 9] + off;
        block_fma(c9, __ldg(un), __ldg(un + 1), __ldg(un + 2), m[k]);
      }
    }
    __syncwarp();
    if (n3 + 2 < 9) issue(n3 + 2, (n3 + 2) % 3);
    __pipeline_commit();
  }
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const double mk[3] = {double(m[k][0]), double(m[k][1]), double(m[k][2])};
    if (!gs_solve_store<float, float>(S, mk, io.f[k], loc, io.y[k], err)) return;
  }
}

static bool stencil_stream_ok(const GridGeo& g) {
  return knob("STENCIL_STREAM", 1) != 0 && g.cd[0][0] % 32 == 0 && g.size[0] % 32 == 0;
}

// zm: neighbours known to be zero (zero-start sweep, common.cuh zero_start_mask): their stencil
// blocks and values are not read -- bit-identical to adding their exact zero products.
template <typename TS, typename TN>
__device__ __forceinline__ bool gs_solve_store(const double S[9], const double m[3], const TN* f, size_t loc, TN* y,
                                               int* err) {
  const double rhs[3] = {double(f[3 * loc]) - m[0], double(f[3 * loc + 1]) - m[1], double(f[3 * loc + 2]) - m[2]};
  const double det = S[0] * (S[4] * S[8] - S[5] * S[7]) - S[1] * (S[3] * S[8] - S[5] * S[6]) +
                     S[2] * (S[3] * S[7] - S[4] * S[6]);
  if (det == 0.0 || !isfinite(det)) {
    atomicExch(err, 1);
    return false;
  }
  double out[3];
  solve3(S, rhs, out);
#pragma unroll
  for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(out[c]);
  return true;
}

template <typename TS, typename TN, bool ZL, int NL, typename TACC = double>
__global__ void __launch_bounds__(128) stencil_gs_fast_kernel(GridGeo g, const TS* __restrict__ st, RhsN<TN> io,
                                                              int color, int* err, unsigned zm) {
  const int h2 = blockIdx.z;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= g.cd[0][0] || h1 >= g.cd[0][1]) return;
  FastAddr fa;
  fast_addr(g, color, h0, h1, h2, fa);
  const unsigned loc = fa.A[0][1] + fa.A[1][1] + fa.A[2][1];
  const TS* row = st + st_index(0, loc);
  TACC m[NL][3] = {};
  double S[9];
  stencil_block(row + 32 * 9 * 13, S);
  const TN* ub[NL][3];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const ZLink<TN> ul = ZL ? io.xl[k] : ZLink<TN>{io.x[k], io.x[k]};
    ub[k][0] = zbase(fa, io.x[k], ul, 0);
    ub[k][1] = io.x[k];
    ub[k][2] = zbase(fa, io.x[k], ul, 2);
  }
#pragma unroll
  for (int n = 0; n < 27; ++n) {
    if (n == 13 || ((zm >> n) & 1u)) continue;
    TACC c9[9];
    stencil_block(row + 32 * 9 * n, c9);
    const size_t off = 3 * (size_t)(fa.A[0][n % 3] + fa.A[1][(n / 3) % 3] + fa.A[2][n / 9]);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const TN* un = ub[k][n / 9] + off;
      block_fma(c9, TACC(__ldg(un)), TACC(__ldg(un + 1)), TACC(__ldg(un + 2)), m[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const double mk[3] = {double(m[k][0]), double(m[k][1]), double(m[k][2])};
    if (!gs_solve_store<TS, TN>(S, mk, io.f[k], loc, io.y[k], err)) return;
  }
}

// Small levels (latency-bound: a few thousand vertices, long per-thread load
// chains): one warp per vertex, lane n < 27 handles neighbour n, partial sums
// reduced with a fixed-order xor shuffle (deterministic).
__device__ __forceinline__ unsigned nbr_loc(const GridGeo& g, int x, int y, int z, int n) {
  const int tx = n % 3 - 1, ty = (n / 3) % 3 - 1, tz = n / 9 - 1;
  int a = x + tx, b = y + ty, c = z + tz;
  a = a < 0 ? a + g.n[0] : (a >= g.n[0] ? a - g.n[0] : a);
  b = b < 0 ? b + g.n[1] : (b >= g.n[1] ? b - g.n[1] : b);
  c = c < 0 ? c + g.n[2] : (c >= g.n[2] ? c - g.n[2] : c);
  return vloc(g, a, b, c);
}

// neighbour n of (x, y, z) in nodal array p; z wraps through the slab links
template <typename TN>
__device__ __forceinline__ const TN* nbr_ptr(const GridGeo& g, const TN* p, const ZLink<TN>& zl, int x, int y, int z,
                                             int n) {
  const int c = z + n / 9 - 1;
  const TN* b = c < 0 ? zl.lo : (c >= g.n[2] ? zl.hi : p);
  return b + 3 * (size_t)nbr_loc(g, x, y, z, n);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename TS, typename TN, int NL>
__device__ __forceinline__ void apply_warp_vertex(const GridGeo& g, const TS* __restrict__ st, const RhsN<TN>& io,
                                                  long long loc, int lane) {
  const int color = color_at(g, loc);
  int vx, vy, vz;
  block_coords(g, color, (unsigned)(loc - g.base[color]), vx, vy, vz);
  double a[NL][3] = {};
  if (lane < 27) {
    double c9[9];
    stencil_block(st + st_index(9 * lane, (unsigned)loc), c9);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const TN* xn = nbr_ptr(g, io.x[k], io.xl[k], vx, vy, vz, lane);
      block_fma(c9, double(xn[0]), double(xn[1]), double(xn[2]), a[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < NL; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) a[k][c] = warp_sum(a[k][c]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NL; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        io.y[k][3 * loc + c] = io.f[k] ? TN(double(io.f[k][3 * loc + c]) - a[k][c]) : TN(a[k][c]);
  }
}

template <typename TS, typename TN, int NL>
__global__ void __launch_bounds__(128) stencil_apply_warp_kernel(GridGeo g, const TS* __restrict__ st, RhsN<TN> io) {
  const long long loc = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (loc >= g.nv) return;
  apply_warp_vertex<TS, TN, NL>(g, st, io, loc, lane);
}

// colour-block vertex i of colour `color` (one warp)
template <typename TS, typename TN, int NL>
__device__ __forceinline__ void gs_warp_vertex(const GridGeo& g, const TS* __restrict__ st, const RhsN<TN>& io,
                                               int color, int* err, unsigned zm, long long i, int lane) {
  int vx, vy, vz;
  block_coords(g, color, (unsigned)i, vx, vy, vz);
  const long long loc = g.base[color] + i;
  double m[NL][3] = {};
  if (lane < 27 && lane != 13 && !((zm >> lane) & 1u)) {
    double c9[9];
    stencil_block(st + st_index(9 * lane, (unsigned)loc), c9);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const TN* un = nbr_ptr(g, io.x[k], io.xl[k], vx, vy, vz, lane);
      block_fma(c9, double(un[0]), double(un[1]), double(un[2]), m[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < NL; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) m[k][c] = warp_sum(m[k][c]);
  if (lane == 0) {
    double S[9];
    stencil_block(st + st_index(9 * 13, (unsigned)loc), S);
#pragma unroll
    for (int k = 0; k < NL; ++k)
      if (!gs_solve_store<TS, TN>(S, m[k], io.f[k], size_t(loc), io.y[k], err)) return;
  }
}

template <typename TS, typename TN, int NL>
__global__ void __launch_bounds__(128) stencil_gs_warp_kernel(GridGeo g, const TS* __restrict__ st, RhsN<TN> io,
                                                              int color, int* err, unsigned zm) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= g.size[color]) return;
  gs_warp_vertex<TS, TN, NL>(g, st, io, color, err, zm, i, lane);
}

// levels with at most this many vertices per colour use warp-per-vertex (default 4096: up to 32^3;
// 64^3 runs 35% faster thread-per-vertex, measured)
static long long warp_vmax() { return (long long)knob("WARP_VMAX", 4096); }
static bool stencil_f32() { return knob("STENCIL_F32", 1) != 0; }

template <typename TS, typename TN, int NL>
static void launch_apply_n(const GridGeo& g, const TS* st, RhsN<TN> io, cudaStream_t s) {
  bool linked = false;
  for (int k = 0; k < NL; ++k) {
    linked = linked || !is_self(io.xl[k], io.x[k]);
    io.xl[k] = resolve(io.xl[k], io.x[k]);
  }
  if (g.nv <= 8 * warp_vmax()) {
    stencil_apply_warp_kernel<TS, TN, NL><<<ceil_div(g.nv * 32, 128), 128, 0, s>>>(g, st, io);
  } else if (fast_ok(g)) {
    const dim3 b = fast_block(g);
    const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), 8 * g.cd[0][2]);
    if constexpr (std::is_same_v<TS, float> && std::is_same_v<TN, float>) {
      if (stencil_f32() && stencil_stream_ok(g) && b.x == 32) {
        if (linked) stencil_apply_stream_kernel<true, NL><<<gr, b, 0, s>>>(g, st, io);
        else stencil_apply_stream_kernel<false, NL><<<gr, b, 0, s>>>(g, st, io);
        IHOM_LAUNCH_CHECK();
        return;
      }
    }
    if (std::is_same_v<TS, float> && std::is_same_v<TN, float> && stencil_f32()) {
      if (linked) stencil_apply_fast_kernel<TS, TN, true, NL, float><<<gr, b, 0, s>>>(g, st, io);
      else stencil_apply_fast_kernel<TS, TN, false, NL, float><<<gr, b, 0, s>>>(g, st, io);
    } else {
      if (linked) stencil_apply_fast_kernel<TS, TN, true, NL><<<gr, b, 0, s>>>(g, st, io);
      else stencil_apply_fast_kernel<TS, TN, false, NL><<<gr, b, 0, s>>>(g, st, io);
    }
  } else {
    if (linked) throw std::invalid_argument("z-slab level needs an even grid");
    stencil_apply_kernel<TS, TN, NL><<<ceil_div(g.nv, 128), 128, 0, s>>>(g, st, io);
  }
  IHOM_LAUNCH_CHECK();
}

template <typename TS, typename TN>
void launch_stencil_apply(const GridGeo& g, const TS* st, const TN* x, const TN* f, TN* y, cudaStream_t s,
                          ZLink<TN> xl) {
  RhsN<TN> io{{x, nullptr}, {xl, {}}, {f, nullptr}, {y, nullptr}};
  launch_apply_n<TS, TN, 1>(g, st, io, s);
}

template <typename TS, typename TN>
void launch_stencil_apply_group(const GridGeo& g, const TS* st, int nl, const TN* const* x, const TN* const* f,
                                TN* const* y, cudaStream_t s, const ZLink<TN>* xl) {
  RhsN<TN> io{};
  for (int k = 0; k < nl; ++k) io.x[k] = x[k], io.xl[k] = xl[k], io.f[k] = f[k], io.y[k] = y[k];
  switch (nl) {
    case 1: launch_apply_n<TS, TN, 1>(g, st, io, s); break;
    case 2: launch_apply_n<TS, TN, 2>(g, st, io, s); break;
    case 3: launch_apply_n<TS, TN, 3>(g, st, io, s); break;
    case 6: launch_apply_n<TS, TN, 6>(g, st, io, s); break;
    default: throw std::invalid_argument("right-hand-side group size must be 1, 2, 3 or 6");
  }
}

// Colour pass of the coarse GS with the determinant check (src/multigrid.cpp:207-239).
template <typename TS, typename TN, int NL>
__global__ void __launch_bounds__(128) stencil_gs_kernel(GridGeo g, const TS* __restrict__ st, RhsN<TN> io,
                                                         int color, int* err, unsigned zm) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.size[color]) return;
  int vx, vy, vz;
  block_coords(g, color, (unsigned)i, vx, vy, vz);
  Nbhd nb;
  gather27(g, vx, vy, vz, nb);
  const long long loc = g.base[color] + i;
  double m[NL][3] = {}, S[9];
  const TS* row0 = st + st_index(0, (unsigned)loc);
  stencil_block(row0 + 32 * 9 * 13, S);
#pragma unroll 3
  for (int n = 0; n < 27; ++n) {
    if (n == 13 || ((zm >> n) & 1u)) continue;
    double c9[9];
    stencil_block(row0 + 32 * 9 * n, c9);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const TN* un = io.x[k] + 3 * (size_t)nb.v[n];
      block_fma(c9, double(un[0]), double(un[1]), double(un[2]), m[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < NL; ++k)
    if (!gs_solve_store<TS, TN>(S, m[k], io.f[k], size_t(loc), io.y[k], err)) return;
}

template <typename TS, typename TN, int NL>
static void launch_gs_n(const GridGeo& g, const TS* st, RhsN<TN> io, int color, int* err, cudaStream_t s,
                        bool zero_start) {
  bool linked = false;
  for (int k = 0; k < NL; ++k) {
    linked = linked || !is_self(io.xl[k], io.x[k]);
    io.xl[k] = resolve(io.xl[k], io.x[k]);
  }
  const unsigned zm = zero_start ? zero_start_mask(color) : 0u;
  if (g.size[color] <= warp_vmax()) {
    stencil_gs_warp_kernel<TS, TN, NL><<<ceil_div(g.size[color] * 32, 128), 128, 0, s>>>(g, st, io, color, err, zm);
  } else if (fast_ok(g)) {
    const dim3 b = fast_block(g);
    const dim3 gr(ceil_div(g.cd[0][0], b.x), ceil_div(g.cd[0][1], b.y), g.cd[0][2]);
    if constexpr (std::is_same_v<TS, float> && std::is_same_v<TN, float>) {
      if (zm == 0u && stencil_f32() && stencil_stream_ok(g) && b.x == 32) {
        if (linked) stencil_gs_stream_kernel<true, NL><<<gr, b, 0, s>>>(g, st, io, color, err);
        else stencil_gs_stream_kernel<false, NL><<<gr, b, 0, s>>>(g, st, io, color, err);
        IHOM_LAUNCH_CHECK();
        return;
      }
    }
    if (std::is_same_v<TS, float> && std::is_same_v<TN, float> && stencil_f32()) {
      if (linked) stencil_gs_fast_kernel<TS, TN, true, NL, float><<<gr, b, 0, s>>>(g, st, io, color, err, zm);
      else stencil_gs_fast_kernel<TS, TN, false, NL, float><<<gr, b, 0, s>>>(g, st, io, color, err, zm);
    } else {
      if (linked) stencil_gs_fast_kernel<TS, TN, true, NL><<<gr, b, 0, s>>>(g, st, io, color, err, zm);
      else stencil_gs_fast_kernel<TS, TN, false, NL><<<gr, b, 0, s>>>(g, st, io, color, err, zm);
    }
  } else {
    if (linked) throw std::invalid_argument("z-slab level needs an even grid");
    stencil_gs_kernel<TS, TN, NL><<<ceil_div(g.size[color], 128), 128, 0, s>>>(g, st, io, color, err, zm);
  }
  IHOM_LAUNCH_CHECK();
}

template <typename TS, typename TN>
void launch_stencil_gs_color(const GridGeo& g, const TS* st, const TN* f, TN* u, int color, int* err,
                             cudaStream_t s, ZLink<TN> ul, bool zero_start) {
  RhsN<TN> io{{u, nullptr}, {ul, {}}, {f, nullptr}, {u, nullptr}};
  launch_gs_n<TS, TN, 1>(g, st, io, color, err, s, zero_start);
}

template <typename TS, typename TN>
void launch_stencil_gs_color_group(const GridGeo& g, const TS* st, int nl, const TN* const* f, TN* const* u,
                                   int color, int* err, cudaStream_t s, const ZLink<TN>* ul, bool zero_start) {
  RhsN<TN> io{};
  for (int k = 0; k < nl; ++k) io.x[k] = u[k], io.xl[k] = ul[k], io.f[k] = f[k], io.y[k] = u[k];
  switch (nl) {
    case 1: launch_gs_n<TS, TN, 1>(g, st, io, color, err, s, zero_start); break;
    case 2: launch_gs_n<TS, TN, 2>(g, st, io, color, err, s, zero_start); break;
    case 3: launch_gs_n<TS, TN, 3>(g, st, io, color, err, s, zero_start); break;
    case 6: launch_gs_n<TS, TN, 6>(g, st, io, color, err, s, zero_start); break;
    default: throw std::invalid_argument("right-hand-side group size must be 1, 2, 3 or 6");
  }
}

// ---------------------------------------------------------------- Galerkin assembly
// Level-1 table: for every output neighbour n a list of (oidx, W[9]) terms,
// flattened; c_eg_start[n] .. c_eg_start[n+1].
constexpr int kMaxEgTerms = 512;
__constant__ int c_eg_start[28];
__constant__ int c_eg_oidx[kMaxEgTerms];
__constant__ double c_eg_w[kMaxEgTerms][9];

// ---- compile-time term structure of the element Galerkin table (tables.cpp ElementGalerkin) ----
// Fine element offset o in {-2..1}^3 contributes to output neighbour delta iff, per axis,
// o in [2 delta - 2, 2 delta + 1] (some local vertex of the element interpolates from v_c and some
// from v_c + delta); terms are ordered by oidx = (ox+2) + 4 (oy+2) + 16 (oz+2) within each n.
// upload_galerkin_tables() checks the host table against this structure.
__host__ __device__ constexpr bool eg_axis_in(int o, int d) { return o >= 2 * d - 2 && o <= 2 * d + 1; }
__host__ __device__ constexpr bool eg_has(int n, int oidx) {
  return eg_axis_in(oidx % 4 - 2, n % 3 - 1) && eg_axis_in((oidx / 4) % 4 - 2, (n / 3) % 3 - 1) &&
         eg_axis_in(oidx / 16 - 2, n / 9 - 1);
}
__host__ __device__ constexpr int eg_rank(int n, int oidx) {  // terms of n before oidx
  int r = 0;
  for (int o = 0; o < oidx; ++o) r += eg_has(n, o) ? 1 : 0;
  return r;
}
__host__ __device__ constexpr int eg_start(int n) {
  int k = 0;
  for (int m = 0; m < n; ++m) k += eg_rank(m, 64);
  return k;
}


void upload_galerkin_tables(const ElementGalerkin& eg, cudaStream_t s) {
  int start[28];
  static int oidx[kMaxEgTerms];
  static double w[kMaxEgTerms][9];
  int k = 0;
  for (int n = 0; n < 27; ++n) {
    start[n] = k;
    for (const auto& t : eg.by_n[size_t(n)]) {
      if (k >= kMaxEgTerms) throw std::logic_error("element Galerkin table overflow");
      oidx[k] = t.oidx;
      for (int e = 0; e < 9; ++e) w[k][e] = t.w[e];
      ++k;
    }
  }
  start[27] = k;
  for (int n = 0; n < 27; ++n) {  // the unrolled kernel hard-codes this structure
    if (start[n] != eg_start(n)) throw std::logic_error("element Galerkin table: unexpected term count");
    for (int i = start[n]; i < start[n + 1]; ++i)
      if (!eg_has(n, oidx[i]) || eg_rank(n, oidx[i]) != i - start[n])
        throw std::logic_error("element Galerkin table: unexpected term order");
  }
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_eg_start, start, sizeof(start), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_eg_oidx, oidx, sizeof(int) * k, 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_eg_w, w, sizeof(double) * 9 * k, 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaStreamSynchronize(s));  // host staging buffers are static
}

// assemble_stencil_from_elements (src/multigrid.cpp:281-305): one thread per
// (coarse vertex, output neighbour n). blockIdx.z = n + 27 (colour + 8 h2): the 27
// neighbours and then the 8 colours of one coarse plane run back to back, so the
// 64 fine coefficients of a region are fetched once and reused from L1/L2. The
// term list of n (<= 64 x (oidx, W[9])) is staged in shared memory (broadcast reads).
constexpr int kMaxEgPerN = 64;
// z-slab form: fine element planes below the slab (2 z - 2, 2 z - 1 < 0) come
// from the slab below (cl.lo); the output goes to gout at halved plane h2 + zoff.
template <typename TC>
__global__ void __launch_bounds__(128) gal_elem_kernel(GridGeo gf, GridGeo gc, const TC* __restrict__ coeff,
                                                       ZLink<TC> cl, GridGeo gout, int zoff, TC* __restrict__ st) {
  __shared__ double w_s[kMaxEgPerN][9];
  __shared__ int o_s[kMaxEgPerN];
  const int n = blockIdx.z % 27;
  const int rest = blockIdx.z / 27;
  const int color = rest & 7, h2 = rest >> 3;
  const int k0 = c_eg_start[n], nt = c_eg_start[n + 1] - k0;
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  for (int i = t; i < nt * 9; i += blockDim.x * blockDim.y) w_s[i / 9][i % 9] = c_eg_w[k0 + i / 9][i % 9];
  for (int i = t; i < nt; i += blockDim.x * blockDim.y) o_s[i] = c_eg_oidx[k0 + i];
  __syncthreads();
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= gc.cd[0][0] || h1 >= gc.cd[0][1]) return;
  const int x = 2 * h0 + (color & 1), y = 2 * h1 + ((color >> 1) & 1), z = 2 * h2 + ((color >> 2) & 1);
  int ex[4], ey[4], ez[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) {  // wrapped fine coordinates 2*vc + o - 2
    ex[o] = wrapi(2 * x + o - 2, gf.n[0]);
    ey[o] = gf.n[0] * wrapi(2 * y + o - 2, gf.n[1]);
    ez[o] = gf.n[0] * gf.n[1] * wrapi(2 * z + o - 2, gf.n[2]);
  }
  const TC* zb[2] = {2 * z - 2 < 0 ? cl.lo : coeff, 2 * z - 1 < 0 ? cl.lo : coeff};  // planes o = 0, 1
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < nt; ++k) {
    const int oi = o_s[k];
    const int oz = oi >> 4;
    const double q = double(__ldg((oz < 2 ? zb[oz] : coeff) + (ex[oi & 3] + ey[(oi >> 2) & 3] + ez[oz])));
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e] += q * w_s[k][e];
  }
  const unsigned loc =
      (unsigned)(color * gout.size[0] + h0 + (long long)gout.cd[0][0] * (h1 + (long long)gout.cd[0][1] * (h2 + zoff)));
#pragma unroll
  for (int e = 0; e < 9; ++e) st[st_index(9 * n + e, loc)] = TC(acc[e]);
}

// Level-1 Galerkin with the term list unrolled at compile time: the fine-coefficient address of
// every term is a fixed register sum, W comes straight from the constant bank as a DFMA operand
// (no shared-memory staging, no dynamic indexing). Same terms, same order, same arithmetic as
// gal_elem_kernel: bit-identical.
template <typename TC, int N, int OI = 0>
__device__ __forceinline__ void gal_elem_terms(const TC* const zb[4], const int ex[4], const int ey[4],
                                               const int ez[4], double acc[9]) {
  if constexpr (OI < 64) {
    if constexpr (eg_has(N, OI)) {
      constexpr int k = eg_start(N) + eg_rank(N, OI);
      const double q = double(__ldg(zb[OI >> 4] + (ex[OI & 3] + ey[(OI >> 2) & 3] + ez[OI >> 4])));
#pragma unroll
      for (int e = 0; e < 9; ++e) acc[e] += q * c_eg_w[k][e];
    }
    gal_elem_terms<TC, N, OI + 1>(zb, ex, ey, ez, acc);
  }
}

template <typename TC, int N>
__device__ __forceinline__ void gal_elem_n(const TC* const zb[4], const int ex[4], const int ey[4], const int ez[4],
                                           TC* __restrict__ st, unsigned loc) {
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  gal_elem_terms<TC, N>(zb, ex, ey, ez, acc);
#pragma unroll
  for (int e = 0; e < 9; ++e) st[st_index(9 * N + e, loc)] = TC(acc[e]);
}

template <typename TC, int N = 0>
__device__ __forceinline__ void gal_elem_dispatch(int n, const TC* const zb[4], const int ex[4], const int ey[4],
                                                  const int ez[4], TC* __restrict__ st, unsigned loc) {
  if constexpr (N < 27) {
    if (n == N) gal_elem_n<TC, N>(zb, ex, ey, ez, st, loc);
    else gal_elem_dispatch<TC, N + 1>(n, zb, ex, ey, ez, st, loc);
  }
}

template <typename TC>
__global__ void __launch_bounds__(128) gal_elem_unrolled_kernel(GridGeo gf, GridGeo gc, const TC* __restrict__ coeff,
                                                                ZLink<TC> cl, GridGeo gout, int zoff,
                                                                TC* __restrict__ st) {
  // n SLOWEST (blockIdx.z = rest + 8 d2 n): the resident blocks run the same n-branch, so the
  // instruction cache holds one ~5 KB unrolled body instead of thrashing over all 27 (ncu:
  // "no_instruction" was the top stall with n fastest); the coefficients are re-read per n from L2/HBM
  // (chunking z so that they stay in L2 across the 27 n was measured no faster: the pass is DFMA-bound).
  const int nrest = 8 * gc.cd[0][2];
  const int n = blockIdx.z / nrest;
  const int rest = blockIdx.z % nrest;
  const int color = rest & 7, h2 = rest >> 3;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= gc.cd[0][0] || h1 >= gc.cd[0][1]) return;
  const int x = 2 * h0 + (color & 1), y = 2 * h1 + ((color >> 1) & 1), z = 2 * h2 + ((color >> 2) & 1);
  int ex[4], ey[4], ez[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    ex[o] = wrapi(2 * x + o - 2, gf.n[0]);
    ey[o] = gf.n[0] * wrapi(2 * y + o - 2, gf.n[1]);
    ez[o] = gf.n[0] * gf.n[1] * wrapi(2 * z + o - 2, gf.n[2]);
  }
  const TC* zb[4] = {2 * z - 2 < 0 ? cl.lo : coeff, 2 * z - 1 < 0 ? cl.lo : coeff, coeff, coeff};
  const unsigned loc =
      (unsigned)(color * gout.size[0] + h0 + (long long)gout.cd[0][0] * (h1 + (long long)gout.cd[0][1] * (h2 + zoff)));
  gal_elem_dispatch<TC>(n, zb, ex, ey, ez, st, loc);
}

// generic (odd coarse grids): one thread per (coarse vertex, n), term list from constant memory
template <typename TC>
__global__ void __launch_bounds__(128) gal_elem_generic_kernel(GridGeo gf, GridGeo gc, const TC* __restrict__ coeff,
                                                               TC* __restrict__ st) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = blockIdx.y;
  if (loc >= gc.nv) return;
  const int color = color_at(gc, loc);
  int x, y, z;
  block_coords(gc, color, (unsigned)(loc - gc.base[color]), x, y, z);
  int ex[4], ey[4], ez[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    ex[o] = wrapi(2 * x + o - 2, gf.n[0]);
    ey[o] = gf.n[0] * wrapi(2 * y + o - 2, gf.n[1]);
    ez[o] = gf.n[0] * gf.n[1] * wrapi(2 * z + o - 2, gf.n[2]);
  }
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = c_eg_start[n]; k < c_eg_start[n + 1]; ++k) {
    const int oi = c_eg_oidx[k];
    const double q = double(__ldg(coeff + (ex[oi & 3] + ey[(oi >> 2) & 3] + ez[oi >> 4])));
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e] += q * c_eg_w[k][e];
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) st[st_index(9 * n + e, (unsigned)loc)] = TC(acc[e]);
}

template <typename TC>
void launch_galerkin_from_elements(const GridGeo& gf, const GridGeo& gc, const TC* coeff, TC* st, cudaStream_t s,
                                   ZLink<TC> cl, const GridGeo* gout, int zoff) {
  if (gc.n[0] % 2 == 0 && gc.n[1] % 2 == 0 && gc.n[2] % 2 == 0) {
    const dim3 b = fast_block(gc);
    const dim3 gr(ceil_div(gc.cd[0][0], b.x), ceil_div(gc.cd[0][1], b.y), 27 * 8 * gc.cd[0][2]);
    if (knob("GAL_UNROLLED", 1))
      gal_elem_unrolled_kernel<TC><<<gr, b, 0, s>>>(gf, gc, coeff, resolve(cl, coeff), gout ? *gout : gc,
                                                    gout ? zoff : 0, st);
    else
      gal_elem_kernel<TC><<<gr, b, 0, s>>>(gf, gc, coeff, resolve(cl, coeff), gout ? *gout : gc, gout ? zoff : 0, st);
  } else {
    if (!is_self(cl, coeff) || gout) throw std::invalid_argument("z-slab Galerkin needs an even coarse grid");
    gal_elem_generic_kernel<TC><<<dim3(ceil_div(gc.nv, 128), 27), 128, 0, s>>>(gf, gc, coeff, st);
  }
  IHOM_LAUNCH_CHECK();
}

// assemble_stencil_from_stencil (src/multigrid.cpp:307-333):
//   [K_vc]_{vc+delta} = sum_{s,t} w(s) w(s+t-2 delta) [K_{2vc+s}]_t
// One thread per (coarse vertex, output neighbour delta): blockIdx.y = delta, so
// every warp walks the same (s, t, w) term list from constant memory
// (2197 terms, grouped by delta in the reference's s-outer/t-inner order) and
// accumulates 9 f64 entries.
constexpr int kMaxSgTerms = 2197;
__constant__ int c_sg_start[28];
__constant__ unsigned short c_sg_st[kMaxSgTerms];  // s | t << 5
__constant__ float c_sg_w[kMaxSgTerms];            // products of 1, 1/2, 1/4, 1/8: exact in f32

static void upload_stencil_galerkin(cudaStream_t s) {
  static std::mutex mu;
  static bool done = false;
  std::lock_guard<std::mutex> lock(mu);  // z-slab threads share the process's constant tables
  if (done) return;
  static int start[28];
  static unsigned short st[kMaxSgTerms];
  static float w[kMaxSgTerms];
  const StencilGalerkin sg;
  int k = 0;
  for (int n = 0; n < 27; ++n) {
    start[n] = k;
    for (const auto& t : sg.by_n[size_t(n)]) {
      st[k] = (unsigned short)(t.s | (t.t << 5));
      w[k] = float(t.w);
      ++k;
    }
  }
  start[27] = k;
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_sg_start, start, sizeof(start), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_sg_st, st, sizeof(unsigned short) * k, 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_sg_w, w, sizeof(float) * k, 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaStreamSynchronize(s));
  done = true;
}

template <typename TS>
__global__ void __launch_bounds__(128) gal_stencil_kernel(GridGeo gf, GridGeo gc, const TS* __restrict__ stf,
                                                          TS* __restrict__ stc) {
  const long long loc = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = blockIdx.y;
  if (loc >= gc.nv) return;
  const int color = color_at(gc, loc);
  int x, y, z;
  block_coords(gc, color, (unsigned)(loc - gc.base[color]), x, y, z);
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int k1 = c_sg_start[n + 1];
  for (int k = c_sg_start[n]; k < k1; ++k) {
    const int st = c_sg_st[k];
    const int s = st & 31, t = st >> 5;
    const unsigned fl = vloc(gf, wrapi(2 * x + s % 3 - 1, gf.n[0]), wrapi(2 * y + (s / 3) % 3 - 1, gf.n[1]),
                             wrapi(2 * z + s / 9 - 1, gf.n[2]));
    const double w = double(c_sg_w[k]);
    const TS* b = stf + st_index(9 * t, fl);
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e] += w * double(__ldg(b + 32 * e));
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) stc[st_index(9 * n + e, (unsigned)loc)] = TS(acc[e]);
}

// Even coarse grid: one thread per (coarse vertex, 3x3 entry e), colour-fastest blocks
// (blockIdx.z = colour + 8 (e + 9 h2)). The thread loads each of the 729 fine values
// [K_{2vc+s}]_t (entry e) once, converts it once and scatters it into every coarse block delta it
// feeds (gal_gen.cuh, tools/gen_galerkin.py): 729 loads + conversions and 2197 f64 FMAs instead of
// 2197 of each; each accumulator still sees the reference's s-outer / t-inner term order.
template <typename TS>
__global__ void __launch_bounds__(128) gal_stencil_fast_kernel(GridGeo gf, GridGeo gc, const TS* __restrict__ stf,
                                                               ZLink<TS> sl, GridGeo gout, int zoff,
                                                               TS* __restrict__ stc) {
  // blockIdx.z = colour + 8 (e + 9 h2): the eight colours of one coarse plane pair run back to back on
  // the same entry e, so the entry-e rows of the five fine planes they read (~35 MB at 512^3) are shared
  // in L2 instead of being re-read from DRAM per colour (ncu: 41 GB read per launch with e outermost)
  const int color = blockIdx.z & 7;
  const int e = (blockIdx.z >> 3) % 9;
  const int h2 = (blockIdx.z >> 3) / 9;
  const int h0 = blockIdx.x * blockDim.x + threadIdx.x, h1 = blockIdx.y * blockDim.y + threadIdx.y;
  if (h0 >= gc.cd[0][0] || h1 >= gc.cd[0][1]) return;
  const int x = 2 * h0 + (color & 1), y = 2 * h1 + ((color >> 1) & 1), z = 2 * h2 + ((color >> 2) & 1);
  FastAddr fa;
  fast_addr(gf, 0, x, y, z, fa);  // fine vertex 2 vc: colour 0 at halved (x, y, z)
  const TS* lo = zbase(fa, stf, sl, 0);  // fine rows of the z-1 plane (fine colour 0: only that one wraps)
  const TS* pb[27];
#pragma unroll
  for (int s = 0; s < 27; ++s)
    pb[s] = (s < 9 ? lo : stf) + st_index(e, fa.A[0][s % 3] + fa.A[1][(s / 3) % 3] + fa.A[2][s / 9]);
  double A[27];
#pragma unroll
  for (int n = 0; n < 27; ++n) A[n] = 0.0;
#define GAL_LD(S, K) double(__ldg(pb[S] + 32 * (K)))
  GAL_TERMS(A)
#undef GAL_LD
  const unsigned loc =
      (unsigned)(color * gout.size[0] + h0 + (long long)gout.cd[0][0] * (h1 + (long long)gout.cd[0][1] * (h2 + zoff)));
#pragma unroll
  for (int n = 0; n < 27; ++n) stc[st_index(9 * n + e, loc)] = TS(A[n]);
}

template <typename TS>
void launch_galerkin_from_stencil(const GridGeo& gf, const GridGeo& gc, const TS* stf, TS* stc, cudaStream_t s,
                                  ZLink<TS> sl, const GridGeo* gout, int zoff) {
  upload_stencil_galerkin(s);
  if (gc.n[0] % 2 == 0 && gc.n[1] % 2 == 0 && gc.n[2] % 2 == 0 && fast_ok(gf)) {
    const dim3 b = fast_block(gc);
    const dim3 gr(ceil_div(gc.cd[0][0], b.x), ceil_div(gc.cd[0][1], b.y), 9 * 8 * gc.cd[0][2]);
    gal_stencil_fast_kernel<TS><<<gr, b, 0, s>>>(gf, gc, stf, resolve(sl, stf), gout ? *gout : gc, gout ? zoff : 0, stc);
  } else {
    if (!is_self(sl, stf) || gout) throw std::invalid_argument("z-slab Galerkin needs even grids");
    gal_stencil_kernel<TS><<<dim3(ceil_div(gc.nv, 128), 27), 128, 0, s>>>(gf, gc, stf, stc);
  }
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- coarsest solve
// One block. Vectors are AoS [loc][3] in the caller's nodal type; the dense matrices are
// in the dof order 3*loc + c of the reference (src/multigrid.cpp:335-366).
constexpr int kCoarseThreads = 512;

__device__ double block_sum_1(double v, double* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) red[t] += red[t + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// x is in dof order; returns sqrt(sum((A x - f)^2)) with f in dof order.
// Row i of M times v, one warp per row: lanes stride the row (coalesced reads of M), fixed-order
// xor-shuffle fold (deterministic). All lanes return the dot product.
__device__ __forceinline__ double warp_row_dot(const double* __restrict__ M, int N, int i, const double* v) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int j = lane; j < N; j += 32) s += M[(size_t)i * N + j] * v[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__device__ double dense_resid(int N, const double* A, const double* x, const double* f, double* r, double* red) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < N; i += nw) {
    const double s = warp_row_dot(A, N, i, x);
    if ((threadIdx.x & 31) == 0) r[i] = f[i] - s;
  }
  __syncthreads();
  double part = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) part += r[i] * r[i];
  return sqrt(block_sum_1(part, red));
}

template <typename TN>
struct CoarseIO {  // the (f, u) pair of each RHS lane; block b solves lane b
  TN* f[kMaxRhsGroup];
  TN* u[kMaxRhsGroup];
};

// One lane's coarsest solve by one block of kCoarseThreads threads (red: kCoarseThreads doubles of shared
// memory); every exit is block-uniform.
template <typename TN>
__device__ void coarsest_lane(int N, long long nv, const double* __restrict__ Ainv, const double* __restrict__ A,
                              const double* __restrict__ Q, int nq, TN* f, TN* u, double negligible, double* work,
                              int* err, double* red) {
  double* fv = work;           // [N] f in dof order
  double* x = work + N;        // [N]
  double* r = work + 2 * N;    // [N]
  // remove_translations(f) (src/multigrid.cpp:81-86, 427)
  for (int c = 0; c < 3; ++c) {
    double part = 0.0;
    for (long long i = threadIdx.x; i < nv; i += blockDim.x) part += double(f[3 * i + c]);
    const double mean = block_sum_1(part, red) / double(nv);
    for (long long i = threadIdx.x; i < nv; i += blockDim.x) fv[3 * i + c] = double(f[3 * i + c]) - mean;
  }
  __syncthreads();
  // deflated near-null modes (floating islands, hierarchy.cpp factor_coarse_dense): f -= q (q . f)
  for (int k = 0; k < nq; ++k) {
    const double* q = Q + (size_t)k * N;
    double part = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) part += q[i] * fv[i];
    const double d = block_sum_1(part, red);
    for (int i = threadIdx.x; i < N; i += blockDim.x) fv[i] -= d * q[i];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) {  // the level's f holds the projected load
    const TN v = TN(fv[i]);
    f[i] = v;
    fv[i] = double(v);
  }
  __syncthreads();
  double part = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) part += fv[i] * fv[i];
  const double fn = sqrt(block_sum_1(part, red));
  if (fn <= negligible) {  // src/multigrid.cpp:430-433
    for (int i = threadIdx.x; i < N; i += blockDim.x) u[i] = TN(0);
    return;
  }
  // x = Ainv f
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < N; i += nw) {
    const double s = warp_row_dot(Ainv, N, i, fv);
    if ((threadIdx.x & 31) == 0) x[i] = s;
  }
  __syncthreads();
  if (fn > 0.0) {  // refinement against the unshifted matrix (src/multigrid.cpp:435-447)
    double rel = dense_resid(N, A, x, fv, r, red) / fn;
    for (int it = 0; it < 3 && rel > 1e-9; ++it) {
      for (int i = warp; i < N; i += nw) {
        const double s = warp_row_dot(Ainv, N, i, r);
        if ((threadIdx.x & 31) == 0) x[i] += s;
      }
      __syncthreads();
      rel = dense_resid(N, A, x, fv, r, red) / fn;
    }
    if (!(rel < 1e-3)) {
      if (threadIdx.x == 0) atomicExch(err, 2);
      return;
    }
  }
  // u = x; remove_translations(u) (src/multigrid.cpp:449-450)
  for (int c = 0; c < 3; ++c) {
    double p2 = 0.0;
    for (long long i = threadIdx.x; i < nv; i += blockDim.x) p2 += x[3 * i + c];
    const double mean = block_sum_1(p2, red) / double(nv);
    for (long long i = threadIdx.x; i < nv; i += blockDim.x) u[3 * i + c] = TN(x[3 * i + c] - mean);
  }
}

template <typename TN>
__global__ void __launch_bounds__(kCoarseThreads) coarsest_kernel(int N, long long nv, const double* __restrict__ Ainv,
                                                                  const double* __restrict__ A,
                                                                  const double* __restrict__ Q, int nq, CoarseIO<TN> io,
                                                                  double negligible, double* work, int* err) {
  __shared__ double red[kCoarseThreads];
  coarsest_lane<TN>(N, nv, Ainv, A, Q, nq, io.f[blockIdx.x], io.u[blockIdx.x], negligible,
                    work + (size_t)blockIdx.x * 3 * N, err, red);
}

template <typename TN>
void launch_coarsest_solve(int ndof, long long nv, const double* Ainv, const double* A, const double* Q, int nq, TN* f,
                           TN* u, double negligible, double* work, int* err, cudaStream_t s) {
  CoarseIO<TN> io{};
  io.f[0] = f;
  io.u[0] = u;
  coarsest_kernel<TN><<<1, kCoarseThreads, 0, s>>>(ndof, nv, Ainv, A, Q, nq, io, negligible, work, err);
  IHOM_LAUNCH_CHECK();
}

void launch_coarsest_solve_group(int ndof, long long nv, const double* Ainv, const double* A, const double* Q, int nq,
                                 int nl, float* const* f, float* const* u, double* work, int* err, cudaStream_t s) {
  if (nl < 1 || nl > kMaxRhsGroup) throw std::invalid_argument("grouped coarsest solve: 1..6 lanes");
  CoarseIO<float> io{};
  for (int k = 0; k < nl; ++k) io.f[k] = f[k], io.u[k] = u[k];
  coarsest_kernel<float><<<nl, kCoarseThreads, 0, s>>>(ndof, nv, Ainv, A, Q, nq, io, 0.0, work, err);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- bottom cycle (one cooperative launch)
bool bottom_level_ok(const GridGeo& g, const GridGeo& gc) {
  if (!fast_ok(g) || g.nv > 8 * warp_vmax() || !transfer_group_ok(g, gc)) return false;
  for (int c = 0; c < 8; ++c)
    if (g.size[c] > warp_vmax() || g.size[c] == 0) return false;
  return true;
}

template <int NL>
__global__ void __launch_bounds__(kCoarseThreads) bottom_cycle_kernel(BottomCycle bc) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[kCoarseThreads];
  const long long nthr = (long long)gridDim.x * blockDim.x, gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nwarp = nthr >> 5, gw = gt >> 5;
  const int lane = threadIdx.x & 31;
  // colour pass c of level L (zm: zero-start mask), then a grid-wide barrier
  auto gs_pass = [&](const BottomLevel& L, int c, unsigned zm) {
    RhsN<float> io{};
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      io.x[k] = L.eu[k];
      io.xl[k] = ZLink<float>{L.eu[k], L.eu[k]};
      io.f[k] = L.ef[k];
      io.y[k] = L.eu[k];
    }
    for (long long i = gw; i < L.g.size[c]; i += nwarp) gs_warp_vertex<float, float, NL>(L.g, L.st, io, c, bc.err, zm, i, lane);
    grid.sync();
  };
  for (int li = 0; li + 1 < bc.nlev; ++li) {  // down: smooth, residual, restrict
    const BottomLevel& L = bc.L[li];
    const BottomLevel& C = bc.L[li + 1];
    if (!L.zs) {
      for (long long t = gt; t < (long long)NL * 3 * L.g.nv; t += nthr) L.eu[t / (3 * L.g.nv)][t % (3 * L.g.nv)] = 0.0f;
      grid.sync();
    }
    for (int sw = 0; sw < bc.pre; ++sw)
      for (int c = 0; c < 8; ++c) gs_pass(L, c, L.zs && sw == 0 ? zero_start_mask(c) : 0u);
    {
      RhsN<float> io{};
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        io.x[k] = L.eu[k];
        io.xl[k] = ZLink<float>{L.eu[k], L.eu[k]};
        io.f[k] = L.ef[k];
        io.y[k] = L.er[k];
      }
      for (long long v = gw; v < L.g.nv; v += nwarp) apply_warp_vertex<float, float, NL>(L.g, L.st, io, v, lane);
    }
    grid.sync();
    const long long nc = C.g.nv, bs = C.g.size[0];
    const int d0 = C.g.cd[0][0], d1 = C.g.cd[0][1];
    for (long long t = gt; t < NL * nc; t += nthr) {
      const int k = int(t / nc);
      const long long r = t % nc, rr = r % bs;
      const int color = int(r / bs), h0 = int(rr % d0), h1 = int((rr / d0) % d1), h2 = int(rr / ((long long)d0 * d1));
      restrict_vertex<float, float>(L.g, L.er[k], ZLink<float>{L.er[k], L.er[k]}, C.ef[k], color, h0, h1, h2, C.g, 0);
    }
    grid.sync();
  }
  if (blockIdx.x < NL) {  // coarsest: block k solves lane k (as the grouped coarsest launch)
    const BottomLevel& C = bc.L[bc.nlev - 1];
    coarsest_lane<float>(bc.N, bc.nvc, bc.Ainv, bc.A, bc.Q, bc.nq, C.ef[blockIdx.x], C.eu[blockIdx.x], 0.0,
                         bc.work + (size_t)blockIdx.x * 3 * bc.N, bc.err, red);
  }
  grid.sync();
  for (int li = bc.nlev - 2; li >= 0; --li) {  // up: prolong-add, smooth
    const BottomLevel& L = bc.L[li];
    const BottomLevel& C = bc.L[li + 1];
    const long long nf = L.g.nv, bs = L.g.size[0];
    const int d0 = L.g.cd[0][0], d1 = L.g.cd[0][1];
    for (long long t = gt; t < NL * nf; t += nthr) {
      const int k = int(t / nf);
      const long long r = t % nf, rr = r % bs;
      const int color = int(r / bs), h0 = int(rr % d0), h1 = int((rr / d0) % d1), h2 = int(rr / ((long long)d0 * d1));
      prolong_add_vertex<float, float>(C.g, L.g, C.eu[k], ZLink<float>{C.eu[k], C.eu[k]}, L.eu[k], color, h0, h1, h2,
                                       0);
    }
    grid.sync();
    for (int sw = 0; sw < bc.post; ++sw)
      for (int c = 0; c < 8; ++c) gs_pass(L, c, 0u);
  }
}

bool launch_bottom_cycle(const BottomCycle& bc, int nl, cudaStream_t s) {
  if (bc.nlev < 2 || bc.nlev > kMaxBottom) throw std::invalid_argument("bottom cycle: 2..6 levels");
  const void* fn = nl == 2 ? (const void*)bottom_cycle_kernel<2>
                 : nl == 3 ? (const void*)bottom_cycle_kernel<3>
                 : nl == 6 ? (const void*)bottom_cycle_kernel<6>
                           : nullptr;
  if (!fn) throw std::invalid_argument("bottom cycle: group of 2, 3 or 6");
  static int blocks[7] = {};
  if (!blocks[nl]) {
    int dev = 0, sms = 0, coop = 0, occ = 0;
    IHOM_CUDA(cudaGetDevice(&dev));
    IHOM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    IHOM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    IHOM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kCoarseThreads, 0));
    blocks[nl] = coop && occ >= 1 ? sms : -1;  // one block per SM: every block co-resident, short barriers
  }
  if (blocks[nl] < 0) return false;
  BottomCycle arg = bc;
  void* args[] = {&arg};
  const cudaError_t e = cudaLaunchCooperativeKernel(fn, blocks[nl], kCoarseThreads, args, 0, s);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    (void)cudaGetLastError();  // a refused configuration, not a sticky error
    blocks[nl] = -1;
    return false;
  }
  IHOM_CUDA(e);
  ++launch_counter();  // counted like every IHOM_LAUNCH_CHECK'd launch (bench gpu_launches)
  return true;
}

// ---------------------------------------------------------------- instantiations
#define INST_T(TN)                                                                                              \
  template void launch_restrict<TN>(const GridGeo&, const GridGeo&, const TN*, TN*, cudaStream_t, ZLink<TN>,   \
                                    const GridGeo*, int);                                                       \
  template void launch_prolong_add<TN>(const GridGeo&, const GridGeo&, const TN*, TN*, cudaStream_t, ZLink<TN>, \
                                       int);
INST_T(double)
INST_T(float)
#undef INST_T
#define INST_S(TS, TN)                                                                                       \
  template void launch_stencil_apply<TS, TN>(const GridGeo&, const TS*, const TN*, const TN*, TN*, cudaStream_t, \
                                             ZLink<TN>);                                                      \
  template void launch_stencil_gs_color<TS, TN>(const GridGeo&, const TS*, const TN*, TN*, int, int*,         \
                                                cudaStream_t, ZLink<TN>, bool);
INST_S(float, double)
INST_S(double, double)
INST_S(float, float)
template void launch_stencil_apply_group<float, float>(const GridGeo&, const float*, int, const float* const*,
                                                       const float* const*, float* const*, cudaStream_t,
                                                       const ZLink<float>*);
template void launch_stencil_gs_color_group<float, float>(const GridGeo&, const float*, int, const float* const*,
                                                          float* const*, int, int*, cudaStream_t,
                                                          const ZLink<float>*, bool);
#undef INST_S
template void launch_galerkin_from_elements<float>(const GridGeo&, const GridGeo&, const float*, float*, cudaStream_t,
                                                   ZLink<float>, const GridGeo*, int);
template void launch_galerkin_from_elements<double>(const GridGeo&, const GridGeo&, const double*, double*,
                                                    cudaStream_t, ZLink<double>, const GridGeo*, int);
template void launch_galerkin_from_stencil<float>(const GridGeo&, const GridGeo&, const float*, float*, cudaStream_t,
                                                  ZLink<float>, const GridGeo*, int);
template void launch_galerkin_from_stencil<double>(const GridGeo&, const GridGeo&, const double*, double*,
                                                   cudaStream_t, ZLink<double>, const GridGeo*, int);
template void launch_coarsest_solve<double>(int, long long, const double*, const double*, const double*, int, double*,
                                            double*, double, double*, int*, cudaStream_t);
template void launch_coarsest_solve<float>(int, long long, const double*, const double*, const double*, int, float*,
                                           float*, double, double*, int*, cudaStream_t);

}  // namespace ihomgpu
