// hsweep_kernels.cuh -- level-0 K.u / residual as a sum-factorised ELEMENT sweep.
//
// Same operator as the vertex-stencil kernels (ku_gen.cuh, sweep_kernels.cuh): y = sum_e q_e K0 u_e
// (src/fem.cpp:98-120), evaluated per element in the per-axis sum/difference basis where K0 has 45
// non-zeros (tools/gen_hada.py, hada_gen.cuh) instead of per vertex as a 27-neighbour stencil
// (243 merged-coefficient products). Every basis change is split per axis and the per-axis partial
// results are shared between the elements / vertices that need them:
//
//   forward   face (x, y of one vertex plane, 4 corners)  ->  element (z: this face +- the face
//             below, kept in registers from the previous plane)
//   middle    w = q_e D/8 u_hat                            (8 class multiplies + 45 terms)
//   inverse   z: element -> upper / lower vertex plane (the upper part waits one plane in
//             registers), y: through a shared-memory exchange with the thread one row up,
//             x: one warp shuffle with the next lane.
//
// FP64 work per vertex drops from ~335 (stencil form) to ~155 operations, shared-memory loads from
// 89 to 18. Rounding differs from the stencil kernels (same operator, different association), so
// this is a separate variant (knob HSWEEP) checked against the oracle at tolerance, not bitwise.
//
// Geometry: a CTA is 32 x BY threads; thread (tx, ty) owns the element column
// (X0 - 1 + tx, Y0 - 1 + ty) and produces the vertex column (X0 + tx, Y0 + ty) for tx < 31,
// ty < BY - 1 (CTA tiles of 31 x (BY - 1) vertices; the u window is 33 x (BY + 1) vertices of one
// plane). The CTA marches up TZ vertex planes; plane z is output one step after its last element
// plane was computed. Periodic wrap / z-slab links are resolved when a window plane is loaded.
// Included by fem_kernels.cu (shares its __constant__ tables; no -rdc).
#pragma once
#include <cuda_pipeline.h>

#include "hada_gen.cuh"

namespace ihomgpu {

template <typename T>
__device__ __forceinline__ T shfl_next(T v) {  // value of the next lane (lane 31 keeps its own)
  return ::__shfl_down_sync(0xffffffffu, v, 1);
}

template <typename TA>
__device__ __forceinline__ TA hada_class(int k);
template <>
__device__ __forceinline__ double hada_class<double>(int k) {
  return c_hada_d[k];
}
template <>
__device__ __forceinline__ float hada_class<float>(int k) {
  return c_hada_f[k];
}

constexpr int kHsX = 32;             // element columns per CTA row (one warp)
constexpr int kHsOX = kHsX - 1;      // output vertices per CTA in x
constexpr int kHsWX = kHsX + 1;      // u window columns
template <int BY>
struct HsGeom {
  static constexpr int WY = BY + 1;
  static constexpr int items = kHsWX * WY;                           // window vertices per plane
  static constexpr int per = (items + kHsX * BY - 1) / (kHsX * BY);  // window items per thread
};

template <typename TN, int BY, bool FUSE>
constexpr int hs_ring() {
  return 3;  // planes s (read), s + 1 (landing), s + 2 (issued into the slot of s - 1)
}
template <typename TN, int BY, bool FUSE>
constexpr size_t hs_smem() {
  return (size_t)hs_ring<TN, BY, FUSE>() * HsGeom<BY>::items * 3 * (sizeof(TN) + (FUSE ? sizeof(float) : 0)) +
         (2 * 6 * BY * kHsX * sizeof(TN) + 3 * 3 * BY * kHsX * sizeof(TN));
}

// grid = (ceil(n0 / 31), ceil(n1 / (BY - 1)), t / TZ); block = (32, BY)
template <typename TC, typename TN, int OUT, int BY, int MINB, bool FUSE>
__global__ void __launch_bounds__(kHsX* BY, MINB)
    l0_hsweep_kernel(GridGeo g, const TC* __restrict__ coeff, ZLink<TC> cl, const TN* __restrict__ u, ZLink<TN> ul,
                     const TN* __restrict__ f, TN* __restrict__ y, float* __restrict__ r32, double* partials, int TZ,
                     const float* __restrict__ e, ZLink<float> el, double* __restrict__ unew) {
  using TA = TN;  // arithmetic and shared-memory value type
  using Geo = HsGeom<BY>;
  constexpr int R = hs_ring<TN, BY, FUSE>();
  constexpr int SLOT = Geo::items * 3;
  extern __shared__ __align__(16) unsigned char hs_raw[];
  TA* us = reinterpret_cast<TA*>(hs_raw);
  TA* xb = us + R * SLOT;                                        // [2][6][BY][32] exchange (y inverse)
  TA* fs = xb + 2 * 6 * BY * kHsX;                               // [3][3][BY][32] f of the output vertex
  float* es = reinterpret_cast<float*>(fs + 3 * 3 * BY * kHsX);  // FUSE: e window ring
  __shared__ double red[kHsX * BY / 32];

  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kHsX + tx;
  const int X0 = blockIdx.x * kHsOX, Y0 = blockIdx.y * (BY - 1), Z0 = blockIdx.z * TZ;
  const int t = g.n[2];
  const unsigned plane = (unsigned)g.cd[0][0] * (unsigned)g.cd[0][1];  // one colour block's halved plane
  // loader bookkeeping, fixed for the march: the window items this thread copies
  unsigned lE[Geo::per], lO[Geo::per];
  int lS[Geo::per];
  [[maybe_unused]] bool lOwn[Geo::per];
#pragma unroll
  for (int r = 0; r < Geo::per; ++r) {
    const int v = tid + r * kHsX * BY;
    lS[r] = -1;
    if (v < Geo::items) {
      const int i = v % kHsWX, j = v / kHsWX;
      const int x = wrapc(X0 - 1 + i, g.n[0]), yy = wrapc(Y0 - 1 + j, g.n[1]);
      lS[r] = 3 * v;
      lOwn[r] = i >= 1 && i <= kHsOX && j >= 1 && j <= BY - 1 && X0 - 1 + i < g.n[0] && Y0 - 1 + j < g.n[1];
      lE[r] = vloc(g, x, yy, 0);
      lO[r] = vloc(g, x, yy, 1);
    }
  }
  auto load_plane = [&](int s, int slot) {  // window plane s <-> local vertex plane Z0 - 1 + s
    const int zl = Z0 - 1 + s;
    const TN* src = zl < 0 ? ul.lo : (zl >= t ? ul.hi : u);
    const float* esrc = nullptr;
    if constexpr (FUSE) esrc = zl < 0 ? el.lo : (zl >= t ? el.hi : e);
    const int z = zl < 0 ? zl + t : (zl >= t ? zl - t : zl);
    const unsigned zoff = (unsigned)(z >> 1) * plane;
    TA* dst = us + slot * SLOT;
#pragma unroll
    for (int r = 0; r < Geo::per; ++r)
      if (lS[r] >= 0) {
        const size_t gl = 3 * (size_t)((z & 1 ? lO[r] : lE[r]) + zoff);
#pragma unroll
        for (int c = 0; c < 3; ++c) __pipeline_memcpy_async(dst + lS[r] + c, src + gl + c, sizeof(TN));
        if constexpr (FUSE) {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            __pipeline_memcpy_async(es + slot * SLOT + lS[r] + c, esrc + gl + c, sizeof(float));
        }
      }
  };
  int rs = 0;  // s % R (window slot of plane s)
  int f3 = 0;  // s % 3 (f slot of output plane s - 3)
  // FUSE: this thread's landed items of window plane s get u += double(e) (the axpy arithmetic); the
  // items this CTA owns (interior columns, vertex planes Z0 .. Z0 + TZ - 1) also go to unew right here
  auto fuse_plane = [&](int s) {
    if constexpr (FUSE) {
      TA* up = us + rs * SLOT;
      const float* ep = es + rs * SLOT;
      const int zl = Z0 - 1 + s;
      const bool zown = s >= 1 && s <= TZ;
      const unsigned zoff = (unsigned)(zl >> 1) * plane;
#pragma unroll
      for (int r = 0; r < Geo::per; ++r)
        if (lS[r] >= 0) {
          TA v[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) v[c] = up[lS[r] + c] + TA(ep[lS[r] + c]);
#pragma unroll
          for (int c = 0; c < 3; ++c) up[lS[r] + c] = v[c];
          if (zown && lOwn[r]) {
            const size_t gl = 3 * (size_t)((zl & 1 ? lO[r] : lE[r]) + zoff);
#pragma unroll
            for (int c = 0; c < 3; ++c) unew[gl + c] = v[c];
          }
        }
    }
  };
  // element coefficient of this thread's column, local element plane ez (>= -1)
  const int ex = wrapc(X0 - 1 + tx, g.n[0]), ey = wrapc(Y0 - 1 + ty, g.n[1]);
  const size_t exy = (size_t)ex + (size_t)g.n[0] * (size_t)ey, eplane = (size_t)g.n[0] * (size_t)g.n[1];
  auto load_q = [&](int ez) -> TC {  // raw: converted where used, so the load is not waited on here
    const TC* src = ez < 0 ? cl.lo : coeff;
    const int z = ez < 0 ? ez + t : ez;
    return __ldg(src + exy + (size_t)z * eplane);
  };
  const bool out_ok = tx < kHsOX && ty < BY - 1 && X0 + tx < g.n[0] && Y0 + ty < g.n[1];
  const int xg = X0 + tx, yg = Y0 + ty;
  const unsigned oE = out_ok ? vloc(g, xg, yg, 0) : 0u, oO = out_ok ? vloc(g, xg, yg, 1) : 0u;
  auto out_loc = [&](int z) { return (size_t)((z & 1 ? oO : oE) + (unsigned)(z >> 1) * plane); };
  // f of this thread's output vertex in plane k (local output index, finalised at step k + 3): copied
  // asynchronously two steps ahead with the window plane of that step (same commit group)
  auto load_f = [&](int k, int slot) {
    if constexpr (OUT != kSwApply) {
      if (out_ok && k >= 0 && k < TZ) {
        const size_t loc = out_loc(Z0 + k);
#pragma unroll
        for (int c = 0; c < 3; ++c)
          __pipeline_memcpy_async(fs + (slot * 3 + c) * BY * kHsX + tid, f + 3 * loc + c, sizeof(TN));
      }
    }
  };

  load_plane(0, 0);
  __pipeline_commit();
  load_plane(1, 1);
  __pipeline_commit();  // f of output planes 0 and 1 ride with window planes 2 and 3
  TC qn = load_q(Z0 - 1);
  // ping-pong register state: faces (this plane / the one below) and upper halves (new / pending)
  TA FA[12], FB[12], UA[12], UB[12], gyu[6];
#pragma unroll
  for (int k = 0; k < 12; ++k) FA[k] = FB[k] = UA[k] = UB[k] = TA(0);
#pragma unroll
  for (int k = 0; k < 6; ++k) gyu[k] = TA(0);
  double ss = 0.0;
  const int last = TZ + 1;  // window planes 0 .. TZ + 1; step s handles window plane s

  // One step. FIN: finalise vertex plane Z0 + s - 3; ELEM: element plane Z0 + s - 2 (needs the face
  // below, Fp); EXCH: its vertex plane Z0 + s - 2 is complete in z (needs the pending upper half Uo).
  auto step = [&](int s, auto FIN, auto FACE, auto ELEM, auto EXCH, TA(&F)[12], const TA(&Fp)[12], TA(&Un)[12],
                  const TA(&Uo)[12]) {
    __pipeline_wait_prior(1);  // window plane s and the f of output plane s - 3 have landed
    if constexpr (decltype(FACE)::value) fuse_plane(s);
    __syncthreads();
    const int rp2 = (rs + 2) % R;
    if (s + 2 <= last) load_plane(s + 2, rp2);
    load_f(s - 1, f3 == 0 ? 2 : f3 - 1);  // finalised at step s + 2
    __pipeline_commit();
    if constexpr (decltype(FIN)::value) {
      // ---- finalise vertex plane Z0 + s - 3 (its y exchange was written in step s - 1)
      const TA* xr = xb + ((s - 1) & 1) * 6 * BY * kHsX;
      const int tyn = ty + 1 < BY ? ty + 1 : ty;  // the last row produces no output
      TA ex6[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) ex6[k] = gyu[k] + xr[(k * BY + tyn) * kHsX + tx];
      TA yv[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const TA S = ex6[c], D = ex6[3 + c];  // tau_x = sum, difference
        const TA up = S + D, lo = S - D;
        yv[c] = up + shfl_next(lo);
      }
      if (out_ok) {
        const size_t loc = out_loc(Z0 + s - 3);
        [[maybe_unused]] const TA* fr = fs + (f3 * 3) * BY * kHsX + tid;
        if constexpr (OUT == kSwDefect) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double r = double(fr[c * BY * kHsX]) - double(yv[c]);
            r32[3 * loc + c] = float(r);
            ss += r * r;
          }
        } else if constexpr (OUT == kSwResidual) {
#pragma unroll
          for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(TA(fr[c * BY * kHsX]) - yv[c]);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(yv[c]);
        }
      }
    }
    if constexpr (decltype(FACE)::value) {
      // ---- forward, face of window plane s: corners (tx, ty) .. (tx + 1, ty + 1)
      const TA* p = us + rs * SLOT + 3 * (ty * kHsWX + tx);
#pragma unroll
      for (int c = 0; c < 3; ++c) {  // F[f*3+c], f = sx + 2 sy
        const TA a = TA(p[c]), b = TA(p[3 + c]), cc = TA(p[3 * kHsWX + c]), d = TA(p[3 * kHsWX + 3 + c]);
        const TA sx0 = b + a, dx0 = b - a, sx1 = d + cc, dx1 = d - cc;
        F[0 * 3 + c] = sx1 + sx0;
        F[2 * 3 + c] = sx1 - sx0;
        F[1 * 3 + c] = dx1 + dx0;
        F[3 * 3 + c] = dx1 - dx0;
      }
    }
    if constexpr (decltype(ELEM)::value) {
      // ---- element plane Z0 + s - 2: u_hat from the faces below (Fp) and above (F)
      const TA q = TA(qn);
      if (s + 1 <= last) qn = load_q(Z0 + s - 1);
      TA uh[24];
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        uh[k] = F[k] + Fp[k];
        uh[12 + k] = F[k] - Fp[k];
      }
      TA qh[kHadaClasses];
#pragma unroll
      for (int k = 0; k < kHadaClasses; ++k) qh[k] = q * hada_class<TA>(k);
      TA w[24];
      hada_apply<TA>(qh, uh, w);
      // ---- inverse z: lower part -> vertex plane Z0 + s - 2, upper part -> Z0 + s - 1 (pending)
      TA gv[12];
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const TA S = k < 3 ? TA(0) : w[k], D = w[12 + k];
        gv[k] = Uo[k] + (k < 3 ? -D : S - D);
        Un[k] = k < 3 ? D : S + D;
      }
      if constexpr (decltype(EXCH)::value) {
        // ---- inverse y of vertex plane Z0 + s - 2: keep the upper half, publish the lower
        TA* xw = xb + (s & 1) * 6 * BY * kHsX;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const TA S = gv[h * 3 + c], D = gv[(2 + h) * 3 + c];
            gyu[h * 3 + c] = S + D;
            xw[((h * 3 + c) * BY + ty) * kHsX + tx] = S - D;
          }
      }
    }
    rs = rs + 1 == R ? 0 : rs + 1;
    f3 = f3 == 2 ? 0 : f3 + 1;
  };
  using T_ = std::true_type;
  using F_ = std::false_type;
  step(0, F_{}, T_{}, F_{}, F_{}, FA, FB, UA, UB);
  step(1, F_{}, T_{}, T_{}, F_{}, FB, FA, UB, UA);
  step(2, F_{}, T_{}, T_{}, T_{}, FA, FB, UA, UB);
  // steady state: steps 3 .. last, two per iteration (the register roles alternate)
  int s = 3;
#pragma unroll 1
  for (; s + 1 <= last; s += 2) {
    step(s, T_{}, T_{}, T_{}, T_{}, FB, FA, UB, UA);
    step(s + 1, T_{}, T_{}, T_{}, T_{}, FA, FB, UA, UB);
  }
  if (s <= last) {
    step(s, T_{}, T_{}, T_{}, T_{}, FB, FA, UB, UA);
    ++s;
  }
  step(s, T_{}, F_{}, F_{}, F_{}, FA, FB, UA, UB);  // s == last + 1: finalise the top plane
  __pipeline_wait_prior(0);
  if constexpr (OUT == kSwDefect) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
    if ((tid & 31) == 0) red[tid >> 5] = ss;
    __syncthreads();
    if (tid == 0) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < kHsX * BY / 32; ++w) sum += red[w];
      partials[blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z)] = sum;
    }
  }
}

}  // namespace ihomgpu

namespace ihomgpu {

constexpr int kHsBY = 8;

bool hsweep_ok(const GridGeo& g, bool f32) {
  if (knob(f32 ? "HSWEEP32" : "HSWEEP", 1) == 0) return false;
  return g.n[0] % 2 == 0 && g.n[1] % 2 == 0 && g.n[2] % 2 == 0 && g.n[0] >= kHsX && g.n[1] >= 2 * kHsBY &&
         g.n[2] >= 4;
}

// planes per CTA: a divisor of the slab's planes minimising (waves) x (steps per CTA), where a CTA
// marches tz + 3 steps and `slots` CTAs are resident at once
static int hsweep_tz(const GridGeo& g, int slots) {
  const long long cols = (long long)ceil_div(g.n[0], kHsOX) * ceil_div(g.n[1], kHsBY - 1);
  int best = g.n[2];
  long long best_cost = -1;
  for (int tz = g.n[2]; tz >= 1; --tz) {
    if (g.n[2] % tz != 0 || (tz < 16 && tz != g.n[2])) continue;
    const long long waves = (cols * (g.n[2] / tz) + slots - 1) / slots;
    const long long cost = waves * (tz + 3);
    if (best_cost < 0 || cost < best_cost) best_cost = cost, best = tz;
  }
  return best;
}

template <typename TC, typename TN, int OUT, bool FUSE>
static long long launch_hsweep(const GridGeo& g, const TC* coeff, ZLink<TC> cl, const TN* u, ZLink<TN> ul,
                               const TN* f, TN* y, float* r32, double* partials, const float* e, ZLink<float> el,
                               double* unew, cudaStream_t s) {
  constexpr size_t sm = hs_smem<TN, kHsBY, FUSE>();
  constexpr int minb = sizeof(TN) == 8 ? 2 : 4;  // f32: 4 CTAs/SM at 64 registers (profiles/kernel_variants_r01.md)
  auto kern = l0_hsweep_kernel<TC, TN, OUT, kHsBY, minb, FUSE>;
  static int per_sm = 0;  // per instantiation
  if (!per_sm) {
    IHOM_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    IHOM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHsX * kHsBY, sm));
    int dev = 0, nsm = 0;
    IHOM_CUDA(cudaGetDevice(&dev));
    IHOM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    per_sm = std::max(1, per_sm) * nsm;
  }
  const int tz = hsweep_tz(g, per_sm);
  const dim3 gr(ceil_div(g.n[0], kHsOX), ceil_div(g.n[1], kHsBY - 1), g.n[2] / tz);
  kern<<<gr, dim3(kHsX, kHsBY), sm, s>>>(g, coeff, cl, u, ul, f, y, r32, partials, tz, e, el, unew);
  IHOM_LAUNCH_CHECK();
  return (long long)gr.x * gr.y * gr.z;
}

}  // namespace ihomgpu


