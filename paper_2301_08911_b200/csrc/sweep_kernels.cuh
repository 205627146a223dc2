// sweep_kernels.cu -- level-0 K.u / residual as a z-plane sweep through shared memory.
//
// Same per-vertex arithmetic as l0_apply_fast_kernel / l0_residual_norm_fast_kernel
// (the generated factored stencil ku_vertex, identical operand order), so every
// output value is bit-identical; what changes is how the 27 neighbours arrive.
//
// The fast kernels read each neighbour straight from HBM/L2 in the colour-block
// AoS layout: three component loads per neighbour at a 12/24-byte lane stride,
// i.e. every L1 sector of a neighbour run is looked up three times, plus a
// 64-bit address per neighbour. ncu (profiles/ncu_r01_l0_stalls.md): the f64
// residual sits at 69% L1 throughput with only 36% issue active -- it is bound
// by L1 wavefronts, not DFMA.
//
// Here a CTA owns a TX x TY column of vertices (actual coordinates, all 8
// colours) over TZ planes and marches up z. A 4-slot ring of shared-memory
// planes holds the (TX+2) x (TY+2) window of u (AoS, like global) for planes
// z-1, z, z+1 while plane z+2 streams in with cp.async; a 3-slot ring holds the
// (TX+1) x (TY+1) element windows of rho^p. Every neighbour is then an LDS at a
// compile-time offset from one of three plane bases (AoS strides of 12 / 24
// bytes are bank-conflict free for 32 consecutive lanes), and the only global
// address arithmetic is the colour-block location of each window vertex,
// computed once per plane. Periodic wrap and z-slab links are resolved while
// loading a plane (the source pointer of plane -1 / t is the slab below /
// above), so the compute loop has no boundary cases at all.
//
// Included by fem_kernels.cu (shares its __constant__ kappa tables; no -rdc).
#pragma once
#include <cuda_pipeline.h>

namespace ihomgpu {

constexpr int kSwTX = 32, kSwTY = 8;                  // vertices per plane per CTA (one per thread)
constexpr int kSwWX = kSwTX + 2, kSwWY = kSwTY + 2;   // u window
constexpr int kSwEX = kSwTX + 1, kSwEY = kSwTY + 1;   // element window
constexpr int kSwUSlot = kSwWX * kSwWY * 3;           // TN values per u plane slot
constexpr int kSwESlot = kSwEX * kSwEY;               // TC values per element plane slot

enum SweepOut { kSwApply = 0, kSwResidual = 1, kSwDefect = 2 };

// Two vertex planes per step (one barrier per two planes): a step needs u planes z-1 .. z+2 and
// element planes z-1 .. z+1 while the next step's two new planes stream in -> rings of 6 and 5.
constexpr int kSwURing = 6, kSwERing = 5;

template <typename TN, typename TC>
constexpr size_t sweep_smem() {
  return sizeof(TN) * kSwURing * kSwUSlot + sizeof(TC) * kSwERing * kSwESlot;
}

__device__ __forceinline__ int wrapc(int c, int n) { return c < 0 ? c + n : (c >= n ? c - n : c); }

// async copy of u plane zl (local index, -1 .. t) of the window into slot buffer dst
template <typename TN>
__device__ __forceinline__ void sweep_load_u(const GridGeo& g, const TN* __restrict__ u, const ZLink<TN>& ul, int X0,
                                             int Y0, int zl, TN* dst) {
  const int t = g.n[2];
  const TN* src = zl < 0 ? ul.lo : (zl >= t ? ul.hi : u);
  const int z = zl < 0 ? zl + t : (zl >= t ? zl - t : zl);
  const int tid = threadIdx.y * kSwTX + threadIdx.x;
  for (int v = tid; v < kSwWX * kSwWY; v += kSwTX * kSwTY) {
    const int i = v % kSwWX, j = v / kSwWX;
    const int x = wrapc(X0 - 1 + i, g.n[0]), y = wrapc(Y0 - 1 + j, g.n[1]);
    const size_t loc = vloc(g, x, y, z);
#pragma unroll
    for (int c = 0; c < 3; ++c) __pipeline_memcpy_async(dst + 3 * v + c, src + 3 * loc + c, sizeof(TN));
  }
}

// async copy of element plane ezl (local, -1 .. t-1) of the window
template <typename TC>
__device__ __forceinline__ void sweep_load_e(const GridGeo& g, const TC* __restrict__ coeff, const ZLink<TC>& cl,
                                             int X0, int Y0, int ezl, TC* dst) {
  const int t = g.n[2];
  const TC* src = ezl < 0 ? cl.lo : coeff;
  const int ez = ezl < 0 ? ezl + t : ezl;
  const int tid = threadIdx.y * kSwTX + threadIdx.x;
  for (int v = tid; v < kSwEX * kSwEY; v += kSwTX * kSwTY) {
    const int i = v % kSwEX, j = v / kSwEX;
    const int x = wrapc(X0 - 1 + i, g.n[0]), y = wrapc(Y0 - 1 + j, g.n[1]);
    const size_t e = (size_t)x + (size_t)g.n[0] * ((size_t)y + (size_t)g.n[1] * ez);
    __pipeline_memcpy_async(dst + v, src + e, sizeof(TC));
  }
}

// grid = (n0 / TX, n1 / TY, t / TZ); block = (TX, TY)
// FUSE (defect residual only): the outer update u += e of the defect-correction cycle is folded in.
// The window planes of the f32 correction e stream in next to those of u; once a thread's copies of a
// plane have landed it adds its own items (u + double(e), the exact axpy arithmetic) in shared memory,
// the step barrier publishes them, the stencil runs on the updated window and every vertex writes its
// updated u to unew -- a second buffer, because the neighbouring CTAs still read the old u of our
// vertices as their halo (the solver swaps the two buffers every cycle).
template <typename TC, typename TN, typename TA, int OUT, int MINB, bool FUSE = false>
__global__ void __launch_bounds__(kSwTX* kSwTY, MINB)
    l0_sweep_kernel(GridGeo g, const TC* __restrict__ coeff, ZLink<TC> cl, const TN* __restrict__ u, ZLink<TN> ul,
                    const TN* __restrict__ f, TN* __restrict__ y, float* __restrict__ r32, double* partials, int TZ,
                    const float* __restrict__ e = nullptr, ZLink<float> el = {}, double* __restrict__ unew = nullptr) {
  extern __shared__ __align__(16) unsigned char sw_raw[];
  TN* us = reinterpret_cast<TN*>(sw_raw);
  TC* es = reinterpret_cast<TC*>(sw_raw + sizeof(TN) * kSwURing * kSwUSlot);
  float* cs = reinterpret_cast<float*>(sw_raw + sizeof(TN) * kSwURing * kSwUSlot + sizeof(TC) * kSwERing * kSwESlot);
  __shared__ double red[kSwTX * kSwTY / 32];
  const int X0 = blockIdx.x * kSwTX, Y0 = blockIdx.y * kSwTY, Z0 = blockIdx.z * TZ;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int xg = X0 + tx, yg = Y0 + ty;
  auto load_u = [&](int zl, int slot) {
    sweep_load_u(g, u, ul, X0, Y0, zl, us + slot * kSwUSlot);
    if constexpr (FUSE) sweep_load_u(g, e, el, X0, Y0, zl, cs + slot * kSwUSlot);
  };
  auto fuse = [&](int slot) {  // this thread's items of a landed plane: u += double(e)
    if constexpr (FUSE) {
      const int tid = threadIdx.y * kSwTX + threadIdx.x;
      TN* up = us + slot * kSwUSlot;
      const float* ep = cs + slot * kSwUSlot;
      for (int v = tid; v < kSwWX * kSwWY; v += kSwTX * kSwTY)
#pragma unroll
        for (int c = 0; c < 3; ++c) up[3 * v + c] += double(ep[3 * v + c]);
    }
  };
  // u plane z sits in slot (z - Z0 + 1) % 6, element plane ez in slot (ez - Z0 + 1) % 5
  for (int P = 0; P < 4; ++P) load_u(Z0 - 1 + P, P);
  for (int E = 0; E < 3; ++E) sweep_load_e(g, coeff, cl, X0, Y0, Z0 - 1 + E, es + E * kSwESlot);
  __pipeline_commit();
  __pipeline_wait_prior(0);
  for (int P = 0; P < 4; ++P) fuse(P);
  __syncthreads();
  double ss = 0.0;
  const int ubase = 3 * ((ty + 1) * kSwWX + tx + 1);
  for (int k = 0; k < TZ; k += 2) {
    if (k + 2 < TZ) {  // planes z+3, z+4 and element planes z+2, z+3 for the next step
      load_u(Z0 + k + 3, (k + 4) % kSwURing);
      load_u(Z0 + k + 4, (k + 5) % kSwURing);
      sweep_load_e(g, coeff, cl, X0, Y0, Z0 + k + 2, es + ((k + 3) % kSwERing) * kSwESlot);
      sweep_load_e(g, coeff, cl, X0, Y0, Z0 + k + 3, es + ((k + 4) % kSwERing) * kSwESlot);
    }
    __pipeline_commit();
#pragma unroll 1
    for (int dz = 0; dz < 2; ++dz) {
      const int kk = k + dz, z = Z0 + kk;
      const TN* p0 = us + (kk % kSwURing) * kSwUSlot + ubase;        // plane z-1
      const TN* p1 = us + ((kk + 1) % kSwURing) * kSwUSlot + ubase;  // plane z
      const TN* p2 = us + ((kk + 2) % kSwURing) * kSwUSlot + ubase;  // plane z+1
      const TC* e0 = es + (kk % kSwERing) * kSwESlot + ty * kSwEX + tx;        // element plane z-1
      const TC* e1 = es + ((kk + 1) % kSwERing) * kSwESlot + ty * kSwEX + tx;  // element plane z
      TA q[8];
#pragma unroll
      for (int ke = 0; ke < 8; ++ke) {
        const TC* eb = (ke >> 2) & 1 ? e1 : e0;
        q[ke] = TA(eb[((ke >> 1) & 1) * kSwEX + (ke & 1)]);
      }
      auto U = [&](int n, int c) -> TA {
        const int t0 = n % 3 - 1, t1 = (n / 3) % 3 - 1, t2 = n / 9;
        const TN* p = t2 == 0 ? p0 : (t2 == 1 ? p1 : p2);
        return TA(p[3 * (t1 * kSwWX + t0) + c]);
      };
      TA acc[3];
      ku_vertex<TA>(q, kappa<TA>(), U, acc);
      const size_t loc = vloc(g, xg, yg, z);
      if constexpr (OUT == kSwDefect) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double r = double(f[3 * loc + c]) - double(acc[c]);
          r32[3 * loc + c] = float(r);
          ss += r * r;
        }
        if constexpr (FUSE) {
#pragma unroll
          for (int c = 0; c < 3; ++c) unew[3 * loc + c] = p1[c];  // the updated u of this vertex
        }
      } else if constexpr (OUT == kSwResidual) {
#pragma unroll
        for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(TA(f[3 * loc + c]) - acc[c]);
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) y[3 * loc + c] = TN(acc[c]);
      }
    }
    __pipeline_wait_prior(0);
    if (k + 2 < TZ) {
      fuse((k + 4) % kSwURing);
      fuse((k + 5) % kSwURing);
    }
    __syncthreads();
  }
  if constexpr (OUT == kSwDefect) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
    const int t = ty * kSwTX + tx;
    if ((t & 31) == 0) red[t >> 5] = ss;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kSwTX * kSwTY / 32; ++w) s += red[w];
      partials[blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z)] = s;
    }
  }
}

// ---------------------------------------------------------------- x-paired f32 sweep (FFMA2)
// Thread (tx, ty) owns the two vertices (X0 + tx, y) and (X0 + 32 + tx, y) of a
// 64 x TY tile; the shared window stores the two halves interleaved as float2
// ([row][col][comp] -> {half 0, half 1}), so every neighbour operand of the
// paired stencil is ONE LDS.64 at a compile-time offset, and the factored
// stencil runs in float2 lane arithmetic (vec2.cuh). Bit-identical to the
// scalar kernels lane by lane.
constexpr int kS2Cols = kSwTX + 2;                       // window columns per half (34)
constexpr int kS2USlot = kS2Cols * kSwWY * 3;            // float2 per u plane slot
constexpr int kS2ECols = kSwTX + 1;                      // element window columns per half (33)
constexpr int kS2ESlot = kS2ECols * kSwEY;               // float2 per element plane slot
constexpr int kS2UItems = 2 * kS2Cols * kSwWY;           // window vertices per plane (both halves)
constexpr int kS2EItems = 2 * kS2ECols * kSwEY;          // window elements per plane
constexpr int kS2UPer = (kS2UItems + kSwTX * kSwTY - 1) / (kSwTX * kSwTY);
constexpr int kS2EPer = (kS2EItems + kSwTX * kSwTY - 1) / (kSwTX * kSwTY);
constexpr size_t kS2Smem = sizeof(float2) * (kSwURing * kS2USlot + kSwERing * kS2ESlot);

// grid = (n0 / 64, n1 / TY, t / TZ); block = (32, TY)
template <int OUT>
__global__ void __launch_bounds__(kSwTX* kSwTY, 2)
    l0_sweep2_kernel(GridGeo g, const float* __restrict__ coeff, ZLink<float> cl, const float* __restrict__ u,
                     ZLink<float> ul, const float* __restrict__ f, float* __restrict__ y, int TZ) {
  extern __shared__ __align__(16) unsigned char sw_raw[];
  float* us = reinterpret_cast<float*>(sw_raw);
  float* es = reinterpret_cast<float*>(sw_raw + sizeof(float2) * kSwURing * kS2USlot);
  const int X0 = blockIdx.x * 2 * kSwTX, Y0 = blockIdx.y * kSwTY, Z0 = blockIdx.z * TZ;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kSwTX + tx;
  const int t = g.n[2];
  const unsigned plane = (unsigned)g.cd[0][0] * (unsigned)g.cd[0][1];  // one colour block's halved plane
  // loader bookkeeping, fixed for the whole march: the window items this thread copies, as
  // (smem float index, location in even-z / odd-z planes at halved z 0)
  unsigned uE[kS2UPer], uO[kS2UPer];
  int uS[kS2UPer];
#pragma unroll
  for (int r = 0; r < kS2UPer; ++r) {
    const int v = tid + r * kSwTX * kSwTY;
    uS[r] = -1;
    if (v < kS2UItems) {
      const int h = v & 1, w = v >> 1, i = w % kS2Cols, j = w / kS2Cols;
      const int x = wrapc(X0 + kSwTX * h + i - 1, g.n[0]), yy = wrapc(Y0 + j - 1, g.n[1]);
      uS[r] = 2 * 3 * w + h;
      uE[r] = vloc(g, x, yy, 0);
      uO[r] = vloc(g, x, yy, 1);
    }
  }
  unsigned eXY[kS2EPer];
  int eS[kS2EPer];
#pragma unroll
  for (int r = 0; r < kS2EPer; ++r) {
    const int v = tid + r * kSwTX * kSwTY;
    eS[r] = -1;
    if (v < kS2EItems) {
      const int h = v & 1, w = v >> 1, i = w % kS2ECols, j = w / kS2ECols;
      const int x = wrapc(X0 + kSwTX * h + i - 1, g.n[0]), yy = wrapc(Y0 + j - 1, g.n[1]);
      eS[r] = 2 * w + h;
      eXY[r] = (unsigned)x + (unsigned)g.n[0] * (unsigned)yy;
    }
  }
  const unsigned eplane = (unsigned)g.n[0] * (unsigned)g.n[1];
  auto load_u = [&](int zl, int slot) {
    const float* src = zl < 0 ? ul.lo : (zl >= t ? ul.hi : u);
    const int z = zl < 0 ? zl + t : (zl >= t ? zl - t : zl);
    const unsigned zoff = (unsigned)(z >> 1) * plane;
    float* dst = us + slot * (2 * kS2USlot);
#pragma unroll
    for (int r = 0; r < kS2UPer; ++r)
      if (uS[r] >= 0) {
        const float* sp = src + 3 * (size_t)((z & 1 ? uO[r] : uE[r]) + zoff);
#pragma unroll
        for (int c = 0; c < 3; ++c) __pipeline_memcpy_async(dst + uS[r] + 2 * c, sp + c, sizeof(float));
      }
  };
  auto load_e = [&](int ezl, int slot) {
    const float* src = ezl < 0 ? cl.lo : coeff;
    const int ez = ezl < 0 ? ezl + t : ezl;
    float* dst = es + slot * (2 * kS2ESlot);
#pragma unroll
    for (int r = 0; r < kS2EPer; ++r)
      if (eS[r] >= 0) __pipeline_memcpy_async(dst + eS[r], src + eXY[r] + (size_t)ez * eplane, sizeof(float));
  };
  for (int P = 0; P < 4; ++P) load_u(Z0 - 1 + P, P);  // u plane z in slot (z - Z0 + 1) % 6
  for (int E = 0; E < 3; ++E) load_e(Z0 - 1 + E, E);  // element plane ez in slot (ez - Z0 + 1) % 5
  __pipeline_commit();
  // output locations of the two vertices (even / odd z at halved z 0)
  const int xa = X0 + tx, xb = X0 + kSwTX + tx, yv = Y0 + ty;
  const unsigned oEa = vloc(g, xa, yv, 0), oOa = vloc(g, xa, yv, 1);
  const unsigned oEb = vloc(g, xb, yv, 0), oOb = vloc(g, xb, yv, 1);
  const float2* U2 = reinterpret_cast<const float2*>(us);
  const float2* E2 = reinterpret_cast<const float2*>(es);
  const int ubase = 3 * ((ty + 1) * kS2Cols + tx + 1);
  __pipeline_wait_prior(0);
  __syncthreads();
  for (int k = 0; k < TZ; k += 2) {
    if (k + 2 < TZ) {
      load_u(Z0 + k + 3, (k + 4) % kSwURing);
      load_u(Z0 + k + 4, (k + 5) % kSwURing);
      load_e(Z0 + k + 2, (k + 3) % kSwERing);
      load_e(Z0 + k + 3, (k + 4) % kSwERing);
    }
    __pipeline_commit();
#pragma unroll 1
    for (int dz = 0; dz < 2; ++dz) {
      const int kk = k + dz, z = Z0 + kk;
      const float2* p0 = U2 + (kk % kSwURing) * kS2USlot + ubase;
      const float2* p1 = U2 + ((kk + 1) % kSwURing) * kS2USlot + ubase;
      const float2* p2 = U2 + ((kk + 2) % kSwURing) * kS2USlot + ubase;
      const float2* e0 = E2 + (kk % kSwERing) * kS2ESlot + ty * kS2ECols + tx;
      const float2* e1 = E2 + ((kk + 1) % kSwERing) * kS2ESlot + ty * kS2ECols + tx;
      float2 q[8];
#pragma unroll
      for (int ke = 0; ke < 8; ++ke) q[ke] = ((ke >> 2) & 1 ? e1 : e0)[((ke >> 1) & 1) * kS2ECols + (ke & 1)];
      auto U = [&](int n, int c) -> float2 {
        const int t0 = n % 3 - 1, t1 = (n / 3) % 3 - 1, t2 = n / 9;
        const float2* p = t2 == 0 ? p0 : (t2 == 1 ? p1 : p2);
        return p[3 * (t1 * kS2Cols + t0) + c];
      };
      float2 acc[3];
      ku_vertex<float2>(q, kappa<float>(), U, acc);
      const unsigned zoff = (unsigned)(z >> 1) * plane;
      const size_t la = (z & 1 ? oOa : oEa) + zoff, lb = (z & 1 ? oOb : oEb) + zoff;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if constexpr (OUT == kSwResidual) {
          y[3 * la + c] = f[3 * la + c] - acc[c].x;
          y[3 * lb + c] = f[3 * lb + c] - acc[c].y;
        } else {
          y[3 * la + c] = acc[c].x;
          y[3 * lb + c] = acc[c].y;
        }
      }
    }
    __pipeline_wait_prior(0);
    __syncthreads();
  }
}

bool sweep2_ok(const GridGeo& g) {
  return knob("L0_SWEEP2", 1) != 0 && g.n[0] % (2 * kSwTX) == 0 && g.n[1] % kSwTY == 0 && g.n[2] % 2 == 0 &&
         g.n[2] >= 4;
}

}  // namespace ihomgpu
#include "hsweep_kernels.cuh"  // sum-factorised element sweep (uses SweepOut / wrapc above)
namespace ihomgpu {

bool sweep_ok(const GridGeo& g) {
  return knob("L0_SWEEP", 1) != 0 && g.n[0] % kSwTX == 0 && g.n[1] % kSwTY == 0 && g.n[2] % 2 == 0 && g.n[2] >= 4 &&
         g.n[0] % 2 == 0 && g.n[1] % 2 == 0;
}

static int sweep_tz(const GridGeo& g) {
  // planes per CTA: enough CTAs for ~4 waves at 2 CTAs/SM, at least 8 planes (halo amortised)
  const long long cols = (long long)(g.n[0] / kSwTX) * (g.n[1] / kSwTY);
  int tz = g.n[2];
  while (tz % 4 == 0 && tz > 8 && cols * (g.n[2] / tz) < 148LL * 2 * 4) tz /= 2;  // stays even
  return tz;
}

template <typename TC, typename TN, typename TA, int OUT>
static long long launch_sweep(const GridGeo& g, const TC* coeff, ZLink<TC> cl, const TN* u, ZLink<TN> ul, const TN* f,
                              TN* y, float* r32, double* partials, cudaStream_t s) {
  const int tz = sweep_tz(g);
  const dim3 gr(g.n[0] / kSwTX, g.n[1] / kSwTY, g.n[2] / tz);
  constexpr size_t sm = sweep_smem<TN, TC>();
  // blocks per SM the register budget targets: f64 2 (128 regs) or 3 (85, knob SWEEP64_MINB); f32 3
  constexpr int minb = sizeof(TA) == 8 ? 2 : 3;
  static bool attr = false;  // per instantiation
  if (!attr) {
    IHOM_CUDA(cudaFuncSetAttribute((const void*)l0_sweep_kernel<TC, TN, TA, OUT, minb>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    IHOM_CUDA(cudaFuncSetAttribute((const void*)l0_sweep_kernel<TC, TN, TA, OUT, 3>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  if (sizeof(TA) == 8 && knob("SWEEP64_MINB", 2) >= 3)
    l0_sweep_kernel<TC, TN, TA, OUT, 3><<<gr, dim3(kSwTX, kSwTY), sm, s>>>(g, coeff, cl, u, ul, f, y, r32, partials, tz);
  else
    l0_sweep_kernel<TC, TN, TA, OUT, minb><<<gr, dim3(kSwTX, kSwTY), sm, s>>>(g, coeff, cl, u, ul, f, y, r32, partials,
                                                                             tz);
  IHOM_LAUNCH_CHECK();
  return (long long)gr.x * gr.y * gr.z;
}

template <typename TC, typename TN, typename TA>
void launch_l0_apply_sweep(const GridGeo& g, const TC* coeff, ZLink<TC> cl, const TN* u, ZLink<TN> ul, const TN* f,
                           TN* y, cudaStream_t s) {
  if constexpr (std::is_same_v<TC, float> && std::is_same_v<TN, float> && std::is_same_v<TA, float>) {
    if (sweep2_ok(g) && !hsweep_ok(g, true)) {
      const long long cols = (long long)(g.n[0] / (2 * kSwTX)) * (g.n[1] / kSwTY);
      int tz = g.n[2];
      while (tz % 4 == 0 && tz > 8 && cols * (g.n[2] / tz) < 148LL * 2 * 4) tz /= 2;  // stays even
      const dim3 gr(g.n[0] / (2 * kSwTX), g.n[1] / kSwTY, g.n[2] / tz);
      static bool attr = false;
      if (!attr) {
        IHOM_CUDA(cudaFuncSetAttribute((const void*)l0_sweep2_kernel<kSwResidual>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kS2Smem));
        IHOM_CUDA(cudaFuncSetAttribute((const void*)l0_sweep2_kernel<kSwApply>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kS2Smem));
        attr = true;
      }
      if (f) l0_sweep2_kernel<kSwResidual><<<gr, dim3(kSwTX, kSwTY), kS2Smem, s>>>(g, coeff, cl, u, ul, f, y, tz);
      else l0_sweep2_kernel<kSwApply><<<gr, dim3(kSwTX, kSwTY), kS2Smem, s>>>(g, coeff, cl, u, ul, f, y, tz);
      IHOM_LAUNCH_CHECK();
      return;
    }
  }
  if constexpr (std::is_same_v<TN, TA>) {
    if (hsweep_ok(g, sizeof(TN) == 4)) {
      if (f) launch_hsweep<TC, TN, kSwResidual, false>(g, coeff, cl, u, ul, f, y, nullptr, nullptr, nullptr, {}, nullptr, s);
      else launch_hsweep<TC, TN, kSwApply, false>(g, coeff, cl, u, ul, f, y, nullptr, nullptr, nullptr, {}, nullptr, s);
      return;
    }
  }
  if (f) launch_sweep<TC, TN, TA, kSwResidual>(g, coeff, cl, u, ul, f, y, nullptr, nullptr, s);
  else launch_sweep<TC, TN, TA, kSwApply>(g, coeff, cl, u, ul, f, y, nullptr, nullptr, s);
}

long long launch_l0_defect_sweep(const GridGeo& g, const float* coeff, ZLink<float> cl, const double* u,
                                 ZLink<double> ul, const double* f, float* r32, double* partials, cudaStream_t s) {
  if (hsweep_ok(g, false))
    return launch_hsweep<float, double, kSwDefect, false>(g, coeff, cl, u, ul, f, nullptr, r32, partials, nullptr, {},
                                                          nullptr, s);
  return launch_sweep<float, double, double, kSwDefect>(g, coeff, cl, u, ul, f, nullptr, r32, partials, s);
}

long long launch_l0_defect_update_sweep(const GridGeo& g, const float* coeff, ZLink<float> cl, const double* u,
                                        ZLink<double> ul, const float* e, ZLink<float> el, double* unew,
                                        const double* f, float* r32, double* partials, cudaStream_t s) {
  if (hsweep_ok(g, false))
    return launch_hsweep<float, double, kSwDefect, true>(g, coeff, resolve(cl, coeff), u, resolve(ul, u), f, nullptr,
                                                         r32, partials, e, resolve(el, e), unew, s);
  const int tz = sweep_tz(g);
  const dim3 gr(g.n[0] / kSwTX, g.n[1] / kSwTY, g.n[2] / tz);
  constexpr size_t sm = sweep_smem<double, float>() + sizeof(float) * kSwURing * kSwUSlot;
  static bool attr = false;
  if (!attr) {
    IHOM_CUDA(cudaFuncSetAttribute((const void*)l0_sweep_kernel<float, double, double, kSwDefect, 2, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  l0_sweep_kernel<float, double, double, kSwDefect, 2, true><<<gr, dim3(kSwTX, kSwTY), sm, s>>>(
      g, coeff, resolve(cl, coeff), u, resolve(ul, u), f, nullptr, r32, partials, tz, e, resolve(el, e), unew);
  IHOM_LAUNCH_CHECK();
  return (long long)gr.x * gr.y * gr.z;
}

template void launch_l0_apply_sweep<float, double, double>(const GridGeo&, const float*, ZLink<float>, const double*,
                                                           ZLink<double>, const double*, double*, cudaStream_t);
template void launch_l0_apply_sweep<double, double, double>(const GridGeo&, const double*, ZLink<double>,
                                                            const double*, ZLink<double>, const double*, double*,
                                                            cudaStream_t);
template void launch_l0_apply_sweep<float, float, float>(const GridGeo&, const float*, ZLink<float>, const float*,
                                                         ZLink<float>, const float*, float*, cudaStream_t);

}  // namespace ihomgpu
