// common.cuh -- shared device/host definitions for the B200 homogenization path.
//
// Layout contract (bit-exact with the reference, inc/grid.hpp:73-78):
//   * vertex storage is colour-major: 8 parity classes, each a dense
//     [hz][hy][hx] block of halved coordinates, x fastest;
//   * nodal fields are AoS (the reference's NodalField, inc/fem.hpp:15-26):
//     comp c of vertex loc at p[3*loc + c] -- one address per neighbour, the
//     three components at immediate offsets;
//   * element fields are x-fastest, eidx = x + n0*(y + n1*z);
//   * coarse stencils are blocked SoA [nv/32][243][32] in T (f32 mixed / f64
//     all-double): entry k = 9*n + 3*r + c of vertex loc at st_index(k, loc),
//     so a warp's 243 coefficient streams form one contiguous block
//     (n = 27-neighbour index x-fastest, inc/fem.hpp:30-35).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace ihomgpu {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::logic_error {
  using std::logic_error::logic_error;
};

#define IHOM_CUDA(call)                                                                         \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      throw ::ihomgpu::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + \
                                 __FILE__ + ":" + std::to_string(__LINE__));                   \
  } while (0)

// Every kernel launch is followed by IHOM_LAUNCH_CHECK(); it also counts launches
// (reported to the bench as gpu_launches).
inline long long& launch_counter() {
  static long long c = 0;
  return c;
}
#define IHOM_LAUNCH_CHECK()           \
  do {                                \
    ++::ihomgpu::launch_counter();    \
    IHOM_CUDA(cudaGetLastError());    \
  } while (0)

// Kernel-variant knobs (measurement / A-B switches, never numerics-changing unless
// documented): the value is the environment variable IHOM_<NAME> when set, else
// the default; ihom_set_knob() overrides it at run time (tests flip variants
// in-process to prove bit-identity). Defined in knobs.cpp.
int knob(const char* name, int dflt);
void set_knob(const char* name, int value);

// Geometry of one periodic grid level (inc/grid.hpp:18-56), passed by value.
struct GridGeo {
  int n[3];
  int cd[8][3];        // colour block dims (n_k - o_k + 1) / 2
  long long base[8];   // colour block base
  long long size[8];   // colour block size
  long long nv;        // vertex count == element count
};

inline GridGeo make_geo(int nx, int ny, int nz) {
  GridGeo g{};
  g.n[0] = nx;
  g.n[1] = ny;
  g.n[2] = nz;
  long long b = 0;
  for (int id = 0; id < 8; ++id) {
    const int o[3] = {id & 1, (id >> 1) & 1, (id >> 2) & 1};
    for (int k = 0; k < 3; ++k) g.cd[id][k] = (g.n[k] - o[k] + 1) / 2;
    g.base[id] = b;
    g.size[id] = (long long)g.cd[id][0] * g.cd[id][1] * g.cd[id][2];
    b += g.size[id];
  }
  g.nv = b;
  return g;
}

__host__ __device__ inline int color_of(int x, int y, int z) { return (x & 1) | ((y & 1) << 1) | ((z & 1) << 2); }

// color_block_location for canonical coordinates (inc/grid.hpp:73-78).
__host__ __device__ inline unsigned vloc(const GridGeo& g, int x, int y, int z) {
  const int id = color_of(x, y, z);
  return (unsigned)(g.base[id] + (x >> 1) + ((long long)(y >> 1) + (long long)(z >> 1) * g.cd[id][1]) * g.cd[id][0]);
}

// Coordinates of the i-th vertex of colour block `color` (inverse of vloc within a block).
__host__ __device__ inline void block_coords(const GridGeo& g, int color, unsigned i, int& x, int& y, int& z) {
  const unsigned d0 = (unsigned)g.cd[color][0], d1 = (unsigned)g.cd[color][1];
  const unsigned hx = i % d0;
  const unsigned t = i / d0;
  const unsigned hy = t % d1, hz = t / d1;
  x = 2 * (int)hx + (color & 1);
  y = 2 * (int)hy + ((color >> 1) & 1);
  z = 2 * (int)hz + ((color >> 2) & 1);
}

// Colour of location loc (inc/grid.hpp:81-92 colour search).
__host__ __device__ inline int color_at(const GridGeo& g, long long loc) {
  int id = 7;
  while (id > 0 && loc < g.base[id]) --id;
  return id;
}

__host__ __device__ inline unsigned eidx(const GridGeo& g, int x, int y, int z) {
  return (unsigned)(x + (long long)g.n[0] * (y + (long long)g.n[1] * z));
}

// gather_neighborhood (src/fem.cpp:37-68): 27 neighbour locations (x fastest,
// 13 = self) and the 8 incident element indices (v - 1 + bits(ke)).
struct Nbhd {
  unsigned v[27];
  unsigned e[8];
};

__device__ __forceinline__ void gather27(const GridGeo& g, int x, int y, int z, Nbhd& nb) {
  int par[3][3], half[3][3], ec[3][2];
  const int c[3] = {x, y, z};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int n = g.n[k], v = c[k];
    const int vm = (v == 0) ? n - 1 : v - 1;
    const int vp = (v + 1 == n) ? 0 : v + 1;
    par[k][0] = vm & 1;
    par[k][1] = v & 1;
    par[k][2] = vp & 1;
    half[k][0] = vm >> 1;
    half[k][1] = v >> 1;
    half[k][2] = vp >> 1;
    ec[k][0] = vm;
    ec[k][1] = v;
  }
#pragma unroll
  for (int t2 = 0; t2 < 3; ++t2)
#pragma unroll
    for (int t1 = 0; t1 < 3; ++t1)
#pragma unroll
      for (int t0 = 0; t0 < 3; ++t0) {
        const int id = par[0][t0] | (par[1][t1] << 1) | (par[2][t2] << 2);
        nb.v[t0 + 3 * t1 + 9 * t2] =
            (unsigned)(g.base[id] + half[0][t0] + (long long)(half[1][t1] + half[2][t2] * g.cd[id][1]) * g.cd[id][0]);
      }
#pragma unroll
  for (int ke = 0; ke < 8; ++ke)
    nb.e[ke] = (unsigned)(ec[0][ke & 1] + g.n[0] * (ec[1][(ke >> 1) & 1] + g.n[1] * ec[2][(ke >> 2) & 1]));
}

// 27-neighbour index of pair (ke, j): offset de + dj - 1 (src/fem.cpp:18-21).
// Zero-start Gauss-Seidel: in the first forward sweep from u = 0, a vertex of
// colour c only sees non-zero values in neighbours of colours < c (already
// updated this sweep); bit n is set for the 27-neighbours of colour > c.
__host__ __device__ constexpr unsigned zero_start_mask(int c) {
  unsigned m = 0u;
  for (int n = 0; n < 27; ++n) {
    const int mk = (n % 3 != 1 ? 1 : 0) | ((n / 3) % 3 != 1 ? 2 : 0) | (n / 9 != 1 ? 4 : 0);
    if ((c ^ mk) > c) m |= 1u << n;
  }
  return m;
}

__host__ __device__ constexpr int pair_ngb(int ke, int j) {
  return ((ke & 1) + (j & 1)) + 3 * (((ke >> 1) & 1) + ((j >> 1) & 1)) + 9 * (((ke >> 2) & 1) + ((j >> 2) & 1));
}

// Partial-pivoting 3x3 solve, src/fem.cpp:72-94: same elimination order and
// pivot choice (first strictly larger |a| wins), written with register row
// swaps instead of an index array so nothing spills to local memory.
template <typename R>
__device__ __forceinline__ void swap_rows(R* a, R* b, R& ra, R& rb, bool doit) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const R t = a[k];
    a[k] = doit ? b[k] : a[k];
    b[k] = doit ? t : b[k];
  }
  const R t = ra;
  ra = doit ? rb : ra;
  rb = doit ? t : rb;
}

// Symmetric positive definite 3x3 solve by the adjugate (one reciprocal, no pivoting or branches): the
// self block S of a vertex is a sum of q-weighted diagonal 3x3 blocks of K0, symmetric bit for bit (both
// triangles are merged by the same operations) and SPD. Used by the level-0 GS (f32 inner cycle and f64
// nodal data), where the partial-pivot solve3 (6 IEEE divisions, pivot selects) was ~15% of the f32
// pass's instructions and more of the f64 one (f64 division is a multi-instruction sequence).
template <typename R>
__device__ __forceinline__ void solve3_spd(const R m[9], const R rhs[3], R out[3]) {
  const R a = m[0], b = m[1], c = m[2], d = m[4], e = m[5], f = m[8];
  const R A = fma(d, f, -e * e), B = fma(c, e, -b * f), C = fma(b, e, -c * d);
  const R D = fma(a, f, -c * c), E = fma(b, c, -a * e), F = fma(a, d, -b * b);
  const R r = R(1) / fma(a, A, fma(b, B, c * C));
  out[0] = fma(A, rhs[0], fma(B, rhs[1], C * rhs[2])) * r;
  out[1] = fma(B, rhs[0], fma(D, rhs[1], E * rhs[2])) * r;
  out[2] = fma(C, rhs[0], fma(E, rhs[1], F * rhs[2])) * r;
}

template <typename R>
__device__ __forceinline__ void solve3(const R m[9], const R rhs[3], R out[3]) {
  R r0[3] = {m[0], m[1], m[2]}, r1[3] = {m[3], m[4], m[5]}, r2[3] = {m[6], m[7], m[8]};
  R b0 = rhs[0], b1 = rhs[1], b2 = rhs[2];
  {  // column 0: pivot row = first strictly largest |a_r0| (swap(piv[0], piv[best]))
    const bool s1 = fabs(r1[0]) > fabs(r0[0]);
    const bool s2 = fabs(r2[0]) > (s1 ? fabs(r1[0]) : fabs(r0[0]));
    swap_rows(r0, r2, b0, b2, s2);
    swap_rows(r0, r1, b0, b1, s1 && !s2);
  }
  {
    const R f1 = r1[0] / r0[0];
#pragma unroll
    for (int k = 0; k < 3; ++k) r1[k] -= f1 * r0[k];
    b1 -= f1 * b0;
    const R f2 = r2[0] / r0[0];
#pragma unroll
    for (int k = 0; k < 3; ++k) r2[k] -= f2 * r0[k];
    b2 -= f2 * b0;
  }
  swap_rows(r1, r2, b1, b2, fabs(r2[1]) > fabs(r1[1]));
  {
    const R f2 = r2[1] / r1[1];
#pragma unroll
    for (int k = 1; k < 3; ++k) r2[k] -= f2 * r1[k];
    b2 -= f2 * b1;
  }
  out[2] = b2 / r2[2];
  out[1] = (b1 - r1[2] * out[2]) / r1[1];
  out[0] = (b0 - r0[1] * out[1] - r0[2] * out[2]) / r0[0];
}

__host__ __device__ __forceinline__ size_t st_index(int k, unsigned loc) {
  return ((size_t)(loc >> 5) * 243 + (size_t)k) * 32 + (loc & 31u);
}
inline size_t stencil_alloc(long long nv) { return (size_t)((nv + 31) / 32) * 32 * 243; }

// On every smoothed level all n_k are even, so the 8 colour blocks share dims
// d_k = n_k/2 and size B = d0 d1 d2 (base[c] = c B). For a vertex of colour
// o = (o0,o1,o2) at halved (h0,h1,h2), neighbour t has location
//   loc(t) = A0[t0] + A1[t1] + A2[t2],
//   A_k[t] = ((o_k ^ (t != 0)) << k) B + s_k * half_k(t),
// half_k(0) = h_k, half_k(-1) = o_k ? h_k : h_k - 1 (wrapped), half_k(+1) = o_k ? h_k + 1 (wrapped) : h_k,
// s = (1, d0, d0 d1). One IADD3 per neighbour; AoS nodal data then gives the three
// components at immediate offsets. Incident elements likewise: e = E0[a] + E1[b] + E2[c].
struct FastAddr {
  unsigned A[3][3];  // [axis][t+1]
  unsigned E[3][2];  // [axis][bit]: element coordinate x-1 (bit 0) or x (bit 1), pre-scaled
  bool zlo, zhi;     // the t2 = -1 / +1 neighbour plane (and, for zlo, the z-1 element plane) wraps
};

// z-slab neighbours of one array. A slab's grid is periodic in x
// and y; in z, reads that wrap through its lower / upper face go to the same
// array of the slab below / above, at the wrapped index (every slab has the
// same local layout, so the wrapped plane of the local layout IS the
// neighbour's boundary plane). The peer array is another slab's buffer on the
// same device or peer memory mapped over NVLink. A periodic single-slab grid
// links every array to itself, which is exactly the old wrap.
template <typename X>
struct ZLink {
  const X* lo = nullptr;
  const X* hi = nullptr;
};
template <typename X>
inline ZLink<X> resolve(ZLink<X> l, const X* self) {
  if (!l.lo) l.lo = self;
  if (!l.hi) l.hi = self;
  return l;
}
template <typename X>
inline bool is_self(const ZLink<X>& l, const X* self) {
  return (!l.lo || l.lo == self) && (!l.hi || l.hi == self);
}

__device__ __forceinline__ void fast_addr(const GridGeo& g, int color, int h0, int h1, int h2, FastAddr& fa) {
  const unsigned B = (unsigned)g.size[0];
  const int h[3] = {h0, h1, h2};
  const unsigned d[3] = {(unsigned)g.cd[0][0], (unsigned)g.cd[0][1], (unsigned)g.cd[0][2]};
  const unsigned sc[3] = {1u, d[0], d[0] * d[1]};
  const unsigned es[3] = {1u, (unsigned)g.n[0], (unsigned)g.n[0] * (unsigned)g.n[1]};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int o = (color >> k) & 1;
    const unsigned hm = o ? (unsigned)h[k] : (h[k] == 0 ? d[k] - 1 : (unsigned)h[k] - 1);
    const unsigned hp = o ? ((unsigned)h[k] + 1 == d[k] ? 0u : (unsigned)h[k] + 1) : (unsigned)h[k];
    const unsigned same = ((unsigned)o << k) * B, other = ((unsigned)(o ^ 1) << k) * B;
    fa.A[k][0] = other + sc[k] * hm;
    fa.A[k][1] = same + sc[k] * (unsigned)h[k];
    fa.A[k][2] = other + sc[k] * hp;
    const int x = 2 * h[k] + o, nk = g.n[k];
    fa.E[k][0] = es[k] * (unsigned)(x == 0 ? nk - 1 : x - 1);
    fa.E[k][1] = es[k] * (unsigned)x;
  }
  const int o2 = (color >> 2) & 1;
  fa.zlo = o2 == 0 && h2 == 0;
  fa.zhi = o2 == 1 && (unsigned)h2 + 1 == d[2];
}

// Base pointer of neighbour plane t2 (0, 1, 2 = z-1, z, z+1) under a z link.
template <typename X>
__device__ __forceinline__ const X* zbase(const FastAddr& fa, const X* self, const ZLink<X>& zl, int t2) {
  return t2 == 0 ? (fa.zlo ? zl.lo : self) : (t2 == 2 ? (fa.zhi ? zl.hi : self) : self);
}

inline bool fast_ok(const GridGeo& g) {
  return g.n[0] % 2 == 0 && g.n[1] % 2 == 0 && g.n[2] % 2 == 0 && g.n[0] >= 8;
}
inline dim3 fast_block(const GridGeo& g) {
  const int d0 = g.cd[0][0];
  const int bx = d0 >= 32 ? 32 : (d0 >= 16 ? 16 : (d0 >= 8 ? 8 : 4));
  return dim3(bx, 128 / bx, 1);
}

inline unsigned ceil_div(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

}  // namespace ihomgpu
