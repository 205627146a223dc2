// hom_kernels.cu -- homogenized tensor and its density sensitivity
// (src/homogenization.cpp:58-144).
//
// Per element the 21 energies E_ij = d_i^T K0 d_j (d_i = chi^i - u^i) are
// evaluated through the quadrature that defines K0 (src/material.cpp:39-69):
// K0 = sum_g w B_g^T C B_g with 2x2x2 Gauss points, so
//   E_ij = sum_g w (e_i - eps(u^i)_g)^T C (e_j - eps(u^j)_g),
// where e_i is the unit engineering strain of the element-relative chi^i
// (src/material.cpp:71-82). Gradients of the trilinear field are formed by
// sum factorisation from nodal differences (d/dx is constant along x), which
// costs ~2.7k flop/element instead of the 3.5k+ of the dense 24x24x6 product.
// Mixed mode reads u through a float snapshot (src/homogenization.cpp:84-85).
#include "kernels.hpp"
#include "hada_gen.cuh"
#include "bulk.cuh"

#include <algorithm>
#include <type_traits>

namespace ihomgpu {

constexpr int kHT = 64;            // threads (elements) per block
constexpr int kGradPerLoad = 36;   // 3 comps x 3 directions x 4 points

__device__ __forceinline__ int wrapp(int c, int n) { return c >= n ? c - n : c; }

// Locations of the 8 corners of element (ex, ey, ez) (x fastest), periodic wrap.
__device__ __forceinline__ void corner_locs(const GridGeo& g, int ex, int ey, int ez, unsigned loc[8]) {
  if (g.n[0] % 2 == 0 && g.n[1] % 2 == 0 && g.n[2] % 2 == 0) {
    // even grid: every colour block has the same dims, so a corner's location is a sum of one
    // per-axis term (colour bit folded in): 6 small tables instead of 8 generic vloc() calls
    const unsigned B = (unsigned)g.size[0], d0 = (unsigned)g.cd[0][0], d01 = d0 * (unsigned)g.cd[0][1];
    unsigned A[3][2];
    const int e3[3] = {ex, ey, ez};
    const unsigned st[3] = {1u, d0, d01};
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int c = wrapp(e3[k] + b, g.n[k]);
        A[k][b] = (unsigned)((c & 1) << k) * B + (unsigned)(c >> 1) * st[k];
      }
#pragma unroll
    for (int j = 0; j < 8; ++j) loc[j] = A[0][j & 1] + A[1][(j >> 1) & 1] + A[2][(j >> 2) & 1];
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      loc[j] = vloc(g, wrapp(ex + (j & 1), g.n[0]), wrapp(ey + ((j >> 1) & 1), g.n[1]), wrapp(ez + ((j >> 2) & 1), g.n[2]));
  }
}

// Computes the 21 upper-triangle energies for element (ex,ey,ez) in arithmetic
// type TE (f64 all-double; f32 in mixed mode, where u is read through the
// reference's f32 snapshot anyway). gs: per-thread smem slice, stride kHT.
// z-slab: the upper vertex plane of the top element layer belongs to the slab
// above (uhi).
template <typename TN, typename TE>
__device__ void element_energies(const GridGeo& g, int ex, int ey, int ez, const TN* const* u, const TN* const* uhi,
                                 bool snap, TE lam, TE mu, TE* gs, TE E[21]) {
  const TE p1 = TE(0.5 + 0.5 / 1.7320508075688772);  // gp[1]; N_a(g) = (a == g) ? p1 : p0
  const TE p0 = TE(0.5 - 0.5 / 1.7320508075688772);
  unsigned loc[8];
  corner_locs(g, ex, ey, ez, loc);
  const bool top = ez + 1 == g.n[2];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const TN* ui = u[i];
    const TN* uz = top ? uhi[i] : u[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      TE U[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double v = double(((j >> 2) & 1 ? uz : ui)[3 * (size_t)loc[j] + c]);
        U[j] = snap ? TE(float(v)) : TE(v);
      }
      // direction k: differences across k at the 4 corners of the other two axes (a,b),
      // then bilinear interpolation to the 4 Gauss points (ga, gb).
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int ka = (k + 1) % 3, kb = (k + 2) % 3;
        const int sk = 1 << k, sa = 1 << ka, sb = 1 << kb;
        TE D[2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int j0 = a * sa + b * sb;
            D[a][b] = U[j0 + sk] - U[j0];
          }
#pragma unroll
        for (int ga = 0; ga < 2; ++ga)
#pragma unroll
          for (int gb = 0; gb < 2; ++gb) {
            TE s = TE(0);
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int b = 0; b < 2; ++b) s += D[a][b] * (a == ga ? p1 : p0) * (b == gb ? p1 : p0);
            gs[(i * kGradPerLoad + (c * 3 + k) * 4 + ga * 2 + gb) * kHT] = s;
          }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 21; ++q) E[q] = TE(0);
  // grad(i, c, k, gx,gy,gz): the two "other" axes of k are (k+1)%3, (k+2)%3.
  auto G = [&](int i, int c, int k, const int gp[3]) {
    const int ga = gp[(k + 1) % 3], gb = gp[(k + 2) % 3];
    return gs[(i * kGradPerLoad + (c * 3 + k) * 4 + ga * 2 + gb) * kHT];
  };
  for (int gq = 0; gq < 8; ++gq) {
    const int gp[3] = {gq & 1, (gq >> 1) & 1, (gq >> 2) & 1};
    TE ed[6][6], sg[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      TE e[6];
      e[0] = -G(i, 0, 0, gp);
      e[1] = -G(i, 1, 1, gp);
      e[2] = -G(i, 2, 2, gp);
      e[3] = -(G(i, 0, 1, gp) + G(i, 1, 0, gp));
      e[4] = -(G(i, 1, 2, gp) + G(i, 2, 1, gp));
      e[5] = -(G(i, 0, 2, gp) + G(i, 2, 0, gp));
      e[i] += TE(1);  // strain of chi^i (engineering order 11,22,33,12,23,13)
      const TE tr = e[0] + e[1] + e[2];
#pragma unroll
      for (int v = 0; v < 6; ++v) ed[i][v] = e[v];
      sg[i][0] = lam * tr + TE(2) * mu * e[0];
      sg[i][1] = lam * tr + TE(2) * mu * e[1];
      sg[i][2] = lam * tr + TE(2) * mu * e[2];
      sg[i][3] = mu * e[3];
      sg[i][4] = mu * e[4];
      sg[i][5] = mu * e[5];
    }
    int q = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = i; j < 6; ++j, ++q) {
        TE s = TE(0);
#pragma unroll
        for (int v = 0; v < 6; ++v) s += ed[i][v] * sg[j][v];
        E[q] += TE(0.125) * s;
      }
  }
}

// ---------------------------------------------------------------- sum/difference-basis energies
// K0 = Hb^T W Hb with W = D/8 the 45-term element stiffness in the per-axis sum/difference basis
// (tools/gen_hada.py, hada_gen.cuh; Hb = per-component 8-point Walsh-Hadamard, H1 = [[1,1],[-1,1]]), so
//   E_ij = d_i^T K0 d_j = d_hat_i^T W d_hat_j,   d_hat = Hb (chi^i - u^i) = chi_hat^i - Hb u^i.
// Per element: 18 butterflies of 24 adds, 6 x 45 terms for W d_hat_j, 21 x 21-term dots (~1.2k flop,
// no shared memory) instead of the quadrature's ~2.7k flop and 864 B of gradients per thread.
// The all-sum entries (sigma = 0) drop out (W annihilates translations).
void upload_modal_tables(const double h[], cudaStream_t s);
__constant__ double c_hw_d[kHadaClasses];
__constant__ float c_hw_f[kHadaClasses];
__constant__ double c_chih_d[6][24];  // Hb chi^i, chi^i element-relative (src/material.cpp:71-82)
__constant__ float c_chih_f[6][24];

void upload_hom_tables(const double hada_classes[], cudaStream_t s) {
  static double wd[kHadaClasses], cd[6][24];
  static float wf[kHadaClasses], cf[6][24];
  for (int k = 0; k < kHadaClasses; ++k) wd[k] = hada_classes[k], wf[k] = float(wd[k]);
  for (int i = 0; i < 6; ++i)
    for (int sg = 0; sg < 8; ++sg)
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int a = 0; a < 8; ++a) {
          double chi[3];
          macro_strain_displacement(i, a & 1, (a >> 1) & 1, (a >> 2) & 1, chi);
          double h = 1.0;  // H1[s][a] = 1 for s = 0; -1 / +1 for s = 1 and a = 0 / 1, per axis
          for (int k = 0; k < 3; ++k)
            if ((sg >> k) & 1) h *= ((a >> k) & 1) ? 1.0 : -1.0;
          acc += h * chi[c];
        }
        cd[i][sg * 3 + c] = acc;
        cf[i][sg * 3 + c] = float(acc);
      }
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_hw_d, wd, sizeof(wd), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_hw_f, wf, sizeof(wf), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_chih_d, cd, sizeof(cd), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_chih_f, cf, sizeof(cf), 0, cudaMemcpyHostToDevice, s));
  // chi is linear in the corner coordinates, so beyond the all-sum entries 0-2 (never read: W annihilates them)
  // H chi lives on the single-bit sigmas 1, 2, 4 (entries 3-8, 12-14): the staged tensor pass keeps only those
  for (int i = 0; i < 6; ++i)
    for (int r = 3; r < 24; ++r)
      if (!((r >= 3 && r <= 8) || (r >= 12 && r <= 14)) && cd[i][r] != 0.0)
        throw std::logic_error("H chi has an entry off the single-bit sigmas");
  upload_modal_tables(hada_classes, s);
}

template <typename TE>
__device__ __forceinline__ TE hw_class(int k) {
  if constexpr (sizeof(TE) == 8) return c_hw_d[k];
  else return c_hw_f[k];
}
template <typename TE>
__device__ __forceinline__ TE chih(int i, int r) {
  if constexpr (sizeof(TE) == 8) return c_chih_d[i][r];
  else return c_chih_f[i][r];
}

template <typename TN, typename TE>
__device__ void element_energies_hada(const GridGeo& g, int ex, int ey, int ez, const TN* const* u,
                                      const TN* const* uhi, bool snap, TE E[21]) {
  unsigned loc[8];
  corner_locs(g, ex, ey, ez, loc);
  const bool top = ez + 1 == g.n[2];
  TE dh[6][24];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const TN* ui = u[i];
    const TN* uz = top ? uhi[i] : u[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      TE V[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double v = double(((j >> 2) & 1 ? uz : ui)[3 * (size_t)loc[j] + c]);
        V[j] = snap ? TE(float(v)) : TE(v);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k)  // in-place butterflies: slot bit k = sigma_k (0 sum, 1 difference)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (!((j >> k) & 1)) {
            const TE a = V[j], b = V[j | (1 << k)];
            V[j] = b + a;
            V[j | (1 << k)] = b - a;
          }
#pragma unroll
      for (int sg = 1; sg < 8; ++sg) dh[i][sg * 3 + c] = chih<TE>(i, sg * 3 + c) - V[sg];
      dh[i][c] = TE(0);  // all-sum entry: never read by W
    }
  }
  TE qh[kHadaClasses];
#pragma unroll
  for (int k = 0; k < kHadaClasses; ++k) qh[k] = hw_class<TE>(k);
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    TE t[24];
    hada_apply<TE>(qh, dh[j], t);
#pragma unroll
    for (int i = 0; i <= j; ++i) {
      TE acc = dh[i][3] * t[3];
#pragma unroll
      for (int r = 4; r < 24; ++r) acc = fma(dh[i][r], t[r], acc);
      E[i * 6 - i * (i - 1) / 2 + (j - i)] = acc;  // upper-triangle row-major (i <= j)
    }
  }
}

__device__ __forceinline__ double block_reduce_h(double v, double* sh) {
  const int t = threadIdx.x;
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
  return r;
}

struct U6 {
  const void* p[6];
  const void* hi[6];  // z-slab: the same fields of the slab above (== p for one periodic domain)
};

// ---------------------------------------------------------------- f64 energies, modal form, element pairs
// W (the 45-term element stiffness in the sum/difference basis, hada_gen.cuh) is block diagonal over the
// 21 non-sum entries: two 3x3 blocks a I + b 11^T ({3,7,14}: h0, h1; {11,16,18}: h5, h6), three 2x2 blocks
// [[h3,h4],[h4,h3]] ({9,20}, {10,17}, {15,19}), three rank-1 blocks h2 [[1,1],[1,1]] ({4,6}, {5,12},
// {8,13}: the rotations, K0's null space) and h7 on {21}, {22}, {23}. With orthonormal eigenvectors,
// W = sum_k l_k v_k v_k^T over 18 modes, so E_ij = d_hat_i^T W d_hat_j = sum_k b_ik b_jk with
// b_ik = sqrt(l_k) v_k . d_hat_i: 18 modal values per load case and a 21 x 18 Gram product.
// Two threads share an element (lanes 2k, 2k+1: load cases 0-2 and 3-5): each forms its three modal
// vectors (54 doubles, no spills), the Gram entries of its own cases, and the cross entries from the
// partner's vectors, exchanged mode by mode with shuffles. Arithmetic f64 throughout; u is rounded to
// f32 precision in mixed mode (the reference's float snapshot, src/homogenization.cpp:84-85) by integer
// round-to-nearest-even on the f64 bits (no conversion instructions; identical to double(float(u)) for
// |u| >= 2^-126).
__constant__ double c_mode[10];  // kP1 kP2 kP3 kQ1 kQ2 kQ3 kR1 kR2 kS kT

void upload_modal_tables(const double h[], cudaStream_t s) {
  double scale = 0.0;
  for (int k = 0; k < kHadaClasses; ++k) scale = std::fmax(scale, std::fabs(h[k]));
  auto root = [scale](double v) {  // eigenvalues of a PSD matrix: rounding-level negatives are zeros
    if (v < -1e-12 * scale) throw std::invalid_argument("element stiffness is not positive semi-definite");
    return v > 0.0 ? std::sqrt(v) : 0.0;
  };
  static double m[10];
  m[0] = root((h[0] + 2.0 * h[1]) / 3.0);
  m[1] = root((h[0] - h[1]) / 2.0);
  m[2] = root((h[0] - h[1]) / 6.0);
  m[3] = root((h[5] + 2.0 * h[6]) / 3.0);
  m[4] = root((h[5] - h[6]) / 2.0);
  m[5] = root((h[5] - h[6]) / 6.0);
  m[6] = root((h[3] + h[4]) / 2.0);
  m[7] = root((h[3] - h[4]) / 2.0);
  m[8] = root(h[2]);
  m[9] = root(h[7]);
  for (int k = 0; k < 10; ++k)
    if (!std::isfinite(m[k])) throw std::invalid_argument("element stiffness is not positive semi-definite");
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_mode, m, sizeof(m), 0, cudaMemcpyHostToDevice, s));
}

__device__ __forceinline__ double snap_f32_bits(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  b += 0x0FFFFFFFull + ((b >> 29) & 1ull);  // round to nearest even at mantissa bit 29
  return __longlong_as_double((long long)(b & ~0x1FFFFFFFull));
}

constexpr int kModes = 18;

// modal vector of one load case from its 8 corner displacements (AoS f64, loc[] / top-plane pointer)
// modal vector (18 values) of one load case from its sum/difference-basis displacement d_hat (entries 3..23)
__device__ __forceinline__ void modal_from_dhat(const double dh[24], double b[kModes]) {
  const double* m = c_mode;
  {  // {3,7,14}
    const double x = dh[3], y = dh[7], z = dh[14];
    b[0] = m[0] * (x + y + z);
    b[1] = m[1] * (x - y);
    b[2] = m[2] * (x + y - 2.0 * z);
  }
  {  // {11,16,18}
    const double x = dh[11], y = dh[16], z = dh[18];
    b[3] = m[3] * (x + y + z);
    b[4] = m[4] * (x - y);
    b[5] = m[5] * (x + y - 2.0 * z);
  }
  b[6] = m[6] * (dh[9] + dh[20]);
  b[7] = m[7] * (dh[9] - dh[20]);
  b[8] = m[6] * (dh[10] + dh[17]);
  b[9] = m[7] * (dh[10] - dh[17]);
  b[10] = m[6] * (dh[15] + dh[19]);
  b[11] = m[7] * (dh[15] - dh[19]);
  b[12] = m[8] * (dh[4] + dh[6]);
  b[13] = m[8] * (dh[5] + dh[12]);
  b[14] = m[8] * (dh[8] + dh[13]);
  b[15] = m[9] * dh[21];
  b[16] = m[9] * dh[22];
  b[17] = m[9] * dh[23];
}

// modal vector of one load case from its 8 corner displacements (AoS, loc[] / top-plane pointer). TU = float:
// the f32 snapshots of the host-staged mode (exactly the values SNAP rounds f64 fields to)
template <bool SNAP, typename TU = double>
__device__ __forceinline__ void modal_vector(const TU* __restrict__ ui, const TU* __restrict__ uz,
                                             const unsigned loc[8], int lc, double b[kModes]) {
  double dh[24];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double V[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double v = double(__ldg(((j >> 2) & 1 ? uz : ui) + 3 * (size_t)loc[j] + c));
      V[j] = SNAP ? snap_f32_bits(v) : v;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (!((j >> k) & 1)) {
          const double a = V[j], bb = V[j | (1 << k)];
          V[j] = bb + a;
          V[j | (1 << k)] = bb - a;
        }
#pragma unroll
    for (int sg = 1; sg < 8; ++sg) dh[sg * 3 + c] = c_chih_d[lc][sg * 3 + c] - V[sg];
  }
  modal_from_dhat(dh, b);
}

// Gram entries of a lane's three modal vectors (eo: 00 01 02 11 12 22) and the cross entries with the
// partner lane (lane ^ x): (own i, partner j) = (0,0) (1,1) (2,2) (0,1) (0,2) (1,2), exchanged mode by mode.
__device__ __forceinline__ void gram_pairs(const double b[3][kModes], int x, double eo[6], double ex[6]) {
#pragma unroll
  for (int q = 0; q < 6; ++q) eo[q] = 0.0, ex[q] = 0.0;
#pragma unroll
  for (int k = 0; k < kModes; ++k) {
    const double p0 = __shfl_xor_sync(0xffffffffu, b[0][k], x);
    const double p1 = __shfl_xor_sync(0xffffffffu, b[1][k], x);
    const double p2 = __shfl_xor_sync(0xffffffffu, b[2][k], x);
    eo[0] = fma(b[0][k], b[0][k], eo[0]);
    eo[1] = fma(b[0][k], b[1][k], eo[1]);
    eo[2] = fma(b[0][k], b[2][k], eo[2]);
    eo[3] = fma(b[1][k], b[1][k], eo[3]);
    eo[4] = fma(b[1][k], b[2][k], eo[4]);
    eo[5] = fma(b[2][k], b[2][k], eo[5]);
    ex[0] = fma(b[0][k], p0, ex[0]);
    ex[1] = fma(b[1][k], p1, ex[1]);
    ex[2] = fma(b[2][k], p2, ex[2]);
    ex[3] = fma(b[0][k], p1, ex[3]);
    ex[4] = fma(b[0][k], p2, ex[4]);
    ex[5] = fma(b[1][k], p2, ex[5]);
  }
}

// Energies of one element shared by a lane pair. Lane role r = lane & 1 owns load cases 3r..3r+2.
// Out: eo[6] Gram entries of the own cases (00 01 02 11 12 22 in local indices), ex[6] cross entries
// (local own i, partner j): (0,0) (1,1) (2,2) (0,1) (0,2) (1,2). The even lane's cross entries are
// (i, 3+j); the odd lane's upper ones are (j, 3+i) with j < i... see energy_index().
template <bool SNAP, typename TU = double>
__device__ __forceinline__ void pair_energies(const U6& uu, const unsigned loc[8], bool top, int role, double eo[6],
                                              double ex[6]) {
  double b[3][kModes];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const TU* ui = static_cast<const TU*>(role ? uu.p[3 + a] : uu.p[a]);
    const TU* uz = top ? static_cast<const TU*>(role ? uu.hi[3 + a] : uu.hi[a]) : ui;
    modal_vector<SNAP, TU>(ui, uz, loc, 3 * role + a, b[a]);
  }
  gram_pairs(b, 1, eo, ex);
}


// Upper-triangle index (i <= j, row-major) of the 21 energies.
__host__ __device__ __forceinline__ constexpr int tri(int i, int j) { return i * 6 - i * (i - 1) / 2 + (j - i); }

// Energy index of slot m (0-5 own, 6-11 cross) for a lane role; -1: not stored by this lane
// (the odd lane's copies of the diagonal cross entries).
__host__ __device__ __forceinline__ constexpr int energy_index(int role, int m) {
  // own slots: (0,0) (0,1) (0,2) (1,1) (1,2) (2,2); cross slots: (0,0) (1,1) (2,2) (0,1) (0,2) (1,2)
  // as (own local i, partner local j)
  const int oi = m == 0 || m == 1 || m == 2 ? 0 : (m == 3 || m == 4 ? 1 : 2);
  const int oj = m == 0 ? 0 : (m == 1 || m == 3 ? 1 : 2);
  const int xi = m == 6 || m == 9 || m == 10 ? 0 : (m == 7 || m == 11 ? 1 : 2);
  const int xj = m == 6 ? 0 : (m == 7 || m == 9 ? 1 : 2);
  return m < 6 ? tri(3 * role + oi, 3 * role + oj)
               : (role == 0 ? tri(xi, 3 + xj)              // even lane: (i, 3+j)
                            : (xi == xj ? -1 : tri(xj, 3 + xi)));  // odd lane: own 3+i, partner j: (j, 3+i)
}

// Element ordering shared by the pair kernels: a block of 128 threads owns a 32 x 2 element column tile
// (x % 32 == 0, y % 2 == 0 grids) and marches up z; else grid-stride over elements. 2 lanes per element.
constexpr int kPT = 128;

template <bool SNAP, typename TU = double>
__global__ void __launch_bounds__(kPT) tensor_pair_kernel(GridGeo g, U6 uu, const double* __restrict__ rho,
                                                          double penal, double* partials, double* __restrict__ ecache) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, role = lane & 1;
  const int slot = (threadIdx.x >> 5) * 16 + (lane >> 1);  // element slot 0..63 of the block
  int eidx[12];
#pragma unroll
  for (int m = 0; m < 12; ++m) eidx[m] = energy_index(role, m);
  double acc[12];
#pragma unroll
  for (int m = 0; m < 12; ++m) acc[m] = 0.0;
  const bool cols = g.n[0] % 32 == 0 && g.n[1] % 2 == 0;
  const long long tiles_x = g.n[0] / 32, ntiles = cols ? tiles_x * (g.n[1] / 2) : 0;
  const long long nsteps = cols ? ((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * g.n[2]
                                : (g.nv - blockIdx.x * 64 + (long long)gridDim.x * 64 - 1) / ((long long)gridDim.x * 64);
  for (long long it = 0; it < nsteps; ++it) {
    int ex, ey, ez;
    long long e;
    bool valid = true;
    if (cols) {
      const long long tile = blockIdx.x + (it / g.n[2]) * gridDim.x;
      ez = int(it % g.n[2]);
      ex = int(tile % tiles_x) * 32 + (slot & 31);
      ey = int(tile / tiles_x) * 2 + (slot >> 5);
      e = ex + (long long)g.n[0] * (ey + (long long)g.n[1] * ez);
    } else {
      e = (long long)blockIdx.x * 64 + slot + it * (long long)gridDim.x * 64;
      valid = e < g.nv;
      const long long ee = valid ? e : 0;  // both lanes of a pair agree; whole pairs idle together
      ex = int(ee % g.n[0]);
      const long long r = ee / g.n[0];
      ey = int(r % g.n[1]);
      ez = int(r / g.n[1]);
    }
    unsigned loc[8];
    corner_locs(g, ex, ey, ez, loc);
    double E[12];
    pair_energies<SNAP, TU>(uu, loc, ez + 1 == g.n[2], role, E, E + 6);
    if (!valid) continue;
    if (ecache) {  // [21][nv]
#pragma unroll
      for (int m = 0; m < 12; ++m)
        if (eidx[m] >= 0) ecache[eidx[m] * g.nv + e] = E[m];
    }
    const double q = penal == 1.0 ? rho[e] : pow(rho[e], penal);  // src/homogenization.cpp:91
#pragma unroll
    for (int m = 0; m < 12; ++m) acc[m] = fma(q, E[m], acc[m]);
  }
  // block sums of the 21 entries (fixed partition and order: deterministic)
  for (int k = 0; k < 21; ++k) {
    double v = 0.0;
#pragma unroll
    for (int m = 0; m < 12; ++m) v += eidx[m] == k ? acc[m] : 0.0;
    const double r = block_reduce_h(v, sh);
    if (threadIdx.x == 0) partials[k * kReducePartials + blockIdx.x] = r;
  }
}

// Sensitivity with the pair energies (no cache): the odd lane hands its 9 stored energies to the even
// lane, which forms sum_ij s_ij E_ij in the cached kernel's order (bit-identical to sens_cached_kernel).
template <bool SNAP, typename TU = double>
__global__ void __launch_bounds__(kPT) sens_pair_kernel(GridGeo g, U6 uu, const double* __restrict__ rho, double penal,
                                                        const double* __restrict__ seed, double inv_m,
                                                        double* __restrict__ out) {
  const int role = threadIdx.x & 1;
  const long long e = ((long long)blockIdx.x * kPT + threadIdx.x) >> 1;
  const bool valid = e < g.nv;
  const long long ee = valid ? e : 0;
  const int ex = int(ee % g.n[0]);
  const long long r = ee / g.n[0];
  const int ey = int(r % g.n[1]), ez = int(r / g.n[1]);
  unsigned loc[8];
  corner_locs(g, ex, ey, ez, loc);
  double E[12];
  pair_energies<SNAP, TU>(uu, loc, ez + 1 == g.n[2], role, E, E + 6);
  double all[21];
#pragma unroll
  for (int m = 0; m < 12; ++m) {
    const double other = __shfl_xor_sync(0xffffffffu, E[m], 1);
    const int k0 = energy_index(0, m), k1 = energy_index(1, m);
    all[k0] = E[m];
    if (k1 >= 0) all[k1] = other;
  }
  if (!valid || role) return;
  double acc = 0.0;  // sum_ij s_ij E_ij, s symmetric (src/homogenization.cpp:120,138-140)
  int q = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i; j < 6; ++j, ++q) acc += (i == j ? 1.0 : 2.0) * seed[i * 6 + j] * all[q];
  out[e] = penal * (penal == 1.0 ? 1.0 : pow(rho[e], penal - 1.0)) * acc * inv_m;
}

// ---------------------------------------------------------------- staged pair tensor pass (bulk copies)
// Same energies as tensor_pair_kernel, for grids with n0 % 32 == 0 and n1 % 2 == 0 (the column tiles):
// a block owns a 32 x 2 element column and marches up z; the six displacement fields of each vertex plane
// of the tile (33 x 3 vertices) are moved into a 3-slot shared-memory ring by the TMA engine
// (cp.async.bulk, 54 contiguous runs per plane, completion counted on one mbarrier per slot), two planes
// ahead of the compute. The corner loads become conflict-free LDS at immediate offsets; in mixed mode each
// staged value is rounded to f32 precision once (not once per incident element). Lanes 0-15 own load
// cases 0-2 of elements 0-15, lanes 16-31 cases 3-5 (partner = lane ^ 16).
// Slot layout (doubles): field f at f*kStFS, row r at r*kStRS, even-x run (17 vertices, the 17th by its
// own 32-byte copy) at 0, odd-x run (16 vertices) at kStP1; vertex k at 3k.
constexpr int kStFS = 312, kStRS = 104, kStP1 = 56, kStPlane = 6 * kStFS;
constexpr uint32_t kStBytes = 6 * 3 * (384 + 32 + 384);
constexpr size_t kStSmem = sizeof(double) * 3 * kStPlane + 3 * sizeof(uint64_t);

bool tensor_stage_ok(const GridGeo& g, const void* const* p, const void* const* hi) {
  if (g.n[0] % 32 || g.n[1] % 2 || g.n[2] % 2 || g.n[2] < 2) return false;
  for (int i = 0; i < 6; ++i)
    if ((reinterpret_cast<uintptr_t>(p[i]) & 15) || (reinterpret_cast<uintptr_t>(hi[i]) & 15)) return false;
  return true;
}

template <bool SNAP>
__global__ void __launch_bounds__(kPT, 3) tensor_stage_kernel(GridGeo g, U6 uu, const double* __restrict__ rho,
                                                           double penal, double* partials,
                                                           double* __restrict__ ecache) {
  extern __shared__ __align__(128) unsigned char st_raw[];
  double* ring = reinterpret_cast<double*>(st_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + 3 * kStPlane);
  __shared__ double chs[6][9];  // chi_hat entries 3-8 and 12-14 (sigma 1, 2, 4); every other entry is 0
  __shared__ double sh[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int role = lane >> 4, j = lane & 15;
  const int xl = 16 * (warp & 1) + j, yl = warp >> 1;
  if (tid < 54) {
    const int r = tid % 9;
    chs[tid / 9][r] = c_chih_d[tid / 9][r < 6 ? 3 + r : 6 + r];
  }
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int n2 = g.n[2];
  const unsigned d0 = (unsigned)g.cd[0][0], d1 = (unsigned)g.cd[0][1], B = (unsigned)g.size[0];
  const long long tiles_x = g.n[0] / 32, ntiles = tiles_x * (g.n[1] / 2);
  int eidx[12];
#pragma unroll
  for (int m = 0; m < 12; ++m) eidx[m] = energy_index(role, m);
  double acc[12];
#pragma unroll
  for (int m = 0; m < 12; ++m) acc[m] = 0.0;
  unsigned phase = 0;  // bit b: parity of the next completion of slot b
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int x0 = int(tile % tiles_x) * 32, y0 = int(tile / tiles_x) * 2;
    // stage vertex plane p (0..n2; n2 = the top plane: plane 0 of the slab above) into slot b: thread 0 arms
    // the slot's mbarrier, threads 0..53 issue one bulk copy each (tx-count may dip below zero until armed)
    auto issue = [&](int p, int b) {
      if (tid == 0) mbar_arrive_expect_tx(&bar[b], kStBytes);
      if (tid >= 54) return;
      const int z = p == n2 ? 0 : p;
      const unsigned pz = (unsigned)z & 1u, h2 = (unsigned)z >> 1;
      const int f = tid / 9, rem = tid % 9, r = rem / 3, part = rem % 3;  // part 0/1: even x (16 + 1), 2: odd x
      int y = y0 + r;
      if (y >= g.n[1]) y -= g.n[1];
      const unsigned px = part == 2 ? 1u : 0u, color = px | (((unsigned)y & 1u) << 1) | (pz << 2);
      unsigned h0 = (unsigned)(x0 >> 1) + (part == 1 ? 16u : 0u);
      if (h0 >= d0) h0 -= d0;
      const size_t loc = (size_t)color * B + h0 + (size_t)d0 * (((unsigned)y >> 1) + (size_t)d1 * h2);
      const double* src = static_cast<const double*>(p == n2 ? uu.hi[f] : uu.p[f]) + 3 * loc;
      double* dst = ring + b * kStPlane + f * kStFS + r * kStRS + (px ? kStP1 : 0) + (part == 1 ? 48 : 0);
      bulk_g2s(dst, src, part == 1 ? 32u : 384u, &bar[b]);
    };
    auto land = [&](int b) {  // wait for slot b; mixed mode rounds the staged values to f32 precision once
      mbar_wait(&bar[b], (phase >> b) & 1u);
      phase ^= 1u << b;
      if constexpr (SNAP) {
        double* sl = ring + b * kStPlane;
        for (int i = tid; i < kStPlane; i += kPT) sl[i] = snap_f32_bits(sl[i]);
        fence_proxy_async_smem();  // these generic writes precede the slot's next bulk copy
      }
    };
    // one barrier per plane step: the step computes from slots z % 3, (z+1) % 3 while plane z+2 lands and is
    // rounded in the third slot; after the barrier slot z % 3 is refilled with plane z+3
    for (int p = 0; p < 3 && p <= n2; ++p) issue(p, p);
    land(0);
    land(1);
    __syncthreads();
    for (int z = 0; z < n2; ++z) {
      const double* bot = ring + (z % 3) * kStPlane;
      const double* top = ring + ((z + 1) % 3) * kStPlane;
      double b[3][kModes];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int f = 3 * role + a;
        double dh[24];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double V[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int x = xl + (jj & 1), r = yl + ((jj >> 1) & 1);
            V[jj] = ((jj >> 2) & 1 ? top : bot)[f * kStFS + r * kStRS + ((x & 1) ? kStP1 : 0) + 3 * (x >> 1) + c];
          }
#pragma unroll
          for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              if (!((jj >> k) & 1)) {
                const double lo = V[jj], hi = V[jj | (1 << k)];
                V[jj] = hi + lo;
                V[jj | (1 << k)] = hi - lo;
              }
#pragma unroll
          for (int sg = 1; sg < 8; ++sg) {
            const int r = sg * 3 + c;
            dh[r] = (r >= 3 && r <= 8) ? chs[f][r - 3] - V[sg] : ((r >= 12 && r <= 14) ? chs[f][r - 6] - V[sg] : -V[sg]);
          }
        }
        modal_from_dhat(dh, b[a]);
      }
      double E[12];
      gram_pairs(b, 16, E, E + 6);
      const int ex = x0 + xl, ey = y0 + yl;
      const long long e = ex + (long long)g.n[0] * (ey + (long long)g.n[1] * z);
      if (ecache) {
#pragma unroll
        for (int m = 0; m < 12; ++m)
          if (eidx[m] >= 0) ecache[eidx[m] * g.nv + e] = E[m];
      }
      const double q = penal == 1.0 ? rho[e] : pow(rho[e], penal);  // src/homogenization.cpp:91
#pragma unroll
      for (int m = 0; m < 12; ++m) acc[m] = fma(q, E[m], acc[m]);
      if (z + 2 <= n2) land((z + 2) % 3);
      __syncthreads();  // slot z % 3 is free, plane z + 2 is staged
      if (z + 3 <= n2) issue(z + 3, z % 3);
    }
  }
  for (int k = 0; k < 21; ++k) {
    double v = 0.0;
#pragma unroll
    for (int m = 0; m < 12; ++m) v += eidx[m] == k ? acc[m] : 0.0;
    const double r = block_reduce_h(v, sh);
    if (threadIdx.x == 0) partials[k * kReducePartials + blockIdx.x] = r;
  }
}

template <typename TN, typename TE, bool HADA>
__global__ void __launch_bounds__(kHT) tensor_kernel(GridGeo g, U6 uu, const double* __restrict__ rho, double penal,
                                                     bool snap, double lam, double mu, double* partials,
                                                     TE* __restrict__ ecache) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  TE* gsm = reinterpret_cast<TE*>(gsm_raw);
  __shared__ double sh[32];
  const TN* u[6];
  const TN* uh[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    u[i] = static_cast<const TN*>(uu.p[i]);
    uh[i] = static_cast<const TN*>(uu.hi[i]);
  }
  double acc[21];
#pragma unroll
  for (int q = 0; q < 21; ++q) acc[q] = 0.0;
  // HADA on x % 32 == 0, y % 2 == 0 grids: a block owns a 32 x 2 element column tile and marches up z,
  // so the upper corner plane of one step is the lower plane of the next (L1/L2 hits instead of the
  // grid-stride order's DRAM re-reads of neighbouring rows' corners)
  const bool cols = HADA && g.n[0] % 32 == 0 && g.n[1] % 2 == 0;
  const long long tiles_x = g.n[0] / 32, ntiles = cols ? tiles_x * (g.n[1] / 2) : 0;
  const long long nsteps = cols ? ((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * g.n[2]
                                : (g.nv - blockIdx.x * kHT + (long long)gridDim.x * kHT - 1) / ((long long)gridDim.x * kHT);
  for (long long it = 0; it < nsteps; ++it) {
    int ex, ey, ez;
    long long e;
    if (cols) {
      const long long tile = blockIdx.x + (it / g.n[2]) * gridDim.x;
      ez = int(it % g.n[2]);
      ex = int(tile % tiles_x) * 32 + int(threadIdx.x & 31);
      ey = int(tile / tiles_x) * 2 + int(threadIdx.x >> 5);
      e = ex + (long long)g.n[0] * (ey + (long long)g.n[1] * ez);
    } else {
      e = (long long)blockIdx.x * kHT + threadIdx.x + it * (long long)gridDim.x * kHT;
      if (e >= g.nv) break;
      ex = int(e % g.n[0]);
      const long long r = e / g.n[0];
      ey = int(r % g.n[1]);
      ez = int(r / g.n[1]);
    }
    TE E[21];
    if constexpr (HADA) element_energies_hada<TN, TE>(g, ex, ey, ez, u, uh, snap, E);
    else element_energies<TN, TE>(g, ex, ey, ez, u, uh, snap, TE(lam), TE(mu), gsm + threadIdx.x, E);
    if (ecache) {  // [21][nv]: the sensitivity pass reuses these instead of recomputing them
#pragma unroll
      for (int k = 0; k < 21; ++k) ecache[k * g.nv + e] = E[k];
    }
    const double q = penal == 1.0 ? rho[e] : pow(rho[e], penal);  // src/homogenization.cpp:91
#pragma unroll
    for (int k = 0; k < 21; ++k) acc[k] += q * double(E[k]);
  }
#pragma unroll
  for (int k = 0; k < 21; ++k) {
    const double r = block_reduce_h(acc[k], sh);
    if (threadIdx.x == 0) partials[k * kReducePartials + blockIdx.x] = r;
  }
}

__global__ void tensor_finalize(const double* partials, int nparts, double* out) {
  __shared__ double sh[32];
  for (int k = 0; k < 21; ++k) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[k * kReducePartials + i];
    const double r = block_reduce_h(s, sh);
    if (threadIdx.x == 0) out[k] = r;
  }
}

static bool htensor() { return knob("HTENSOR", 1) != 0; }

// Element energies of the mixed mode: the reference rounds u to f32 and forms d, K0 d and the dots in
// f64 (src/homogenization.cpp:84-94, 132-140) -- TE = double here too. ENERGY_F32=1 selects the
// all-f32 energy arithmetic (faster, not the reference's precision; off by default).
bool energy_f32(bool snap) { return snap && knob("ENERGY_F32", 0) != 0; }

static size_t grad_smem(bool f32) { return (f32 ? sizeof(float) : sizeof(double)) * 6 * kGradPerLoad * kHT; }

static void set_smem(const void* fn, bool f32) {
  IHOM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grad_smem(f32)));
}

template <typename TN>
void launch_effective_tensor(const GridGeo& g, const TN* const u[6], const double* rho, double penal, bool snap,
                             double lam, double mu, double* partials, double* c21, cudaStream_t s,
                             const TN* const* uhi, void* ecache) {
  long long blocks = (g.nv + kHT - 1) / kHT;
  if (blocks > kReducePartials) blocks = kReducePartials;
  U6 uu;
  for (int i = 0; i < 6; ++i) {
    uu.p[i] = u[i];
    uu.hi[i] = uhi ? uhi[i] : u[i];
  }
  const bool te32 = energy_f32(snap);
  if constexpr (std::is_same_v<TN, float>) {  // f32 snapshots (host-staged displacements): f64 energies
    if (te32) throw std::invalid_argument("f32 displacement snapshots take the f64 energy path");
    blocks = std::min<long long>((g.nv + 63) / 64, kReducePartials);
    tensor_pair_kernel<false, float><<<(unsigned)blocks, kPT, 0, s>>>(g, uu, rho, penal, partials,
                                                                     static_cast<double*>(ecache));
  } else if (htensor() && !te32 && tensor_stage_ok(g, uu.p, uu.hi)) {  // f64 energies, bulk-staged column tiles
    static int occ = 0;
    if (!occ) {
      IHOM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tensor_stage_kernel<true>, kPT, kStSmem));
      int dev = 0, sms = 0;
      IHOM_CUDA(cudaGetDevice(&dev));
      IHOM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      occ = std::max(1, occ) * sms;
    }
    const long long ntiles = (long long)(g.n[0] / 32) * (g.n[1] / 2);
    blocks = std::min<long long>(std::min<long long>(ntiles, occ), kReducePartials);
    if (snap)
      tensor_stage_kernel<true><<<(unsigned)blocks, kPT, kStSmem, s>>>(g, uu, rho, penal, partials,
                                                                       static_cast<double*>(ecache));
    else
      tensor_stage_kernel<false><<<(unsigned)blocks, kPT, kStSmem, s>>>(g, uu, rho, penal, partials,
                                                                        static_cast<double*>(ecache));
  } else if (htensor() && !te32) {  // f64 energies: modal form, two lanes per element
    blocks = (g.nv + 63) / 64;
    if (blocks > kReducePartials) blocks = kReducePartials;
    if (snap)
      tensor_pair_kernel<true><<<(unsigned)blocks, kPT, 0, s>>>(g, uu, rho, penal, partials, static_cast<double*>(ecache));
    else
      tensor_pair_kernel<false><<<(unsigned)blocks, kPT, 0, s>>>(g, uu, rho, penal, partials, static_cast<double*>(ecache));
  } else if (htensor()) {  // sum/difference-basis energies: no gradient scratch in shared memory
    if (te32)
      tensor_kernel<TN, float, true><<<(unsigned)blocks, kHT, 0, s>>>(g, uu, rho, penal, snap, lam, mu, partials,
                                                                      static_cast<float*>(ecache));
    else
      tensor_kernel<TN, double, true><<<(unsigned)blocks, kHT, 0, s>>>(g, uu, rho, penal, snap, lam, mu, partials,
                                                                       static_cast<double*>(ecache));
  } else if (te32) {
    set_smem((const void*)tensor_kernel<TN, float, false>, true);
    tensor_kernel<TN, float, false><<<(unsigned)blocks, kHT, grad_smem(true), s>>>(g, uu, rho, penal, snap, lam, mu,
                                                                                    partials,
                                                                                    static_cast<float*>(ecache));
  } else {
    set_smem((const void*)tensor_kernel<TN, double, false>, false);
    tensor_kernel<TN, double, false><<<(unsigned)blocks, kHT, grad_smem(false), s>>>(g, uu, rho, penal, snap, lam, mu,
                                                                                      partials,
                                                                                      static_cast<double*>(ecache));
  }
  IHOM_LAUNCH_CHECK();
  tensor_finalize<<<1, 256, 0, s>>>(partials, (int)blocks, c21);
  IHOM_LAUNCH_CHECK();
}

template <typename TN, typename TE, bool HADA>
__global__ void __launch_bounds__(kHT) sens_kernel(GridGeo g, U6 uu, const double* __restrict__ rho, double penal,
                                                   bool snap, double lam, double mu, const double* __restrict__ seed,
                                                   double inv_m, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  TE* gsm = reinterpret_cast<TE*>(gsm_raw);
  const TN* u[6];
  const TN* uh[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    u[i] = static_cast<const TN*>(uu.p[i]);
    uh[i] = static_cast<const TN*>(uu.hi[i]);
  }
  const long long e = (long long)blockIdx.x * kHT + threadIdx.x;
  if (e >= g.nv) return;
  const int ex = int(e % g.n[0]);
  const long long r = e / g.n[0];
  const int ey = int(r % g.n[1]), ez = int(r / g.n[1]);
  TE E[21];
  if constexpr (HADA) element_energies_hada<TN, TE>(g, ex, ey, ez, u, uh, snap, E);
  else element_energies<TN, TE>(g, ex, ey, ez, u, uh, snap, TE(lam), TE(mu), gsm + threadIdx.x, E);
  double acc = 0.0;  // sum_ij s_ij E_ij with s symmetric (src/homogenization.cpp:120,138-140)
  int q = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i; j < 6; ++j, ++q) acc += (i == j ? 1.0 : 2.0) * seed[i * 6 + j] * double(E[q]);
  out[e] = penal * (penal == 1.0 ? 1.0 : pow(rho[e], penal - 1.0)) * acc * inv_m;  // :141 (1/M over the whole grid)
}

// Sensitivity from the energies the tensor pass cached: identical arithmetic on identical E values.
template <typename TE>
__global__ void sens_cached_kernel(long long nv, const TE* __restrict__ ecache, const double* __restrict__ rho,
                                   double penal, const double* __restrict__ seed, double inv_m, double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nv) return;
  double acc = 0.0;
  int q = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i; j < 6; ++j, ++q) acc += (i == j ? 1.0 : 2.0) * seed[i * 6 + j] * double(ecache[q * nv + e]);
  out[e] = penal * (penal == 1.0 ? 1.0 : pow(rho[e], penal - 1.0)) * acc * inv_m;
}

void launch_sensitivity_cached(long long nv, const void* ecache, bool f32, const double* rho, double penal,
                               const double* sym_seed36, double* out, cudaStream_t s, long long m_total) {
  const double inv_m = 1.0 / double(m_total > 0 ? m_total : nv);
  if (f32)
    sens_cached_kernel<float><<<ceil_div(nv, 256), 256, 0, s>>>(nv, static_cast<const float*>(ecache), rho, penal,
                                                                 sym_seed36, inv_m, out);
  else
    sens_cached_kernel<double><<<ceil_div(nv, 256), 256, 0, s>>>(nv, static_cast<const double*>(ecache), rho, penal,
                                                                  sym_seed36, inv_m, out);
  IHOM_LAUNCH_CHECK();
}

template <typename TN>
void launch_tensor_sensitivity(const GridGeo& g, const TN* const u[6], const double* rho, double penal, bool snap,
                               double lam, double mu, const double* sym_seed36, double* out, cudaStream_t s,
                               const TN* const* uhi, long long m_total) {
  U6 uu;
  for (int i = 0; i < 6; ++i) {
    uu.p[i] = u[i];
    uu.hi[i] = uhi ? uhi[i] : u[i];
  }
  const double inv_m = 1.0 / double(m_total > 0 ? m_total : g.nv);
  const bool te32 = energy_f32(snap);
  if constexpr (std::is_same_v<TN, float>) {  // f32 snapshots (host-staged displacements)
    if (te32) throw std::invalid_argument("f32 displacement snapshots take the f64 energy path");
    sens_pair_kernel<false, float><<<ceil_div(2 * g.nv, kPT), kPT, 0, s>>>(g, uu, rho, penal, sym_seed36, inv_m, out);
  } else if (htensor() && !te32) {
    if (snap)
      sens_pair_kernel<true><<<ceil_div(2 * g.nv, kPT), kPT, 0, s>>>(g, uu, rho, penal, sym_seed36, inv_m, out);
    else
      sens_pair_kernel<false><<<ceil_div(2 * g.nv, kPT), kPT, 0, s>>>(g, uu, rho, penal, sym_seed36, inv_m, out);
  } else if (htensor()) {
    if (te32)
      sens_kernel<TN, float, true><<<ceil_div(g.nv, kHT), kHT, 0, s>>>(g, uu, rho, penal, snap, lam, mu, sym_seed36,
                                                                       inv_m, out);
    else
      sens_kernel<TN, double, true><<<ceil_div(g.nv, kHT), kHT, 0, s>>>(g, uu, rho, penal, snap, lam, mu, sym_seed36,
                                                                        inv_m, out);
  } else if (te32) {
    set_smem((const void*)sens_kernel<TN, float, false>, true);
    sens_kernel<TN, float, false><<<ceil_div(g.nv, kHT), kHT, grad_smem(true), s>>>(g, uu, rho, penal, snap, lam, mu,
                                                                                    sym_seed36, inv_m, out);
  } else {
    set_smem((const void*)sens_kernel<TN, double, false>, false);
    sens_kernel<TN, double, false><<<ceil_div(g.nv, kHT), kHT, grad_smem(false), s>>>(g, uu, rho, penal, snap, lam,
                                                                                      mu, sym_seed36, inv_m, out);
  }
  IHOM_LAUNCH_CHECK();
}

template void launch_effective_tensor<double>(const GridGeo&, const double* const[6], const double*, double, bool,
                                              double, double, double*, double*, cudaStream_t, const double* const*,
                                              void*);
template void launch_tensor_sensitivity<double>(const GridGeo&, const double* const[6], const double*, double, bool,
                                                double, double, const double*, double*, cudaStream_t,
                                                const double* const*, long long);
template void launch_effective_tensor<float>(const GridGeo&, const float* const[6], const double*, double, bool, double,
                                             double, double*, double*, cudaStream_t, const float* const*, void*);
template void launch_tensor_sensitivity<float>(const GridGeo&, const float* const[6], const double*, double, bool,
                                               double, double, const double*, double*, cudaStream_t,
                                               const float* const*, long long);

}  // namespace ihomgpu
