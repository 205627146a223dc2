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
    const double q = pow(rho[e], penal);  // src/homogenization.cpp:91
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
  if (htensor()) {  // sum/difference-basis energies: no gradient scratch in shared memory
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
  out[e] = penal * pow(rho[e], penal - 1.0) * acc * inv_m;  // :141 (1/M over the whole grid)
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
  out[e] = penal * pow(rho[e], penal - 1.0) * acc * inv_m;
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
  if (htensor()) {
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

}  // namespace ihomgpu
