// density_kernels.cu -- design-side kernels of the iteration:
//   radial_filter / DensityExpr eval+backward  (src/density.cpp:23-83)
//   symmetrize                                 (src/density.cpp:100-150)
//   OC trial / bisection reductions            (src/oc.cpp:14-77)
//   sensitivity_filter                         (src/oc.cpp:79-111)
//   clamp_bounds, field_mean                   (src/runner.cpp:47-49, src/density.cpp:11-14)
// Element fields are f64, x-fastest.
#include "density.hpp"
#include "kernels.hpp"
#include "profiler.hpp"

#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace ihomgpu {

constexpr int kMaxTaps = 343;  // radius < 4
__constant__ int c_tap_d[kMaxTaps][3];
__constant__ double c_tap_w[kMaxTaps];
constexpr int kMaxOps = 48;
__constant__ int c_sym_perm[kMaxOps][3];
__constant__ int c_sym_flip[kMaxOps][3];

// kernel_taps (src/density.cpp:23-45): kernel 0 = linear, 1 = spline4; normalised.
// sensitivity_filter taps (src/oc.cpp:85-96): linear cone, NOT normalised (wsum returned).
static std::vector<Tap> make_taps(double radius, int kernel, bool normalise, double* wsum) {
  std::vector<Tap> taps;
  const int r = int(std::floor(radius));
  for (int dz = -r; dz <= r; ++dz)
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        const double dist = std::sqrt(double(dx * dx + dy * dy + dz * dz));
        double w;
        if (normalise) {
          if (dist > radius) continue;
          if (kernel == 0) {
            w = radius - dist;
          } else {
            const double q = 1.0 - (dist / radius) * (dist / radius);
            w = q * q;
          }
        } else {
          w = radius - dist;
        }
        if (w > 0.0) taps.push_back({{dx, dy, dz}, w});
      }
  double total = 0.0;
  for (const auto& t : taps) total += t.w;
  if (normalise)
    for (auto& t : taps) t.w /= total;
  if (wsum) *wsum = total;
  if ((int)taps.size() > kMaxTaps) throw std::invalid_argument("filter radius too large (max 3.99)");
  return taps;
}

static void upload_taps(const std::vector<Tap>& taps, cudaStream_t s) {
  static int d[kMaxTaps][3];
  static double w[kMaxTaps];
  for (size_t i = 0; i < taps.size(); ++i) {
    for (int k = 0; k < 3; ++k) d[i][k] = taps[i].d[k];
    w[i] = taps[i].w;
  }
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_tap_d, d, sizeof(int) * 3 * taps.size(), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_tap_w, w, sizeof(double) * taps.size(), 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaStreamSynchronize(s));
}

__device__ __forceinline__ int wrapd(int c, int n) {
  c %= n;
  return c < 0 ? c + n : c;
}

// mode 0: out = conv(f); mode 1: out = conv(rho*f) / (max(rho,rmin)*wsum)  (sensitivity filter)
// z-slab: taps below / above the slab read the neighbours' planes (fl, rl).
__global__ void filter_kernel(int nx, int ny, int nz, int ntaps, const double* __restrict__ f,
                              const double* __restrict__ rho, double wsum, int mode, double* __restrict__ out,
                              ZLink<double> fl, ZLink<double> rl) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long m = (long long)nx * ny * nz;
  if (i >= m) return;
  const int x = int(i % nx);
  const long long r = i / nx;
  const int y = int(r % ny), z = int(r / ny);
  double s = 0.0;
  for (int t = 0; t < ntaps; ++t) {
    const int zz = z + c_tap_d[t][2];
    const long long k = wrapd(x + c_tap_d[t][0], nx) +
                        (long long)nx * (wrapd(y + c_tap_d[t][1], ny) + (long long)ny * wrapd(zz, nz));
    const double* fb = zz < 0 ? fl.lo : (zz >= nz ? fl.hi : f);
    if (mode == 0) {
      s += c_tap_w[t] * fb[k];
    } else {
      const double* rb = zz < 0 ? rl.lo : (zz >= nz ? rl.hi : rho);
      s += c_tap_w[t] * rb[k] * fb[k];
    }
  }
  out[i] = mode == 0 ? s : s / (fmax(rho[i], kRhoMin) * wsum);
}

// Fast path: the taps of radius r live in a (2R+1)^3 cube of constant weights
// (zero outside the ball); per-axis wrapped offsets are computed once per thread,
// so every tap is one IADD3 + load (no modulo per tap).
__constant__ double c_cube_w[7 * 7 * 7];
// NZ elements per thread (planes z, z + nz/NZ, ...): independent tap chains interleaved for latency
// hiding; every element keeps its own z, y, x tap order (bit-identical to NZ = 1).
template <int R, int NZ = 1>
__global__ void __launch_bounds__(256) filter_cube_kernel(int nx, int ny, int nz, const double* __restrict__ f,
                                                          ZLink<double> fl, double* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= nx) return;
  int X[2 * R + 1], Y[2 * R + 1], Z[NZ][2 * R + 1];
  const double* zb[NZ][2 * R + 1];  // z-slab: planes beyond the slab come from its neighbours
  int zs[NZ];
#pragma unroll
  for (int k = 0; k < NZ; ++k) zs[k] = blockIdx.z + k * (nz / NZ);
#pragma unroll
  for (int d = -R; d <= R; ++d) {
    X[d + R] = wrapd(x + d, nx);
    Y[d + R] = nx * wrapd(y + d, ny);
#pragma unroll
    for (int k = 0; k < NZ; ++k) {
      const int z = zs[k];
      Z[k][d + R] = nx * ny * wrapd(z + d, nz);
      zb[k][d + R] = z + d < 0 ? fl.lo : (z + d >= nz ? fl.hi : f);
    }
  }
  double s[NZ];
#pragma unroll
  for (int k = 0; k < NZ; ++k) s[k] = 0.0;
#pragma unroll
  for (int dz = 0; dz <= 2 * R; ++dz)
#pragma unroll
    for (int dy = 0; dy <= 2 * R; ++dy)
#pragma unroll
      for (int dx = 0; dx <= 2 * R; ++dx) {
        const double w = c_cube_w[(dz * (2 * R + 1) + dy) * (2 * R + 1) + dx];
        if (w != 0.0) {
#pragma unroll
          for (int k = 0; k < NZ; ++k)  // kernel_taps order: z, y, x
            s[k] += w * __ldg(zb[k][dz] + (size_t)(X[dx] + Y[dy] + Z[k][dz]));
        }
      }
#pragma unroll
  for (int k = 0; k < NZ; ++k) out[x + (size_t)nx * (y + (size_t)ny * zs[k])] = s[k];
}

static std::mutex g_const_mu;  // host staging of the constant-memory tap tables (z-slab threads)

static bool filter_cube(const int n[3], const std::vector<Tap>& taps, double radius, const double* f, double* out,
                        cudaStream_t s, ZLink<double> fl) {
  // the cube spans the taps actually present (w > 0): at the default r = 2 the spline/linear taps are
  // exactly the 3^3 cube (the (+-2,0,0) offsets have w = 0 and are dropped, kernel_taps), so the R = 1
  // kernel runs 27 iterations instead of 125 -- same taps in the same z, y, x order: bit-identical
  int R = 0;
  for (const auto& t : taps)
    for (int k = 0; k < 3; ++k) R = std::max(R, std::abs(t.d[k]));
  if (R < 1 || R > 3 || n[0] < 2 * R + 1 || n[1] < 2 * R + 1 || n[2] < 2 * R + 1) return false;
  std::lock_guard<std::mutex> lock(g_const_mu);
  static double cube[7 * 7 * 7];
  const int W = 2 * R + 1;
  for (int i = 0; i < W * W * W; ++i) cube[i] = 0.0;
  for (const auto& t : taps) cube[((t.d[2] + R) * W + (t.d[1] + R)) * W + (t.d[0] + R)] = t.w;
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_cube_w, cube, sizeof(double) * W * W * W, 0, cudaMemcpyHostToDevice, s));
  const dim3 b(256), g(ceil_div(n[0], 256), n[1], n[2]);
  fl = resolve(fl, f);
  if (R == 1 && n[2] % 4 == 0 && knob("FILTER_NZ", 1) != 0)
    filter_cube_kernel<1, 4><<<dim3(g.x, g.y, n[2] / 4), b, 0, s>>>(n[0], n[1], n[2], f, fl, out);
  else if (R == 1) filter_cube_kernel<1><<<g, b, 0, s>>>(n[0], n[1], n[2], f, fl, out);
  else if (R == 2) filter_cube_kernel<2><<<g, b, 0, s>>>(n[0], n[1], n[2], f, fl, out);
  else filter_cube_kernel<3><<<g, b, 0, s>>>(n[0], n[1], n[2], f, fl, out);
  IHOM_LAUNCH_CHECK();
  IHOM_CUDA(cudaStreamSynchronize(s));  // cube staging buffer is static
  return true;
}

void radial_filter(const int n[3], const double* f, double radius, int kernel, double* out, cudaStream_t s,
                   ZLink<double> fl) {
  const long long m = (long long)n[0] * n[1] * n[2];
  if (radius < 1.0) {
    IHOM_CUDA(cudaMemcpyAsync(out, f, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    return;
  }
  const auto taps = make_taps(radius, kernel, true, nullptr);
  if (!is_self(fl, f) && int(std::floor(radius)) > n[2]) throw std::invalid_argument("filter radius exceeds the z-slab");
  ProfScope p(s, "filter", double(m) * 16.0);
  if (filter_cube(n, taps, radius, f, out, s, fl)) return;
  std::lock_guard<std::mutex> lock(g_const_mu);
  upload_taps(taps, s);
  filter_kernel<<<ceil_div(m, 256), 256, 0, s>>>(n[0], n[1], n[2], (int)taps.size(), f, nullptr, 1.0, 0, out,
                                                 resolve(fl, f), ZLink<double>{f, f});
  IHOM_LAUNCH_CHECK();
  IHOM_CUDA(cudaStreamSynchronize(s));
}

void sensitivity_filter(const int n[3], const double* sens, const double* rho, double radius, double* out,
                        cudaStream_t s, ZLink<double> sl, ZLink<double> rl) {
  const long long m = (long long)n[0] * n[1] * n[2];
  if (radius < 1.0) {
    IHOM_CUDA(cudaMemcpyAsync(out, sens, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    return;
  }
  double wsum = 0.0;
  const auto taps = make_taps(radius, 0, false, &wsum);
  if (!is_self(sl, sens) && int(std::floor(radius)) > n[2]) throw std::invalid_argument("filter radius exceeds the z-slab");
  std::lock_guard<std::mutex> lock(g_const_mu);
  upload_taps(taps, s);
  ProfScope p(s, "filter", double(m) * 24.0);
  filter_kernel<<<ceil_div(m, 256), 256, 0, s>>>(n[0], n[1], n[2], (int)taps.size(), sens, rho, wsum, 1, out,
                                                 resolve(sl, sens), resolve(rl, rho));
  IHOM_LAUNCH_CHECK();
  IHOM_CUDA(cudaStreamSynchronize(s));
}

// x^k for a small integer k by repeated multiplication (the SIMP exponent 3 of the default config):
// the f64 pow() is a log/exp sequence ~10x the cost of this memory-bound pass; both are within an
// ulp or two of the reference's std::pow
__device__ __forceinline__ double ipow(double x, int k) {
  double r = 1.0;
  for (int j = 0; j < k; ++j) r *= x;
  return r;
}

// out = x^p  /  out = g * p * x^(p-1); ip > 0: p == ip exactly (integer exponent <= 4)
__global__ void pow_kernel(const double* __restrict__ x, const double* __restrict__ g, double p, int ip, long long m,
                           double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (ip > 0) out[i] = g ? g[i] * p * ipow(x[i], ip - 1) : ipow(x[i], ip);
  else out[i] = g ? g[i] * p * pow(x[i], p - 1.0) : pow(x[i], p);
}

static int int_exponent(double p) {
  return (knob("POW_INT", 1) != 0 && p >= 1.0 && p <= 4.0 && p == double(int(p))) ? int(p) : 0;
}

void pow_field(const double* x, double p, long long m, double* out, cudaStream_t s) {
  ProfScope ps(s, "pow", double(m) * 16.0);
  pow_kernel<<<ceil_div(m, 256), 256, 0, s>>>(x, nullptr, p, int_exponent(p), m, out);
  IHOM_LAUNCH_CHECK();
}

void pow_backward(const double* x, const double* g, double p, long long m, double* out, cudaStream_t s) {
  ProfScope ps(s, "pow", double(m) * 24.0);
  pow_kernel<<<ceil_div(m, 256), 256, 0, s>>>(x, g, p, int_exponent(p), m, out);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- symmetrize
static int symmetry_group(int sym, int perm[kMaxOps][3], int flip[kMaxOps][3]) {
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  int k = 0;
  auto push = [&](const int* p, int m) {
    for (int a = 0; a < 3; ++a) {
      perm[k][a] = p[a];
      flip[k][a] = (m >> a) & 1;
    }
    ++k;
  };
  auto sign = [](const int* p) {
    int s = 1;
    for (int i = 0; i < 3; ++i)
      for (int j = i + 1; j < 3; ++j)
        if (p[i] > p[j]) s = -s;
    return s;
  };
  switch (sym) {  // src/density.cpp:100-127
    case 1:
      for (int m = 0; m < 8; ++m) push(perms[0], m);
      break;
    case 2:
      for (const auto& p : perms)
        for (int m = 0; m < 8; ++m) push(p, m);
      break;
    case 3:
      for (const auto& p : perms)
        for (int m = 0; m < 8; ++m) {
          const int nflip = (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1);
          if (sign(p) * ((nflip % 2) ? -1 : 1) == 1) push(p, m);
        }
      break;
    default:
      throw std::invalid_argument("unknown symmetry");
  }
  return k;
}

__global__ void symmetrize_kernel(int nx, int ny, int nz, int nops, const double* __restrict__ in,
                                  double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long m = (long long)nx * ny * nz;
  if (i >= m) return;
  const int n[3] = {nx, ny, nz};
  int e[3];
  e[0] = int(i % nx);
  const long long r = i / nx;
  e[1] = int(r % ny);
  e[2] = int(r / ny);
  double s = 0.0;
  for (int o = 0; o < nops; ++o) {
    int q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      q[k] = e[c_sym_perm[o][k]];
      if (c_sym_flip[o][k]) q[k] = n[k] - 1 - q[k];
    }
    s += in[q[0] + (long long)nx * (q[1] + (long long)ny * q[2])];
  }
  out[i] = s * (1.0 / double(nops));
}

// reflect3 / first half of reflect6: average over the 8 axis flips. One thread
// per element of the octant [0, ceil(n/2))^3 reads the 8 mirror images once and
// writes the average to all of them (the result is flip-invariant).
__global__ void flip_avg_kernel(int nx, int ny, int nz, const double* __restrict__ in, double* __restrict__ out) {
  const int hx = (nx + 1) / 2, hy = (ny + 1) / 2, hz = (nz + 1) / 2;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)hx * hy * hz) return;
  const int x = int(i % hx);
  const long long r = i / hx;
  const int y = int(r % hy), z = int(r / hy);
  const int xs[2] = {x, nx - 1 - x}, ys[2] = {y, ny - 1 - y}, zs[2] = {z, nz - 1 - z};
  double sum = 0.0;
#pragma unroll
  for (int m = 0; m < 8; ++m)  // reference op order within one permutation: m = fx | fy<<1 | fz<<2
    sum += in[xs[m & 1] + (long long)nx * (ys[(m >> 1) & 1] + (long long)ny * zs[(m >> 2) & 1])];
  const double v = sum * 0.125;
#pragma unroll
  for (int m = 0; m < 8; ++m)
    out[xs[m & 1] + (long long)nx * (ys[(m >> 1) & 1] + (long long)ny * zs[(m >> 2) & 1])] = v;
}

// Second half of reflect6: average over the 6 axis permutations on a cubic grid,
// tiled 8^3. A CTA owns an orbit representative tile B (bx <= by <= bz), stages
// the 6 permuted source tiles in shared memory (coalesced 64-byte rows), averages,
// and writes the (permutation-invariant) result to all 6 image tiles.
constexpr int kPT = 8;
__global__ void __launch_bounds__(512) perm_avg_kernel(int n, const double* __restrict__ in, double* __restrict__ out) {
  __shared__ double tile[6][kPT * kPT * kPT];
  __shared__ double avg[kPT * kPT * kPT];
  const int nt = n / kPT;
  // decode the representative tile from blockIdx.x over all (bx,by,bz) with bx<=by<=bz
  int b[3];
  {
    int k = blockIdx.x, bz = 0;
    while (k >= (bz + 1) * (bz + 2) / 2) {
      k -= (bz + 1) * (bz + 2) / 2;
      ++bz;
    }
    int by = 0;
    while (k >= by + 1) {
      k -= by + 1;
      ++by;
    }
    b[0] = k;
    b[1] = by;
    b[2] = bz;
  }
  if (b[2] >= nt) return;
  const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const int t = threadIdx.x;
  const int l[3] = {t % kPT, (t / kPT) % kPT, t / (kPT * kPT)};
#pragma unroll
  for (int p = 0; p < 6; ++p) {  // source tile p(B), element l (x fastest): coalesced rows
    const int sb[3] = {b[perm[p][0]], b[perm[p][1]], b[perm[p][2]]};
    tile[p][t] = in[(sb[0] * kPT + l[0]) + (long long)n * ((sb[1] * kPT + l[1]) + (long long)n * (sb[2] * kPT + l[2]))];
  }
  __syncthreads();
  double sum = 0.0;
#pragma unroll
  for (int p = 0; p < 6; ++p) {  // image of e = (B, l) under p lies in tile p(B) at local (l[p0], l[p1], l[p2])
    const int a = l[perm[p][0]], bb = l[perm[p][1]], c = l[perm[p][2]];
    sum += tile[p][a + kPT * (bb + kPT * c)];
  }
  avg[t] = sum * (1.0 / 6.0);
  __syncthreads();
#pragma unroll
  for (int p = 0; p < 6; ++p) {  // out at p(e) = avg(e): thread writes image-tile element (a,b,c) = t
    const int sb[3] = {b[perm[p][0]], b[perm[p][1]], b[perm[p][2]]};
    int e[3];
    e[perm[p][0]] = l[0];
    e[perm[p][1]] = l[1];
    e[perm[p][2]] = l[2];
    out[(sb[0] * kPT + l[0]) + (long long)n * ((sb[1] * kPT + l[1]) + (long long)n * (sb[2] * kPT + l[2]))] =
        avg[e[0] + kPT * (e[1] + kPT * e[2])];
  }
}

void symmetrize(const int n[3], double* field, int sym, double* scratch, cudaStream_t s) {
  if (sym == 0) return;
  if (sym != 1 && (n[0] != n[1] || n[1] != n[2]))
    throw std::invalid_argument("reflect6/rotate3 symmetry requires a cubic grid");
  const long long m = (long long)n[0] * n[1] * n[2];
  if (sym == 1 || (sym == 2 && n[0] % kPT == 0)) {  // factored fast path (src/density.cpp:100-150 group)
    const long long oct = (long long)((n[0] + 1) / 2) * ((n[1] + 1) / 2) * ((n[2] + 1) / 2);
    ProfScope p(s, "symmetrize", double(m) * 16.0 * (sym == 2 ? 2.0 : 1.0));
    flip_avg_kernel<<<ceil_div(oct, 256), 256, 0, s>>>(n[0], n[1], n[2], field, sym == 2 ? scratch : scratch);
    IHOM_LAUNCH_CHECK();
    if (sym == 1) {
      IHOM_CUDA(cudaMemcpyAsync(field, scratch, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    } else {
      const int nt = n[0] / kPT;
      const int reps = nt * (nt + 1) * (nt + 2) / 6;
      perm_avg_kernel<<<reps, kPT * kPT * kPT, 0, s>>>(n[0], scratch, field);
      IHOM_LAUNCH_CHECK();
    }
    return;
  }
  std::lock_guard<std::mutex> lock(g_const_mu);
  static int perm[kMaxOps][3], flip[kMaxOps][3];
  const int nops = symmetry_group(sym, perm, flip);
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_sym_perm, perm, sizeof(int) * 3 * nops, 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyToSymbolAsync(c_sym_flip, flip, sizeof(int) * 3 * nops, 0, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyAsync(scratch, field, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
  {
    ProfScope p(s, "symmetrize", double(m) * 16.0);
    symmetrize_kernel<<<ceil_div(m, 256), 256, 0, s>>>(n[0], n[1], n[2], nops, scratch, field);
  }
  IHOM_LAUNCH_CHECK();
  IHOM_CUDA(cudaStreamSynchronize(s));  // constant staging buffers are static
}

// ---- z-slab symmetrize: gather form over every slab's copy (peer memory).
// Element e of this slab = global (x, y, z0 + zl); a global element (a, b, c)
// lives on slab c / t at local plane c % t.
__device__ __forceinline__ double slab_at(const PeerTable& in, int n0, int n1, int t, int a, int b, int c) {
  const int owner = c / t;
  return static_cast<const double*>(in.p[owner])[a + (long long)n0 * (b + (long long)n1 * (c - owner * t))];
}

// 8 axis flips, summed from the octant representative in flip_avg_kernel's
// order -- bitwise the single-domain result.
__global__ void flip_gather_kernel(int n0, int n1, int n2, int t, int z0, PeerTable in, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n0 * n1 * t) return;
  const int x = int(i % n0);
  const long long r = i / n0;
  const int y = int(r % n1), z = z0 + int(r / n1);
  const int rx = min(x, n0 - 1 - x), ry = min(y, n1 - 1 - y), rz = min(z, n2 - 1 - z);
  const int xs[2] = {rx, n0 - 1 - rx}, ys[2] = {ry, n1 - 1 - ry}, zs[2] = {rz, n2 - 1 - rz};
  double sum = 0.0;
#pragma unroll
  for (int m = 0; m < 8; ++m) sum += slab_at(in, n0, n1, t, xs[m & 1], ys[(m >> 1) & 1], zs[(m >> 2) & 1]);
  out[i] = sum * 0.125;
}

// 6 axis permutations (cubic grid), summed from the sorted-coordinate
// representative of the orbit: every orbit member gets the same bits.
__global__ void perm_gather_kernel(int n, int t, int z0, PeerTable in, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n * n * t) return;
  int e[3];
  e[0] = int(i % n);
  const long long r = i / n;
  e[1] = int(r % n);
  e[2] = z0 + int(r / n);
  int a = e[0], b = e[1], c = e[2], tmp;  // sort ascending
  if (a > b) { tmp = a; a = b; b = tmp; }
  if (b > c) { tmp = b; b = c; c = tmp; }
  if (a > b) { tmp = a; a = b; b = tmp; }
  const int rep[3] = {a, b, c};
  const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  double sum = 0.0;
#pragma unroll
  for (int p = 0; p < 6; ++p) sum += slab_at(in, n, n, t, rep[perm[p][0]], rep[perm[p][1]], rep[perm[p][2]]);
  out[i] = sum * (1.0 / 6.0);
}

// generic group (rotate3, odd sizes): symmetrize_kernel's op order
__global__ void sym_gather_kernel(int n0, int n1, int n2, int t, int z0, int nops, PeerTable in,
                                  double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n0 * n1 * t) return;
  const int n[3] = {n0, n1, n2};
  int e[3];
  e[0] = int(i % n0);
  const long long r = i / n0;
  e[1] = int(r % n1);
  e[2] = z0 + int(r / n1);
  double sum = 0.0;
  for (int o = 0; o < nops; ++o) {
    int q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      q[k] = e[c_sym_perm[o][k]];
      if (c_sym_flip[o][k]) q[k] = n[k] - 1 - q[k];
    }
    sum += slab_at(in, n0, n1, t, q[0], q[1], q[2]);
  }
  out[i] = sum * (1.0 / double(nops));
}

void symmetrize_slab(const int n[3], const Slab& slab, double* field, PeerTable fpeers, double* scratch,
                     PeerTable speers, int sym, cudaStream_t s) {
  if (sym == 0) return;
  if (sym != 1 && (n[0] != n[1] || n[1] != n[2]))
    throw std::invalid_argument("reflect6/rotate3 symmetry requires a cubic grid");
  const int t = n[2] / slab.nranks, z0 = slab.rank * t;
  const long long m = (long long)n[0] * n[1] * t;
  ProfScope p(s, "symmetrize", double(m) * 16.0 * (sym == 2 ? 2.0 : 1.0));
  slab.sync(s);  // every slab's field is current
  if (sym == 1 || sym == 2) {
    flip_gather_kernel<<<ceil_div(m, 256), 256, 0, s>>>(n[0], n[1], n[2], t, z0, fpeers, scratch);
    IHOM_LAUNCH_CHECK();
    if (sym == 1) {
      slab.sync(s);  // nobody overwrites its field while others still gather from it
      IHOM_CUDA(cudaMemcpyAsync(field, scratch, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    } else {
      slab.sync(s);
      perm_gather_kernel<<<ceil_div(m, 256), 256, 0, s>>>(n[0], t, z0, speers, field);
      IHOM_LAUNCH_CHECK();
    }
  } else {
    {
      // the operator tables live in process-wide __constant__ memory shared by every slab thread of a
      // local fabric: upload + gather under the lock, and release it BEFORE the slab barrier (a thread
      // waiting at the barrier while holding it would stall the others on the lock: deadlock)
      std::lock_guard<std::mutex> lock(g_const_mu);
      static int perm[kMaxOps][3], flip[kMaxOps][3];
      const int nops = symmetry_group(sym, perm, flip);
      IHOM_CUDA(cudaMemcpyToSymbolAsync(c_sym_perm, perm, sizeof(int) * 3 * nops, 0, cudaMemcpyHostToDevice, s));
      IHOM_CUDA(cudaMemcpyToSymbolAsync(c_sym_flip, flip, sizeof(int) * 3 * nops, 0, cudaMemcpyHostToDevice, s));
      sym_gather_kernel<<<ceil_div(m, 256), 256, 0, s>>>(n[0], n[1], n[2], t, z0, nops, fpeers, scratch);
      IHOM_LAUNCH_CHECK();
      IHOM_CUDA(cudaStreamSynchronize(s));
    }
    slab.sync(s);
    IHOM_CUDA(cudaMemcpyAsync(field, scratch, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
  }
  slab.sync(s);  // the symmetrized field is final on every slab
}

__global__ void clamp_kernel(double* f, long long m, double lo, double hi) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) f[i] = fmin(fmax(f[i], lo), hi);
}

void clamp_field(double* f, long long m, double lo, double hi, cudaStream_t s) {
  ProfScope p(s, "vector", double(m) * 16.0);
  clamp_kernel<<<ceil_div(m, 256), 256, 0, s>>>(f, m, lo, hi);
  IHOM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- reductions for OC
constexpr int kDT = 256;

__device__ __forceinline__ double block_reduce_d(double v, double* sh, bool is_max) {
  const int t = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_down_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : v + w;
  }
  if ((t & 31) == 0) sh[t >> 5] = v;
  __syncthreads();
  double r = is_max ? -INFINITY : 0.0;
  if (t < 32) {
    r = (t < (int)(blockDim.x >> 5)) ? sh[t] : r;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_down_sync(0xffffffffu, r, o);
      r = is_max ? fmax(r, w) : r + w;
    }
  }
  __syncthreads();
  return r;
}

static int dgrid(long long n) {
  long long g = (n + kDT * 8 - 1) / (kDT * 8);
  if (g < 1) g = 1;
  if (g > kReducePartials) g = kReducePartials;
  return int(g);
}

__global__ void finalize_d(const double* partials, int nparts, bool is_max, double* out) {
  __shared__ double sh[32];
  double s = is_max ? -INFINITY : 0.0;
  for (int i = threadIdx.x; i < nparts; i += kDT) s = is_max ? fmax(s, partials[i]) : s + partials[i];
  const double r = block_reduce_d(s, sh, is_max);
  if (threadIdx.x == 0) *out = r;
}

__global__ void sum_kernel(const double* __restrict__ f, long long m, double* partials) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kDT + threadIdx.x; i < m; i += (long long)gridDim.x * kDT) s += f[i];
  const double r = block_reduce_d(s, sh, false);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

void field_sum(const double* f, long long m, double* partials, double* out, cudaStream_t s, const Slab& slab) {
  const int g = dgrid(m);
  ProfScope p(s, "reduce", double(m) * 8.0);
  sum_kernel<<<g, kDT, 0, s>>>(f, m, partials);
  IHOM_LAUNCH_CHECK();
  finalize_d<<<1, kDT, 0, s>>>(partials, g, false, out);
  IHOM_LAUNCH_CHECK();
  slab.allreduce(out, 1, false, s);
}

// max(1e-30, -g) over the field plus a non-finite flag (src/oc.cpp:29-38)
__global__ void oc_scale_kernel(const double* __restrict__ g, long long m, double* partials, int* bad) {
  __shared__ double sh[32];
  double s = 1e-30;
  for (long long i = (long long)blockIdx.x * kDT + threadIdx.x; i < m; i += (long long)gridDim.x * kDT) {
    const double v = g[i];
    if (!isfinite(v)) atomicExch(bad, 1);
    s = fmax(s, fmax(1e-30, -v));
  }
  const double r = block_reduce_d(s, sh, true);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

struct OCParams {
  double damp, step, lo, hi;
};

// ---------------------------------------------------------------- device-resident OC bisection
// oc_update (src/oc.cpp:27-77). The geometric bisection runs on the device: every pass evaluates the means
// of a depth-3 subtree of the bisection (7 trial lambdas, and lo0/hi0 on the first pass) in one sweep over
// rho and sqrt(b0), then one thread walks the subtree exactly as the sequential loop would (same
// sqrt(lo*hi) midpoints, same stop rule, same 60-trial cap) and leaves the bracket or the final lambda in
// device memory. Passes run in batches with one 8-byte read of the done flag per batch (usually one batch
// per update, versus one blocking read-back per trial before).
// Per element a trial is x = clamp(clamp(rho * sqrt(b0) * lambda^-1/2, rho -+ step), [rho_min, 1])
// (the two clamps fused into one interval):
// sqrt(b0) is formed once per update instead of sqrt(b0 / lambda) per trial (the reference's
// rho * pow(b0 / lambda, 0.5), src/oc.cpp:18; same value to an ulp).
constexpr int kOcTree = 7;           // lambdas per pass (depth-3 subtree)
constexpr int kOcSlots = 2 + kOcTree;  // + lo0, hi0 on the first pass
constexpr int kOcMaxPasses = 22;     // 2 bracket trials + 60 bisection trials, 3 per pass

struct OcState {  // device scratch (doubles)
  double lo, hi, lambda, mean, trials, done, ok, pass;
};

// sb = sqrt(max(1e-30, -g) / scale) into `sb` (src/oc.cpp:35-41, the normaliser on the device)
__global__ void oc_prep_kernel(const double* __restrict__ g, long long m, const double* scale, double* sb) {
  const double inv = 1.0 / *scale;
  for (long long i = (long long)blockIdx.x * kDT + threadIdx.x; i < m; i += (long long)gridDim.x * kDT)
    sb[i] = sqrt(fmax(1e-30, -g[i]) * inv);
}

// the same two clamps as one (rho lies in [lo, hi], so [rho - step, rho + step] meets [lo, hi] and
// clamp(clamp(x, a, b), c, d) == clamp(x, max(a, c), min(b, d)) exactly)
__device__ __forceinline__ void oc_bounds(double rho, OCParams p, double& lo, double& hi) {
  lo = fmax(rho - p.step, p.lo);
  hi = fmin(rho + p.step, p.hi);
}

// the lambdas of a pass: slots 0/1 = lo0/hi0 (first pass only), slots 2.. = the subtree in level order
// (node k's children: 2k+1 when mean > V (lo = lambda_k), 2k+2 otherwise (hi = lambda_k))
__device__ __forceinline__ void oc_pass_lambdas(const OcState& st, double lam[kOcSlots]) {
  lam[0] = 1e-12;
  lam[1] = 1e12;
  double lo[kOcTree], hi[kOcTree];
  lo[0] = st.lo;
  hi[0] = st.hi;
#pragma unroll
  for (int k = 0; k < kOcTree; ++k) {
    lam[2 + k] = sqrt(lo[k] * hi[k]);
    if (2 * k + 2 < kOcTree) {
      lo[2 * k + 1] = lam[2 + k], hi[2 * k + 1] = hi[k];
      lo[2 * k + 2] = lo[k], hi[2 * k + 2] = lam[2 + k];
    }
  }
}

__global__ void oc_pass_kernel(const double* __restrict__ rho, const double* __restrict__ sb, long long m,
                               const OcState* st, OCParams p, double* partials) {
  __shared__ double sh[32];
  const OcState S = *st;
  if (S.done != 0.0) return;
  const bool first = S.pass == 0.0;
  double lam[kOcSlots], rl[kOcSlots], acc[kOcSlots];
  oc_pass_lambdas(S, lam);
#pragma unroll
  for (int k = 0; k < kOcSlots; ++k) rl[k] = 1.0 / sqrt(lam[k]), acc[k] = 0.0;
  for (long long i = (long long)blockIdx.x * kDT + threadIdx.x; i < m; i += (long long)gridDim.x * kDT) {
    const double r = rho[i], base = r * sb[i];
    double lo, hi;
    oc_bounds(r, p, lo, hi);
#pragma unroll
    for (int k = 0; k < kOcSlots; ++k)
      if (first || k >= 2) acc[k] += fmin(fmax(base * rl[k], lo), hi);
  }
#pragma unroll
  for (int k = 0; k < kOcSlots; ++k) {
    const double v = block_reduce_d(acc[k], sh, false);
    if (threadIdx.x == 0) partials[k * kReducePartials + blockIdx.x] = v;
  }
}

__global__ void oc_sums_kernel(const double* partials, int nparts, const OcState* st, double* sums) {
  __shared__ double sh[32];
  if (st->done != 0.0) return;
  for (int k = 0; k < kOcSlots; ++k) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kDT) v += partials[k * kReducePartials + i];
    const double r = block_reduce_d(v, sh, false);
    if (threadIdx.x == 0) sums[k] = r;
  }
}

// the sequential loop of src/oc.cpp:44-76 over this pass's means
__device__ void oc_decide_kernel_body(OcState* st, const double* sums, double count, double volume, double tol) {
  OcState S = *st;
  if (S.done != 0.0) return;
  double lam[kOcSlots];
  oc_pass_lambdas(S, lam);
  if (S.pass == 0.0) {
    const double mean_lo = sums[0] / count;
    if (volume >= mean_lo) {  // even the maximal move stays at or under target
      S.done = 1.0, S.lambda = lam[0], S.mean = mean_lo, S.ok = fabs(mean_lo - volume) <= tol;
      *st = S;
      return;
    }
    const double mean_hi = sums[1] / count;
    if (volume <= mean_hi) {  // cannot shrink below target within the step limit
      S.done = 1.0, S.lambda = lam[1], S.mean = mean_hi, S.ok = fabs(mean_hi - volume) <= tol;
      *st = S;
      return;
    }
  }
  int k = 0;
  while (k < kOcTree) {
    const double mean = sums[2 + k] / count;
    S.trials += 1.0;
    S.lambda = lam[2 + k];
    S.mean = mean;
    if (fabs(mean - volume) <= tol) {
      S.done = 1.0, S.ok = 1.0;
      break;
    }
    if (mean > volume) S.lo = lam[2 + k], k = 2 * k + 1;
    else S.hi = lam[2 + k], k = 2 * k + 2;
    if (S.trials >= 60.0) {  // cap: the last trial's field, ok iff within tolerance (src/oc.cpp:72-75)
      S.done = 1.0, S.ok = 0.0;
      break;
    }
  }
  S.pass += 1.0;
  *st = S;
}

__global__ void oc_decide_kernel(OcState* st, const double* sums, double count, double volume, double tol) {
  oc_decide_kernel_body(st, sums, count, volume, tol);
}

// one domain: the sums and the walk in one launch (slabs fold the sums across ranks in between)
__global__ void oc_sums_decide_kernel(const double* partials, int nparts, OcState* st, double* sums, double count,
                                      double volume, double tol) {
  __shared__ double sh[32];
  if (st->done != 0.0) return;
  for (int k = 0; k < kOcSlots; ++k) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kDT) v += partials[k * kReducePartials + i];
    const double r = block_reduce_d(v, sh, false);
    if (threadIdx.x == 0) sums[k] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) oc_decide_kernel_body(st, sums, count, volume, tol);
}

__global__ void oc_write_kernel(const double* __restrict__ rho, double* sbout, long long m, const OcState* st,
                                OCParams p) {
  const double rl = 1.0 / sqrt(st->lambda);
  for (long long i = (long long)blockIdx.x * kDT + threadIdx.x; i < m; i += (long long)gridDim.x * kDT) {
    const double r = rho[i];
    double lo, hi;
    oc_bounds(r, p, lo, hi);
    sbout[i] = fmin(fmax(r * sbout[i] * rl, lo), hi);  // sbout holds sqrt(b0) on entry, the update on exit
  }
}

OCResult oc_update(long long m, const double* rho, const double* g, const OCConfig& cfg, double* out, Workspace& ws,
                   cudaStream_t s, const Slab& slab, long long m_total) {
  const int grid = dgrid(m);
  const double count = double(m_total > 0 ? m_total : m);
  IHOM_CUDA(cudaMemsetAsync(ws.flag, 0, sizeof(int), s));
  oc_scale_kernel<<<grid, kDT, 0, s>>>(g, m, ws.partials, ws.flag);
  IHOM_LAUNCH_CHECK();
  finalize_d<<<1, kDT, 0, s>>>(ws.partials, grid, true, ws.scalar);
  IHOM_LAUNCH_CHECK();
  // max scale and the non-finite flag over all slabs (ws.scalars[62..63]); scale back into ws.scalar
  launch_int_to_double(ws.flag, ws.scalars + 62, s);
  IHOM_CUDA(cudaMemcpyAsync(ws.scalars + 63, ws.scalar, sizeof(double), cudaMemcpyDeviceToDevice, s));
  slab.allreduce(ws.scalars + 62, 2, true, s);
  IHOM_CUDA(cudaMemcpyAsync(ws.scalar, ws.scalars + 63, sizeof(double), cudaMemcpyDeviceToDevice, s));
  {
    ProfScope pt(s, "oc_trial", double(m) * 16.0);
    oc_prep_kernel<<<grid, kDT, 0, s>>>(g, m, ws.scalar, out);  // out = sqrt(b0) until the final write
    IHOM_LAUNCH_CHECK();
  }
  OcState init{1e-12, 1e12, 1e-12, 0.0, 0.0, 0.0, 1.0, 0.0};
  OcState* st = reinterpret_cast<OcState*>(ws.scalars);  // scalars[0..7]
  double* sums = ws.scalars + 16;                          // scalars[16..24]
  IHOM_CUDA(cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  const OCParams p{cfg.damp, cfg.step_limit, cfg.min_density, 1.0};
  if (cfg.damp != 0.5) throw std::invalid_argument("the device OC update implements damp = 0.5 (src/oc.cpp:18)");
  // passes in batches (6 first: a typical update needs 5-7), one 8-byte read of the done flag per batch;
  // passes queued after termination exit at once
  for (int pass = 0; pass < kOcMaxPasses;) {
    const int batch = pass == 0 ? 6 : 4;
    for (int b = 0; b < batch && pass < kOcMaxPasses; ++b, ++pass) {
      ProfScope pt(s, "oc_trial", double(m) * 16.0);
      oc_pass_kernel<<<grid, kDT, 0, s>>>(rho, out, m, st, p, ws.partials);
      IHOM_LAUNCH_CHECK();
      if (slab.on()) {
        oc_sums_kernel<<<1, kDT, 0, s>>>(ws.partials, grid, st, sums);
        IHOM_LAUNCH_CHECK();
        slab.allreduce(sums, kOcSlots, false, s);
        oc_decide_kernel<<<1, 1, 0, s>>>(st, sums, count, cfg.volume, cfg.bisect_tol);
      } else {
        oc_sums_decide_kernel<<<1, kDT, 0, s>>>(ws.partials, grid, st, sums, count, cfg.volume, cfg.bisect_tol);
      }
      IHOM_LAUNCH_CHECK();
    }
    double done = 0.0;
    IHOM_CUDA(cudaMemcpyAsync(&done, &st->done, sizeof(double), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    if (done != 0.0) break;
  }
  {
    ProfScope pt(s, "oc_trial", double(m) * 24.0);
    oc_write_kernel<<<grid, kDT, 0, s>>>(rho, out, m, st, p);
    IHOM_LAUNCH_CHECK();
  }
  OcState fin{};
  int bad = 0;
  IHOM_CUDA(cudaMemcpyAsync(&fin, st, sizeof(fin), cudaMemcpyDeviceToHost, s));
  double flag = 0.0;
  IHOM_CUDA(cudaMemcpyAsync(&flag, ws.scalars + 62, sizeof(double), cudaMemcpyDeviceToHost, s));
  double scale = 0.0;
  IHOM_CUDA(cudaMemcpyAsync(&scale, ws.scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
  IHOM_CUDA(cudaStreamSynchronize(s));
  bad = flag != 0.0;
  if (bad) throw std::invalid_argument("non-finite sensitivity");
  OCResult res;
  res.lambda = fin.lambda * scale;
  res.bisection_ok = fin.ok != 0.0;
  res.trials = int(fin.trials);
  return res;
}

}  // namespace ihomgpu

namespace ihomgpu {

// ---------------------------------------------------------------- trig init
// init_trig (src/density.cpp:169-259): the random weights and rotation are
// drawn on the host with the reference's counter-based splitmix64 stream;
// the Q_n basis evaluation and the sigmoid-offset bisection run on device.
constexpr int kMaxTrigW = 48 + 48 * 49 / 2;
__constant__ double c_trig_w[kMaxTrigW];
__constant__ double c_trig_rot[9];

// z-slab: elements [0, nx ny t) of the slab starting at global plane z0
__global__ void trig_eval_kernel(int nx, int ny, int nz, int planes, int z0, int basis_n, double* __restrict__ y) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long m = (long long)nx * ny * planes;
  if (i >= m) return;
  const int n[3] = {nx, ny, nz};
  int e[3];
  e[0] = int(i % nx);
  const long long r = i / nx;
  e[1] = int(r % ny);
  e[2] = z0 + int(r / ny);
  double xb[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    xb[a] = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) xb[a] += c_trig_rot[a * 3 + k] * ((e[k] + 0.5) / double(n[k]) - 0.5);
  }
  double t[48];
  const int nt = 6 * basis_n;
  for (int ax = 0, j = 0; ax < 3; ++ax)
    for (int k = 1; k <= basis_n; ++k) {
      t[j++] = cos(2.0 * M_PI * k * xb[ax]);
      t[j++] = sin(2.0 * M_PI * k * xb[ax]);
    }
  double s = 0.0;
  int j = 0;
  for (int a = 0; a < nt; ++a) s += c_trig_w[j++] * t[a];
  for (int a = 0; a < nt; ++a)
    for (int b = a; b < nt; ++b) s += c_trig_w[j++] * t[a] * t[b];
  y[i] = s;
}

__global__ void minmax_kernel(const double* __restrict__ y, long long m, double* partials) {
  __shared__ double sh[32];
  double lo = INFINITY, hi = -INFINITY;
  for (long long i = (long long)blockIdx.x * kDT + threadIdx.x; i < m; i += (long long)gridDim.x * kDT) {
    lo = fmin(lo, y[i]);
    hi = fmax(hi, y[i]);
  }
  const double rhi = block_reduce_d(hi, sh, true);
  const double rlo = -block_reduce_d(-lo, sh, true);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = rhi;
    partials[kReducePartials + blockIdx.x] = rlo;
  }
}

__global__ void project_kernel(const double* __restrict__ y, long long m, double vhat, double k, double mu,
                               double* __restrict__ rho, double* partials) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * kDT + threadIdx.x; i < m; i += (long long)gridDim.x * kDT) {
    const double v = kRhoMin + vhat / (1.0 + exp(-k * (y[i] - mu)));
    rho[i] = v;
    s += v;
  }
  const double r = block_reduce_d(s, sh, false);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

static std::uint64_t splitmix64(std::uint64_t x) {  // src/density.cpp:154-159
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d449bd133111ebULL;
  return x ^ (x >> 31);
}
static double uniform_pm1(std::uint64_t seed, std::uint64_t counter) {  // :162-165
  const std::uint64_t h = splitmix64(splitmix64(seed) ^ (counter * 0xd1b54a32d192ed03ULL + 1));
  return double(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

bool init_trig(const int n[3], int basis_n, std::uint64_t seed, double volume, double sigmoid_k, double* rho,
               double* scratch, Workspace& ws, cudaStream_t s, const Slab& slab) {
  if (basis_n < 1 || basis_n > 8) throw std::invalid_argument("trig basis order must be in [1, 8]");
  if (!(volume > kRhoMin && volume <= 1.0)) throw std::invalid_argument("volume fraction out of range");
  const int t = n[2] / slab.nranks, z0 = slab.rank * t;
  const long long m = (long long)n[0] * n[1] * t;
  const double count = double((long long)n[0] * n[1] * n[2]);
  const int nt = 6 * basis_n;
  const int nq = nt + nt * (nt + 1) / 2;
  std::vector<double> w(static_cast<size_t>(nq));
  for (int j = 0; j < nq; ++j) w[size_t(j)] = uniform_pm1(seed, std::uint64_t(j));
  double q[4], qn = 0.0;
  for (int j = 0; j < 4; ++j) {
    q[j] = uniform_pm1(seed, std::uint64_t(nq + j));
    qn += q[j] * q[j];
  }
  if (qn < 1e-12) {
    q[0] = 1.0;
    q[1] = q[2] = q[3] = 0.0;
    qn = 1.0;
  }
  qn = std::sqrt(qn);
  for (double& c : q) c /= qn;
  const double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
  const double rot[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy),
                         2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx),
                         2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)};
  {
    std::lock_guard<std::mutex> lock(g_const_mu);
    IHOM_CUDA(cudaMemcpyToSymbolAsync(c_trig_w, w.data(), sizeof(double) * nq, 0, cudaMemcpyHostToDevice, s));
    IHOM_CUDA(cudaMemcpyToSymbolAsync(c_trig_rot, rot, sizeof(rot), 0, cudaMemcpyHostToDevice, s));
    trig_eval_kernel<<<ceil_div(m, 128), 128, 0, s>>>(n[0], n[1], n[2], t, z0, basis_n, scratch);
    IHOM_LAUNCH_CHECK();
    IHOM_CUDA(cudaStreamSynchronize(s));
  }
  double* y = scratch;
  const int grid = dgrid(m);
  minmax_kernel<<<grid, kDT, 0, s>>>(y, m, ws.partials);
  IHOM_LAUNCH_CHECK();
  finalize_d<<<1, kDT, 0, s>>>(ws.partials, grid, true, ws.scalar);
  // min = -max(-x): reuse finalize on the second half
  std::vector<double> mins(static_cast<size_t>(grid));
  double yhi = 0.0;
  IHOM_CUDA(cudaMemcpyAsync(&yhi, ws.scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
  IHOM_CUDA(cudaMemcpyAsync(mins.data(), ws.partials + kReducePartials, sizeof(double) * grid, cudaMemcpyDeviceToHost, s));
  IHOM_CUDA(cudaStreamSynchronize(s));
  double ylo = mins[0];
  for (double v : mins) ylo = std::min(ylo, v);
  if (slab.on()) {  // global extremes: max over slabs of (yhi, -ylo)
    const double ext[2] = {yhi, -ylo};
    IHOM_CUDA(cudaMemcpyAsync(ws.scalars + 60, ext, sizeof(ext), cudaMemcpyHostToDevice, s));
    slab.allreduce(ws.scalars + 60, 2, true, s);
    double g2[2];
    IHOM_CUDA(cudaMemcpyAsync(g2, ws.scalars + 60, sizeof(g2), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    yhi = g2[0];
    ylo = -g2[1];
  }
  const double vhat = std::min(1.5 * volume, 1.0 - kRhoMin);
  const double k = sigmoid_k;
  auto project = [&](double mu) {
    project_kernel<<<grid, kDT, 0, s>>>(y, m, vhat, k, mu, rho, ws.partials);
    IHOM_LAUNCH_CHECK();
    finalize_d<<<1, kDT, 0, s>>>(ws.partials, grid, false, ws.scalar2);
    slab.allreduce(ws.scalar2, 1, false, s);
    double sum = 0.0;
    IHOM_CUDA(cudaMemcpyAsync(&sum, ws.scalar2, sizeof(double), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    return sum / count;
  };
  auto constant = [&]() {
    std::vector<double> c(size_t(m), volume);
    IHOM_CUDA(cudaMemcpyAsync(rho, c.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
  };
  double lo = ylo - 45.0 / k, hi = yhi + 45.0 / k;
  if (!(project(lo) >= volume && project(hi) <= volume)) {
    constant();
    return true;
  }
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double mean = project(mid);
    if (std::abs(mean - volume) <= 1e-4) return false;
    (mean > volume ? lo : hi) = mid;
  }
  if (std::abs(project(0.5 * (lo + hi)) - volume) <= 1e-4) return false;
  constant();
  return true;
}

}  // namespace ihomgpu
