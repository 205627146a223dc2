// ihom_oracle.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Eigen-free CPU restatement of the reference inverse-homogenization hot path
// (/root/reference/proj, abbreviated below: inc/ = proj/include/ihom/, src/ =
// proj/src/). Every function cites the reference file:line it restates. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library.
//
// Parity pins:
//   * density/filter/symmetrize/init_trig/OC are checked BIT-EXACT against the
//     reference's own src/density.cpp + src/oc.cpp compiled into oracle/_ref/;
//   * K0, full-solid C^H, uniform-rho_min, laminate, objective values and the
//     sparse direct (energy identity) oracle reproduce the reference's
//     known-answer tests (tests/test_material.cpp, tests/test_homogenization.cpp,
//     tests/test_objective.cpp, tests/test_runner.cpp);
//   * Eigen (absent here) is replaced by plain loops; the coarsest LDLT by the
//     same diagonal-pivoting LDL^T on a dense matrix (rounding-level difference).
//   * ONE DEVIATION (g_coarse_project, default on, orc_set_coarse_project(0) restores
//     the reference): the coarsest operator is projected onto the translation-free
//     subspace before factoring, see project_translations().
//
// Layouts follow the reference exactly: nodal fields AoS a[3*loc+c] in the
// colour-block order of inc/grid.hpp:73-78, element fields x-fastest.

#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

using I3 = std::array<int, 3>;
using i64 = std::int64_t;

// ---------------------------------------------------------------- parallel
// inc/parallel.hpp:29-56
template <class F>
void parallel_for(i64 n, F&& body) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) body(i);
}

template <class F>
double block_sum(i64 n, F&& term) {
  constexpr i64 kBlock = 4096;
  if (n <= 0) return 0.0;
  const i64 nb = (n + kBlock - 1) / kBlock;
  std::vector<double> partial(size_t(nb), 0.0);
#pragma omp parallel for schedule(static)
  for (i64 b = 0; b < nb; ++b) {
    const i64 lo = b * kBlock, hi = std::min(n, lo + kBlock);
    double s = 0.0;
    for (i64 i = lo; i < hi; ++i) s += term(i);
    partial[size_t(b)] = s;
  }
  for (i64 stride = 1; stride < nb; stride *= 2)
    for (i64 b = 0; b + stride < nb; b += 2 * stride) partial[size_t(b)] += partial[size_t(b + stride)];
  return partial[0];
}

// -------------------------------------------------------------------- grid
// inc/grid.hpp:11-116
inline I3 color_origin(int id) { return {id & 1, (id >> 1) & 1, (id >> 2) & 1}; }

struct Grid {
  I3 n{0, 0, 0};
  std::array<I3, 8> cdim{};
  std::array<i64, 8> cbase{}, csize{};
  Grid() = default;
  explicit Grid(I3 r) : n(r) {  // inc/grid.hpp:29-42
    for (int k = 0; k < 3; ++k)
      if (n[k] < 4) throw std::invalid_argument("grid resolution must be >= 4 per axis");
    i64 base = 0;
    for (int id = 0; id < 8; ++id) {
      const I3 o = color_origin(id);
      for (int k = 0; k < 3; ++k) cdim[id][k] = (n[k] - o[k] + 1) / 2;
      cbase[id] = base;
      csize[id] = i64(cdim[id][0]) * cdim[id][1] * cdim[id][2];
      base += csize[id];
    }
  }
  i64 nv() const { return i64(n[0]) * n[1] * n[2]; }
  bool even() const { return n[0] % 2 == 0 && n[1] % 2 == 0 && n[2] % 2 == 0; }
  bool can_coarsen() const { return even() && n[0] / 2 >= 4 && n[1] / 2 >= 4 && n[2] / 2 >= 4; }
  Grid coarsened() const { return Grid({n[0] / 2, n[1] / 2, n[2] / 2}); }
};

inline I3 wrap(I3 c, const Grid& g) {  // inc/grid.hpp:58-64
  for (int k = 0; k < 3; ++k) {
    c[k] %= g.n[k];
    if (c[k] < 0) c[k] += g.n[k];
  }
  return c;
}
inline int color_of(const I3& v) { return (v[0] & 1) | ((v[1] & 1) << 1) | ((v[2] & 1) << 2); }
inline i64 loc_of(const I3& v, const Grid& g) {  // inc/grid.hpp:73-78
  const int id = color_of(v);
  const I3& d = g.cdim[id];
  return g.cbase[id] + (v[0] >> 1) + (i64(v[1] >> 1) + i64(v[2] >> 1) * d[1]) * d[0];
}
inline I3 vertex_at(i64 loc, const Grid& g) {  // inc/grid.hpp:81-92
  int id = 7;
  while (id > 0 && loc < g.cbase[id]) --id;
  i64 r = loc - g.cbase[id];
  const I3& d = g.cdim[id];
  const I3 o = color_origin(id);
  const int i0 = int(r % d[0]);
  r /= d[0];
  const int i1 = int(r % d[1]);
  const int i2 = int(r / d[1]);
  return {2 * i0 + o[0], 2 * i1 + o[1], 2 * i2 + o[2]};
}
inline I3 lvo(int j) { return {j & 1, (j >> 1) & 1, (j >> 2) & 1}; }  // inc/grid.hpp:95
inline std::array<I3, 8> element_vertices(const I3& e, const Grid& g) {  // :97-104
  std::array<I3, 8> out;
  for (int j = 0; j < 8; ++j) {
    const I3 d = lvo(j);
    out[j] = wrap({e[0] + d[0], e[1] + d[1], e[2] + d[2]}, g);
  }
  return out;
}
inline i64 eidx(const I3& e, const Grid& g) { return e[0] + i64(g.n[0]) * (e[1] + i64(g.n[1]) * e[2]); }
inline I3 element_at(i64 idx, const Grid& g) {  // :112-116
  const int x = int(idx % g.n[0]);
  idx /= g.n[0];
  return {x, int(idx % g.n[1]), int(idx / g.n[1])};
}

// ---------------------------------------------------------------- material
// src/material.cpp:7-82
struct Material {
  double E = 1.0, nu = 0.3;
  double lambda() const { return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)); }
  double mu() const { return E / (2.0 * (1.0 + nu)); }
  void elasticity(double c[6][6]) const {
    std::memset(c, 0, sizeof(double) * 36);
    const double l = lambda(), m = mu();
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) c[i][j] = l;
      c[i][i] = l + 2.0 * m;
      c[3 + i][3 + i] = m;
    }
  }
};

struct K0 {
  double k[24][24];
};

K0 element_stiffness(const Material& mat) {  // src/material.cpp:39-69
  double c[6][6];
  mat.elasticity(c);
  double k[24][24] = {};
  const double gp[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  const double w = 1.0 / 8.0;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int ci = 0; ci < 2; ++ci) {
        const double p[3] = {gp[a], gp[b], gp[ci]};
        double grad[8][3];
        for (int j = 0; j < 8; ++j) {  // shape_gradients, src/material.cpp:22-35
          const I3 d = lvo(j);
          double f[3], g[3];
          for (int kk = 0; kk < 3; ++kk) {
            f[kk] = d[kk] ? p[kk] : 1.0 - p[kk];
            g[kk] = d[kk] ? 1.0 : -1.0;
          }
          grad[j][0] = g[0] * f[1] * f[2];
          grad[j][1] = f[0] * g[1] * f[2];
          grad[j][2] = f[0] * f[1] * g[2];
        }
        double B[6][24] = {};
        for (int j = 0; j < 8; ++j) {
          const int col = 3 * j;
          B[0][col + 0] = grad[j][0];
          B[1][col + 1] = grad[j][1];
          B[2][col + 2] = grad[j][2];
          B[3][col + 0] = grad[j][1];
          B[3][col + 1] = grad[j][0];
          B[4][col + 1] = grad[j][2];
          B[4][col + 2] = grad[j][1];
          B[5][col + 0] = grad[j][2];
          B[5][col + 2] = grad[j][0];
        }
        double CB[6][24];
        for (int r = 0; r < 6; ++r)
          for (int q = 0; q < 24; ++q) {
            double s = 0.0;
            for (int t = 0; t < 6; ++t) s += c[r][t] * B[t][q];
            CB[r][q] = s;
          }
        for (int r = 0; r < 24; ++r)
          for (int q = 0; q < 24; ++q) {
            double s = 0.0;
            for (int t = 0; t < 6; ++t) s += B[t][r] * CB[t][q];
            k[r][q] += w * s;
          }
      }
  K0 out;
  for (int r = 0; r < 24; ++r)
    for (int q = 0; q < 24; ++q) out.k[r][q] = 0.5 * (k[r][q] + k[q][r]);
  return out;
}

void macro_strain_displacement(int i, const I3& x, double out[3]) {  // src/material.cpp:71-82
  const double x0 = x[0], x1 = x[1], x2 = x[2];
  switch (i) {
    case 0: out[0] = x0; out[1] = 0; out[2] = 0; return;
    case 1: out[0] = 0; out[1] = x1; out[2] = 0; return;
    case 2: out[0] = 0; out[1] = 0; out[2] = x2; return;
    case 3: out[0] = x1 / 2.0; out[1] = x0 / 2.0; out[2] = 0; return;
    case 4: out[0] = 0; out[1] = x2 / 2.0; out[2] = x1 / 2.0; return;
    case 5: out[0] = x2 / 2.0; out[1] = 0; out[2] = x0 / 2.0; return;
    default: throw std::invalid_argument("macro strain index must be in [0, 6)");
  }
}

// --------------------------------------------------------------------- fem
// inc/fem.hpp:30-133, src/fem.cpp:10-156
inline int neighbor_index(const I3& t) { return (t[0] + 1) + 3 * (t[1] + 1) + 9 * (t[2] + 1); }
inline I3 neighbor_offset(int idx) { return {idx % 3 - 1, (idx / 3) % 3 - 1, idx / 9 - 1}; }

struct Tables {  // inc/fem.hpp:45-65, src/fem.cpp:10-35
  double blk[8][8][9];
  float blk_f[8][8][9];
  int ngb[8][8];
  double fmacro[8][6][3];
  std::array<std::vector<std::pair<int, int>>, 27> groups;
  explicit Tables(const K0& ks) {
    for (int ke = 0; ke < 8; ++ke) {
      const int row = 7 - ke;
      const I3 de = lvo(ke);
      for (int j = 0; j < 8; ++j) {
        const I3 dj = lvo(j);
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) {
            const double x = ks.k[3 * row + r][3 * j + c];
            blk[ke][j][3 * r + c] = x;
            blk_f[ke][j][3 * r + c] = float(x);
          }
        ngb[ke][j] = neighbor_index({de[0] + dj[0] - 1, de[1] + dj[1] - 1, de[2] + dj[2] - 1});
        groups[size_t(ngb[ke][j])].push_back({ke, j});
      }
      for (int i = 0; i < 6; ++i) {
        double acc[3] = {0, 0, 0};
        for (int j = 0; j < 8; ++j) {
          double chi[3];
          macro_strain_displacement(i, lvo(j), chi);
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) acc[r] += blk[ke][j][3 * r + c] * chi[c];
        }
        for (int r = 0; r < 3; ++r) fmacro[ke][i][r] = acc[r];
      }
    }
  }
  template <typename T>
  const T* flat() const {
    if constexpr (sizeof(T) == sizeof(float)) return &blk_f[0][0][0];
    else return &blk[0][0][0];
  }
};

struct Nbhd {
  i64 vloc[27];
  i64 eix[8];
};

void gather_neighborhood(const Grid& g, const I3& v, Nbhd& nb) {  // src/fem.cpp:37-68
  int par[3][3], half[3][3], ec[3][2];
  for (int k = 0; k < 3; ++k) {
    const int n = g.n[k], x = v[k];
    const int xm = (x == 0) ? n - 1 : x - 1;
    const int xp = (x + 1 == n) ? 0 : x + 1;
    par[k][0] = xm & 1; par[k][1] = x & 1; par[k][2] = xp & 1;
    half[k][0] = xm >> 1; half[k][1] = x >> 1; half[k][2] = xp >> 1;
    ec[k][0] = xm; ec[k][1] = x;
  }
  int idx = 0;
  for (int t2 = 0; t2 < 3; ++t2)
    for (int t1 = 0; t1 < 3; ++t1)
      for (int t0 = 0; t0 < 3; ++t0, ++idx) {
        const int id = par[0][t0] | (par[1][t1] << 1) | (par[2][t2] << 2);
        const I3& d = g.cdim[id];
        nb.vloc[idx] = g.cbase[id] + half[0][t0] + (i64(half[1][t1]) + i64(half[2][t2]) * d[1]) * d[0];
      }
  for (int ke = 0; ke < 8; ++ke)
    nb.eix[ke] = ec[0][ke & 1] + i64(g.n[0]) * (ec[1][(ke >> 1) & 1] + i64(g.n[1]) * ec[2][(ke >> 2) & 1]);
}

void solve3(const double m[9], const double rhs[3], double out[3]) {  // src/fem.cpp:72-94
  double a[9];
  std::memcpy(a, m, sizeof(a));
  double b[3] = {rhs[0], rhs[1], rhs[2]};
  int piv[3] = {0, 1, 2};
  for (int c = 0; c < 3; ++c) {
    int best = c;
    for (int r = c + 1; r < 3; ++r)
      if (std::abs(a[3 * piv[r] + c]) > std::abs(a[3 * piv[best] + c])) best = r;
    std::swap(piv[c], piv[best]);
    const double d = a[3 * piv[c] + c];
    for (int r = c + 1; r < 3; ++r) {
      const double fac = a[3 * piv[r] + c] / d;
      for (int cc = c; cc < 3; ++cc) a[3 * piv[r] + cc] -= fac * a[3 * piv[c] + cc];
      b[piv[r]] -= fac * b[piv[c]];
    }
  }
  for (int c = 2; c >= 0; --c) {
    double s = b[piv[c]];
    for (int cc = c + 1; cc < 3; ++cc) s -= a[3 * piv[c] + cc] * out[cc];
    out[c] = s / a[3 * piv[c] + c];
  }
}

template <typename T>
inline void vertex_apply(const Tables& tab, const T* coeff, const Nbhd& nb, const double* u, double y[3]) {
  // inc/fem.hpp:86-105
  const T* blocks = tab.flat<T>();
  y[0] = y[1] = y[2] = 0.0;
  T q[8];
  for (int ke = 0; ke < 8; ++ke) q[ke] = coeff[nb.eix[ke]];
  for (int n = 0; n < 27; ++n) {
    T c[9] = {};
    for (const auto& pr : tab.groups[size_t(n)]) {
      const T w = q[pr.first];
      const T* b = blocks + (pr.first * 8 + pr.second) * 9;
      for (int e = 0; e < 9; ++e) c[e] += w * b[e];
    }
    const double* un = u + 3 * nb.vloc[n];
    y[0] += double(c[0]) * un[0] + double(c[1]) * un[1] + double(c[2]) * un[2];
    y[1] += double(c[3]) * un[0] + double(c[4]) * un[1] + double(c[5]) * un[2];
    y[2] += double(c[6]) * un[0] + double(c[7]) * un[1] + double(c[8]) * un[2];
  }
}

template <typename T>
inline void vertex_split_apply(const Tables& tab, const T* coeff, const Nbhd& nb, const double* u,
                               double s[9], double m[3]) {  // inc/fem.hpp:109-133
  const T* blocks = tab.flat<T>();
  m[0] = m[1] = m[2] = 0.0;
  T q[8];
  for (int ke = 0; ke < 8; ++ke) q[ke] = coeff[nb.eix[ke]];
  for (int n = 0; n < 27; ++n) {
    T c[9] = {};
    for (const auto& pr : tab.groups[size_t(n)]) {
      const T w = q[pr.first];
      const T* b = blocks + (pr.first * 8 + pr.second) * 9;
      for (int e = 0; e < 9; ++e) c[e] += w * b[e];
    }
    if (n == 13) {
      for (int e = 0; e < 9; ++e) s[e] = double(c[e]);
      continue;
    }
    const double* un = u + 3 * nb.vloc[n];
    m[0] += double(c[0]) * un[0] + double(c[1]) * un[1] + double(c[2]) * un[2];
    m[1] += double(c[3]) * un[0] + double(c[4]) * un[1] + double(c[5]) * un[2];
    m[2] += double(c[6]) * un[0] + double(c[7]) * un[1] + double(c[8]) * un[2];
  }
}

template <typename T>
void apply_kernel(const Grid& g, const Tables& tab, const T* coeff, const double* u, double* y) {
  parallel_for(g.nv(), [&](i64 loc) {  // src/fem.cpp:98-106
    Nbhd nb;
    gather_neighborhood(g, vertex_at(loc, g), nb);
    vertex_apply(tab, coeff, nb, u, y + 3 * loc);
  });
}

template <typename T>
void residual_kernel(const Grid& g, const Tables& tab, const T* coeff, const double* u, const double* f,
                     double* r) {
  parallel_for(g.nv(), [&](i64 loc) {  // src/fem.cpp:108-120
    Nbhd nb;
    gather_neighborhood(g, vertex_at(loc, g), nb);
    double y[3];
    vertex_apply(tab, coeff, nb, u, y);
    for (int c = 0; c < 3; ++c) r[3 * loc + c] = f[3 * loc + c] - y[c];
  });
}

template <typename T>
void gs_kernel(const Grid& g, const Tables& tab, const T* coeff, const double* f, double* u) {
  for (int color = 0; color < 8; ++color) {  // src/fem.cpp:122-137
    const i64 base = g.cbase[color];
    parallel_for(g.csize[color], [&](i64 i) {
      const i64 loc = base + i;
      Nbhd nb;
      gather_neighborhood(g, vertex_at(loc, g), nb);
      double s[9], m[3];
      vertex_split_apply(tab, coeff, nb, u, s, m);
      const double rhs[3] = {f[3 * loc] - m[0], f[3 * loc + 1] - m[1], f[3 * loc + 2] - m[2]};
      solve3(s, rhs, u + 3 * loc);
    });
  }
}

template <typename T>
void macro_force_kernel(const Grid& g, const Tables& tab, const T* coeff, int load, double* f) {
  parallel_for(g.nv(), [&](i64 loc) {  // src/fem.cpp:139-156
    Nbhd nb;
    gather_neighborhood(g, vertex_at(loc, g), nb);
    double y[3] = {0, 0, 0};
    for (int ke = 0; ke < 8; ++ke) {
      const double q = double(coeff[nb.eix[ke]]);
      for (int c = 0; c < 3; ++c) y[c] += q * tab.fmacro[ke][load][c];
    }
    for (int c = 0; c < 3; ++c) f[3 * loc + c] = y[c];
  });
}

// --------------------------------------------------------------- multigrid
// src/multigrid.cpp:12-94
inline double tw1(int c) {
  const int a = c < 0 ? -c : c;
  return a >= 2 ? 0.0 : (2.0 - a) / 2.0;
}

struct Field {  // inc/fem.hpp:15-26
  Grid grid;
  std::vector<double> a;
  Field() = default;
  explicit Field(const Grid& g) : grid(g), a(size_t(3 * g.nv()), 0.0) {}
  void zero() { std::fill(a.begin(), a.end(), 0.0); }
};

void restrict_field(const Field& fr, Field& cf) {  // src/multigrid.cpp:19-41
  const Grid& gc = cf.grid;
  const Grid& gf = fr.grid;
  parallel_for(gc.nv(), [&](i64 loc) {
    const I3 vc = vertex_at(loc, gc);
    double acc[3] = {0, 0, 0};
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const double w = tw1(dx) * tw1(dy) * tw1(dz);
          const I3 vf = wrap({2 * vc[0] + dx, 2 * vc[1] + dy, 2 * vc[2] + dz}, gf);
          const double* rv = fr.a.data() + 3 * loc_of(vf, gf);
          for (int c = 0; c < 3; ++c) acc[c] += w * rv[c];
        }
    for (int c = 0; c < 3; ++c) cf.a[size_t(3 * loc + c)] = acc[c];
  });
}

void prolong_add(const Field& cu, Field& fu) {  // src/multigrid.cpp:43-79
  const Grid& gc = cu.grid;
  const Grid& gf = fu.grid;
  parallel_for(gf.nv(), [&](i64 loc) {
    const I3 vf = vertex_at(loc, gf);
    double acc[3] = {0, 0, 0};
    int base[3], cnt[3];
    double w1[3];
    for (int k = 0; k < 3; ++k) {
      if (vf[k] % 2 == 0) { base[k] = vf[k] / 2; cnt[k] = 1; w1[k] = 1.0; }
      else { base[k] = (vf[k] - 1) / 2; cnt[k] = 2; w1[k] = 0.5; }
    }
    for (int a = 0; a < cnt[0]; ++a)
      for (int b = 0; b < cnt[1]; ++b)
        for (int c = 0; c < cnt[2]; ++c) {
          const I3 vc = wrap({base[0] + a, base[1] + b, base[2] + c}, gc);
          const double w = w1[0] * w1[1] * w1[2];
          const double* uv = cu.a.data() + 3 * loc_of(vc, gc);
          for (int d = 0; d < 3; ++d) acc[d] += w * uv[d];
        }
    for (int d = 0; d < 3; ++d) fu.a[size_t(3 * loc + d)] += acc[d];
  });
}

void remove_translations(Field& f) {  // src/multigrid.cpp:81-86
  const i64 nv = f.grid.nv();
  for (int c = 0; c < 3; ++c) {
    const double mean = block_sum(nv, [&](i64 i) { return f.a[size_t(3 * i + c)]; }) / double(nv);
    parallel_for(nv, [&](i64 i) { f.a[size_t(3 * i + c)] -= mean; });
  }
}
double field_dot(const Field& a, const Field& b) {  // :88-91
  return block_sum(i64(a.a.size()), [&](i64 i) { return a.a[size_t(i)] * b.a[size_t(i)]; });
}
double field_norm(const Field& f) { return std::sqrt(field_dot(f, f)); }

struct ElementGalerkinTable {  // src/multigrid.cpp:102-149
  struct Term { int ngb; double w[9]; };
  std::array<std::vector<Term>, 64> terms;
  explicit ElementGalerkinTable(const K0& ks) {
    for (int oz = -2; oz <= 1; ++oz)
      for (int oy = -2; oy <= 1; ++oy)
        for (int ox = -2; ox <= 1; ++ox) {
          const int oidx = (ox + 2) + 4 * ((oy + 2) + 4 * (oz + 2));
          for (int n = 0; n < 27; ++n) {
            const I3 delta = neighbor_offset(n);
            double acc[9] = {};
            bool any = false;
            for (int i = 0; i < 8; ++i) {
              const I3 di = lvo(i);
              const double wi = tw1(ox + di[0]) * tw1(oy + di[1]) * tw1(oz + di[2]);
              if (wi == 0.0) continue;
              for (int j = 0; j < 8; ++j) {
                const I3 dj = lvo(j);
                const double wj = tw1(ox + dj[0] - 2 * delta[0]) * tw1(oy + dj[1] - 2 * delta[1]) *
                                  tw1(oz + dj[2] - 2 * delta[2]);
                if (wj == 0.0) continue;
                any = true;
                for (int r = 0; r < 3; ++r)
                  for (int c = 0; c < 3; ++c) acc[3 * r + c] += wi * wj * ks.k[3 * i + r][3 * j + c];
              }
            }
            if (any) {
              Term t;
              t.ngb = n;
              for (int e = 0; e < 9; ++e) t.w[e] = acc[e];
              terms[size_t(oidx)].push_back(t);
            }
          }
        }
  }
};

struct StencilGalerkinTable {  // src/multigrid.cpp:151-182
  struct Term { int s, t; double w; };
  std::array<std::vector<Term>, 27> terms;
  StencilGalerkinTable() {
    for (int n = 0; n < 27; ++n) {
      const I3 delta = neighbor_offset(n);
      for (int s = 0; s < 27; ++s) {
        const I3 so = neighbor_offset(s);
        const double ws = tw1(so[0]) * tw1(so[1]) * tw1(so[2]);
        for (int t = 0; t < 27; ++t) {
          const I3 to = neighbor_offset(t);
          const double wt = tw1(so[0] + to[0] - 2 * delta[0]) * tw1(so[1] + to[1] - 2 * delta[1]) *
                            tw1(so[2] + to[2] - 2 * delta[2]);
          if (ws * wt != 0.0) terms[size_t(n)].push_back({s, t, ws * wt});
        }
      }
    }
  }
};

template <typename T>
void stencil_apply(const Grid& g, const std::vector<T>& st, const double* x, double* y) {
  parallel_for(g.nv(), [&](i64 loc) {  // src/multigrid.cpp:186-205
    Nbhd nb;
    gather_neighborhood(g, vertex_at(loc, g), nb);
    const T* row = st.data() + 243 * loc;
    double acc[3] = {0, 0, 0};
    for (int n = 0; n < 27; ++n) {
      const double* xn = x + 3 * nb.vloc[n];
      const T* b = row + 9 * n;
      acc[0] += double(b[0]) * xn[0] + double(b[1]) * xn[1] + double(b[2]) * xn[2];
      acc[1] += double(b[3]) * xn[0] + double(b[4]) * xn[1] + double(b[5]) * xn[2];
      acc[2] += double(b[6]) * xn[0] + double(b[7]) * xn[1] + double(b[8]) * xn[2];
    }
    for (int c = 0; c < 3; ++c) y[3 * loc + c] = acc[c];
  });
}

template <typename T>
void stencil_gs(const Grid& g, const std::vector<T>& st, const double* f, double* u) {
  for (int color = 0; color < 8; ++color) {  // src/multigrid.cpp:207-239
    const i64 base = g.cbase[color];
    parallel_for(g.csize[color], [&](i64 i) {
      const i64 loc = base + i;
      Nbhd nb;
      gather_neighborhood(g, vertex_at(loc, g), nb);
      const T* row = st.data() + 243 * loc;
      double m[3] = {0, 0, 0}, s[9];
      for (int n = 0; n < 27; ++n) {
        const T* b = row + 9 * n;
        if (n == 13) {
          for (int e = 0; e < 9; ++e) s[e] = double(b[e]);
          continue;
        }
        const double* un = u + 3 * nb.vloc[n];
        m[0] += double(b[0]) * un[0] + double(b[1]) * un[1] + double(b[2]) * un[2];
        m[1] += double(b[3]) * un[0] + double(b[4]) * un[1] + double(b[5]) * un[2];
        m[2] += double(b[6]) * un[0] + double(b[7]) * un[1] + double(b[8]) * un[2];
      }
      const double rhs[3] = {f[3 * loc] - m[0], f[3 * loc + 1] - m[1], f[3 * loc + 2] - m[2]};
      const double det = s[0] * (s[4] * s[8] - s[5] * s[7]) - s[1] * (s[3] * s[8] - s[5] * s[6]) +
                         s[2] * (s[3] * s[7] - s[4] * s[6]);
      if (det == 0.0 || !std::isfinite(det)) throw std::runtime_error("non-invertible coarse stencil diagonal");
      solve3(s, rhs, u + 3 * loc);
    });
  }
}

struct SolverOptions {  // inc/multigrid.hpp:22-27
  double tol = 1e-2;
  int max_cycles = 50;
  int pre_sweeps = 1;
  int post_sweeps = 1;
};
struct SolveStats {  // inc/multigrid.hpp:29-33
  int cycles = 0;
  double rel_residual = 0.0;
  bool converged = false;
};

template <typename T>
struct Level {  // inc/multigrid.hpp:38-46
  Grid grid;
  Field u, f, r;
  std::vector<T> coeff, stencil;
  explicit Level(const Grid& g) : grid(g), u(g), f(g), r(g) {}
};

// Coarsest-operator deviation switch (default on): project the assembled operator onto the
// translation-free subspace, a <- P a P (P = I - (1/nv) sum_c t_c t_c^T), before the shift.
// The reference factors the raw operator (src/multigrid.cpp:368-383); with f32 Galerkin
// stencils A t_c ~ 1e-7 op_scale and on designs with floating islands its refinement stalls
// above the 1e-3 gate and throws (src/multigrid.cpp:446-447) -- 0 restores that behaviour.
int g_coarse_project = 1;

void project_translations(std::vector<double>& a, i64 nv) {
  const i64 N = 3 * nv;
  std::vector<double> b(a.size());
  // row means of every component block (aP), then column means ((aP) -> P(aP))
  for (i64 i = 0; i < N; ++i) {
    double m[3] = {0, 0, 0};
    for (i64 j = 0; j < N; ++j) m[j % 3] += a[size_t(i * N + j)];
    for (i64 j = 0; j < N; ++j) b[size_t(i * N + j)] = a[size_t(i * N + j)] - m[j % 3] / double(nv);
  }
  for (i64 j = 0; j < N; ++j) {
    double m[3] = {0, 0, 0};
    for (i64 i = 0; i < N; ++i) m[i % 3] += b[size_t(i * N + j)];
    for (i64 i = 0; i < N; ++i) a[size_t(i * N + j)] = b[size_t(i * N + j)] - m[i % 3] / double(nv);
  }
  for (i64 i = 0; i < N; ++i)
    for (i64 j = 0; j < i; ++j) {
      const double s = 0.5 * (a[size_t(i * N + j)] + a[size_t(j * N + i)]);
      a[size_t(i * N + j)] = a[size_t(j * N + i)] = s;
    }
}

// Dense LDL^T with symmetric diagonal pivoting: Eigen::LDLT's algorithm
// (src/multigrid.cpp:380 coarse_ldlt_.compute), pivot = largest remaining |diagonal|.
struct DenseLDLT {
  int n = 0;
  std::vector<double> L;  // unit lower below the diagonal, D on the diagonal
  std::vector<int> perm;  // position -> original index
  void compute(std::vector<double> a, int dim) {
    n = dim;
    perm.resize(size_t(n));
    for (int i = 0; i < n; ++i) perm[size_t(i)] = i;
    for (int k = 0; k < n; ++k) {
      int p = k;
      for (int i = k + 1; i < n; ++i)
        if (std::fabs(a[size_t(i) * n + i]) > std::fabs(a[size_t(p) * n + p])) p = i;
      if (p != k) {
        for (int j = 0; j < n; ++j) std::swap(a[size_t(k) * n + j], a[size_t(p) * n + j]);
        for (int i = 0; i < n; ++i) std::swap(a[size_t(i) * n + k], a[size_t(i) * n + p]);
        std::swap(perm[size_t(k)], perm[size_t(p)]);
      }
      double d = a[size_t(k) * n + k];
      for (int j = 0; j < k; ++j) d -= a[size_t(k) * n + j] * a[size_t(k) * n + j] * a[size_t(j) * n + j];
      if (!(std::fabs(d) > 0.0) || !std::isfinite(d)) throw std::runtime_error("coarsest-level factorization failed");
      a[size_t(k) * n + k] = d;
      for (int i = k + 1; i < n; ++i) {
        double s = a[size_t(i) * n + k];
        for (int j = 0; j < k; ++j) s -= a[size_t(i) * n + j] * a[size_t(k) * n + j] * a[size_t(j) * n + j];
        a[size_t(i) * n + k] = s / d;
      }
    }
    L = std::move(a);
  }
  std::vector<double> solve(const std::vector<double>& b) const {
    std::vector<double> y(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) y[size_t(i)] = b[size_t(perm[size_t(i)])];
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < i; ++k) y[size_t(i)] -= L[size_t(i) * n + k] * y[size_t(k)];
    for (int i = 0; i < n; ++i) y[size_t(i)] /= L[size_t(i) * n + i];
    for (int i = n - 1; i >= 0; --i)
      for (int k = i + 1; k < n; ++k) y[size_t(i)] -= L[size_t(k) * n + i] * y[size_t(k)];
    std::vector<double> x(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) x[size_t(perm[size_t(i)])] = y[size_t(i)];
    return x;
  }
};

// Coarsest dense solve (src/multigrid.cpp:368-383 factor, :426-451 solve) on an assembled
// operator `raw` in dof order 3*loc + c. solve() takes the translation-free load and returns the
// relative residual after refinement; the caller applies the 1e-3 singularity gate.
std::string g_dump_path;  // non-empty: dump (raw operator, load) of a failing coarsest solve here

struct CoarseSolver {
  i64 nv = 0;
  double op_scale = 0.0;
  std::vector<double> raw, cmat;
  std::vector<std::vector<double>> nulls;  // deflated near-null directions (orthonormal, translation-free)
  DenseLDLT ldlt;
  // The deviation (g_coarse_project) also deflates near-null modes beyond the translations: trailing
  // pivots of the diagonal-pivoted LDL^T below 1e-6 op_scale (floating islands of the design, ~1e-8 op_scale:
  // under the f32 stencils' resolution, so their amplified solution components are rounding noise) give
  // directions v = Pm^T L^-T e_k; orthonormalised against the translations they are projected off the
  // operator and the load and shifted like the translations.
  void factor(std::vector<double> a, i64 nverts) {
    nv = nverts;
    const i64 N = 3 * nv;
    raw = a;
    double dsum = 0.0;
    for (i64 i = 0; i < N; ++i) dsum += a[size_t(i * N + i)];
    op_scale = dsum / double(N);  // :373
    nulls.clear();
    auto shifted = [&](const std::vector<double>& m) {  // :374-379 deflation shift (+ near-null modes)
      std::vector<double> b = m;
      for (i64 i = 0; i < nv; ++i)
        for (i64 j = 0; j < nv; ++j)
          for (int c = 0; c < 3; ++c) b[size_t((3 * i + c) * N + 3 * j + c)] += op_scale / double(nv);
      for (const auto& q : nulls)
        for (i64 i = 0; i < N; ++i)
          for (i64 j = 0; j < N; ++j) b[size_t(i * N + j)] += op_scale * q[size_t(i)] * q[size_t(j)];
      return b;
    };
    if (g_coarse_project) {
      project_translations(a, nv);
      DenseLDLT probe;
      probe.compute(shifted(a), int(N));
      for (int k = 0; k < int(N); ++k) {
        if (!(std::fabs(probe.L[size_t(k) * N + k]) < 1e-6 * op_scale)) continue;
        std::vector<double> y(static_cast<size_t>(N), 0.0);  // L^T y = e_k
        y[size_t(k)] = 1.0;
        for (int i = k - 1; i >= 0; --i)
          for (int j = i + 1; j <= k; ++j) y[size_t(i)] -= probe.L[size_t(j) * N + i] * y[size_t(j)];
        std::vector<double> v(static_cast<size_t>(N));
        for (i64 i = 0; i < N; ++i) v[size_t(probe.perm[size_t(i)])] = y[size_t(i)];
        for (int rep = 0; rep < 2; ++rep) {
          for (int c = 0; c < 3; ++c) {
            double m = 0.0;
            for (i64 i = 0; i < nv; ++i) m += v[size_t(3 * i + c)];
            for (i64 i = 0; i < nv; ++i) v[size_t(3 * i + c)] -= m / double(nv);
          }
          for (const auto& q : nulls) {
            double d = 0.0;
            for (i64 i = 0; i < N; ++i) d += q[size_t(i)] * v[size_t(i)];
            for (i64 i = 0; i < N; ++i) v[size_t(i)] -= d * q[size_t(i)];
          }
        }
        double nn = 0.0;
        for (double t : v) nn += t * t;
        if (!(nn > 0.0)) continue;
        for (double& t : v) t /= std::sqrt(nn);
        nulls.push_back(std::move(v));
      }
      for (const auto& q : nulls) {  // a <- (I - q q^T) a (I - q q^T)
        std::vector<double> aq(size_t(N), 0.0);
        for (i64 i = 0; i < N; ++i)
          for (i64 j = 0; j < N; ++j) aq[size_t(i)] += a[size_t(i * N + j)] * q[size_t(j)];
        double qaq = 0.0;
        for (i64 i = 0; i < N; ++i) qaq += q[size_t(i)] * aq[size_t(i)];
        for (i64 i = 0; i < N; ++i)
          for (i64 j = 0; j < N; ++j)
            a[size_t(i * N + j)] += qaq * q[size_t(i)] * q[size_t(j)] - aq[size_t(i)] * q[size_t(j)] - q[size_t(i)] * aq[size_t(j)];
      }
      if (!nulls.empty())
        for (i64 i = 0; i < N; ++i)
          for (i64 j = 0; j < i; ++j) {
            const double t = 0.5 * (a[size_t(i * N + j)] + a[size_t(j * N + i)]);
            a[size_t(i * N + j)] = a[size_t(j * N + i)] = t;
          }
    }
    cmat = a;
    ldlt.compute(shifted(a), int(N));
  }
  void project_load(std::vector<double>& fv) const {  // f -= q (q . f) over the deflated modes
    for (const auto& q : nulls) {
      double d = 0.0;
      for (size_t i = 0; i < fv.size(); ++i) d += q[i] * fv[i];
      for (size_t i = 0; i < fv.size(); ++i) fv[i] -= d * q[i];
    }
  }
  std::vector<double> mul(const std::vector<double>& x) const {
    const size_t N = x.size();
    std::vector<double> y(N, 0.0);
    for (size_t i = 0; i < N; ++i) {
      double s = 0.0;
      for (size_t j = 0; j < N; ++j) s += cmat[i * N + j] * x[j];
      y[i] = s;
    }
    return y;
  }
  double resid(const std::vector<double>& x, const std::vector<double>& f) const {
    const std::vector<double> ax = mul(x);
    double s = 0.0;
    for (size_t i = 0; i < f.size(); ++i) s += (ax[i] - f[i]) * (ax[i] - f[i]);
    return std::sqrt(s);
  }
  double solve(const std::vector<double>& fv, double fn, std::vector<double>& x) const {  // :434-447
    x = ldlt.solve(fv);
    double rel = resid(x, fv) / fn;
    for (int it = 0; it < 3 && rel > 1e-9; ++it) {
      const std::vector<double> ax = mul(x);
      std::vector<double> r(fv.size());
      for (size_t i = 0; i < r.size(); ++i) r[i] = fv[i] - ax[i];
      const std::vector<double> dx = ldlt.solve(r);
      for (size_t i = 0; i < x.size(); ++i) x[i] += dx[i];
      rel = resid(x, fv) / fn;
    }
    return rel;
  }
  void dump(const std::vector<double>& fv) const {
    if (g_dump_path.empty()) return;
    FILE* fp = std::fopen(g_dump_path.c_str(), "wb");
    if (!fp) return;
    const long long hdr[2] = {nv, 3 * nv};
    std::fwrite(hdr, sizeof(hdr), 1, fp);
    std::fwrite(raw.data(), sizeof(double), raw.size(), fp);
    std::fwrite(fv.data(), sizeof(double), fv.size(), fp);
    std::fclose(fp);
  }
};

template <typename T>
class Hierarchy {  // inc/multigrid.hpp:53-93, src/multigrid.cpp:245-501
 public:
  Hierarchy(const Grid& root, const Material& mat, double penal)
      : penal_(penal), ks_(element_stiffness(mat)), tab_(ks_) {
    Grid g = root;
    levels_.emplace_back(g);
    while (g.can_coarsen()) {
      g = g.coarsened();
      levels_.emplace_back(g);
    }
    for (size_t l = 1; l < levels_.size(); ++l) levels_[l].stencil.assign(size_t(243 * levels_[l].grid.nv()), T(0));
  }
  int num_levels() const { return int(levels_.size()); }
  Level<T>& level(int l) { return levels_[size_t(l)]; }
  const Tables& tables() const { return tab_; }
  const K0& ks() const { return ks_; }
  double op_scale() const { return op_scale_; }
  const Grid& level0_grid() const { return levels_[0].grid; }

  void set_density(const std::vector<double>& rho) {  // src/multigrid.cpp:263-279
    Level<T>& l0 = levels_[0];
    if (i64(rho.size()) != l0.grid.nv()) throw std::invalid_argument("density resolution does not match the hierarchy");
    l0.coeff.resize(size_t(l0.grid.nv()));
    const double p = penal_;
    parallel_for(l0.grid.nv(), [&](i64 i) { l0.coeff[size_t(i)] = T(std::pow(double(T(rho[size_t(i)])), p)); });
    if (levels_.size() > 1) {
      assemble_from_elements(1);
      for (int l = 2; l < num_levels(); ++l) assemble_from_stencil(l);
    }
    factor_coarsest();
    density_set_ = true;
  }

  void apply(int l, const Field& x, Field& y) const {  // :392-398
    const Level<T>& lev = levels_[size_t(l)];
    if (l == 0) apply_kernel<T>(lev.grid, tab_, lev.coeff.data(), x.a.data(), y.a.data());
    else stencil_apply<T>(lev.grid, lev.stencil, x.a.data(), y.a.data());
  }
  void relax(int l, int sweeps) {  // :400-408
    Level<T>& lev = levels_[size_t(l)];
    for (int s = 0; s < sweeps; ++s) {
      if (l == 0) gs_kernel<T>(lev.grid, tab_, lev.coeff.data(), lev.f.a.data(), lev.u.a.data());
      else stencil_gs<T>(lev.grid, lev.stencil, lev.f.a.data(), lev.u.a.data());
    }
  }
  void compute_residual(int l) {  // :410-424
    Level<T>& lev = levels_[size_t(l)];
    if (l == 0) residual_kernel<T>(lev.grid, tab_, lev.coeff.data(), lev.u.a.data(), lev.f.a.data(), lev.r.a.data());
    else {
      stencil_apply<T>(lev.grid, lev.stencil, lev.u.a.data(), lev.r.a.data());
      parallel_for(i64(lev.r.a.size()), [&](i64 i) { lev.r.a[size_t(i)] = lev.f.a[size_t(i)] - lev.r.a[size_t(i)]; });
    }
  }
  double negligible_load(const Field& f) const { return 1e-12 * op_scale_ * std::sqrt(double(f.a.size())); }

  void coarsest_solve() {  // :426-451
    Level<T>& lev = levels_.back();
    remove_translations(lev.f);
    coarse_.project_load(lev.f.a);
    const std::vector<double>& fv = lev.f.a;
    double fn = 0.0;
    for (double x : fv) fn += x * x;
    fn = std::sqrt(fn);
    if (fn <= negligible_load(lev.f)) {
      lev.u.zero();
      return;
    }
    std::vector<double> x;
    if (fn > 0.0) {
      const double rel = coarse_.solve(fv, fn, x);
      if (!(rel < 1e-3)) {
        coarse_.dump(fv);
        throw std::runtime_error("coarsest operator is singular beyond translations");
      }
    } else {
      x = coarse_.ldlt.solve(fv);
    }
    lev.u.a = x;
    remove_translations(lev.u);
  }

  double v_cycle(const SolverOptions& opts) {  // :453-472
    if (!density_set_) throw std::logic_error("set_density before v_cycle");
    const int lmax = num_levels() - 1;
    for (int l = 0; l < lmax; ++l) {
      if (l > 0) levels_[size_t(l)].u.zero();
      relax(l, opts.pre_sweeps);
      compute_residual(l);
      restrict_field(levels_[size_t(l)].r, levels_[size_t(l + 1)].f);
    }
    if (lmax > 0) levels_[size_t(lmax)].u.zero();
    coarsest_solve();
    for (int l = lmax - 1; l >= 0; --l) {
      prolong_add(levels_[size_t(l + 1)].u, levels_[size_t(l)].u);
      relax(l, opts.post_sweeps);
    }
    compute_residual(0);
    const double fn = field_norm(levels_[0].f);
    return fn > 0.0 ? field_norm(levels_[0].r) / fn : 0.0;
  }

  SolveStats solve(const Field& fload, Field& u, const SolverOptions& opts) {  // :474-501
    if (!density_set_) throw std::logic_error("set_density before solve");
    Level<T>& l0 = levels_[0];
    l0.f.a = fload.a;
    remove_translations(l0.f);
    l0.u.a = u.a;
    SolveStats st;
    const double fn = field_norm(l0.f);
    if (fn <= negligible_load(l0.f)) {
      u.zero();
      l0.u.zero();
      st.converged = true;
      return st;
    }
    compute_residual(0);
    st.rel_residual = field_norm(l0.r) / fn;
    while (st.rel_residual > opts.tol && st.cycles < opts.max_cycles) {
      st.rel_residual = v_cycle(opts);
      ++st.cycles;
    }
    st.converged = st.rel_residual <= opts.tol;
    remove_translations(l0.u);
    u.a = l0.u.a;
    return st;
  }


 private:
  void assemble_from_elements(int coarse) {  // :281-305
    const ElementGalerkinTable table(ks_);
    Level<T>& lc = levels_[size_t(coarse)];
    const Level<T>& lf = levels_[size_t(coarse - 1)];
    const Grid& gc = lc.grid;
    const Grid& gf = lf.grid;
    parallel_for(gc.nv(), [&](i64 loc) {
      const I3 vc = vertex_at(loc, gc);
      double acc[27][9] = {};
      for (int oz = -2; oz <= 1; ++oz)
        for (int oy = -2; oy <= 1; ++oy)
          for (int ox = -2; ox <= 1; ++ox) {
            const I3 ef = wrap({2 * vc[0] + ox, 2 * vc[1] + oy, 2 * vc[2] + oz}, gf);
            const double q = double(lf.coeff[size_t(eidx(ef, gf))]);
            const int oidx = (ox + 2) + 4 * ((oy + 2) + 4 * (oz + 2));
            for (const auto& t : table.terms[size_t(oidx)])
              for (int e = 0; e < 9; ++e) acc[t.ngb][e] += q * t.w[e];
          }
      T* row = lc.stencil.data() + 243 * loc;
      for (int n = 0; n < 27; ++n)
        for (int e = 0; e < 9; ++e) row[9 * n + e] = T(acc[n][e]);
    });
  }
  void assemble_from_stencil(int coarse) {  // :307-333
    static const StencilGalerkinTable table;
    Level<T>& lc = levels_[size_t(coarse)];
    const Level<T>& lf = levels_[size_t(coarse - 1)];
    const Grid& gc = lc.grid;
    const Grid& gf = lf.grid;
    parallel_for(gc.nv(), [&](i64 loc) {
      const I3 vc = vertex_at(loc, gc);
      i64 fl[27];
      for (int s = 0; s < 27; ++s) {
        const I3 so = neighbor_offset(s);
        fl[s] = loc_of(wrap({2 * vc[0] + so[0], 2 * vc[1] + so[1], 2 * vc[2] + so[2]}, gf), gf);
      }
      T* row = lc.stencil.data() + 243 * loc;
      for (int n = 0; n < 27; ++n) {
        double acc[9] = {};
        for (const auto& t : table.terms[size_t(n)]) {
          const T* b = lf.stencil.data() + 243 * fl[t.s] + 9 * t.t;
          for (int e = 0; e < 9; ++e) acc[e] += t.w * double(b[e]);
        }
        for (int e = 0; e < 9; ++e) row[9 * n + e] = T(acc[e]);
      }
    });
  }
  std::vector<double> assemble_dense(int l) const {  // :335-366
    const Level<T>& lev = levels_[size_t(l)];
    const Grid& g = lev.grid;
    const i64 nv = g.nv();
    const i64 N = 3 * nv;
    std::vector<double> a(size_t(N * N), 0.0);
    if (l == 0) {
      for (i64 ei = 0; ei < nv; ++ei) {
        const I3 e = element_at(ei, g);
        const double q = double(lev.coeff[size_t(ei)]);
        const auto verts = element_vertices(e, g);
        i64 locs[8];
        for (int j = 0; j < 8; ++j) locs[j] = loc_of(verts[j], g);
        for (int i = 0; i < 8; ++i)
          for (int j = 0; j < 8; ++j)
            for (int r = 0; r < 3; ++r)
              for (int c = 0; c < 3; ++c)
                a[size_t((3 * locs[i] + r) * N + 3 * locs[j] + c)] += q * ks_.k[3 * i + r][3 * j + c];
      }
    } else {
      for (i64 loc = 0; loc < nv; ++loc) {
        const I3 v = vertex_at(loc, g);
        const T* row = lev.stencil.data() + 243 * loc;
        for (int n = 0; n < 27; ++n) {
          const I3 t = neighbor_offset(n);
          const i64 wl = loc_of(wrap({v[0] + t[0], v[1] + t[1], v[2] + t[2]}, g), g);
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) a[size_t((3 * loc + r) * N + 3 * wl + c)] += double(row[9 * n + 3 * r + c]);
        }
      }
    }
    return a;
  }
  void factor_coarsest() {  // :368-383 (op_scale_ = mean diagonal, :373)
    const int lc = num_levels() - 1;
    coarse_.factor(assemble_dense(lc), levels_[size_t(lc)].grid.nv());
    op_scale_ = coarse_.op_scale;
  }

  double penal_;
  K0 ks_;
  Tables tab_;
  std::vector<Level<T>> levels_;
  CoarseSolver coarse_;
  double op_scale_ = 0.0;
  bool density_set_ = false;
};

// ----------------------------------------------------------- homogenization
// inc/homogenization.hpp:26-51, src/homogenization.cpp:16-144
struct CellSolveStats {
  int total_cycles = 0;
  double worst_residual = 0.0;
  int worst_load = -1;
  bool converged = true;
};

struct ChiTable {  // src/homogenization.cpp:44-54
  double chi[6][24];
  ChiTable() {
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 8; ++j) {
        double x[3];
        macro_strain_displacement(i, lvo(j), x);
        for (int c = 0; c < 3; ++c) chi[i][3 * j + c] = x[c];
      }
  }
};

template <typename T>
class Homogenizer {
 public:
  Homogenizer(I3 reso, const Material& mat, double penal, const SolverOptions& opts)
      : hier_(Grid(reso), mat, penal), opts_(opts), penal_(penal) {
    for (auto& u : u_) u = Field(hier_.level(0).grid);
  }
  void set_density(const std::vector<double>& rho) {
    rho_ = rho;
    hier_.set_density(rho);
    density_set_ = true;
  }
  CellSolveStats solve_cell_problems() {  // src/homogenization.cpp:23-40
    if (!density_set_) throw std::logic_error("set_density before solve_cell_problems");
    Level<T>& l0 = hier_.level(0);
    Field f(l0.grid);
    CellSolveStats out;
    for (int i = 0; i < 6; ++i) {
      macro_force_kernel<T>(l0.grid, hier_.tables(), l0.coeff.data(), i, f.a.data());
      const SolveStats s = hier_.solve(f, u_[size_t(i)], opts_);
      out.total_cycles += s.cycles;
      if (s.rel_residual >= out.worst_residual) {
        out.worst_residual = s.rel_residual;
        out.worst_load = i;
      }
      if (!s.converged) out.converged = false;
    }
    return out;
  }
  void gather_d(const Grid& g, i64 ei, const ChiTable& chi, double d[24][6]) const {
    const I3 e = element_at(ei, g);
    const auto verts = element_vertices(e, g);
    for (int j = 0; j < 8; ++j) {
      const i64 loc = loc_of(verts[j], g);
      for (int i = 0; i < 6; ++i) {
        const double* uu = u_[size_t(i)].a.data() + 3 * loc;
        for (int c = 0; c < 3; ++c) {
          const double uval = std::is_same_v<T, float> ? double(float(uu[c])) : uu[c];
          d[3 * j + c][i] = chi.chi[i][3 * j + c] - uval;
        }
      }
    }
  }
  void effective_tensor(double C[36]) const {  // src/homogenization.cpp:58-111
    static const ChiTable chi;
    const Grid& g = hier_.level0_grid();
    const i64 m = g.nv();
    const K0& k0 = hier_.ks();
    constexpr i64 kBlock = 512;
    const i64 nb = (m + kBlock - 1) / kBlock;
    std::vector<std::array<double, 21>> partial(static_cast<size_t>(nb));
    parallel_for(nb, [&](i64 blk) {
      std::array<double, 21> acc{};
      const i64 lo = blk * kBlock, hi = std::min(m, lo + kBlock);
      double d[24][6], kd[24][6];
      for (i64 ei = lo; ei < hi; ++ei) {
        gather_d(g, ei, chi, d);
        for (int r = 0; r < 24; ++r)
          for (int i = 0; i < 6; ++i) {
            double s = 0.0;
            for (int k = 0; k < 24; ++k) s += k0.k[r][k] * d[k][i];
            kd[r][i] = s;
          }
        const double q = std::pow(rho_[size_t(ei)], penal_);
        int idx = 0;
        for (int i = 0; i < 6; ++i)
          for (int j = i; j < 6; ++j, ++idx) {
            double s = 0.0;
            for (int r = 0; r < 24; ++r) s += d[r][i] * kd[r][j];
            acc[size_t(idx)] += q * s;
          }
      }
      partial[size_t(blk)] = acc;
    });
    std::array<double, 21> total{};
    for (i64 b = 0; b < nb; ++b)
      for (int k = 0; k < 21; ++k) total[size_t(k)] += partial[size_t(b)][size_t(k)];
    int idx = 0;
    for (int i = 0; i < 6; ++i)
      for (int j = i; j < 6; ++j, ++idx) {
        C[i * 6 + j] = total[size_t(idx)] / double(m);
        C[j * 6 + i] = C[i * 6 + j];
      }
  }
  void tensor_sensitivity(const double seed[36], double* out) const {  // :113-144
    static const ChiTable chi;
    const Grid& g = hier_.level0_grid();
    const i64 m = g.nv();
    const K0& k0 = hier_.ks();
    double s[6][6];
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) s[i][j] = 0.5 * (seed[i * 6 + j] + seed[j * 6 + i]);
    parallel_for(m, [&](i64 ei) {
      double d[24][6], kd[24][6];
      gather_d(g, ei, chi, d);
      for (int r = 0; r < 24; ++r)
        for (int i = 0; i < 6; ++i) {
          double t = 0.0;
          for (int k = 0; k < 24; ++k) t += k0.k[r][k] * d[k][i];
          kd[r][i] = t;
        }
      double acc = 0.0;
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
          double t = 0.0;
          for (int r = 0; r < 24; ++r) t += d[r][i] * kd[r][j];
          acc += s[i][j] * t;
        }
      out[ei] = penal_ * std::pow(rho_[size_t(ei)], penal_ - 1.0) * acc / double(m);
    });
  }
  Field& displacement(int i) { return u_[size_t(i)]; }
  Hierarchy<T>& hierarchy() { return hier_; }
  SolverOptions& options() { return opts_; }

 private:
  Hierarchy<T> hier_;
  SolverOptions opts_;
  double penal_;
  std::vector<double> rho_;
  std::array<Field, 6> u_;
  bool density_set_ = false;
};

// ----------------------------------------------------------------- density
// inc/density.hpp, src/density.cpp:11-265
constexpr double kRhoMin = 0.001;

double field_mean(const double* f, i64 n) {  // src/density.cpp:11-14
  if (n == 0) return 0.0;
  return block_sum(n, [&](i64 i) { return f[i]; }) / double(n);
}

struct Tap { int d[3]; double w; };

std::vector<Tap> kernel_taps(double radius, int kernel) {  // src/density.cpp:23-45; kernel 0=linear 1=spline4
  std::vector<Tap> taps;
  const int r = int(std::floor(radius));
  for (int dz = -r; dz <= r; ++dz)
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        const double dist = std::sqrt(double(dx * dx + dy * dy + dz * dz));
        if (dist > radius) continue;
        double w;
        if (kernel == 0) w = radius - dist;
        else {
          const double q = 1.0 - (dist / radius) * (dist / radius);
          w = q * q;
        }
        if (w > 0.0) taps.push_back({{dx, dy, dz}, w});
      }
  double total = 0.0;
  for (const auto& t : taps) total += t.w;
  for (auto& t : taps) t.w /= total;
  return taps;
}

void radial_filter(const I3& n, const double* f, double radius, int kernel, double* out) {  // :48-63
  const i64 m = i64(n[0]) * n[1] * n[2];
  if (radius < 1.0) {
    std::memcpy(out, f, sizeof(double) * size_t(m));
    return;
  }
  const auto taps = kernel_taps(radius, kernel);
  const Grid g(n);
  parallel_for(m, [&](i64 i) {
    const I3 e = element_at(i, g);
    double s = 0.0;
    for (const auto& t : taps) s += t.w * f[eidx(wrap({e[0] + t.d[0], e[1] + t.d[1], e[2] + t.d[2]}, g), g)];
    out[i] = s;
  });
}

struct GroupOp { int perm[3]; bool flip[3]; };

std::vector<GroupOp> symmetry_group(int sym) {  // src/density.cpp:100-127; 0 none 1 reflect3 2 reflect6 3 rotate3
  std::vector<GroupOp> ops;
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  auto sign = [](const int p[3]) {
    int s = 1;
    for (int i = 0; i < 3; ++i)
      for (int j = i + 1; j < 3; ++j)
        if (p[i] > p[j]) s = -s;
    return s;
  };
  switch (sym) {
    case 0: ops.push_back({{0, 1, 2}, {false, false, false}}); break;
    case 1:
      for (int m = 0; m < 8; ++m) ops.push_back({{0, 1, 2}, {bool(m & 1), bool(m & 2), bool(m & 4)}});
      break;
    case 2:
      for (const auto& p : perms)
        for (int m = 0; m < 8; ++m) ops.push_back({{p[0], p[1], p[2]}, {bool(m & 1), bool(m & 2), bool(m & 4)}});
      break;
    case 3:
      for (const auto& p : perms)
        for (int m = 0; m < 8; ++m) {
          const int nflip = (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1);
          if (sign(p) * ((nflip % 2) ? -1 : 1) == 1)
            ops.push_back({{p[0], p[1], p[2]}, {bool(m & 1), bool(m & 2), bool(m & 4)}});
        }
      break;
    default: throw std::invalid_argument("unknown symmetry");
  }
  return ops;
}

void symmetrize(double* field, const I3& n, int sym) {  // src/density.cpp:131-150
  if (sym == 0) return;
  if (sym != 1 && (n[0] != n[1] || n[1] != n[2]))
    throw std::invalid_argument("reflect6/rotate3 symmetry requires a cubic grid");
  const auto ops = symmetry_group(sym);
  const Grid g(n);
  const i64 m = g.nv();
  std::vector<double> in(field, field + m);
  const double inv = 1.0 / double(ops.size());
  parallel_for(m, [&](i64 i) {
    const I3 e = element_at(i, g);
    double s = 0.0;
    for (const auto& op : ops) {
      I3 q{e[op.perm[0]], e[op.perm[1]], e[op.perm[2]]};
      for (int k = 0; k < 3; ++k)
        if (op.flip[k]) q[k] = n[k] - 1 - q[k];
      s += in[size_t(eidx(q, g))];
    }
    field[i] = s * inv;
  });
}

std::uint64_t splitmix64(std::uint64_t x) {  // src/density.cpp:154-159
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d449bd133111ebULL;
  return x ^ (x >> 31);
}
double uniform_pm1(std::uint64_t seed, std::uint64_t counter) {  // :162-165
  const std::uint64_t h = splitmix64(splitmix64(seed) ^ (counter * 0xd1b54a32d192ed03ULL + 1));
  return double(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// src/density.cpp:169-259. Returns fallback flag.
bool init_trig(int basis_n, std::uint64_t seed, double volume, double sigmoid_k, const I3& reso, double* rho) {
  if (basis_n < 1 || basis_n > 8) throw std::invalid_argument("trig basis order must be in [1, 8]");
  if (!(volume > kRhoMin && volume <= 1.0)) throw std::invalid_argument("volume fraction out of range");
  const Grid g(reso);
  const i64 m = g.nv();
  const int nt = 6 * basis_n;
  const int nq = nt + nt * (nt + 1) / 2;
  std::vector<double> w(static_cast<size_t>(nq));
  for (int j = 0; j < nq; ++j) w[size_t(j)] = uniform_pm1(seed, std::uint64_t(j));
  double q[4], qn = 0.0;
  for (int j = 0; j < 4; ++j) {
    q[j] = uniform_pm1(seed, std::uint64_t(nq + j));
    qn += q[j] * q[j];
  }
  if (qn < 1e-12) { q[0] = 1.0; q[1] = q[2] = q[3] = 0.0; qn = 1.0; }
  qn = std::sqrt(qn);
  for (double& c : q) c /= qn;
  const double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
  const double rot[3][3] = {{1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy)},
                            {2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx)},
                            {2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)}};
  std::vector<double> y(static_cast<size_t>(m));
  parallel_for(m, [&](i64 i) {
    const I3 e = element_at(i, g);
    double xb[3];
    for (int r = 0; r < 3; ++r) {
      xb[r] = 0.0;
      for (int k = 0; k < 3; ++k) xb[r] += rot[r][k] * ((e[k] + 0.5) / double(g.n[k]) - 0.5);
    }
    double t[48];
    for (int ax = 0, j = 0; ax < 3; ++ax)
      for (int k = 1; k <= basis_n; ++k) {
        t[j++] = std::cos(2.0 * M_PI * k * xb[ax]);
        t[j++] = std::sin(2.0 * M_PI * k * xb[ax]);
      }
    double s = 0.0;
    int j = 0;
    for (int a = 0; a < nt; ++a) s += w[size_t(j++)] * t[a];
    for (int a = 0; a < nt; ++a)
      for (int b = a; b < nt; ++b) s += w[size_t(j++)] * t[a] * t[b];
    y[size_t(i)] = s;
  });
  const double vhat = std::min(1.5 * volume, 1.0 - kRhoMin);
  const double k = sigmoid_k;
  auto project = [&](double mu) {
    parallel_for(m, [&](i64 i) { rho[i] = kRhoMin + vhat / (1.0 + std::exp(-k * (y[size_t(i)] - mu))); });
    return field_mean(rho, m);
  };
  auto constant = [&]() {
    for (i64 i = 0; i < m; ++i) rho[i] = volume;
  };
  double ylo = y[0], yhi = y[0];
  for (i64 i = 1; i < m; ++i) {
    ylo = std::min(ylo, y[size_t(i)]);
    yhi = std::max(yhi, y[size_t(i)]);
  }
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
  project(0.5 * (lo + hi));
  if (std::abs(field_mean(rho, m) - volume) <= 1e-4) return false;
  constant();
  return true;
}

// ---------------------------------------------------------------------- oc
// inc/oc.hpp:10-61, src/oc.cpp:14-111
struct OCConfig {
  double min_density = kRhoMin, step_limit = 0.05, damp = 0.5, volume = 0.3, bisect_tol = 1e-6;
};

void oc_trial(i64 m, const double* rho, const std::vector<double>& b0, const OCConfig& cfg, double lambda,
              double* out) {  // src/oc.cpp:14-23
  const double damp = cfg.damp, step = cfg.step_limit;
  parallel_for(m, [&](i64 i) {
    double x = rho[i] * std::pow(b0[size_t(i)] / lambda, damp);
    x = std::clamp(x, rho[i] - step, rho[i] + step);
    out[i] = std::clamp(x, cfg.min_density, 1.0);
  });
}

// src/oc.cpp:27-77. returns bisection_ok
bool oc_update(i64 m, const double* rho, const double* sens, const OCConfig& cfg, double* out, double* lambda_out) {
  for (i64 i = 0; i < m; ++i)
    if (!std::isfinite(sens[i])) throw std::invalid_argument("non-finite sensitivity");
  constexpr double kSensFloor = 1e-30;
  std::vector<double> b0(static_cast<size_t>(m));
  double scale = kSensFloor;
  for (i64 i = 0; i < m; ++i) scale = std::max(scale, std::max(kSensFloor, -sens[i]));
  parallel_for(m, [&](i64 i) { b0[size_t(i)] = std::max(kSensFloor, -sens[i]) / scale; });
  const double lo0 = 1e-12, hi0 = 1e12;
  oc_trial(m, rho, b0, cfg, lo0, out);
  const double mean_lo = field_mean(out, m);
  if (cfg.volume >= mean_lo) {
    *lambda_out = lo0 * scale;
    return std::abs(mean_lo - cfg.volume) <= cfg.bisect_tol;
  }
  oc_trial(m, rho, b0, cfg, hi0, out);
  const double mean_hi = field_mean(out, m);
  if (cfg.volume <= mean_hi) {
    *lambda_out = hi0 * scale;
    return std::abs(mean_hi - cfg.volume) <= cfg.bisect_tol;
  }
  double lo = lo0, hi = hi0, lambda = lo0;
  for (int it = 0; it < 60; ++it) {
    lambda = std::sqrt(lo * hi);
    oc_trial(m, rho, b0, cfg, lambda, out);
    const double mean = field_mean(out, m);
    if (std::abs(mean - cfg.volume) <= cfg.bisect_tol) {
      *lambda_out = lambda * scale;
      return true;
    }
    (mean > cfg.volume ? lo : hi) = lambda;
  }
  *lambda_out = lambda * scale;
  return std::abs(field_mean(out, m) - cfg.volume) <= cfg.bisect_tol;
}

void sensitivity_filter(const I3& n, const double* sens, const double* rho, double radius, double* out) {
  const i64 m = i64(n[0]) * n[1] * n[2];  // src/oc.cpp:79-111
  if (radius < 1.0) {
    std::memcpy(out, sens, sizeof(double) * size_t(m));
    return;
  }
  const Grid g(n);
  const int r = int(std::floor(radius));
  std::vector<Tap> taps;
  for (int dz = -r; dz <= r; ++dz)
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        const double dist = std::sqrt(double(dx * dx + dy * dy + dz * dz));
        const double w = radius - dist;
        if (w > 0.0) taps.push_back({{dx, dy, dz}, w});
      }
  double wsum = 0.0;
  for (const auto& t : taps) wsum += t.w;
  parallel_for(m, [&](i64 i) {
    const I3 e = element_at(i, g);
    double acc = 0.0;
    for (const auto& t : taps) {
      const i64 k = eidx(wrap({e[0] + t.d[0], e[1] + t.d[1], e[2] + t.d[2]}, g), g);
      acc += t.w * rho[k] * sens[k];
    }
    out[i] = acc / (std::max(rho[i], kRhoMin) * wsum);
  });
}

struct ConvergeChecker {  // inc/oc.hpp:35-61
  double threshold = 5e-4;
  int required = 3, hits = 0;
  double prev = 0.0;
  bool has_prev = false;
  bool update(double f) {
    if (has_prev) {
      const double rel = std::abs(f - prev) / std::max(std::abs(prev), 1e-12);
      hits = rel < threshold ? hits + 1 : 0;
    }
    prev = f;
    has_prev = true;
    return hits >= required;
  }
};

// --------------------------------------------------------------- objective
// src/objective.cpp:5-270 (DAG with memoised eval, reverse-mode backward,
// eager constant folding)
enum class Op { kConst, kEntry, kAdd, kSub, kMul, kDiv, kPow, kLog, kExp, kNeg };
struct Node {
  Op op;
  double value = 0.0;
  int i = 0, j = 0;
  std::shared_ptr<const Node> a, b;
};
using NP = std::shared_ptr<const Node>;
NP mk(Op op, double v, int i, int j, NP a, NP b) {
  auto n = std::make_shared<Node>();
  n->op = op; n->value = v; n->i = i; n->j = j; n->a = std::move(a); n->b = std::move(b);
  return n;
}
struct Ex {
  NP n;
  static Ex c(double v) { return {mk(Op::kConst, v, 0, 0, nullptr, nullptr)}; }
  static Ex e(int i, int j) { return {mk(Op::kEntry, 0, i, j, nullptr, nullptr)}; }
};
bool bc(const Ex& a, const Ex& b) { return a.n->op == Op::kConst && b.n->op == Op::kConst; }
Ex operator+(const Ex& a, const Ex& b) { return bc(a, b) ? Ex::c(a.n->value + b.n->value) : Ex{mk(Op::kAdd, 0, 0, 0, a.n, b.n)}; }
Ex operator-(const Ex& a, const Ex& b) { return bc(a, b) ? Ex::c(a.n->value - b.n->value) : Ex{mk(Op::kSub, 0, 0, 0, a.n, b.n)}; }
Ex operator*(const Ex& a, const Ex& b) { return bc(a, b) ? Ex::c(a.n->value * b.n->value) : Ex{mk(Op::kMul, 0, 0, 0, a.n, b.n)}; }
Ex operator/(const Ex& a, const Ex& b) { return bc(a, b) ? Ex::c(a.n->value / b.n->value) : Ex{mk(Op::kDiv, 0, 0, 0, a.n, b.n)}; }
Ex operator-(const Ex& a) { return a.n->op == Op::kConst ? Ex::c(-a.n->value) : Ex{mk(Op::kNeg, 0, 0, 0, a.n, nullptr)}; }
Ex epow(const Ex& a, double e) { return a.n->op == Op::kConst ? Ex::c(std::pow(a.n->value, e)) : Ex{mk(Op::kPow, e, 0, 0, a.n, nullptr)}; }
Ex elog(const Ex& a) { return a.n->op == Op::kConst ? Ex::c(std::log(a.n->value)) : Ex{mk(Op::kLog, 0, 0, 0, a.n, nullptr)}; }

double ev(const Node* n, const double* C, std::unordered_map<const Node*, double>& memo) {
  auto it = memo.find(n);
  if (it != memo.end()) return it->second;
  double v = 0.0;
  switch (n->op) {
    case Op::kConst: v = n->value; break;
    case Op::kEntry: v = C[n->i * 6 + n->j]; break;
    case Op::kAdd: v = ev(n->a.get(), C, memo) + ev(n->b.get(), C, memo); break;
    case Op::kSub: v = ev(n->a.get(), C, memo) - ev(n->b.get(), C, memo); break;
    case Op::kMul: v = ev(n->a.get(), C, memo) * ev(n->b.get(), C, memo); break;
    case Op::kDiv: {
      const double den = ev(n->b.get(), C, memo);
      if (den == 0.0) throw std::runtime_error("division by zero");
      v = ev(n->a.get(), C, memo) / den;
      break;
    }
    case Op::kPow: {
      const double base = ev(n->a.get(), C, memo);
      if (base < 0.0 && n->value != std::floor(n->value)) throw std::runtime_error("fractional power of negative value");
      if (base == 0.0 && n->value < 1.0 && n->value != 0.0) throw std::runtime_error("non-positive base of power");
      v = std::pow(base, n->value);
      break;
    }
    case Op::kLog: {
      const double x = ev(n->a.get(), C, memo);
      if (!(x > 0.0)) throw std::runtime_error("log of non-positive value");
      v = std::log(x);
      break;
    }
    case Op::kExp: v = std::exp(ev(n->a.get(), C, memo)); break;
    case Op::kNeg: v = -ev(n->a.get(), C, memo); break;
  }
  memo.emplace(n, v);
  return v;
}
void topo(const Node* n, std::unordered_map<const Node*, bool>& seen, std::vector<const Node*>& order) {
  if (seen.count(n)) return;
  seen.emplace(n, true);
  if (n->a) topo(n->a.get(), seen, order);
  if (n->b) topo(n->b.get(), seen, order);
  order.push_back(n);
}
double eval_expr(const Ex& x, const double* C) {
  std::unordered_map<const Node*, double> memo;
  return ev(x.n.get(), C, memo);
}
void backward_expr(const Ex& x, double seed, const double* C, double* G) {  // src/objective.cpp:132-180
  std::unordered_map<const Node*, double> values;
  ev(x.n.get(), C, values);
  std::unordered_map<const Node*, bool> seen;
  std::vector<const Node*> order;
  topo(x.n.get(), seen, order);
  std::unordered_map<const Node*, double> adj;
  adj[x.n.get()] = seed;
  for (int k = 0; k < 36; ++k) G[k] = 0.0;
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    const Node* n = *it;
    auto ai = adj.find(n);
    if (ai == adj.end()) continue;
    const double g = ai->second;
    switch (n->op) {
      case Op::kConst: break;
      case Op::kEntry: G[n->i * 6 + n->j] += g; break;
      case Op::kAdd: adj[n->a.get()] += g; adj[n->b.get()] += g; break;
      case Op::kSub: adj[n->a.get()] += g; adj[n->b.get()] -= g; break;
      case Op::kMul:
        adj[n->a.get()] += g * values.at(n->b.get());
        adj[n->b.get()] += g * values.at(n->a.get());
        break;
      case Op::kDiv: {
        const double bv = values.at(n->b.get());
        adj[n->a.get()] += g / bv;
        adj[n->b.get()] -= g * values.at(n->a.get()) / (bv * bv);
        break;
      }
      case Op::kPow: adj[n->a.get()] += g * n->value * std::pow(values.at(n->a.get()), n->value - 1.0); break;
      case Op::kLog: adj[n->a.get()] += g / values.at(n->a.get()); break;
      case Op::kExp: adj[n->a.get()] += g * values.at(n); break;
      case Op::kNeg: adj[n->a.get()] -= g; break;
    }
  }
}
// src/objective.cpp:238-260; obj 0 bulk 1 shear 2 npr_relaxed 3 npr_log
Ex make_objective(int obj, double beta, double eta, double tau, double gamma, int iter) {
  switch (obj) {
    case 0: {
      const Ex diag = Ex::e(0, 0) + Ex::e(1, 1) + Ex::e(2, 2);
      const Ex off = Ex::e(0, 1) + Ex::e(0, 2) + Ex::e(1, 2);
      return -((diag + Ex::c(2.0) * off) / Ex::c(9.0));
    }
    case 1: return -((Ex::e(3, 3) + Ex::e(4, 4) + Ex::e(5, 5)) / Ex::c(3.0));
    case 2: {
      if (!(beta > 0.0 && beta < 1.0)) throw std::invalid_argument("npr-relaxed beta must lie in (0,1)");
      const Ex off = Ex::e(0, 1) + Ex::e(0, 2) + Ex::e(1, 2);
      const Ex diag = Ex::e(0, 0) + Ex::e(1, 1) + Ex::e(2, 2);
      return off - Ex::c(std::pow(beta, double(iter))) * diag;
    }
    case 3: {
      const Ex off = Ex::e(0, 1) + Ex::e(1, 2) + Ex::e(2, 0);
      const Ex diag = Ex::e(0, 0) + Ex::e(1, 1) + Ex::e(2, 2);
      return elog(Ex::c(1.0) + Ex::c(eta) * off / diag) + Ex::c(tau) * epow(diag, gamma);
    }
    default: throw std::invalid_argument("unknown objective");
  }
}

}  // namespace orc

// ================================================================ C API
// Plain pointers; nodal fields AoS [3*nv] in colour-block order; element
// fields x-fastest. Errors: return code != 0 and orc_last_error() text.
using namespace orc;

static thread_local std::string g_err;

#define ORC_TRY(...)                        \
  try {                                     \
    __VA_ARGS__;                                   \
    return 0;                               \
  } catch (const std::invalid_argument& e) { \
    g_err = e.what();                       \
    return 1;                               \
  } catch (const std::runtime_error& e) {   \
    g_err = e.what();                       \
    return 2;                               \
  } catch (const std::exception& e) {       \
    g_err = e.what();                       \
    return 3;                               \
  }

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_set_coarse_project(int on) {
  g_coarse_project = on != 0;
  return 0;
}
int orc_set_coarse_dump(const char* path) {
  g_dump_path = path ? path : "";
  return 0;
}
// Standalone coarsest solve of an assembled operator (fixtures): projection/shift/LDLT/refinement
// exactly as the hierarchy's; f is made translation-free first (src/multigrid.cpp:427).
int orc_coarse_dense_solve(long long nv, const double* raw, const double* f, double* x_out, double* rel_out) {
  ORC_TRY({
    const i64 N = 3 * nv;
    CoarseSolver cs;
    cs.factor(std::vector<double>(raw, raw + N * N), nv);
    std::vector<double> fv(f, f + N);
    for (int c = 0; c < 3; ++c) {
      double m = 0.0;
      for (i64 i = 0; i < nv; ++i) m += fv[size_t(3 * i + c)];
      m /= double(nv);
      for (i64 i = 0; i < nv; ++i) fv[size_t(3 * i + c)] -= m;
    }
    cs.project_load(fv);
    double fn = 0.0;
    for (double v : fv) fn += v * v;
    fn = std::sqrt(fn);
    std::vector<double> x;
    *rel_out = cs.solve(fv, fn, x);
    std::copy(x.begin(), x.end(), x_out);
  })
}
int orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

int orc_k0(double E, double nu, double* out576) {
  ORC_TRY({
    Material m{E, nu};
    const K0 k = element_stiffness(m);
    std::memcpy(out576, &k.k[0][0], sizeof(double) * 576);
  })
}

int orc_grid_info(int nx, int ny, int nz, long long* cbase8, int* cdim24) {
  ORC_TRY({
    const Grid g({nx, ny, nz});
    for (int c = 0; c < 8; ++c) {
      cbase8[c] = g.cbase[c];
      for (int k = 0; k < 3; ++k) cdim24[3 * c + k] = g.cdim[c][k];
    }
  })
}

// Location of every vertex, enumerated x-fastest over (x,y,z).
int orc_grid_locs(int nx, int ny, int nz, long long* out) {
  ORC_TRY({
    const Grid g({nx, ny, nz});
    i64 k = 0;
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) out[k++] = loc_of({x, y, z}, g);
  })
}

int orc_fem_tables(double E, double nu, double* fmacro144, int* ngb64) {
  ORC_TRY({
    const Tables t(element_stiffness(Material{E, nu}));
    std::memcpy(fmacro144, &t.fmacro[0][0][0], sizeof(double) * 144);
    std::memcpy(ngb64, &t.ngb[0][0], sizeof(int) * 64);
  })
}

// which: 0 apply (y=Ku), 1 residual (r=f-Ku; f in), 2 one GS sweep (u in/out, f in),
// 3 macro force load (=extra) into out. coeff is the element coefficient (already rho^p)
// given in f64; mixed=1 rounds it to f32 and runs the T=float path.
int orc_fem(int nx, int ny, int nz, double E, double nu, int mixed, int which, int extra, const double* coeff,
            double* u, const double* f, double* out) {
  ORC_TRY({
    const Grid g({nx, ny, nz});
    const Tables t(element_stiffness(Material{E, nu}));
    const i64 m = g.nv();
    auto run = [&](auto tag) {
      using T = decltype(tag);
      std::vector<T> c(static_cast<size_t>(m));
      for (i64 i = 0; i < m; ++i) c[size_t(i)] = T(coeff[i]);
      switch (which) {
        case 0: apply_kernel<T>(g, t, c.data(), u, out); break;
        case 1: residual_kernel<T>(g, t, c.data(), u, f, out); break;
        case 2: gs_kernel<T>(g, t, c.data(), f, u); break;
        case 3: macro_force_kernel<T>(g, t, c.data(), extra, out); break;
        default: throw std::invalid_argument("bad fem op");
      }
    };
    if (mixed) run(float{});
    else run(double{});
  })
}

int orc_restrict(int nx, int ny, int nz, const double* fine, double* coarse) {
  ORC_TRY({
    Field fr(Grid({nx, ny, nz}));
    std::memcpy(fr.a.data(), fine, sizeof(double) * fr.a.size());
    Field cf(fr.grid.coarsened());
    restrict_field(fr, cf);
    std::memcpy(coarse, cf.a.data(), sizeof(double) * cf.a.size());
  })
}

int orc_prolong_add(int nx, int ny, int nz, const double* coarse, double* fine) {
  ORC_TRY({
    Field fu(Grid({nx, ny, nz}));
    std::memcpy(fu.a.data(), fine, sizeof(double) * fu.a.size());
    Field cu(fu.grid.coarsened());
    std::memcpy(cu.a.data(), coarse, sizeof(double) * cu.a.size());
    prolong_add(cu, fu);
    std::memcpy(fine, fu.a.data(), sizeof(double) * fu.a.size());
  })
}

// ---- hierarchy / homogenizer handles
struct OrcHom {
  int mixed;
  std::unique_ptr<Homogenizer<float>> hf;
  std::unique_ptr<Homogenizer<double>> hd;
};

void* orc_hom_create(int nx, int ny, int nz, double E, double nu, double penal, int mixed, double tol,
                     int max_cycles) {
  try {
    SolverOptions o;
    o.tol = tol;
    o.max_cycles = max_cycles;
    auto* h = new OrcHom{mixed, nullptr, nullptr};
    if (mixed) h->hf = std::make_unique<Homogenizer<float>>(I3{nx, ny, nz}, Material{E, nu}, penal, o);
    else h->hd = std::make_unique<Homogenizer<double>>(I3{nx, ny, nz}, Material{E, nu}, penal, o);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void orc_hom_destroy(void* p) { delete static_cast<OrcHom*>(p); }

#define HOM_DISPATCH(p, ...)                   \
  OrcHom* H = static_cast<OrcHom*>(p);         \
  if (H->mixed) {                              \
    auto& hom = *H->hf;                        \
    __VA_ARGS__;                               \
  } else {                                     \
    auto& hom = *H->hd;                        \
    __VA_ARGS__;                               \
  }

int orc_hom_set_density(void* p, const double* rho, long long m) {
  ORC_TRY({ HOM_DISPATCH(p, hom.set_density(std::vector<double>(rho, rho + m))) })
}
int orc_hom_solve(void* p, int* total_cycles, double* worst_residual, int* worst_load, int* converged) {
  ORC_TRY({
    HOM_DISPATCH(p, {
      const CellSolveStats s = hom.solve_cell_problems();
      *total_cycles = s.total_cycles;
      *worst_residual = s.worst_residual;
      *worst_load = s.worst_load;
      *converged = s.converged ? 1 : 0;
    })
  })
}
int orc_hom_tensor(void* p, double* C36) { ORC_TRY({ HOM_DISPATCH(p, hom.effective_tensor(C36)) }) }
int orc_hom_sensitivity(void* p, const double* seed36, double* out) {
  ORC_TRY({ HOM_DISPATCH(p, hom.tensor_sensitivity(seed36, out)) })
}
int orc_hom_get_u(void* p, int i, double* out) {
  ORC_TRY({ HOM_DISPATCH(p, {
    const Field& f = hom.displacement(i);
    std::memcpy(out, f.a.data(), sizeof(double) * f.a.size());
  }) })
}
int orc_hom_set_u(void* p, int i, const double* in) {
  ORC_TRY({ HOM_DISPATCH(p, {
    Field& f = hom.displacement(i);
    std::memcpy(f.a.data(), in, sizeof(double) * f.a.size());
  }) })
}
int orc_hom_num_levels(void* p) {
  OrcHom* H = static_cast<OrcHom*>(p);
  return H->mixed ? H->hf->hierarchy().num_levels() : H->hd->hierarchy().num_levels();
}
// Level-l stencil (243 per vertex, loc-major) as f64.
int orc_hom_get_stencil(void* p, int l, double* out) {
  ORC_TRY({ HOM_DISPATCH(p, {
    auto& lev = hom.hierarchy().level(l);
    for (size_t i = 0; i < lev.stencil.size(); ++i) out[i] = double(lev.stencil[i]);
  }) })
}
// Hierarchy-level ops for parity tests: set level-0 f/u, run one v-cycle, read fields.
int orc_hom_level_field(void* p, int l, int which, int write, double* buf) {
  ORC_TRY({ HOM_DISPATCH(p, {
    auto& lev = hom.hierarchy().level(l);
    Field& f = which == 0 ? lev.u : (which == 1 ? lev.f : lev.r);
    if (write) std::memcpy(f.a.data(), buf, sizeof(double) * f.a.size());
    else std::memcpy(buf, f.a.data(), sizeof(double) * f.a.size());
  }) })
}
int orc_hom_vcycle(void* p, double* rel) {
  ORC_TRY({ HOM_DISPATCH(p, { *rel = hom.hierarchy().v_cycle(hom.options()); }) })
}
int orc_hom_relax(void* p, int l, int sweeps) { ORC_TRY({ HOM_DISPATCH(p, hom.hierarchy().relax(l, sweeps)) }) }
int orc_hom_residual(void* p, int l) { ORC_TRY({ HOM_DISPATCH(p, hom.hierarchy().compute_residual(l)) }) }
int orc_hom_coarsest_solve(void* p) { ORC_TRY({ HOM_DISPATCH(p, hom.hierarchy().coarsest_solve()) }) }
int orc_hom_hsolve(void* p, const double* f, double* u, int* cycles, double* rel, int* conv) {
  ORC_TRY({ HOM_DISPATCH(p, {
    Field ff(hom.hierarchy().level(0).grid), uu(hom.hierarchy().level(0).grid);
    std::memcpy(ff.a.data(), f, sizeof(double) * ff.a.size());
    std::memcpy(uu.a.data(), u, sizeof(double) * uu.a.size());
    const SolveStats s = hom.hierarchy().solve(ff, uu, hom.options());
    std::memcpy(u, uu.a.data(), sizeof(double) * uu.a.size());
    *cycles = s.cycles;
    *rel = s.rel_residual;
    *conv = s.converged;
  }) })
}
double orc_hom_op_scale(void* p) {
  OrcHom* H = static_cast<OrcHom*>(p);
  return H->mixed ? H->hf->hierarchy().op_scale() : H->hd->hierarchy().op_scale();
}

// ---- density side
double orc_field_mean(const double* f, long long m) { return field_mean(f, m); }
int orc_radial_filter(int nx, int ny, int nz, const double* f, double radius, int kernel, double* out) {
  ORC_TRY(radial_filter({nx, ny, nz}, f, radius, kernel, out))
}
int orc_symmetrize(int nx, int ny, int nz, double* f, int sym) { ORC_TRY(symmetrize(f, {nx, ny, nz}, sym)) }
int orc_init_trig(int nx, int ny, int nz, int basis_n, unsigned long long seed, double volume, double sigmoid_k,
                  double* rho, int* fallback) {
  ORC_TRY({ *fallback = init_trig(basis_n, seed, volume, sigmoid_k, {nx, ny, nz}, rho) ? 1 : 0; })
}
int orc_oc_update(long long m, const double* rho, const double* sens, double volume, double step, double damp,
                  double min_density, double bisect_tol, double* out, double* lambda, int* ok) {
  ORC_TRY({
    OCConfig c;
    c.volume = volume;
    c.step_limit = step;
    c.damp = damp;
    c.min_density = min_density;
    c.bisect_tol = bisect_tol;
    *ok = oc_update(m, rho, sens, c, out, lambda) ? 1 : 0;
  })
}
int orc_sensitivity_filter(int nx, int ny, int nz, const double* sens, const double* rho, double radius,
                           double* out) {
  ORC_TRY(sensitivity_filter({nx, ny, nz}, sens, rho, radius, out))
}
int orc_objective(int obj, double beta, double eta, double tau, double gamma, int iter, const double* C36,
                  double* value, double* grad36) {
  ORC_TRY({
    const Ex x = make_objective(obj, beta, eta, tau, gamma, iter);
    *value = eval_expr(x, C36);
    if (grad36) backward_expr(x, 1.0, C36, grad36);
  })
}

// ---- the optimisation loop, src/runner.cpp:51-136
struct OrcRunConfig {
  int reso;
  double vol, youngs, poisson;
  int obj;
  double beta, eta, tau, gamma, penal, filter_radius;
  int filter_placement;  // 0 density 1 sensitivity
  int kernel;            // 0 linear 1 spline4
  int sym;               // 0 none 1 reflect3 2 reflect6 3 rotate3
  int init;              // 0 constant 1 trig
  int basis_n;
  unsigned long long seed;
  int max_iter;
  double step, damp, tol;
  int max_cycles;
  int mixed;
};
struct OrcIterRecord {
  int iter;
  double objective, volume;
  int cycles;
  double residual, ms;
  double C[36];
};

// records must hold max_iter entries; returns the number written in *nrec.
// flags: bit0 solver_failed, bit1 converged, bit2 init_fallback, bit3 oc_warning
int orc_run(const OrcRunConfig* cfg, OrcIterRecord* records, int* nrec, double* rho_out, int* flags) {
  ORC_TRY({
    auto impl = [&](auto tag) {
      using T = decltype(tag);
      const I3 reso{cfg->reso, cfg->reso, cfg->reso};
      const i64 m = i64(cfg->reso) * cfg->reso * cfg->reso;
      SolverOptions so;
      so.tol = cfg->tol;
      so.max_cycles = cfg->max_cycles;
      Homogenizer<T> hom(reso, Material{cfg->youngs, cfg->poisson}, 1.0, so);
      std::vector<double> rho(static_cast<size_t>(m));
      *flags = 0;
      if (cfg->init == 0) {
        for (auto& x : rho) x = cfg->vol;
      } else {
        if (init_trig(cfg->basis_n, cfg->seed, cfg->vol, 15.0, reso, rho.data())) *flags |= 4;
      }
      auto clamp_bounds = [&](std::vector<double>& f) {
        parallel_for(m, [&](i64 i) { f[size_t(i)] = std::clamp(f[size_t(i)], kRhoMin, 1.0); });
      };
      if (cfg->sym != 0) {
        symmetrize(rho.data(), reso, cfg->sym);
        clamp_bounds(rho);
      }
      const bool dfilt = cfg->filter_placement == 0 && cfg->filter_radius >= 1.0;
      OCConfig oc;
      oc.volume = cfg->vol;
      oc.step_limit = cfg->step;
      oc.damp = cfg->damp;
      ConvergeChecker conv;
      std::vector<double> pre(static_cast<size_t>(m)), phys(static_cast<size_t>(m)), grad(static_cast<size_t>(m)), gd(static_cast<size_t>(m)), tmp(static_cast<size_t>(m)),
          next(static_cast<size_t>(m));
      *nrec = 0;
      for (int iter = 0; iter < cfg->max_iter; ++iter) {
        const auto t0 = std::chrono::steady_clock::now();
        // DensityExpr::eval, src/density.cpp:65-72
        if (dfilt) radial_filter(reso, rho.data(), cfg->filter_radius, cfg->kernel, pre.data());
        else pre = rho;
        const double p = cfg->penal;
        parallel_for(m, [&](i64 i) { phys[size_t(i)] = std::pow(pre[size_t(i)], p); });
        hom.set_density(phys);
        const CellSolveStats st = hom.solve_cell_problems();
        OrcIterRecord& rec = records[*nrec];
        hom.effective_tensor(rec.C);
        const Ex obj = make_objective(cfg->obj, cfg->beta, cfg->eta, cfg->tau, cfg->gamma, iter);
        const double fval = eval_expr(obj, rec.C);
        rec.iter = iter;
        rec.objective = fval;
        rec.volume = field_mean(rho.data(), m);
        rec.cycles = st.total_cycles;
        rec.residual = st.worst_residual;
        rec.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++*nrec;
        if (!st.converged) {
          *flags |= 1;
          break;
        }
        if (conv.update(fval)) {
          *flags |= 2;
          break;
        }
        if (iter + 1 == cfg->max_iter) break;
        double seed[36];
        backward_expr(obj, 1.0, rec.C, seed);
        hom.tensor_sensitivity(seed, grad.data());
        // DensityExpr::backward, src/density.cpp:74-83
        parallel_for(m, [&](i64 i) { tmp[size_t(i)] = grad[size_t(i)] * p * std::pow(pre[size_t(i)], p - 1.0); });
        if (dfilt) radial_filter(reso, tmp.data(), cfg->filter_radius, cfg->kernel, gd.data());
        else gd = tmp;
        if (cfg->filter_placement == 1 && cfg->filter_radius >= 1.0) {
          sensitivity_filter(reso, gd.data(), rho.data(), cfg->filter_radius, tmp.data());
          gd = tmp;
        }
        symmetrize(gd.data(), reso, cfg->sym);
        double lam;
        if (!oc_update(m, rho.data(), gd.data(), oc, next.data(), &lam)) *flags |= 8;
        rho.swap(next);
        if (cfg->sym != 0) {
          symmetrize(rho.data(), reso, cfg->sym);
          clamp_bounds(rho);
        }
        // full-iteration wall time (the reference's rec.ms stops after the objective, src/runner.cpp:98)
        rec.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      }
      std::memcpy(rho_out, rho.data(), sizeof(double) * size_t(m));
    };
    if (cfg->mixed) impl(float{});
    else impl(double{});
  })
}

}  // extern "C"
