// tables.cpp -- see tables.hpp. Pure host C++ (no Eigen).
#include "tables.hpp"

#include <cmath>
#include <cstring>
#include <stdexcept>

namespace ihomgpu {

namespace {
inline void lvo(int j, int d[3]) {  // inc/grid.hpp:95
  d[0] = j & 1;
  d[1] = (j >> 1) & 1;
  d[2] = (j >> 2) & 1;
}
inline double tw1(int c) {  // src/multigrid.cpp:12-15
  const int a = c < 0 ? -c : c;
  return a >= 2 ? 0.0 : (2.0 - a) / 2.0;
}
inline void noff(int idx, int t[3]) {  // inc/fem.hpp:33-35
  t[0] = idx % 3 - 1;
  t[1] = (idx / 3) % 3 - 1;
  t[2] = idx / 9 - 1;
}
}  // namespace

void validate_material(const Material& m) {
  if (!(m.youngs > 0.0)) throw std::invalid_argument("Young's modulus must be positive");
  if (!(m.poisson > -1.0 && m.poisson < 0.5)) throw std::invalid_argument("Poisson's ratio must lie in (-1, 0.5)");
}

K0Matrix element_stiffness(const Material& mat) {  // src/material.cpp:39-69
  validate_material(mat);
  const double l = mat.lambda(), m = mat.mu();
  double c[6][6] = {};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) c[i][j] = l;
    c[i][i] = l + 2.0 * m;
    c[3 + i][3 + i] = m;
  }
  double k[24][24] = {};
  const double gp[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int q = 0; q < 2; ++q) {
        const double p[3] = {gp[a], gp[b], gp[q]};
        double grad[8][3];
        for (int j = 0; j < 8; ++j) {
          int d[3];
          lvo(j, d);
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
          B[0][col] = grad[j][0];
          B[1][col + 1] = grad[j][1];
          B[2][col + 2] = grad[j][2];
          B[3][col] = grad[j][1];
          B[3][col + 1] = grad[j][0];
          B[4][col + 1] = grad[j][2];
          B[4][col + 2] = grad[j][1];
          B[5][col] = grad[j][2];
          B[5][col + 2] = grad[j][0];
        }
        double CB[6][24];
        for (int r = 0; r < 6; ++r)
          for (int s = 0; s < 24; ++s) {
            double acc = 0.0;
            for (int t = 0; t < 6; ++t) acc += c[r][t] * B[t][s];
            CB[r][s] = acc;
          }
        for (int r = 0; r < 24; ++r)
          for (int s = 0; s < 24; ++s) {
            double acc = 0.0;
            for (int t = 0; t < 6; ++t) acc += B[t][r] * CB[t][s];
            k[r][s] += 0.125 * acc;
          }
      }
  K0Matrix out;
  for (int r = 0; r < 24; ++r)
    for (int s = 0; s < 24; ++s) out.k[r][s] = 0.5 * (k[r][s] + k[s][r]);
  return out;
}

void macro_strain_displacement(int i, int x0, int x1, int x2, double out[3]) {  // src/material.cpp:71-82
  out[0] = out[1] = out[2] = 0.0;
  switch (i) {
    case 0: out[0] = x0; break;
    case 1: out[1] = x1; break;
    case 2: out[2] = x2; break;
    case 3: out[0] = x1 / 2.0; out[1] = x0 / 2.0; break;
    case 4: out[1] = x2 / 2.0; out[2] = x1 / 2.0; break;
    case 5: out[0] = x2 / 2.0; out[2] = x0 / 2.0; break;
    default: throw std::invalid_argument("macro strain index must be in [0, 6)");
  }
}

StiffnessTables::StiffnessTables(const K0Matrix& ks) {  // src/fem.cpp:10-35
  for (int ke = 0; ke < 8; ++ke) {
    const int row = 7 - ke;
    for (int j = 0; j < 8; ++j)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          blk[ke][j][3 * r + c] = ks.k[3 * row + r][3 * j + c];
          blk_f[ke][j][3 * r + c] = float(ks.k[3 * row + r][3 * j + c]);
        }
    for (int i = 0; i < 6; ++i) {
      double acc[3] = {0, 0, 0};
      for (int j = 0; j < 8; ++j) {
        int d[3];
        lvo(j, d);
        double chi[3];
        macro_strain_displacement(i, d[0], d[1], d[2], chi);
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) acc[r] += blk[ke][j][3 * r + c] * chi[c];
      }
      for (int r = 0; r < 3; ++r) fmacro[ke][i][r] = acc[r];
    }
  }
}

ElementGalerkin::ElementGalerkin(const K0Matrix& ks) {  // src/multigrid.cpp:102-149, regrouped by n
  for (int oz = -2; oz <= 1; ++oz)
    for (int oy = -2; oy <= 1; ++oy)
      for (int ox = -2; ox <= 1; ++ox) {
        const int oidx = (ox + 2) + 4 * ((oy + 2) + 4 * (oz + 2));
        for (int n = 0; n < 27; ++n) {
          int delta[3];
          noff(n, delta);
          double acc[9] = {};
          bool any = false;
          for (int i = 0; i < 8; ++i) {
            int di[3];
            lvo(i, di);
            const double wi = tw1(ox + di[0]) * tw1(oy + di[1]) * tw1(oz + di[2]);
            if (wi == 0.0) continue;
            for (int j = 0; j < 8; ++j) {
              int dj[3];
              lvo(j, dj);
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
            t.oidx = oidx;
            std::memcpy(t.w, acc, sizeof(acc));
            by_n[size_t(n)].push_back(t);
          }
        }
      }
}

StencilGalerkin::StencilGalerkin() {  // src/multigrid.cpp:151-182
  for (int n = 0; n < 27; ++n) {
    int delta[3];
    noff(n, delta);
    for (int s = 0; s < 27; ++s) {
      int so[3];
      noff(s, so);
      const double ws = tw1(so[0]) * tw1(so[1]) * tw1(so[2]);
      for (int t = 0; t < 27; ++t) {
        int to[3];
        noff(t, to);
        const double wt = tw1(so[0] + to[0] - 2 * delta[0]) * tw1(so[1] + to[1] - 2 * delta[1]) *
                          tw1(so[2] + to[2] - 2 * delta[2]);
        if (ws * wt != 0.0) by_n[size_t(n)].push_back({s, t, ws * wt});
      }
    }
  }
}

}  // namespace ihomgpu
