// tables.hpp -- host-side constant tables, computed once per material and
// uploaded to __constant__ memory ("host-computed once").
//
//   K0        24x24 unit-element stiffness, src/material.cpp:39-69
//   blk       blk[ke][j] = K0 block (7-ke, j), src/fem.cpp:10-23
//   fmacro    fmacro[ke][i] = sum_j blk[ke][j] chi^i(j), src/fem.cpp:24-33
//   egal      level-1 Galerkin weights W(o, delta), src/multigrid.cpp:102-149
//   sgal      level>=2 Galerkin weights w(s) w(s+t-2 delta), src/multigrid.cpp:151-182
#pragma once

#include <array>
#include <vector>

namespace ihomgpu {

struct Material {
  double youngs = 1.0, poisson = 0.3;
  double lambda() const { return youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)); }
  double mu() const { return youngs / (2.0 * (1.0 + poisson)); }
};

void validate_material(const Material& m);  // inc/material.hpp:23-25

struct K0Matrix {
  double k[24][24];
};

K0Matrix element_stiffness(const Material& m);
void macro_strain_displacement(int i, int x0, int x1, int x2, double out[3]);

struct StiffnessTables {
  double blk[8][8][9];
  float blk_f[8][8][9];
  double fmacro[8][6][3];
  explicit StiffnessTables(const K0Matrix& k);
};

// Level-1 Galerkin table grouped by output neighbour n: terms[n] lists
// (fine-element offset index oidx in [0,64), 9 weights).
struct ElementGalerkin {
  struct Term {
    int oidx;
    double w[9];
  };
  std::array<std::vector<Term>, 27> by_n;
  explicit ElementGalerkin(const K0Matrix& k);
};

// Stencil-to-stencil table grouped by coarse neighbour n: (s, t, w).
struct StencilGalerkin {
  struct Term {
    int s, t;
    double w;
  };
  std::array<std::vector<Term>, 27> by_n;
  StencilGalerkin();
};

}  // namespace ihomgpu
