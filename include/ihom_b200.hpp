// ihom_b200.hpp -- header-only C++ wrapper over the C ABI (ihom_b200.h) that
// mirrors the reference API (proj/include/ihom/*.hpp) so a reference caller
// switches by changing the namespace (and the precision template argument into
// a constructor argument):
//
//   ihom::Homogenizer<float> hom(reso, mat, penal, opts);   // reference (CPU), inc/homogenization.hpp:29
//   ihom::gpu::Homogenizer   hom(reso, mat, penal, opts);   // this library (B200), Precision::mixed
//
// IVec3, BaseMaterial and SolverOptions have the reference's fields and
// validation (inc/grid.hpp:9, inc/material.hpp:17-35, inc/multigrid.hpp:22-27).
//
// Exceptions are re-raised with the reference's types (std::invalid_argument,
// std::runtime_error, std::logic_error) from the C status codes.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ihom_b200.h"

namespace ihom {
namespace gpu {

inline void check(int rc) {
  if (rc == IHOM_OK) return;
  const std::string msg = ihom_last_error();
  switch (rc) {
    case IHOM_E_INVALID: throw std::invalid_argument(msg);
    case IHOM_E_STATE: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

enum class Precision { mixed, all_double };  // the reference's Homogenizer<float> / Homogenizer<double>

using IVec3 = std::array<int, 3>;  // inc/grid.hpp:9

struct BaseMaterial {  // inc/material.hpp:17-35
  double youngs = 1.0;
  double poisson = 0.3;
  BaseMaterial() = default;
  BaseMaterial(double e, double nu) : youngs(e), poisson(nu) {
    if (!(e > 0.0)) throw std::invalid_argument("Young's modulus must be positive");
    if (!(nu > -1.0 && nu < 0.5)) throw std::invalid_argument("Poisson's ratio must lie in (-1, 0.5)");
  }
  double lambda() const { return youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)); }
  double mu() const { return youngs / (2.0 * (1.0 + poisson)); }
};

struct SolverOptions {  // inc/multigrid.hpp:22-27 (+ the solver mode of this library)
  double tol = 1e-2;
  int max_cycles = 50;
  int pre_sweeps = 1;
  int post_sweeps = 1;
  int mode = IHOM_SOLVER_VCYCLE;
};

struct CellSolveStats {  // inc/homogenization.hpp:13-18
  int total_cycles = 0;
  double worst_residual = 0.0;
  int worst_load = -1;
  bool converged = true;
};

using Matrix6 = std::array<double, 36>;  // row-major 6x6 (Voigt 11,22,33,12,23,13)

// Device twin of ihom::Homogenizer<T> (inc/homogenization.hpp:26-51). Density
// and sensitivity vectors are host std::vector<double> (x-fastest elements);
// raw device pointers are accepted by the *_device overloads.
class Homogenizer {
 public:
  // inc/homogenization.hpp:29: Homogenizer(IVec3 reso, const BaseMaterial& mat, double penal, const SolverOptions&)
  Homogenizer(IVec3 reso, const BaseMaterial& mat, double penal, const SolverOptions& o,
              Precision p = Precision::mixed, int device = 0) {
    ihom_desc d{{reso[0], reso[1], reso[2]}, mat.youngs, mat.poisson, penal,
                p == Precision::mixed ? IHOM_MIXED : IHOM_ALL_DOUBLE, device};
    ihom_solver_opts so{o.tol, o.max_cycles, o.pre_sweeps, o.post_sweeps, o.mode};
    ctx_ = ihom_create(&d, &so);
    if (!ctx_) throw std::invalid_argument(ihom_last_error());
    nv_ = (long long)reso[0] * reso[1] * reso[2];
  }
  ~Homogenizer() { ihom_destroy(ctx_); }
  Homogenizer(const Homogenizer&) = delete;
  Homogenizer& operator=(const Homogenizer&) = delete;

  void set_density(const std::vector<double>& rho_phys) { check(ihom_set_density(ctx_, rho_phys.data(), IHOM_HOST)); }
  void set_density_device(const double* rho_phys) { check(ihom_set_density(ctx_, rho_phys, IHOM_DEVICE)); }
  CellSolveStats solve_cell_problems() {
    ihom_cell_stats s{};
    check(ihom_solve_cell_problems(ctx_, &s));
    return {s.total_cycles, s.worst_residual, s.worst_load, s.converged != 0};
  }
  Matrix6 effective_tensor() {
    Matrix6 c{};
    check(ihom_effective_tensor(ctx_, c.data()));
    return c;
  }
  std::vector<double> tensor_sensitivity(const Matrix6& seed) {
    std::vector<double> out(static_cast<size_t>(nv_));
    check(ihom_tensor_sensitivity(ctx_, seed.data(), out.data(), IHOM_HOST));
    return out;
  }
  std::vector<double> displacement(int i) {  // AoS [nv][3], colour-block vertex order
    std::vector<double> out(static_cast<size_t>(3 * nv_));
    check(ihom_get_displacement(ctx_, i, out.data(), IHOM_HOST));
    return out;
  }
  void set_displacement(int i, const std::vector<double>& u) {
    check(ihom_set_displacement(ctx_, i, u.data(), IHOM_HOST));
  }
  // where the six fields live: 0 device-resident, 2 / 1 host-staged (memory lever)
  int host_staged() {
    const int v = ihom_host_staged(ctx_);
    if (v < 0) check(IHOM_E_STATE);
    return v;
  }
  ihom_ctx* handle() { return ctx_; }

 private:
  ihom_ctx* ctx_ = nullptr;
  long long nv_ = 0;
};

// radial_filter / symmetrize / oc_update (inc/density.hpp:36-69, inc/oc.hpp:27-33)
inline std::vector<double> radial_filter(std::array<int, 3> n, const std::vector<double>& f, double radius,
                                         int kernel = IHOM_KERNEL_SPLINE4) {
  std::vector<double> out(f.size());
  check(ihom_radial_filter(n.data(), f.data(), radius, kernel, out.data(), IHOM_HOST));
  return out;
}
inline void symmetrize(std::vector<double>& field, std::array<int, 3> n, int sym) {
  check(ihom_symmetrize(n.data(), field.data(), sym, IHOM_HOST));
}
struct OCResult {
  std::vector<double> rho;
  double lambda = 0.0;
  bool bisection_ok = true;
};
inline OCResult oc_update(const std::vector<double>& rho, const std::vector<double>& sens, const ihom_oc_config& cfg) {
  OCResult r;
  r.rho.resize(rho.size());
  int ok = 0;
  check(ihom_oc_update((long long)rho.size(), rho.data(), sens.data(), &cfg, r.rho.data(), &r.lambda, &ok,
                       IHOM_HOST));
  r.bisection_ok = ok != 0;
  return r;
}

}  // namespace gpu
}  // namespace ihom
