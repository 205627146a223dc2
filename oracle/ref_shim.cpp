// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers that expose the UNMODIFIED reference density/OC code
// (/root/reference/proj/src/density.cpp, src/oc.cpp, compiled from where they
// lie by oracle/Makefile into oracle/_ref/libihom_ref.so) so the tests can pin
// the oracle restatement bit-for-bit and bench.py can time the reference's own
// CPU code for the density side of the iteration. Only these two translation
// units build without Eigen; nothing here is product code.

#include <cstring>
#include <optional>
#include <stdexcept>

#include "ihom/density.hpp"
#include "ihom/oc.hpp"
#include "ihom/parallel.hpp"

using namespace ihom;

namespace {
DensityField make(int nx, int ny, int nz, const double* p) {
  DensityField f({nx, ny, nz});
  std::memcpy(f.v.data(), p, sizeof(double) * f.v.size());
  return f;
}
FilterKernel kern(int k) { return k == 0 ? FilterKernel::linear : FilterKernel::spline4; }
Symmetry symm(int s) {
  switch (s) {
    case 1: return Symmetry::reflect3;
    case 2: return Symmetry::reflect6;
    case 3: return Symmetry::rotate3;
    default: return Symmetry::none;
  }
}
}  // namespace

extern "C" {

void ref_set_workers(int n) { set_worker_count(n); }

double ref_field_mean(int nx, int ny, int nz, const double* f) { return field_mean(make(nx, ny, nz, f)); }

void ref_radial_filter(int nx, int ny, int nz, const double* f, double radius, int kernel, double* out) {
  const DensityField r = radial_filter(make(nx, ny, nz, f), radius, kern(kernel));
  std::memcpy(out, r.v.data(), sizeof(double) * r.v.size());
}

// radius < 0: pow only. g_phys may be null (eval only).
void ref_density_expr(int nx, int ny, int nz, double radius, int kernel, double exponent, const double* design,
                      double* phys, const double* g_phys, double* g_design) {
  DensityExpr e = radius < 0 ? DensityExpr::pow_only(exponent) : DensityExpr(radius, kern(kernel), exponent);
  const DensityField out = e.eval(make(nx, ny, nz, design));
  std::memcpy(phys, out.v.data(), sizeof(double) * out.v.size());
  if (g_phys) {
    const std::vector<double> g(g_phys, g_phys + out.v.size());
    const std::vector<double> gd = e.backward(g);
    std::memcpy(g_design, gd.data(), sizeof(double) * gd.size());
  }
}

int ref_symmetrize(int nx, int ny, int nz, double* f, int sym) {
  try {
    std::vector<double> v(f, f + std::size_t(nx) * ny * nz);
    symmetrize(v, {nx, ny, nz}, symm(sym));
    std::memcpy(f, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

int ref_init_trig(int nx, int ny, int nz, int basis_n, unsigned long long seed, double volume, double k,
                  double* rho) {
  TrigInitSpec s;
  s.basis_n = basis_n;
  s.seed = seed;
  s.volume = volume;
  s.sigmoid_k = k;
  const TrigInitResult r = init_trig(s, {nx, ny, nz});
  std::memcpy(rho, r.field.v.data(), sizeof(double) * r.field.v.size());
  return r.fallback ? 1 : 0;
}

int ref_oc_update(int nx, int ny, int nz, const double* rho, const double* sens, double volume, double step,
                  double damp, double* out, double* lambda) {
  OCConfig c;
  c.volume = volume;
  c.step_limit = step;
  c.damp = damp;
  const OCResult r = oc_update(make(nx, ny, nz, rho), make(nx, ny, nz, sens), c);
  std::memcpy(out, r.rho.v.data(), sizeof(double) * r.rho.v.size());
  *lambda = r.lambda;
  return r.bisection_ok ? 1 : 0;
}

void ref_sensitivity_filter(int nx, int ny, int nz, const double* sens, const double* rho, double radius,
                            double* out) {
  const DensityField r = sensitivity_filter(make(nx, ny, nz, sens), make(nx, ny, nz, rho), radius);
  std::memcpy(out, r.v.data(), sizeof(double) * r.v.size());
}

}  // extern "C"
