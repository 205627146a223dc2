// density.hpp -- design-side device operations (see density_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "fabric.hpp"

namespace ihomgpu {

constexpr double kRhoMin = 0.001;  // inc/density.hpp:12

struct Tap {
  int d[3];
  double w;
};

// Scratch shared by reductions: partial sums, two scalars, a flag.
struct Workspace {
  double* partials = nullptr;  // >= 21 * kReducePartials doubles
  double* scalar = nullptr;
  double* scalar2 = nullptr;
  double* scalars = nullptr;   // 64 doubles of general scratch
  int* flag = nullptr;
};

struct OCConfig {  // inc/oc.hpp:10-16
  double min_density = kRhoMin;
  double step_limit = 0.05;
  double damp = 0.5;
  double volume = 0.3;
  double bisect_tol = 1e-6;
};

struct OCResult {  // inc/oc.hpp:18-22
  double lambda = 0.0;
  bool bisection_ok = true;
  int trials = 0;
};

// z-slab forms: n = this slab's dims (n0, n1, t) for the filters; the links
// reach the slabs below / above. Defaults = one periodic domain.
void radial_filter(const int n[3], const double* f, double radius, int kernel, double* out, cudaStream_t s,
                   ZLink<double> fl = {});
void sensitivity_filter(const int n[3], const double* sens, const double* rho, double radius, double* out,
                        cudaStream_t s, ZLink<double> sl = {}, ZLink<double> rl = {});
void pow_field(const double* x, double p, long long m, double* out, cudaStream_t s);
void pow_backward(const double* x, const double* g, double p, long long m, double* out, cudaStream_t s);
void symmetrize(const int n[3], double* field, int sym, double* scratch, cudaStream_t s);
// n = global dims; field / scratch = this slab's planes; peers = every slab's copy
void symmetrize_slab(const int n[3], const Slab& slab, double* field, PeerTable fpeers, double* scratch,
                     PeerTable speers, int sym, cudaStream_t s);
void clamp_field(double* f, long long m, double lo, double hi, cudaStream_t s);
void field_sum(const double* f, long long m, double* partials, double* out, cudaStream_t s, const Slab& slab = {});
// n = global dims; rho / scratch = this slab's planes
bool init_trig(const int n[3], int basis_n, std::uint64_t seed, double volume, double sigmoid_k, double* rho,
               double* scratch, Workspace& ws, cudaStream_t s, const Slab& slab = {});
// m = this slab's elements, m_total = the whole grid's (the volume mean)
// Device-resident bisection (density_kernels.cu); `out` (not aliasing rho or g) doubles as scratch.
OCResult oc_update(long long m, const double* rho, const double* g, const OCConfig& cfg, double* out, Workspace& ws,
                   cudaStream_t s, const Slab& slab = {}, long long m_total = 0);

}  // namespace ihomgpu
