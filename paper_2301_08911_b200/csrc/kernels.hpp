// kernels.hpp -- host-callable launchers for every device kernel of the hot
// path. All launchers are asynchronous on the given stream; templates are
// instantiated explicitly in the .cu files for the supported type sets.
//
// Type parameters: TC = element-coefficient / stencil storage (float in mixed
// mode, double in all-double mode); TN = nodal storage; TA = arithmetic type
// of the merged stencil.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "fabric.hpp"
#include "tables.hpp"

namespace ihomgpu {

// ---- constant tables (one upload per material; cheap, idempotent) ----
void upload_fem_tables(const StiffnessTables& t, const K0Matrix& k, cudaStream_t s);
void upload_galerkin_tables(const ElementGalerkin& eg, cudaStream_t s);
void upload_hom_tables(const double hada_classes[], cudaStream_t s);  // hom_kernels.cu (from upload_fem_tables)
void upload_gs_group_tables(const float kappa_f[], cudaStream_t s);    // gs_group_kernels.cu (idem)

// ---- level 0, matrix-free (src/fem.cpp:98-156, src/multigrid.cpp:263-279) ----
template <typename TC>
void launch_coeff(const double* rho, TC* coeff, long long m, double penal, cudaStream_t s);

// y = K u (f == nullptr) or y = f - K u, over all vertices.
template <typename TC, typename TN, typename TA>
void launch_l0_apply(const GridGeo& g, const TC* coeff, const TN* u, const TN* f, TN* y, cudaStream_t s,
                     ZLink<TC> cl = {}, ZLink<TN> ul = {});

// One colour pass of the 8-colour Gauss-Seidel (src/fem.cpp:122-137).
template <typename TC, typename TN, typename TA>
void launch_l0_gs_color(const GridGeo& g, const TC* coeff, const TN* f, TN* u, int color, cudaStream_t s,
                        ZLink<TC> cl = {}, ZLink<TN> ul = {}, bool zero_start = false);
// fused pass of colours ca and ca ^ 1 (f32 inner fields): one CTA per row, bit-identical to the two passes

// true if launch_l0_gs_color takes the zero-start path on this grid (it then never reads colours > c
// during the first sweep, so u need not be cleared before it)
template <typename TC, typename TN, typename TA>
bool l0_gs_zero_start_ok(const GridGeo& g);

// z-plane sweep variants (sweep_kernels.cuh): shared-memory plane ring, bit-identical outputs
bool sweep_ok(const GridGeo& g);
template <typename TC, typename TN, typename TA>
void launch_l0_apply_sweep(const GridGeo& g, const TC* coeff, ZLink<TC> cl, const TN* u, ZLink<TN> ul, const TN* f,
                           TN* y, cudaStream_t s);
long long launch_l0_defect_sweep(const GridGeo& g, const float* coeff, ZLink<float> cl, const double* u,
                                 ZLink<double> ul, const double* f, float* r32, double* partials, cudaStream_t s);
// the same with the defect-correction update folded in: unew = u + e (f32 e), r32 = float(f - K unew)
long long launch_l0_defect_update_sweep(const GridGeo& g, const float* coeff, ZLink<float> cl, const double* u,
                                        ZLink<double> ul, const float* e, ZLink<float> el, double* unew,
                                        const double* f, float* r32, double* partials, cudaStream_t s);
// Fused defect residual: r32 = float(f - K u) (f64 arithmetic), per-block |r|^2 partials; returns #partials.
template <typename TC>
long long launch_l0_residual_norm(const GridGeo& g, const TC* coeff, const double* u, const double* f, float* r32,
                                  double* partials, cudaStream_t s, ZLink<TC> cl = {}, ZLink<double> ul = {});

// Colour passes `color` and color + 1 (color even) of the f32 level-0 GS in one launch (blocks own whole
// rows; bitwise the two separate passes). Knob GS_PAIR.
bool l0_gs_pair_ok(const GridGeo& g);
void launch_l0_gs_pair(const GridGeo& g, const float* coeff, const float* f, float* u, int color, cudaStream_t s,
                       ZLink<float> cl, ZLink<float> ul, bool zero_start);
template <typename TC>
void launch_macro_force(const GridGeo& g, const TC* coeff, int load, double* f, cudaStream_t s, ZLink<TC> cl = {});
// macro force plus the component sums of f (sums[3]) from per-block partials of the same pass
// (block_sums: 3 macro_force_sums_blocks(g) doubles); even grids only (fast_ok)
long long macro_force_sums_blocks(const GridGeo& g);
template <typename TC>
void launch_macro_force_sums(const GridGeo& g, const TC* coeff, int load, double* f, double* block_sums,
                             double* partials, double* sums, cudaStream_t s, ZLink<TC> cl = {},
                             unsigned* ticket = nullptr);

// ---- transfer (src/multigrid.cpp:12-79) ----
// z-slab arguments: rl / cl link the source array to the slabs
// below / above; gout + zoff redirect the coarse output of a restriction (or
// Galerkin product) into the replicated global coarse level at this slab's
// first halved plane zoff; a prolongation from the replicated level reads it
// at coarse plane offset zoff. Defaults = one periodic domain.
template <typename TN>
void launch_restrict(const GridGeo& gf, const GridGeo& gc, const TN* rf, TN* fc, cudaStream_t s, ZLink<TN> rl = {},
                     const GridGeo* gout = nullptr, int zoff = 0);
template <typename TN>
void launch_prolong_add(const GridGeo& gc, const GridGeo& gf, const TN* uc, TN* uf, cudaStream_t s,
                        ZLink<TN> cl = {}, int zoff = 0);

// the same for the RHS lanes of a lockstep group in one launch (f32 inner fields, TRANSFER_F32, even
// grids; per-lane arithmetic identical to one launch per lane)
bool transfer_group_ok(const GridGeo& gf, const GridGeo& gc);
void launch_restrict_group(const GridGeo& gf, const GridGeo& gc, int nl, const float* const* rf,
                           const ZLink<float>* rl, float* const* fc, cudaStream_t s);
void launch_prolong_add_group(const GridGeo& gc, const GridGeo& gf, int nl, const float* const* uc,
                              const ZLink<float>* cl, float* const* uf, cudaStream_t s);

// ---- coarse levels (src/multigrid.cpp:186-239, 281-333) ----
template <typename TS, typename TN>
void launch_stencil_apply(const GridGeo& g, const TS* st, const TN* x, const TN* f, TN* y, cudaStream_t s,
                          ZLink<TN> xl = {});
template <typename TS, typename TN>
void launch_stencil_gs_color(const GridGeo& g, const TS* st, const TN* f, TN* u, int color, int* err,
                             cudaStream_t s, ZLink<TN> ul = {}, bool zero_start = false);
// the same for nl = 1, 2, 3 or 6 right-hand sides in lockstep (each stencil block read once for all;
// per-RHS arithmetic identical to the single launches)
constexpr int kMaxRhsGroup = 6;
template <typename TS, typename TN>
void launch_stencil_apply_group(const GridGeo& g, const TS* st, int nl, const TN* const* x, const TN* const* f,
                                TN* const* y, cudaStream_t s, const ZLink<TN>* xl);
template <typename TS, typename TN>
void launch_stencil_gs_color_group(const GridGeo& g, const TS* st, int nl, const TN* const* f, TN* const* u,
                                   int color, int* err, cudaStream_t s, const ZLink<TN>* ul, bool zero_start = false);
template <typename TC>
void launch_galerkin_from_elements(const GridGeo& gf, const GridGeo& gc, const TC* coeff, TC* st, cudaStream_t s,
                                   ZLink<TC> cl = {}, const GridGeo* gout = nullptr, int zoff = 0);
template <typename TS>
void launch_galerkin_from_stencil(const GridGeo& gf, const GridGeo& gc, const TS* stf, TS* stc, cudaStream_t s,
                                  ZLink<TS> sl = {}, const GridGeo* gout = nullptr, int zoff = 0);

// Coarsest level: x = Ainv f with <=3 refinement steps against A, translation
// projection in/out, singularity flag (src/multigrid.cpp:426-451). Single block.
template <typename TN>
void launch_coarsest_solve(int ndof, long long nv, const double* Ainv, const double* A, const double* Q, int nq, TN* f,
                           TN* u, double negligible, double* work, int* err, cudaStream_t s);
// every RHS lane of a lockstep group (f32 inner fields, block per lane; work: nl * 3 ndof doubles)
// Bottom of the grouped inner V-cycle in one cooperative launch (levels whose colour passes are
// warp-per-vertex, <= 32^3, down to the coarsest): the same per-vertex kernels in the same order as the
// level-by-level launches, grid-wide barriers between the passes (bitwise the same results).
constexpr int kMaxBottom = 6;
struct BottomLevel {
  GridGeo g;
  const float* st;  // stencils (unused on the coarsest level)
  float* eu[kMaxRhsGroup];
  float* ef[kMaxRhsGroup];
  float* er[kMaxRhsGroup];
  int zs;           // zero-start pre-smoothing (else e is cleared first)
};
struct BottomCycle {
  int nlev;  // levels [lb, lmax]; L[nlev - 1] is the coarsest
  BottomLevel L[kMaxBottom];
  int pre, post;
  int N;
  long long nvc;
  const double* Ainv;
  const double* A;
  const double* Q;
  int nq;
  double* work;  // 3 N per lane
  int* err;
};
bool bottom_level_ok(const GridGeo& g, const GridGeo& gc);  // level g (next coarser gc) can run inside
bool launch_bottom_cycle(const BottomCycle& bc, int nl, cudaStream_t s);  // false: launch refused (too large)
void launch_coarsest_solve_group(int ndof, long long nv, const double* Ainv, const double* A, const double* Q, int nq,
                                 int nl, float* const* f, float* const* u, double* work, int* err, cudaStream_t s);

// ---- reductions (deterministic: fixed partition per size, fixed fold order) ----
// sums of the three AoS components: out[3]
template <typename TN>
void launch_comp_sums(const TN* x, long long nv, double* partials, double* out, cudaStream_t s,
                      unsigned* ticket = nullptr);  // ticket: fold the partials in the last block (one launch)
// out[c] = fold of the per-block partials (c < ncomp), the second stage of every reduction here
void launch_finalize(const double* partials, int nparts, int ncomp, double* out, cudaStream_t s);
// out[0] = dot(a, b) over n entries
template <typename TN>
void launch_dot(const TN* a, const TN* b, long long n, double* partials, double* out, cudaStream_t s,
                unsigned* ticket = nullptr);
// x[3 i + c] -= sums[c] / count (count = vertices of the whole grid; default nv)
template <typename TN>
void launch_sub_means(TN* x, long long nv, const double* sums, cudaStream_t s, long long count = 0);
// dst = src - mean (per component), the in-place variant's arithmetic
// x -= per-component mean (sums / count) and out = ||x||^2, bitwise launch_sub_means + launch_dot
void launch_sub_means_norm(double* x, long long nv, const double* sums, double* partials, double* out,
                           cudaStream_t s, long long count = 0, unsigned* ticket = nullptr);
void launch_sub_means_copy(const double* src, double* dst, long long nv, const double* sums, cudaStream_t s,
                           long long count = 0);
void launch_int_to_double(const int* in, double* out, cudaStream_t s);
// z-slab: copy the planes of the replicated level g owned by the other slabs (planes per slab)
template <typename X>
void launch_gather_owned(const GridGeo& g, PeerTable peers, int planes, int me, int per_vertex, X* dst,
                         cudaStream_t s);
// u += e (f64 += TN)
template <typename TN>
void launch_axpy_update(double* u, const TN* e, long long n, cudaStream_t s);
// y = (TO) x
template <typename TI, typename TO>
void launch_convert(const TI* x, TO* y, long long n, cudaStream_t s);
constexpr int kReducePartials = 1184;  // 8 * 148: capacity of the partials buffer (per component)
void launch_sum(const double* a, long long n, double* partials, double* out, cudaStream_t s,
                unsigned* ticket = nullptr);
// MG-PCG helpers
void launch_dot_df(const double* a, const float* b, long long n, double* partials, double* out, cudaStream_t s);
void launch_pcg_p(double* p, const float* z, const double* beta, long long n, bool first, cudaStream_t s);
void launch_pcg_ur(double* u, double* r, const double* p, const double* q, const double* alpha, float* r32,
                   long long n, double* partials, double* out, cudaStream_t s);
void launch_ratio(const double* num, const double* den, double* out, cudaStream_t s);
void launch_grid_locs(const GridGeo& g, long long* out, long long* out27, cudaStream_t s);
void copy_nodal(const double* in, double* out, long long nv, cudaStream_t s);

// ---- homogenization (src/homogenization.cpp:58-144) ----
// partial sums (21 per block) of q_e * d_i^T K0 d_j; finalized into C[21].
template <typename TN>
void launch_effective_tensor(const GridGeo& g, const TN* const u[6], const double* rho, double penal, bool snap_f32,
                             double lambda, double mu, double* partials, double* c21, cudaStream_t s,
                             const TN* const* uhi = nullptr, void* ecache = nullptr);
// ecache: optional [21][nv] per-element energies written by the tensor pass (TE = f32 when snap_f32, else f64);
// the sensitivity then reads them instead of recomputing (bit-identical).
// true when the mixed-mode element energies run in f32 (knob ENERGY_F32; default: f64 like the reference)
bool energy_f32(bool snap);
void launch_sensitivity_cached(long long nv, const void* ecache, bool f32, const double* rho, double penal,
                               const double* sym_seed36, double* out, cudaStream_t s, long long m_total);
// z-slab: uhi = the six fields of the slab above; m_total = elements of the whole grid (the 1/M factor)
template <typename TN>
void launch_tensor_sensitivity(const GridGeo& g, const TN* const u[6], const double* rho, double penal,
                               bool snap_f32, double lambda, double mu, const double* sym_seed36, double* out,
                               cudaStream_t s, const TN* const* uhi = nullptr, long long m_total = 0);

}  // namespace ihomgpu
