/* ihom_b200.h -- C ABI of the B200-native inverse-homogenization hot path.
 *
 * The reference (/root/reference/proj) is a C++ library with no FFI; each entry
 * point below replaces the reference interface cited beside it, with plain
 * pointers/sizes and status codes instead of C++ types and exceptions
 * (SURVEY.md 8b). A C++ maintainer binds it through include/ihom_b200.hpp
 * (ihom::gpu::Homogenizer etc., same method names as the reference);
 * Python binds it with ctypes (paper_2301_08911_b200/__init__.py).
 *
 * Conventions
 *   - Nodal fields cross the boundary as AoS f64 [3*nv] in the reference's
 *     colour-block vertex order (inc/fem.hpp:15-26); element fields as f64
 *     [nx*ny*nz], x fastest (inc/density.hpp:20-31).
 *   - `where`: IHOM_HOST (pointer is host memory; copied in/out inside the call)
 *     or IHOM_DEVICE (pointer is CUDA device memory on the context's device).
 *   - Every call is stream-ordered on the context stream and synchronous at
 *     return. One host thread per context.
 *   - Errors: the reference's exceptions map to status codes; the message is
 *     available from ihom_last_error() (thread-local).
 *       std::invalid_argument -> IHOM_E_INVALID
 *       std::runtime_error (numerical: singular blocks, LDLT, coarsest) -> IHOM_E_NUMERIC
 *       std::logic_error (call order)  -> IHOM_E_STATE
 *       ihom::EvalError (objective domain) -> IHOM_E_EVAL
 *       CUDA failure -> IHOM_E_CUDA
 */
#ifndef IHOM_B200_H_
#define IHOM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  IHOM_OK = 0,
  IHOM_E_INVALID = 1,
  IHOM_E_NUMERIC = 2,
  IHOM_E_STATE = 3,
  IHOM_E_CUDA = 4,
  IHOM_E_EVAL = 5,
  IHOM_E_INTERNAL = 6
};
enum { IHOM_HOST = 0, IHOM_DEVICE = 1 };
enum { IHOM_MIXED = 0, IHOM_ALL_DOUBLE = 1 };          /* inc/config.hpp Precision */
enum { IHOM_SOLVER_VCYCLE = 0, IHOM_SOLVER_MIXED_DEFECT = 1, IHOM_SOLVER_PCG = 2 };
enum { IHOM_SYM_NONE = 0, IHOM_SYM_REFLECT3 = 1, IHOM_SYM_REFLECT6 = 2, IHOM_SYM_ROTATE3 = 3 };
enum { IHOM_KERNEL_LINEAR = 0, IHOM_KERNEL_SPLINE4 = 1 };
enum { IHOM_OBJ_BULK = 0, IHOM_OBJ_SHEAR = 1, IHOM_OBJ_NPR_RELAXED = 2, IHOM_OBJ_NPR_LOG = 3 };

typedef struct ihom_ctx ihom_ctx;

/* Homogenizer<T>(reso, mat, penal, opts), inc/homogenization.hpp:29 */
typedef struct {
  int n[3];
  double youngs, poisson; /* BaseMaterial, inc/material.hpp:17-35 */
  double penal;           /* SIMP exponent applied inside the homogenizer */
  int precision;          /* IHOM_MIXED (T=float) | IHOM_ALL_DOUBLE (T=double) */
  int device;             /* CUDA ordinal */
} ihom_desc;

/* SolverOptions, inc/multigrid.hpp:22-27 (+ mode) */
typedef struct {
  double tol;
  int max_cycles, pre_sweeps, post_sweeps;
  int mode; /* IHOM_SOLVER_* */
} ihom_solver_opts;

/* CellSolveStats, inc/homogenization.hpp:13-18 */
typedef struct {
  int total_cycles;
  double worst_residual;
  int worst_load;
  int converged;
} ihom_cell_stats;

/* SolveStats, inc/multigrid.hpp:29-33 */
typedef struct {
  int cycles;
  double rel_residual;
  int converged;
} ihom_solve_stats;

const char* ihom_last_error(void);
const char* ihom_version(void);

/* ---- Homogenizer (inc/homogenization.hpp:26-51) ---- */
ihom_ctx* ihom_create(const ihom_desc* desc, const ihom_solver_opts* opts);
void ihom_destroy(ihom_ctx* ctx);
int ihom_set_solver(ihom_ctx* ctx, const ihom_solver_opts* opts);                 /* options() */
int ihom_set_density(ihom_ctx* ctx, const double* rho_phys, int where);          /* set_density */
int ihom_solve_cell_problems(ihom_ctx* ctx, ihom_cell_stats* stats);              /* solve_cell_problems */
int ihom_effective_tensor(ihom_ctx* ctx, double C[36]);                           /* effective_tensor */
int ihom_tensor_sensitivity(ihom_ctx* ctx, const double seed[36], double* out, int where); /* tensor_sensitivity */
int ihom_get_displacement(ihom_ctx* ctx, int load, double* u_aos, int where);     /* displacement(i) */
int ihom_set_displacement(ihom_ctx* ctx, int load, const double* u_aos, int where);
/* Displacement storage (memory lever; no reference counterpart -- the paper keeps the six fields in
 * host-backed unified memory): 0 device-resident f64; 2 pinned-host f64 with f32
 * evaluation snapshots; 1 pinned-host f32 snapshots only. Knob U_HOST (-1 never, 0 auto when the
 * device-resident layout does not fit, 1 / 2 forced). -1 on error. */
int ihom_host_staged(ihom_ctx* ctx);

/* ---- z-slab decomposition ----
 * A grid of n[2] z planes is split into nranks slabs of t = n[2] / nranks
 * planes (t a multiple of 4); slab r holds planes [r t, (r+1) t) of every
 * element / vertex field (x-fastest elements; nodal fields in the slab's own
 * colour-block order). Slabs read across their faces directly from the
 * neighbours' memory: a LOCAL fabric keeps all slabs of a grid in this process
 * on one device (one host thread per slab); an IPC fabric maps one slab per
 * process over NVLink, exchanging CUDA IPC handles through the caller's
 * host allgather (e.g. torch.distributed). Every ihom_*_slab context call is
 * collective over the slabs of its fabric. The reference has no distributed
 * mode; this replaces nothing and keeps every per-slab result equal to the
 * single-domain one up to the order of the cross-slab sums. */
typedef struct ihom_fabric ihom_fabric;
typedef void (*ihom_allgather_fn)(const void* send, void* recv, size_t bytes, void* user);
ihom_fabric* ihom_fabric_local(int nranks, int device);
ihom_fabric* ihom_fabric_ipc(int rank, int nranks, int device, ihom_allgather_fn allgather, void* user);
void ihom_fabric_destroy(ihom_fabric* f);
ihom_ctx* ihom_create_slab(const ihom_desc* desc, const ihom_solver_opts* opts, ihom_fabric* f, int rank);
int ihom_slab_info(ihom_ctx* ctx, int* z0, int* planes, int* nranks);

/* ---- Hierarchy (inc/multigrid.hpp:53-93), via hierarchy() ---- */
int ihom_num_levels(ihom_ctx* ctx);
int ihom_level_dims(ihom_ctx* ctx, int level, int n[3]);
/* which: 0 = u, 1 = f, 2 = r; write != 0 uploads buf, else downloads. AoS host buffers. */
int ihom_level_field(ihom_ctx* ctx, int level, int which, int write, double* buf_aos);
int ihom_apply(ihom_ctx* ctx, int level, const double* x_aos, double* y_aos);     /* apply(l, x, y) */
int ihom_relax(ihom_ctx* ctx, int level, int sweeps);                              /* relax */
int ihom_compute_residual(ihom_ctx* ctx, int level);                               /* compute_residual */
int ihom_coarsest_solve(ihom_ctx* ctx);                                            /* coarsest_solve */
/* Coarsest-level dense solve of a caller-assembled operator (raw [3nv][3nv], dof order 3*loc+c)
   for load f [3nv]: factor_coarsest + coarsest_solve (src/multigrid.cpp:368-451) with the device
   kernel; x = translation-free solution, rel = ||A'x - Pf|| / ||Pf|| (A' the projected operator). */
int ihom_coarse_dense_solve(long long nv, const double* raw, const double* f, double* x, double* rel);
int ihom_v_cycle(ihom_ctx* ctx, double* rel);                                      /* v_cycle */
int ihom_solve(ihom_ctx* ctx, const double* f_aos, double* u_aos, ihom_solve_stats* st); /* solve(f, u, opts) */
int ihom_get_stencil(ihom_ctx* ctx, int level, double* out /* [nv][27][3][3] */);
int ihom_get_coeff(ihom_ctx* ctx, double* out /* [nv] */);
int ihom_macro_force(ihom_ctx* ctx, int load, double* f_aos);                      /* macro_force_kernel */
double ihom_op_scale(ihom_ctx* ctx);
long long ihom_kernel_launches(ihom_ctx* ctx);

/* colour-block location of every vertex (x-fastest enumeration) and, if nbr27 != NULL, the 27
   neighbour locations of every location (inc/grid.hpp:73-92, src/fem.cpp:37-68). Host outputs. */
int ihom_grid_locs(const int n[3], long long* locs, long long* nbr27);

/* restrict_residual_field (dir 0: out[coarse] = R in[fine]) / prolong_add_field (dir 1: out[fine] += P in[coarse])
   (inc/multigrid.hpp:13-20, src/multigrid.cpp:19-79) on the even fine grid nf; AoS host buffers in
   colour-block order; f32 != 0 runs the f32 inner-cycle transfer kernels (TRANSFER_F32), else f64. */
int ihom_transfer(const int nf[3], int dir, int f32, const double* in, double* out);

/* ---- density pipeline (inc/density.hpp:36-69, inc/oc.hpp:27-33) ---- */
int ihom_radial_filter(const int n[3], const double* f, double radius, int kernel, double* out, int where);
/* DensityExpr: radius < 1 (or < 0) means pow only. eval: phys = filter(design)^p, keeps pre in pre_out (may be null).
   backward: g_design = filter(g_phys * p * pre^(p-1)). */
int ihom_density_expr_eval(const int n[3], double radius, int kernel, double exponent, const double* design,
                           double* phys, double* pre_out, int where);
int ihom_density_expr_backward(const int n[3], double radius, int kernel, double exponent, const double* pre,
                               const double* g_phys, double* g_design, int where);
int ihom_symmetrize(const int n[3], double* field, int sym, int where);
int ihom_field_mean(const double* f, long long m, double* mean, int where);
/* oc_update: returns lambda, bisection_ok; trials = number of bisection trials (diagnostic) */
typedef struct {
  double min_density, step_limit, damp, volume, bisect_tol;
} ihom_oc_config;
int ihom_oc_update(long long m, const double* rho, const double* sens, const ihom_oc_config* cfg, double* out,
                   double* lambda, int* bisection_ok, int where);
int ihom_sensitivity_filter(const int n[3], const double* sens, const double* rho, double radius, double* out,
                            int where);
int ihom_init_trig(const int n[3], int basis_n, uint64_t seed, double volume, double sigmoid_k, double* rho,
                   int* fallback); /* host output; src/density.cpp:169-259 */

/* ---- objectives (src/objective.cpp:238-268) ---- */
int ihom_objective(int obj, double beta, double eta, double tau, double gamma, int iter, const double C[36],
                   double* value, double grad[36]);

/* ---- the optimisation loop (src/runner.cpp:51-136) ---- */
typedef struct { /* RunConfig, inc/config.hpp:15-42 */
  int reso;
  double vol, youngs, poisson;
  int obj;
  double beta, eta, tau, gamma, penal, filter_radius;
  int filter_placement; /* 0 density, 1 sensitivity */
  int kernel;           /* IHOM_KERNEL_* */
  int sym;              /* IHOM_SYM_* */
  int init;             /* 0 constant, 1 trig, 2 from init_rho */
  int basis_n;
  uint64_t seed;
  int max_iter;
  double step, damp, tol;
  int max_cycles;
  int precision; /* IHOM_MIXED | IHOM_ALL_DOUBLE */
  int solver_mode;
  int device;
} ihom_run_config;

typedef struct { /* IterationRecord, inc/runner.hpp:12-19 (+ tensor, OC diagnostics) */
  int iter;
  double objective, volume;
  int cycles;
  double residual, ms;
  double C[36];
  double lambda;
  int oc_trials;
} ihom_iter_record;

/* Observer (inc/runner.hpp:36-38): called after every density update with the
   record and (host copies of) prev/next design fields; return 0 to stop. */
typedef int (*ihom_observer)(int iter, const double* prev, const double* next, const ihom_iter_record* rec,
                             void* user);

/* flags: bit0 solver_failed, bit1 converged, bit2 init_fallback, bit3 oc_warning */
int ihom_run_optimization(const ihom_run_config* cfg, const double* init_rho /* host, may be null */,
                          ihom_iter_record* records, int capacity, int* nrec, double* rho_out /* host */,
                          int* flags, ihom_observer obs, void* user);

/* Stepping interface to the same loop: one optimisation iteration per call.
   rho_in (optional) replaces the current design before the iteration; rho_out (optional)
   receives the updated design; both live in `where` memory. status: 0 = design updated,
   1 = solver failed, 2 = converged, 3 = last iteration (no update in cases 1-3). */
typedef struct ihom_opt ihom_opt;
ihom_opt* ihom_opt_create(const ihom_run_config* cfg, const double* init_rho /* host, may be null */);
/* z-slab `rank` of the run over fabric f: designs in / out are that slab's
 * elements (global planes [rank t, (rank+1) t)); every call is collective. */
ihom_opt* ihom_opt_create_slab(const ihom_run_config* cfg, const double* init_rho, ihom_fabric* f, int rank);
void ihom_opt_destroy(ihom_opt* opt);
int ihom_opt_step(ihom_opt* opt, const double* rho_in, double* rho_out, int where, ihom_iter_record* rec,
                  int* status);
int ihom_opt_design(ihom_opt* opt, double* out, int where);
int ihom_opt_flags(ihom_opt* opt);
long long ihom_opt_launches(ihom_opt* opt);
void* ihom_opt_stream(ihom_opt* opt); /* the cudaStream_t every kernel of this optimiser runs on */

/* Multi-GPU (one process per GPU): load case i is solved by rank owner6[i] (NULL: i % nranks)
   and broadcast to every rank over NCCL; C^H, sensitivities and the design update then run
   identically on all ranks. uid128 = ncclUniqueId bytes from ihom_nccl_unique_id on rank 0. */
int ihom_nccl_unique_id(void* out128);
int ihom_opt_set_comm(ihom_opt* opt, const void* uid128, int rank, int nranks, const int* owner6);
int ihom_set_comm(ihom_ctx* ctx, const void* uid128, int rank, int nranks, const int* owner6);

/* Per-kernel-family device time (CUDA events on the launching stream) and algorithmic bytes. */
int ihom_profile_enable(int on); /* enabling resets the totals */
int ihom_profile_count(void);
long long ihom_launch_count(void); /* kernels launched by this library since load */
/* Runs one kernel family `reps` times on the context's current data (isolated timing / ncu target):
   l0_gs_f64|f32, l0_residual_f64|f32, l1_gs_*, l1_residual_*, vcycle_f64|f32, set_density, tensor, sensitivity. */
int ihom_bench_op(ihom_ctx* ctx, const char* op, int reps);
int ihom_profile_get(int index, char* family, int cap, long long* launches, double* ms, double* bytes);
/* Kernel-variant knobs (A/B switches; default = environment IHOM_<name>, else built-in):
   L0_PAIR (paired FFMA2 level-0 f32 kernels, 1), PAIR_MINB (3|4), L0_GS2 (1), RES_MINB (3),
   L0_KERNEL (0 fast | 1 smem-tiled). Every variant computes bit-identical results. */
int ihom_set_knob(const char* name, int value);
int ihom_get_knob(const char* name, int dflt);

#ifdef __cplusplus
}
#endif

#endif /* IHOM_B200_H_ */
