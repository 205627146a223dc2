// hierarchy.hpp -- device-resident geometric multigrid hierarchy and the
// homogenizer that drives the six periodic cell problems.
//
// Mirrors ihom::Hierarchy<T> (inc/multigrid.hpp:53-93) and
// ihom::Homogenizer<T> (inc/homogenization.hpp:26-51): same method names,
// same semantics, T = coefficient/stencil storage (float: mixed, double:
// all-double). Nodal data are f64 AoS [loc][3] in device memory.
//
// Two solver modes:
//   kVCycle    -- the reference's stationary V-cycle iteration, step for step
//                 (src/multigrid.cpp:453-501), f64 nodal data throughout;
//   kPCG (mixed precision) -- conjugate gradients on K u = f in f64, preconditioned
//                 by one symmetric inner V-cycle (f32; post-smoothing in reverse
//                 colour order so the preconditioner is SPD), same stopping rule;
//   kMixedDefect (mixed precision only) -- the same V-cycle in defect-correction
//                 form: the outer residual r = f - K u and the update u += e
//                 are f64, the inner V-cycle on K e = r runs on f32 nodal data
//                 (identical to the reference's cycle in exact arithmetic;
//                 see DESIGN.md "solver modes").
#pragma once

#include <array>
#include <future>
#include <memory>
#include <string>
#include <vector>

#include "comm.hpp"
#include "common.cuh"
#include "density.hpp"
#include "fabric.hpp"
#include "kernels.hpp"
#include "tables.hpp"

namespace ihomgpu {

// Coarsest-level dense factorisation (src/multigrid.cpp:368-383): a (dof order 3*loc+c, raw
// assembly in, projected operator out unless knob COARSE_PROJECT=0), explicit inverse of the
// deflated matrix via pivoted LDL^T. Returns op_scale (mean diagonal of the raw operator).
// Near-null modes beyond the translations (|pivot| < 1e-6 op_scale) are deflated too: their orthonormal
// directions go to *q ([m][3nv]) and *m; the device solve projects the load off them.
double factor_coarse_dense(std::vector<double>& a, long long nv, std::vector<double>& inv,
                           std::vector<double>* q = nullptr, int* m = nullptr);

enum SolverMode { kVCycle = 0, kMixedDefect = 1, kPCG = 2 };

struct SolverOptions {  // inc/multigrid.hpp:22-27
  double tol = 1e-2;
  int max_cycles = 50;
  int pre_sweeps = 1;
  int post_sweeps = 1;
  int mode = kVCycle;
};

struct SolveStats {  // inc/multigrid.hpp:29-33
  int cycles = 0;
  double rel_residual = 0.0;
  bool converged = false;
};

struct CellSolveStats {  // inc/homogenization.hpp:13-18
  int total_cycles = 0;
  double worst_residual = 0.0;
  int worst_load = -1;
  bool converged = true;
};

// RAII device buffer.
template <typename X>
struct DevBuf {
  X* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) IHOM_CUDA(cudaMalloc(&p, sizeof(X) * count));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p;
    n = o.n;
    o.p = nullptr;
    o.n = 0;
    return *this;
  }
};

template <typename X>
ZLink<X> neighbours(const std::vector<void*>& all, int rank) {
  const int n = int(all.size());
  return {static_cast<const X*>(all[size_t((rank + n - 1) % n)]), static_cast<const X*>(all[size_t((rank + 1) % n)])};
}
inline PeerTable peer_table(const std::vector<void*>& all) {
  PeerTable t{};
  for (size_t r = 0; r < all.size(); ++r) t.p[r] = all[r];
  return t;
}

template <typename T>
class Hierarchy {
 public:
  using value_type = T;
  // n = dims of the WHOLE grid; with a slab only planes [rank t, (rank+1) t) are stored
  // lean: host-staged-displacement layout (memory lever): 0 never, 1 when the device-resident
  // layout would not fit this device's free HBM (decided collectively over the slabs), 2 always. A lean
  // hierarchy (mixed precision, even grids) allocates no level-0 f64 r and no f64 u/f/r on coarser
  // levels (the mixed_defect solver never reads them), no ping-pong u and no lockstep RHS slots.
  Hierarchy(const int n[3], const Material& mat, double penal, cudaStream_t s, Slab slab = {}, int lean = 0);
  ~Hierarchy() {
    quiesce();
    try {
      join_coarsest();
    } catch (...) {
    }
    if (h_pinned_) cudaFreeHost(h_pinned_);
    if (h_coarse_) cudaFreeHost(h_coarse_);
    if (s_fact_) cudaStreamDestroy(s_fact_);
    if (ev_fact_) cudaEventDestroy(ev_fact_);
  }
  // z-slab teardown is collective: no slab frees buffers its neighbours may still read
  void quiesce() noexcept {
    try {
      sync();
      cudaStreamSynchronize(s_);
    } catch (...) {
    }
  }
  Hierarchy(const Hierarchy&) = delete;
  Hierarchy& operator=(const Hierarchy&) = delete;

  void set_density(const double* rho_phys_dev);
  void bind_tables();  // re-upload this hierarchy's constant tables (shared per process)
  int num_levels() const { return int(levels_.size()); }
  const GridGeo& geo(int l) const { return levels_[size_t(l)].g; }

  // Reference operations on the f64 level fields.
  void apply(int l, const double* x, double* y);  // y = K_l x
  void relax(int l, int sweeps, bool zero_start = false);  // zero_start: u == 0 on entry (first sweep skips it)
  void compute_residual(int l);
  void coarsest_solve();
  double v_cycle(const SolverOptions& opts);
  // Solve K u = f with l0.f already holding the load; u is the warm start /
  // result buffer (bound as level-0 u for the duration of the call; ul = its
  // z-slab links).
  SolveStats solve_bound(double* u, const SolverOptions& opts, ZLink<double> ul = {});
  // ---- lockstep groups of right-hand sides (RHS_PAIRS on; RHS_GROUP = 2, 3 or 6 cell problems): a
  // group shares every coarse-level stencil read. The inactive RHSs' per-RHS fields and solver state
  // live in slots_ and are swapped in by select_rhs(); every level-0 operation runs per RHS exactly as
  // in a single solve.
  bool pair_ok(const SolverOptions& opts) const;
  int group_size(const SolverOptions& opts);  // 1 (no grouping), 2, 3 or 6; collective on z-slabs
  void select_rhs(int k);
  int current_rhs() const { return cur_rhs_; }
  // solve K u_k = f_k for k < G (f_k = level_f(0) of RHS k); stats per RHS, identical to G solve_bound calls
  void solve_bound_group(int G, double* const* u, const SolverOptions& opts, const ZLink<double>* ul, SolveStats* st);


  // level_f(0) of the current RHS = macro force of load (src/fem.cpp:145-150). On even grids the
  // component sums of f come out of the same pass and the next project_norm0 of that f uses them.
  void macro_force(int load);
  double* level_u(int l) { return l == 0 && u0_bound_ ? u0_bound_ : levels_[size_t(l)].u.p; }
  ZLink<double> ulink(int l) const { return l == 0 && u0_bound_ ? u0l_ : levels_[size_t(l)].ul; }
  double* level_f(int l) {  // handed out for writing: level 0's macro-force sums no longer describe it
    if (l == 0) msum_f_[cur_rhs_] = nullptr;
    return levels_[size_t(l)].f.p;
  }
  double* level_r(int l) { return levels_[size_t(l)].r.p; }
  const T* stencil(int l) const { return levels_[size_t(l)].st.p; }
  const T* coeff() const { return coeff_.p; }
  double op_scale() const { return op_scale_; }
  double negligible_load(long long ndof) const;

  // Deterministic device reductions used by the solver (over all slabs).
  void remove_translations(double* f, int l);
  double project_norm0(double* f);  // remove_translations(f, 0) + norm(f) in one pass fewer
  void remove_translations_to(const double* src, double* dst, int l);
  double norm(const double* x, long long n);

  // z-slab plumbing
  const Slab& slab() const { return slab_; }
  bool sharded(int l) const { return levels_[size_t(l)].sharded; }
  long long global_nv(int l) const { return levels_[size_t(l)].nv_global; }
  void sync();                                     // fabric barrier (no-op on one domain)
  void sync_halo();                                // barrier with the z-neighbour slabs only
  void allreduce(double* dev, int n, bool is_max = false);  // over slabs, rank-order fold
  template <typename X>
  ZLink<X> link(X* p) {                            // collective: this buffer on the slabs below / above
    if (!slab_.on()) return {p, p};
    return neighbours<X>(slab_.fab->exchange(slab_.rank, p), slab_.rank);
  }
  const ZLink<T>& coeff_link() const { return coeff_l_; }

  bool lean() const { return lean_; }
  void ensure_inner();
  float* inner_e(int l) { return levels_[size_t(l)].eu.p; }  // f32 inner fields of the live RHS
  float* inner_f(int l) { return levels_[size_t(l)].ef.p; }
  float* inner_r(int l) { return levels_[size_t(l)].er.p; }

  // Runs one kernel family `reps` times on the current level data (benchmark / ncu target).
  void bench_op(const std::string& op, int reps);
  cudaStream_t stream() const { return s_; }
  Workspace& workspace() { return ws_; }
  const K0Matrix& k0() const { return k0_; }
  const Material& material() const { return mat_; }
  long long launches() const { return launches_; }

 private:
  struct Level {
    GridGeo g;                    // sharded: this slab's planes; replicated: the whole level
    bool sharded = false;
    long long nv_global = 0;
    DevBuf<double> u, f, r;
    DevBuf<T> st;                 // coarse stencil, blocked [nv/32][243][32] (st_index)
    DevBuf<float> eu, ef, er;     // f32 inner-cycle fields (kMixedDefect)
    ZLink<double> ul, rl;         // z-slab links (sharded levels)
    ZLink<float> eul, erl;
    ZLink<T> stl;
    PeerTable fpeer{}, efpeer{}, stpeer{};  // first replicated level: every slab's copy
  };
  // the first replicated level L (slab mode): its planes owned by this slab
  // are produced from the sharded level above, then gathered from the owners
  int first_replicated() const { return rep0_; }
  GridGeo transition_geo() const;  // this slab's share of level rep0_ (kernel iteration space)
  int transition_zoff_h() const;   // its first halved plane in the replicated level
  template <typename X>
  void gather_owned(int l, X* dst, PeerTable peers, int per_vertex);
  void restrict_to(int l, const double* r, double* f);   // level l -> l+1 (f64 fields)
  void restrict_to_f32(int l);
  void prolong_from(int l, const double* uc, double* u, ZLink<double> cl);
  void factor_coarsest();
  void check_error(const char* where);
  double v_cycle_defect(const SolverOptions& opts);
  void relax_f32(int l, int sweeps, bool reverse = false, bool zero_start = false);
  bool zero_start_ok(int l) const;  // the level's GS kernels support a zero-start first sweep
  void inner_vcycle(const SolverOptions& opts, bool symmetric);  // eu0 ~= K^-1 ef0 from zero
  SolveStats solve_pcg(double* u, const SolverOptions& opts);
  void residual_f32(int l);
  void coarsest_f32();
  double defect_residual(bool update = false, double* slot = nullptr);  // ef0 = float(f0 - K u0), returns
                                                // ||f0 - K u0||; update: u0 += e0 first, folded into the same
                                                // sweep; slot: leave this slab's ||r||^2 there, no read-back
  bool fused_update_ok() const;                 // the defect sweep can fold in the u += e update
  bool decide_lean(int request);                // constructor: the lean layout (collective on z-slabs)
  void restore_home();                          // end of a solve: the result back in the bound buffer

  Material mat_;
  double penal_;
  K0Matrix k0_;
  cudaStream_t s_;
  Slab slab_;
  int rep0_ = 1 << 30;      // first replicated level (slab mode)
  ZLink<T> coeff_l_{};
  ZLink<double> u0l_{};     // links of the bound level-0 u
  std::vector<Level> levels_;
  DevBuf<T> coeff_;
  DevBuf<double> Ainv_, A_, cwork_, Q_;
  int nnull_ = 0;  // deflated near-null modes of the coarsest operator (rows of Q_)
  // The coarsest factorisation runs on a host worker thread while the stream carries on (set_density
  // returns with the GPU busy); join_coarsest() makes the first coarsest solve of a density wait for it.
  std::future<int> fact_;          // -> nnull
  cudaStream_t s_fact_ = nullptr;  // uploads of the factorisation
  cudaEvent_t ev_fact_ = nullptr;  // recorded on s_fact_ after the uploads
  void* h_coarse_ = nullptr;       // pinned staging of the coarsest stencil / coefficients
  size_t h_coarse_bytes_ = 0;
  bool fact_joined_ = true;
  void join_coarsest();
  int ndof_c_ = 0;
  double op_scale_ = 0.0;
  bool density_set_ = false;
  bool inner_ready_ = false;
  struct RhsSlot {  // another RHS of a lockstep group (see select_rhs)
    std::vector<DevBuf<float>> eu, ef, er;
    std::vector<ZLink<float>> eul, erl;
    std::vector<PeerTable> efpeer;
    DevBuf<double> f0;
    DevBuf<double> ualt;
    ZLink<double> ualtl{};
    double* u0_bound = nullptr;
    double* u_home = nullptr;
    ZLink<double> u0l{}, u_home_l{};
    double fnorm0 = 0.0;
    bool ready = false;
  };
  std::vector<RhsSlot> slots_;
  int where_[6] = {-1, 0, 1, 2, 3, 4};  // slot holding RHS k's fields (-1: live in the levels)
  int cur_rhs_ = 0;
  int group_auto_ = 0;  // automatic group size, decided on first use
  void ensure_group(int G);
  void swap_live(RhsSlot& o);
  RhsSlot* slot_of(int k) { return k == cur_rhs_ ? nullptr : &slots_[size_t(where_[k])]; }
  void inner_down(int l, const SolverOptions& opts);  // pre-smooth, residual, restrict (current RHS)
  void inner_prolong(int l);                          // e_l += I e_{l+1} (current RHS)
  void inner_coarsest();
  void inner_vcycle_group(int G, const SolverOptions& opts, const bool* act);
  void relax_f32_group(int G, int l, int sweeps, bool zero_start);
  void residual_f32_group(int G, int l);
  double finish_defect_cycle(double* slot = nullptr);  // u += e (fused or not), the new residual; returns ||r||
                                                       // (slot: deferred, see defect_residual)
  void finish_defect_cycles(int G, const bool* act, double* rn);  // all active RHSs, one read-back
  bool transfer_group(int G, int l, bool down);                   // grouped level >= 1 transfer
  int bottom_start(int G) const;                                  // first level of the bottom cycle
  bool bottom_cycle(int G, int lb, const SolverOptions& opts);    // levels lb .. coarsest, one launch
  bool bottom_ok_ = true;                                         // cooperative launch accepted so far
  double* u0_bound_ = nullptr;
  double* u_home_ = nullptr;  // the caller's buffer of the current solve (u0_bound_ may be u_alt_)
  ZLink<double> u_home_l_{};
  DevBuf<double> u_alt_;      // second level-0 u buffer of the fused update (ping-pong)
  ZLink<double> u_alt_l_{};
  double fnorm0_ = 0.0;
  const double* msum_f_[kMaxRhsGroup] = {};  // f whose component sums macro_force left (per RHS)
  DevBuf<double> mf_part_;                    // macro-force block sums (3 per block)
  bool lean_ = false;
  DevBuf<double> red_;   // partials + scalars
  DevBuf<int> err_;
  DevBuf<unsigned> ticket_;  // last-block reduction counter (reduce.cuh finalize_in_last_block), kept zero
  DevBuf<double> npart_;  // per-block |r|^2 partials of the fused defect residual
  DevBuf<double> pcg_p_, pcg_q_, pcg_s_;  // PCG direction, K p, device scalars
  Workspace ws_;
  double* h_pinned_ = nullptr;  // small pinned read-back buffer
  long long launches_ = 0;
};

template <typename T>
class Homogenizer {
 public:
  Homogenizer(const int n[3], const Material& mat, double penal, const SolverOptions& opts, cudaStream_t s,
              Slab slab = {});
  ~Homogenizer();
  Homogenizer(const Homogenizer&) = delete;
  Homogenizer& operator=(const Homogenizer&) = delete;

  void set_density(const double* rho_phys_dev);
  CellSolveStats solve_cell_problems();
  void effective_tensor(double C[36]);
  void tensor_sensitivity(const double seed[36], double* out_dev);

  // load case i's displacement field (3 nv doubles) from / into a device buffer
  void read_displacement(int i, double* dst_dev);
  void write_displacement(int i, const double* src_dev);
  // Memory lever (the paper keeps the six fields in host-backed unified memory and evaluates
  // from f32 copies): 0 = six device-resident f64 fields; 2 = host-staged: the
  // f64 fields live in pinned host memory, each solve stages its warm start in and the result out, and
  // C^H / sensitivities read f32 snapshots placed in the level-0 buffers the solver has released;
  // 1 = as 2 with only the f32 snapshots on the host (warm starts from them). Knob U_HOST: -1 never,
  // 0 (default) when the device-resident layout does not fit, 1 / 2 forced.
  int host_staged() const { return host_u_; }
  // Multi-GPU: load case i is solved by rank owner[i], then broadcast to all ranks.
  void set_comm(Comm* c, const int owner[6]) {
    comm_ = c;
    for (int i = 0; i < 6; ++i) owner_[i] = owner ? owner[i] : (c ? i % c->size() : 0);
  }
  Hierarchy<T>& hierarchy() { return hier_; }
  SolverOptions& options() { return opts_; }
  const double* density() const { return rho_.p; }
  long long nv() const { return hier_.geo(0).nv; }

 private:
  Hierarchy<T> hier_;
  SolverOptions opts_;
  double penal_;
  DevBuf<double> rho_;
  std::array<DevBuf<double>, 6> u_;
  std::array<ZLink<double>, 6> ul_{};  // z-slab links of the six fields
  DevBuf<double> seed_;
  DevBuf<double> stats_;  // per-load (cycles, rel, converged) for the multi-GPU combine
  bool density_set_ = false;
  // per-element energies of the last effective_tensor() (knob ENERGY_CACHE, default on): [21][nv]
  DevBuf<unsigned char> ecache_;
  bool ecache_valid_ = false;
  bool ecache_skip_ = false;  // not enough HBM for the energy cache (decided once)
  // host-staged displacements (host_u_ > 0)
  int host_u_ = 0;
  std::array<double*, 6> hu64_{};  // pinned f64 fields (mode 2)
  std::array<float*, 6> hu32_{};   // pinned f32 snapshots
  std::array<float*, 6> snap_{};   // device snapshot slots: halves of level-0 u, inner e0 / f0, halves of f0
  std::array<ZLink<float>, 6> snapl_{};
  bool snaps_ready_ = false;
  cudaStream_t cs_ = nullptr;   // copy stream: a solve's write-back overlaps the next solve's stage-in
  cudaEvent_t ev_solved_ = nullptr, ev_staged_out_ = nullptr;
  // mode 2: the f32 snapshot of field i is made on the host from its f64 write-back (ev_back_[i]) by a
  // worker, so only the f64 field crosses PCIe device -> host
  std::array<cudaEvent_t, 6> ev_back_{};
  std::array<std::future<void>, 6> conv_;
  void join_conversions();
  CellSolveStats solve_host_staged();
  void ensure_snapshots();
  Comm* comm_ = nullptr;
  int owner_[6] = {0, 0, 0, 0, 0, 0};
};

}  // namespace ihomgpu
