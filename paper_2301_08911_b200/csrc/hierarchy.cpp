// hierarchy.cpp -- host orchestration of the device multigrid hierarchy and
// the homogenizer (src/multigrid.cpp:245-501, src/homogenization.cpp:16-144).
#include "hierarchy.hpp"

#include "profiler.hpp"

#include <cmath>
#include <cstring>
#include <mutex>
#include <thread>
#include <type_traits>

namespace ihomgpu {

namespace {

constexpr int kRedDoubles = 21 * kReducePartials + 128;
constexpr int kMacroSums = 72;  // ws_.scalars[72 .. 72 + 3 kMaxRhsGroup): component sums left by macro_force

// Dense assembly of a level operator in the reference dof order 3*loc + c
// (src/multigrid.cpp:335-366).
std::vector<double> assemble_dense_l0(const GridGeo& g, const std::vector<double>& coeff, const K0Matrix& k0) {
  const long long nv = g.nv, N = 3 * nv;
  std::vector<double> a(size_t(N * N), 0.0);
  for (long long ei = 0; ei < nv; ++ei) {
    const int ex = int(ei % g.n[0]);
    const long long r = ei / g.n[0];
    const int ey = int(r % g.n[1]), ez = int(r / g.n[1]);
    long long locs[8];
    for (int j = 0; j < 8; ++j)
      locs[j] = vloc(g, (ex + (j & 1)) % g.n[0], (ey + ((j >> 1) & 1)) % g.n[1], (ez + ((j >> 2) & 1)) % g.n[2]);
    const double q = coeff[size_t(ei)];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j)
        for (int rr = 0; rr < 3; ++rr)
          for (int c = 0; c < 3; ++c)
            a[size_t((3 * locs[i] + rr) * N + 3 * locs[j] + c)] += q * k0.k[3 * i + rr][3 * j + c];
  }
  return a;
}

template <typename T>
std::vector<double> assemble_dense_stencil(const GridGeo& g, const std::vector<T>& st) {
  const long long nv = g.nv, N = 3 * nv;
  std::vector<double> a(size_t(N * N), 0.0);
  for (long long loc = 0; loc < nv; ++loc) {
    const int color = color_at(g, loc);
    int x, y, z;
    block_coords(g, color, (unsigned)(loc - g.base[color]), x, y, z);
    for (int n = 0; n < 27; ++n) {
      const int tx = n % 3 - 1, ty = (n / 3) % 3 - 1, tz = n / 9 - 1;
      const long long wl = vloc(g, (x + tx + g.n[0]) % g.n[0], (y + ty + g.n[1]) % g.n[1], (z + tz + g.n[2]) % g.n[2]);
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          a[size_t((3 * loc + r) * N + 3 * wl + c)] += double(st[st_index(9 * n + 3 * r + c, (unsigned)loc)]);
    }
  }
  return a;
}

// Translation projection of the coarsest operator: a <- P a P, P = I - (1/nv) sum_c t_c t_c^T
// (t_c = unit translation of component c), then symmetrised. The f32 Galerkin stencils leave
// A*t_c at ~1e-7 op_scale; on designs with floating islands (near-null modes ~1e-8 op_scale)
// that leak makes the reference's refinement stall above its 1e-3 gate
// (src/multigrid.cpp:441-447). Projection makes the deflated system exactly consistent.
// Knob COARSE_PROJECT=0 restores the reference (unprojected) operator.
void project_translations(std::vector<double>& a, long long nv) {
  const long long N = 3 * nv;
  const double inv_nv = 1.0 / double(nv);
  for (long long i = 0; i < N; ++i) {  // a P: subtract per-component row means
    double* row = a.data() + size_t(i * N);
    double m[3] = {0.0, 0.0, 0.0};
    for (long long j = 0; j < nv; ++j)
      for (int c = 0; c < 3; ++c) m[c] += row[3 * j + c];
    for (int c = 0; c < 3; ++c) m[c] *= inv_nv;
    for (long long j = 0; j < nv; ++j)
      for (int c = 0; c < 3; ++c) row[3 * j + c] -= m[c];
  }
  std::vector<double> m(size_t(3 * N), 0.0);  // P (aP): per-component column means
  for (long long i = 0; i < nv; ++i)
    for (int r = 0; r < 3; ++r) {
      const double* row = a.data() + size_t((3 * i + r) * N);
      double* mr = m.data() + size_t(r * N);
      for (long long k = 0; k < N; ++k) mr[k] += row[k];
    }
  for (auto& v : m) v *= inv_nv;
  for (long long i = 0; i < nv; ++i)
    for (int r = 0; r < 3; ++r) {
      double* row = a.data() + size_t((3 * i + r) * N);
      const double* mr = m.data() + size_t(r * N);
      for (long long k = 0; k < N; ++k) row[k] -= mr[k];
    }
  for (long long i = 0; i < N; ++i)
    for (long long j = i + 1; j < N; ++j) {
      const double s = 0.5 * (a[size_t(i * N + j)] + a[size_t(j * N + i)]);
      a[size_t(i * N + j)] = s;
      a[size_t(j * N + i)] = s;
    }
}

// Symmetric LDL^T with diagonal pivoting (the algorithm of Eigen::LDLT, which the reference
// uses at src/multigrid.cpp:380: at step k the largest remaining |diagonal| is swapped in). Unlike a
// Cholesky it tolerates the slightly indefinite near-null modes f32 stencils produce; it fails only on
// an exactly zero or non-finite pivot (Eigen's NumericalIssue).
struct Ldlt {
  int n = 0;
  std::vector<double> a;  // unit L below the diagonal, D on it (permuted order)
  std::vector<int> perm;  // position -> original index
  void factor(std::vector<double> m, int N) {
    n = N;
    a = std::move(m);
    perm.resize(size_t(n));
    for (int i = 0; i < n; ++i) perm[size_t(i)] = i;
    auto A = [&](int i, int j) -> double& { return a[size_t(i) * n + j]; };
    std::vector<double> t(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
      int p = k;
      double best = std::fabs(A(k, k));
      for (int i = k + 1; i < n; ++i)
        if (std::fabs(A(i, i)) > best) best = std::fabs(A(i, i)), p = i;
      if (p != k) {  // symmetric swap of rows and columns k <-> p
        for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
        for (int i = 0; i < n; ++i) std::swap(A(i, k), A(i, p));
        std::swap(perm[size_t(k)], perm[size_t(p)]);
      }
      for (int j = 0; j < k; ++j) t[size_t(j)] = A(k, j) * A(j, j);  // left-looking column k
      double d = A(k, k);
      for (int j = 0; j < k; ++j) d -= A(k, j) * t[size_t(j)];
      if (!(std::fabs(d) > 0.0) || !std::isfinite(d)) throw NumericError("coarsest-level factorization failed");
      A(k, k) = d;
      for (int i = k + 1; i < n; ++i) {
        double s = A(i, k);
        for (int j = 0; j < k; ++j) s -= A(i, j) * t[size_t(j)];
        A(i, k) = s / d;
      }
    }
  }
  double pivot(int k) const { return a[size_t(k) * n + k]; }
  // Pm^T L^-T e_k: the near-null direction of a tiny trailing pivot k (diagonal pivoting is rank-revealing)
  std::vector<double> null_direction(int k) const {
    std::vector<double> y(static_cast<size_t>(n), 0.0), v(static_cast<size_t>(n));
    y[size_t(k)] = 1.0;
    for (int i = k - 1; i >= 0; --i) {
      double s = 0.0;
      for (int j = i + 1; j <= k; ++j) s -= a[size_t(j) * n + i] * y[size_t(j)];
      y[size_t(i)] = s;
    }
    for (int i = 0; i < n; ++i) v[size_t(perm[size_t(i)])] = y[size_t(i)];
    return v;
  }
  // explicit inverse A^-1 = Pm^T L^-T D^-1 L^-1 Pm (for the device matvecs)
  std::vector<double> inverse() const {
    std::vector<double> W(size_t(n) * n, 0.0);  // W = L^-1 (unit lower), column by column
    for (int j = 0; j < n; ++j) {
      W[size_t(j) * n + j] = 1.0;
      for (int i = j + 1; i < n; ++i) {
        double s = 0.0;
        for (int k = j; k < i; ++k) s -= a[size_t(i) * n + k] * W[size_t(k) * n + j];
        W[size_t(i) * n + j] = s;
      }
    }
    std::vector<double> inv(size_t(n) * n, 0.0);  // W^T D^-1 W, scattered through the permutation
    for (int i = 0; i < n; ++i)
      for (int j = i; j < n; ++j) {
        double s = 0.0;
        for (int k = j; k < n; ++k) s += W[size_t(k) * n + i] * W[size_t(k) * n + j] / pivot(k);
        inv[size_t(perm[size_t(i)]) * n + perm[size_t(j)]] = s;
        inv[size_t(perm[size_t(j)]) * n + perm[size_t(i)]] = s;
      }
    return inv;
  }
};

// a <- (I - Q Q^T) a (I - Q Q^T) for orthonormal columns q (each length N), symmetrised.
void project_out(std::vector<double>& a, const std::vector<std::vector<double>>& Q, long long N) {
  for (const auto& q : Q) {
    std::vector<double> aq(size_t(N), 0.0);  // a q
    for (long long i = 0; i < N; ++i) {
      double s = 0.0;
      for (long long j = 0; j < N; ++j) s += a[size_t(i * N + j)] * q[size_t(j)];
      aq[size_t(i)] = s;
    }
    double qaq = 0.0;
    for (long long i = 0; i < N; ++i) qaq += q[size_t(i)] * aq[size_t(i)];
    // (I - qq^T) a (I - qq^T) = a - aq q^T - q (aq)^T + (q^T a q) q q^T
    for (long long i = 0; i < N; ++i)
      for (long long j = 0; j < N; ++j)
        a[size_t(i * N + j)] += -aq[size_t(i)] * q[size_t(j)] - q[size_t(i)] * aq[size_t(j)] +
                                qaq * q[size_t(i)] * q[size_t(j)];
  }
  for (long long i = 0; i < N; ++i)
    for (long long j = i + 1; j < N; ++j) {
      const double v = 0.5 * (a[size_t(i * N + j)] + a[size_t(j * N + i)]);
      a[size_t(i * N + j)] = a[size_t(j * N + i)] = v;
    }
}

// Algorithmic bytes, sN = nodal bytes, sC = coefficient/stencil bytes.
double gs_l0_bytes(const GridGeo& g, int c, double sN, double sC) {
  // other colours' u (7/8 of 3 comps) + all element coefficients + f_c read + u_c write
  return double(g.nv) * (7.0 / 8.0 * 3.0 * sN + sC) + double(g.size[c]) * 6.0 * sN;
}
double gs_coarse_bytes(const GridGeo& g, int c, double sN, double sC) {
  return double(g.size[c]) * (243.0 * sC + 6.0 * sN) + double(g.nv - g.size[c]) * 3.0 * sN;
}
// zero-start pass (first sweep from u = 0): only colours < c hold data -- c of the 7 other colour
// blocks are read, and a coarse vertex reads the stencil blocks of its non-zero neighbours only
double gs_l0_bytes_zs(const GridGeo& g, int c, double sN, double sC) {
  return double(g.nv) * (double(c) / 8.0 * 3.0 * sN + sC) + double(g.size[c]) * 6.0 * sN;
}
// colour pair (c, c + 1), f32: the other colours' u once (colour c + 1 old for pass c; zero start: the
// colours < c, and c + 1 is a known zero), every coefficient once, f and the update of both colours
double gs_l0_pair_bytes(const GridGeo& g, int c, bool zs) {
  const double others = zs ? double(c) / 8.0 : 7.0 / 8.0;
  return double(g.nv) * (others * 12.0 + 4.0) + double(g.size[c] + g.size[c + 1]) * 24.0;
}
double gs_coarse_bytes_zs(const GridGeo& g, int c, double sN, double sC) {
  const int live = 27 - __builtin_popcount(zero_start_mask(c));
  double others = 0.0;
  for (int k = 0; k < c; ++k) others += double(g.size[k]);
  return double(g.size[c]) * (9.0 * live * sC + 6.0 * sN) + others * 3.0 * sN;
}
double resid_l0_bytes(const GridGeo& g, double sN, double sC, bool with_f) {
  return double(g.nv) * ((with_f ? 9.0 : 6.0) * sN + sC);
}
double resid_coarse_bytes(const GridGeo& g, double sN, double sC, bool with_f) {
  return double(g.nv) * (243.0 * sC + (with_f ? 9.0 : 6.0) * sN);
}

// Free HBM as seen by the memory levers; knob HBM_LIMIT_MB > 0 caps it (tests exercise the low-memory
// paths on a large GPU with it).
size_t hbm_free_limit(size_t free_b) {
  const int mb = knob("HBM_LIMIT_MB", 0);
  return mb > 0 ? std::min(free_b, size_t(mb) << 20) : free_b;
}

bool can_coarsen(const GridGeo& g) {  // inc/grid.hpp:47-51
  for (int k = 0; k < 3; ++k)
    if (g.n[k] % 2 != 0 || g.n[k] / 2 < 4) return false;
  return true;
}

}  // namespace

// ============================================================== Hierarchy
template <typename T>
Hierarchy<T>::Hierarchy(const int n[3], const Material& mat, double penal, cudaStream_t s, Slab slab, int lean)
    : mat_(mat), penal_(penal), s_(s), slab_(slab) {
  for (int k = 0; k < 3; ++k)
    if (n[k] < 4) throw std::invalid_argument("grid resolution must be >= 4 per axis");
  if ((long long)n[0] * n[1] * n[2] >= (1LL << 31)) throw std::invalid_argument("grid too large for 32-bit vertex indexing");
  int t = n[2];
  if (slab_.on()) {  // z-slab constraints
    if (slab_.rank < 0 || slab_.rank >= slab_.nranks || slab_.nranks != slab_.fab->size())
      throw std::invalid_argument("bad z-slab rank / count");
    if (n[2] % slab_.nranks != 0) throw std::invalid_argument("z planes must divide evenly among the slabs");
    t = n[2] / slab_.nranks;
    if (t % 4 != 0) throw std::invalid_argument("each z-slab needs a multiple of 4 planes");
    if (n[0] % 2 != 0 || n[1] % 2 != 0 || n[0] < 8) throw std::invalid_argument("z-slabs need even x/y dims, x >= 8");
  }
  k0_ = element_stiffness(mat);
  bind_tables();
  GridGeo g = make_geo(n[0], n[1], n[2]);
  std::vector<GridGeo> global{g};
  while (can_coarsen(g)) {
    g = make_geo(g.n[0] / 2, g.n[1] / 2, g.n[2] / 2);
    global.push_back(g);
  }
  if (global.back().nv > 343) throw std::invalid_argument("coarsest level larger than 7^3 is not supported");
  bool sharding = slab_.on();
  for (size_t l = 0; l < global.size(); ++l) {
    levels_.emplace_back();
    Level& L = levels_.back();
    const GridGeo& G = global[l];
    L.nv_global = G.nv;
    // level l is split into slabs while every slab keeps >= 4 planes (a multiple of 4,
    // so the restriction into the next level stays on even colour blocks) and the
    // even-grid kernels apply; below, every slab holds the whole (small) level.
    sharding = sharding && (t % (4 << l) == 0) && G.n[0] % 2 == 0 && G.n[1] % 2 == 0 && G.n[0] >= 8;
    L.sharded = sharding;
    L.g = sharding ? make_geo(G.n[0], G.n[1], t >> l) : G;
    if (slab_.on() && !sharding && rep0_ > int(l)) rep0_ = int(l);
  }
  if (slab_.on() && !levels_[0].sharded) throw std::invalid_argument("level 0 cannot be split into these slabs");
  red_.alloc(kRedDoubles);
  err_.alloc(1);
  IHOM_CUDA(cudaMemsetAsync(err_.p, 0, sizeof(int), s_));
  ticket_.alloc(1);
  IHOM_CUDA(cudaMemsetAsync(ticket_.p, 0, sizeof(unsigned), s_));
  ws_.partials = red_.p;
  ws_.scalar = red_.p + 21 * kReducePartials;
  ws_.scalar2 = ws_.scalar + 1;
  ws_.scalars = ws_.scalar + 8;
  ws_.flag = err_.p;
  IHOM_CUDA(cudaMallocHost(&h_pinned_, 64 * sizeof(double)));
  lean_ = decide_lean(lean);
  for (size_t l = 0; l < levels_.size(); ++l) {
    Level& L = levels_[l];
    const size_t n3 = size_t(3 * L.g.nv);
    // lean: the f64 fields the mixed_defect solver never touches are not allocated (level 0 keeps u and f;
    // the replicated transition level keeps f, whose peer table is exchanged below)
    const bool keep_u = !lean_ || l == 0, keep_f = keep_u || (slab_.on() && int(l) == rep0_), keep_r = !lean_;
    if (keep_u) L.u.alloc(n3);
    if (keep_f) L.f.alloc(n3);
    if (keep_r) L.r.alloc(n3);
    if (keep_u) IHOM_CUDA(cudaMemsetAsync(L.u.p, 0, sizeof(double) * n3, s_));
    if (keep_f) IHOM_CUDA(cudaMemsetAsync(L.f.p, 0, sizeof(double) * n3, s_));
    if (keep_r) IHOM_CUDA(cudaMemsetAsync(L.r.p, 0, sizeof(double) * n3, s_));
    if (l > 0) L.st.alloc(stencil_alloc(L.g.nv));
  }
  coeff_.alloc(size_t(levels_[0].g.nv));
  ndof_c_ = int(3 * levels_.back().g.nv);
  cwork_.alloc(size_t(3 * ndof_c_));
  IHOM_CUDA(cudaStreamSynchronize(s_));
  if (slab_.on()) {  // collective, same order on every slab
    coeff_l_ = link(coeff_.p);
    for (size_t l = 0; l < levels_.size(); ++l) {
      Level& L = levels_[l];
      if (L.sharded) {
        if (L.u.p) L.ul = link(L.u.p);
        if (L.r.p) L.rl = link(L.r.p);
        if (l > 0) L.stl = link(L.st.p);
      } else if (int(l) == rep0_) {
        L.fpeer = peer_table(slab_.fab->exchange(slab_.rank, L.f.p));
        L.stpeer = peer_table(slab_.fab->exchange(slab_.rank, L.st.p));
      }
    }
  }
}

// Bytes per level-0 vertex of the device-resident layout at group size 1 without the energy cache
// (distributed.py memory_plan): six f64 displacements, level-0 f64 u/f/r and ping-pong u, f32 inner
// fields, coefficients, level >= 1 stencils, the density-side fields.
constexpr double kResidentBytesPerVertex = 144 + 96 + 41 + 4 + 139 + 64;

template <typename T>
bool Hierarchy<T>::decide_lean(int request) {
  if (request <= 0 || !std::is_same_v<T, float> || !fast_ok(levels_[0].g) || levels_.size() < 2) return false;
  double want = request >= 2 ? 1.0 : 0.0;
  if (request == 1) {
    int dev = 0;
    IHOM_CUDA(cudaGetDevice(&dev));
    double share = 1.0;
    if (slab_.on()) {  // slabs sharing this device split its free memory (one-hot by device ordinal)
      double h[16] = {};
      h[dev & 15] = 1.0;
      IHOM_CUDA(cudaMemcpyAsync(ws_.scalars + 32, h, sizeof(h), cudaMemcpyHostToDevice, s_));
      allreduce(ws_.scalars + 32, 16, false);
      IHOM_CUDA(cudaMemcpyAsync(h, ws_.scalars + 32, sizeof(h), cudaMemcpyDeviceToHost, s_));
      IHOM_CUDA(cudaStreamSynchronize(s_));
      share = std::max(1.0, h[dev & 15]);
    }
    size_t free_b = 0, total_b = 0;
    IHOM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    free_b = hbm_free_limit(free_b);
    const double need = kResidentBytesPerVertex * double(levels_[0].g.nv) + 4e9 / share;
    want = need > double(free_b) / share ? 1.0 : 0.0;
  }
  if (slab_.on()) {  // every slab takes the same layout
    IHOM_CUDA(cudaMemcpyAsync(ws_.scalars + 32, &want, sizeof(double), cudaMemcpyHostToDevice, s_));
    allreduce(ws_.scalars + 32, 1, true);
    IHOM_CUDA(cudaMemcpyAsync(&want, ws_.scalars + 32, sizeof(double), cudaMemcpyDeviceToHost, s_));
    IHOM_CUDA(cudaStreamSynchronize(s_));
  }
  return want > 0.5;
}

template <typename T>
GridGeo Hierarchy<T>::transition_geo() const {
  const GridGeo& f = levels_[size_t(rep0_ - 1)].g;
  return make_geo(f.n[0] / 2, f.n[1] / 2, f.n[2] / 2);
}

template <typename T>
int Hierarchy<T>::transition_zoff_h() const {
  return slab_.rank * (levels_[size_t(rep0_ - 1)].g.n[2] / 4);
}

template <typename T>
void Hierarchy<T>::sync() {
  if (slab_.on()) slab_.fab->barrier(slab_.rank, s_);
}

template <typename T>
void Hierarchy<T>::sync_halo() {  // a sharded level's kernel reads / overwrites only the z-neighbour slabs' planes
  if (slab_.on()) slab_.fab->barrier(slab_.rank, s_, true);
}

template <typename T>
void Hierarchy<T>::allreduce(double* dev, int n, bool is_max) {
  if (slab_.on()) slab_.fab->allreduce(slab_.rank, dev, n, is_max, s_);
}

template <typename T>
template <typename X>
void Hierarchy<T>::gather_owned(int l, X* dst, PeerTable peers, int per_vertex) {
  sync();  // every owner's planes written
  {
    ProfScope p(s_, "slab_gather", double(levels_[size_t(l)].g.nv) * per_vertex * sizeof(X));
    launch_gather_owned<X>(levels_[size_t(l)].g, peers, levels_[size_t(l - 1)].g.n[2] / 2, slab_.rank, per_vertex,
                           dst, s_);
  }
  ++launches_;
  sync();  // nobody rewrites its planes while others still read them
}

template <typename T>
void Hierarchy<T>::restrict_to(int l, const double* r, double* f) {
  Level& F = levels_[size_t(l)];
  Level& C = levels_[size_t(l + 1)];
  const ZLink<double> rl = F.rl;
  if (F.sharded) sync_halo();
  {
    ProfScope p(s_, "restrict", double(F.g.nv) * 27.0);
    if (!(F.sharded && !C.sharded)) {
      launch_restrict<double>(F.g, C.g, r, f, s_, F.sharded ? rl : ZLink<double>{});
    } else {
      const GridGeo gc = transition_geo();
      launch_restrict<double>(F.g, gc, r, f, s_, rl, &C.g, transition_zoff_h());
    }
  }
  ++launches_;
  if (slab_.on() && !C.sharded && F.sharded) gather_owned<double>(l + 1, f, C.fpeer, 3);
}

template <typename T>
void Hierarchy<T>::restrict_to_f32(int l) {
  Level& F = levels_[size_t(l)];
  Level& C = levels_[size_t(l + 1)];
  if (F.sharded) sync_halo();
  {
    ProfScope p(s_, "restrict", double(F.g.nv) * 13.5);
    if (!(F.sharded && !C.sharded)) {
      launch_restrict<float>(F.g, C.g, F.er.p, C.ef.p, s_, F.sharded ? F.erl : ZLink<float>{});
    } else {
      const GridGeo gc = transition_geo();
      launch_restrict<float>(F.g, gc, F.er.p, C.ef.p, s_, F.erl, &C.g, transition_zoff_h());
    }
  }
  ++launches_;
  if (slab_.on() && !C.sharded && F.sharded) gather_owned<float>(l + 1, C.ef.p, C.efpeer, 3);
}

template <typename T>
void Hierarchy<T>::prolong_from(int l, const double* uc, double* u, ZLink<double> cl) {
  Level& F = levels_[size_t(l)];
  Level& C = levels_[size_t(l + 1)];
  if (F.sharded) sync_halo();
  {
    ProfScope p(s_, "prolong", double(F.g.nv) * 51.0);
    if (!(F.sharded && !C.sharded)) launch_prolong_add<double>(C.g, F.g, uc, u, s_, C.sharded ? cl : ZLink<double>{});
    else launch_prolong_add<double>(C.g, F.g, uc, u, s_, {}, slab_.rank * (F.g.n[2] / 2));
  }
  ++launches_;
}

template <typename T>
void Hierarchy<T>::bind_tables() {
  static std::mutex mu;  // z-slab threads of one process share the constant tables
  std::lock_guard<std::mutex> lock(mu);
  const StiffnessTables tab(k0_);
  upload_fem_tables(tab, k0_, s_);
  upload_galerkin_tables(ElementGalerkin(k0_), s_);
}

template <typename T>
void Hierarchy<T>::set_density(const double* rho) {  // src/multigrid.cpp:263-279
  const GridGeo& g0 = levels_[0].g;
  {
    ProfScope p(s_, "coeff", double(g0.nv) * (8.0 + sizeof(T)));
    launch_coeff<T>(rho, coeff_.p, g0.nv, penal_, s_);
  }
  launches_ += 1;
  for (size_t l = 1; l < levels_.size(); ++l) {
    Level& F = levels_[l - 1];
    Level& C = levels_[l];
    const bool transition = slab_.on() && F.sharded && !C.sharded;
    const GridGeo gc = transition ? transition_geo() : C.g;
    const GridGeo* gout = transition ? &C.g : nullptr;
    const int zoff = transition ? transition_zoff_h() : 0;
    if (F.sharded) sync_halo();
    if (l == 1) {
      ProfScope p(s_, "galerkin_l1", double(g0.nv) * sizeof(T) + double(gc.nv) * 243.0 * sizeof(T));
      launch_galerkin_from_elements<T>(g0, gc, coeff_.p, C.st.p, s_, F.sharded ? coeff_l_ : ZLink<T>{}, gout, zoff);
    } else {
      ProfScope p(s_, "galerkin_coarse", double(F.g.nv + gc.nv) * 243.0 * sizeof(T));
      launch_galerkin_from_stencil<T>(F.g, gc, F.st.p, C.st.p, s_, F.sharded ? F.stl : ZLink<T>{}, gout, zoff);
    }
    ++launches_;
    if (transition) gather_owned<T>(int(l), C.st.p, C.stpeer, 243);
  }
  factor_coarsest();
  density_set_ = true;
}

double factor_coarse_dense(std::vector<double>& a, long long nv, std::vector<double>& inv, std::vector<double>* qout,
                           int* mout) {
  const long long N = 3 * nv;
  double dsum = 0.0;
  for (long long i = 0; i < N; ++i) dsum += a[size_t(i * N + i)];
  const double op_scale = dsum / double(N);  // mean diagonal (src/multigrid.cpp:373)
  const double shift = op_scale / double(nv);  // deflation shift (src/multigrid.cpp:374-379)
  auto shifted = [&](const std::vector<std::vector<double>>& Q) {
    std::vector<double> b = a;
    for (long long i = 0; i < nv; ++i)
      for (long long j = 0; j < nv; ++j)
        for (int c = 0; c < 3; ++c) b[size_t((3 * i + c) * N + 3 * j + c)] += shift;
    for (const auto& q : Q)
      for (long long i = 0; i < N; ++i)
        for (long long j = 0; j < N; ++j) b[size_t(i * N + j)] += op_scale * q[size_t(i)] * q[size_t(j)];
    return b;
  };
  std::vector<std::vector<double>> Q;
  Ldlt f;
  if (knob("COARSE_PROJECT", 1) != 0) {
    project_translations(a, nv);
    // Near-null modes beyond the translations (floating islands of the design: modes ~1e-8 op_scale,
    // below the f32 stencils' resolution) are deflated like the translations: trailing pivots of the
    // pivoted LDL^T below kNearNull op_scale give their directions, orthonormalised against the
    // translations; the operator is projected off them and shifted on them, the load projected.
    constexpr double kNearNull = 1e-6;
    f.factor(shifted(Q), int(N));
    for (int k = 0; k < int(N); ++k)
      if (std::fabs(f.pivot(k)) < kNearNull * op_scale) {
        std::vector<double> v = f.null_direction(k);
        for (int pass = 0; pass < 2; ++pass) {  // twice-iterated Gram-Schmidt
          for (int c = 0; c < 3; ++c) {
            double m = 0.0;
            for (long long i = 0; i < nv; ++i) m += v[size_t(3 * i + c)];
            m /= double(nv);
            for (long long i = 0; i < nv; ++i) v[size_t(3 * i + c)] -= m;
          }
          for (const auto& q : Q) {
            double d = 0.0;
            for (long long i = 0; i < N; ++i) d += q[size_t(i)] * v[size_t(i)];
            for (long long i = 0; i < N; ++i) v[size_t(i)] -= d * q[size_t(i)];
          }
        }
        double nrm = 0.0;
        for (double x : v) nrm += x * x;
        nrm = std::sqrt(nrm);
        if (!(nrm > 0.0)) continue;
        for (double& x : v) x /= nrm;
        Q.push_back(std::move(v));
      }
    if (!Q.empty()) {
      project_out(a, Q, N);
      f.factor(shifted(Q), int(N));
    }
  } else {
    f.factor(shifted(Q), int(N));
  }
  inv = f.inverse();
  if (qout) {
    qout->clear();
    for (const auto& q : Q) qout->insert(qout->end(), q.begin(), q.end());
  }
  if (mout) *mout = int(Q.size());
  return op_scale;
}

template <typename T>
void Hierarchy<T>::factor_coarsest() {  // src/multigrid.cpp:368-383
  join_coarsest();  // a previous density's factorisation is done with the staging buffers
  const int lc = num_levels() - 1;
  const GridGeo g = levels_[size_t(lc)].g;
  const long long N = 3 * g.nv;
  const size_t bytes = lc == 0 ? sizeof(T) * size_t(g.nv) : sizeof(T) * stencil_alloc(g.nv);
  if (h_coarse_bytes_ < bytes) {
    if (h_coarse_) IHOM_CUDA(cudaFreeHost(h_coarse_));
    IHOM_CUDA(cudaMallocHost(&h_coarse_, bytes));
    h_coarse_bytes_ = bytes;
  }
  if (!s_fact_) {
    IHOM_CUDA(cudaStreamCreateWithFlags(&s_fact_, cudaStreamNonBlocking));
    IHOM_CUDA(cudaEventCreateWithFlags(&ev_fact_, cudaEventDisableTiming));
  }
  if (A_.n != size_t(N * N)) {  // fixed-size device buffers: no per-density (device-synchronising) reallocation
    A_.alloc(size_t(N * N));
    Ainv_.alloc(size_t(N * N));
    Q_.alloc(size_t(N * N));
  }
  IHOM_CUDA(cudaMemcpyAsync(h_coarse_, lc == 0 ? static_cast<const void*>(coeff_.p) : levels_[size_t(lc)].st.p, bytes,
                            cudaMemcpyDeviceToHost, s_));
  IHOM_CUDA(cudaStreamSynchronize(s_));
  // op_scale (mean diagonal, src/multigrid.cpp:373) now: the solves' negligible-load tests need it first
  std::vector<double> a;
  if (lc == 0) {
    const T* c = static_cast<const T*>(h_coarse_);
    a = assemble_dense_l0(g, std::vector<double>(c, c + g.nv), k0_);
  } else {
    const T* st = static_cast<const T*>(h_coarse_);
    a = assemble_dense_stencil<T>(g, std::vector<T>(st, st + stencil_alloc(g.nv)));
  }
  double dsum = 0.0;
  for (long long i = 0; i < N; ++i) dsum += a[size_t(i * N + i)];
  op_scale_ = dsum / double(N);
  int dev = 0;
  IHOM_CUDA(cudaGetDevice(&dev));
  fact_joined_ = false;
  fact_ = std::async(std::launch::async, [this, dev, nv = g.nv, a = std::move(a)]() mutable {
    IHOM_CUDA(cudaSetDevice(dev));
    std::vector<double> inv, q;
    int m = 0;
    factor_coarse_dense(a, nv, inv, &q, &m);
    IHOM_CUDA(cudaMemcpyAsync(A_.p, a.data(), sizeof(double) * a.size(), cudaMemcpyHostToDevice, s_fact_));
    IHOM_CUDA(cudaMemcpyAsync(Ainv_.p, inv.data(), sizeof(double) * inv.size(), cudaMemcpyHostToDevice, s_fact_));
    if (m > 0) IHOM_CUDA(cudaMemcpyAsync(Q_.p, q.data(), sizeof(double) * q.size(), cudaMemcpyHostToDevice, s_fact_));
    IHOM_CUDA(cudaEventRecord(ev_fact_, s_fact_));
    IHOM_CUDA(cudaStreamSynchronize(s_fact_));  // the host vectors die with this task
    return m;
  });
}

template <typename T>
void Hierarchy<T>::join_coarsest() {
  if (fact_joined_) return;
  fact_joined_ = true;
  nnull_ = fact_.get();  // rethrows a failed factorisation (NumericError) here
  IHOM_CUDA(cudaStreamWaitEvent(s_, ev_fact_, 0));
}

template <typename T>
double Hierarchy<T>::negligible_load(long long ndof) const {  // src/multigrid.cpp:388-390
  return 1e-12 * op_scale_ * std::sqrt(double(ndof));
}

template <typename T>
void Hierarchy<T>::check_error(const char* where) {
  int e = 0;
  if (slab_.on()) slab_.fab->check(slab_.rank);  // a timed-out barrier (dead or diverged peer) surfaces here
  if (slab_.on()) {  // collective: every slab throws together (or none does)
    launch_int_to_double(err_.p, ws_.scalars + 60, s_);
    allreduce(ws_.scalars + 60, 1, true);
    IHOM_CUDA(cudaMemcpyAsync(h_pinned_, ws_.scalars + 60, sizeof(double), cudaMemcpyDeviceToHost, s_));
    IHOM_CUDA(cudaStreamSynchronize(s_));
    e = int(h_pinned_[0]);
  } else {
    IHOM_CUDA(cudaMemcpyAsync(&e, err_.p, sizeof(int), cudaMemcpyDeviceToHost, s_));
    IHOM_CUDA(cudaStreamSynchronize(s_));
  }
  if (e) {
    IHOM_CUDA(cudaMemsetAsync(err_.p, 0, sizeof(int), s_));
    if (e == 1) throw NumericError(std::string("non-invertible coarse stencil diagonal (") + where + ")");
    throw NumericError(std::string("coarsest operator is singular beyond translations (") + where + ")");
  }
}

template <typename T>
void Hierarchy<T>::remove_translations(double* f, int l) {  // src/multigrid.cpp:81-86
  const Level& L = levels_[size_t(l)];
  const long long nv = L.g.nv;
  {
    ProfScope p(s_, "reduce", double(nv) * 24.0);
    launch_comp_sums<double>(f, nv, ws_.partials, ws_.scalars, s_, ticket_.p);
  }
  if (L.sharded) allreduce(ws_.scalars, 3);  // component sums over the whole grid
  {
    ProfScope p(s_, "vector", double(nv) * 48.0);
    launch_sub_means<double>(f, nv, ws_.scalars, s_, L.nv_global);
  }
  launches_ += 2;
}

// remove_translations of src written into dst (the fused-update solve ends in the other buffer):
// the same sums and the same per-entry fma as the in-place version
template <typename T>
void Hierarchy<T>::remove_translations_to(const double* src, double* dst, int l) {
  const Level& L = levels_[size_t(l)];
  const long long nv = L.g.nv;
  {
    ProfScope p(s_, "reduce", double(nv) * 24.0);
    launch_comp_sums<double>(src, nv, ws_.partials, ws_.scalars, s_, ticket_.p);
  }
  if (L.sharded) allreduce(ws_.scalars, 3);
  {
    ProfScope p(s_, "vector", double(nv) * 48.0);
    launch_sub_means_copy(src, dst, nv, ws_.scalars, s_, L.nv_global);
  }
  launches_ += 2;
}

// remove_translations(f, 0) followed by norm(f): one pass fewer over f, bitwise the same results.
template <typename T>
double Hierarchy<T>::project_norm0(double* f) {
  const Level& L = levels_[0];
  const long long nv = L.g.nv;
  if (knob("PROJECT_NORM", 1) == 0) {
    remove_translations(f, 0);
    return norm(f, 3 * nv);
  }
  double* sums = ws_.scalars;
  if (msum_f_[cur_rhs_] == f) {  // the sums came out of the macro-force pass
    sums = ws_.scalars + kMacroSums + 3 * cur_rhs_;
  } else {
    ProfScope p(s_, "reduce", double(nv) * 24.0);
    launch_comp_sums<double>(f, nv, ws_.partials, sums, s_, ticket_.p);
    ++launches_;
  }
  msum_f_[cur_rhs_] = nullptr;
  if (L.sharded) allreduce(sums, 3);
  {
    ProfScope p(s_, "vector", double(nv) * 48.0);
    launch_sub_means_norm(f, nv, sums, ws_.partials, ws_.scalars + 4, s_, L.nv_global, ticket_.p);
  }
  ++launches_;
  allreduce(ws_.scalars + 4, 1);
  IHOM_CUDA(cudaMemcpyAsync(h_pinned_, ws_.scalars + 4, sizeof(double), cudaMemcpyDeviceToHost, s_));
  IHOM_CUDA(cudaStreamSynchronize(s_));
  return std::sqrt(h_pinned_[0]);
}

template <typename T>
void Hierarchy<T>::macro_force(int load) {  // src/fem.cpp:145-150
  Level& L0 = levels_[0];
  const ZLink<T> cl = slab_.on() ? coeff_l_ : ZLink<T>{};
  ProfScope p(s_, "macro_force", double(L0.g.nv) * (24.0 + sizeof(T)));
  if (fast_ok(L0.g) && knob("MACRO_SUMS", 1)) {
    const size_t nb = size_t(3 * macro_force_sums_blocks(L0.g));
    if (mf_part_.n < nb) mf_part_.alloc(nb);
    launch_macro_force_sums<T>(L0.g, coeff_.p, load, L0.f.p, mf_part_.p, ws_.partials,
                               ws_.scalars + kMacroSums + 3 * cur_rhs_, s_, cl, ticket_.p);
    msum_f_[cur_rhs_] = L0.f.p;
    launches_ += 2;
  } else {
    launch_macro_force<T>(L0.g, coeff_.p, load, L0.f.p, s_, cl);
    msum_f_[cur_rhs_] = nullptr;
    ++launches_;
  }
}

template <typename T>
double Hierarchy<T>::norm(const double* x, long long n) {  // src/multigrid.cpp:88-94
  {
    ProfScope p(s_, "reduce", double(n) * 8.0);
    launch_dot<double>(x, x, n, ws_.partials, ws_.scalars + 4, s_, ticket_.p);
  }
  ++launches_;
  allreduce(ws_.scalars + 4, 1);  // level-0 fields only: split over the slabs
  IHOM_CUDA(cudaMemcpyAsync(h_pinned_, ws_.scalars + 4, sizeof(double), cudaMemcpyDeviceToHost, s_));
  IHOM_CUDA(cudaStreamSynchronize(s_));
  return std::sqrt(h_pinned_[0]);
}

template <typename T>
void Hierarchy<T>::apply(int l, const double* x, double* y) {  // src/multigrid.cpp:392-398
  const Level& L = levels_[size_t(l)];
  if (L.sharded) throw std::invalid_argument("apply() on a z-slab level: use the solver operations");
  if (l == 0) {
    ProfScope p(s_, "l0_apply", resid_l0_bytes(L.g, 8, sizeof(T), false));
    launch_l0_apply<T, double, double>(L.g, coeff_.p, x, nullptr, y, s_);
  } else {
    ProfScope p(s_, "coarse_apply", resid_coarse_bytes(L.g, 8, sizeof(T), false));
    launch_stencil_apply<T, double>(L.g, L.st.p, x, nullptr, y, s_);
  }
  ++launches_;
}

template <typename T>
void Hierarchy<T>::relax(int l, int sweeps, bool zero_start) {  // src/multigrid.cpp:400-408
  Level& L = levels_[size_t(l)];
  double* u = level_u(l);
  const ZLink<double> ul = L.sharded ? ulink(l) : ZLink<double>{};
  if (zero_start && l == 0) throw std::logic_error("zero-start sweeps exist on the coarse levels only");
  for (int sw = 0; sw < sweeps; ++sw)
    for (int c = 0; c < 8; ++c) {
      if (L.g.size[c] == 0) continue;
      if (L.sharded) sync_halo();  // colour c-1 of the neighbouring slabs is final
      const bool zs = zero_start && sw == 0;
      if (l == 0) {
        ProfScope p(s_, "l0_gs_f64", gs_l0_bytes(L.g, c, 8, sizeof(T)));
        launch_l0_gs_color<T, double, double>(L.g, coeff_.p, L.f.p, u, c, s_, L.sharded ? coeff_l_ : ZLink<T>{}, ul);
      } else {
        ProfScope p(s_, l == 1 ? "l1_gs_f64" : "coarse_gs_f64",
                    zs ? gs_coarse_bytes_zs(L.g, c, 8, sizeof(T)) : gs_coarse_bytes(L.g, c, 8, sizeof(T)));
        launch_stencil_gs_color<T, double>(L.g, L.st.p, L.f.p, u, c, err_.p, s_, ul, zs);
      }
      ++launches_;
    }
}

template <typename T>
void Hierarchy<T>::compute_residual(int l) {  // src/multigrid.cpp:410-424
  Level& L = levels_[size_t(l)];
  if (L.sharded) sync_halo();
  const ZLink<double> ul = L.sharded ? ulink(l) : ZLink<double>{};
  if (l == 0) {
    ProfScope p(s_, "l0_residual_f64", resid_l0_bytes(L.g, 8, sizeof(T), true));
    launch_l0_apply<T, double, double>(L.g, coeff_.p, level_u(0), L.f.p, L.r.p, s_, L.sharded ? coeff_l_ : ZLink<T>{},
                                       ul);
  } else {
    ProfScope p(s_, l == 1 ? "l1_residual_f64" : "coarse_residual_f64", resid_coarse_bytes(L.g, 8, sizeof(T), true));
    launch_stencil_apply<T, double>(L.g, L.st.p, L.u.p, L.f.p, L.r.p, s_, ul);
  }
  ++launches_;
}

template <typename T>
void Hierarchy<T>::coarsest_solve() {  // src/multigrid.cpp:426-451
  join_coarsest();
  const int lc = num_levels() - 1;
  Level& L = levels_[size_t(lc)];
  ProfScope p(s_, "coarsest", 0.0);
  launch_coarsest_solve<double>(ndof_c_, L.g.nv, Ainv_.p, A_.p, Q_.p, nnull_, L.f.p, level_u(lc), negligible_load(ndof_c_),
                                cwork_.p, err_.p, s_);
  ++launches_;
}

template <typename T>
double Hierarchy<T>::v_cycle(const SolverOptions& opts) {  // src/multigrid.cpp:453-472
  if (!density_set_) throw StateError("set_density before v_cycle");
  if (opts.mode == kMixedDefect && std::is_same_v<T, float>) return v_cycle_defect(opts);
  const int lmax = num_levels() - 1;
  for (int l = 0; l < lmax; ++l) {
    const bool zs = l > 0 && opts.pre_sweeps > 0 && zero_start_ok(l);
    if (l > 0 && !zs)
      IHOM_CUDA(cudaMemsetAsync(levels_[size_t(l)].u.p, 0, sizeof(double) * 3 * levels_[size_t(l)].g.nv, s_));
    relax(l, opts.pre_sweeps, zs);
    compute_residual(l);
    restrict_to(l, levels_[size_t(l)].r.p, levels_[size_t(l + 1)].f.p);
  }
  if (lmax > 0) IHOM_CUDA(cudaMemsetAsync(levels_[size_t(lmax)].u.p, 0, sizeof(double) * 3 * levels_[size_t(lmax)].g.nv, s_));
  coarsest_solve();
  for (int l = lmax - 1; l >= 0; --l) {
    prolong_from(l, levels_[size_t(l + 1)].u.p, level_u(l), levels_[size_t(l + 1)].ul);
    relax(l, opts.post_sweeps);
  }
  compute_residual(0);
  const long long n0 = 3 * levels_[0].g.nv;
  // ||f_0|| is constant inside solve() unless the coarsest solve (lmax == 0) re-projects f_0
  const double fn = (u0_bound_ && lmax > 0) ? fnorm0_ : norm(levels_[0].f.p, n0);
  const double rn = norm(levels_[0].r.p, n0);
  check_error("v_cycle");
  return fn > 0.0 ? rn / fn : 0.0;
}

// ---- mixed-precision defect-correction cycle (kMixedDefect) ----
template <typename T>
void Hierarchy<T>::ensure_inner() {
  if (inner_ready_) return;
  for (auto& L : levels_) {
    const size_t n3 = size_t(3 * L.g.nv);
    L.eu.alloc(n3);
    L.ef.alloc(n3);
    L.er.alloc(n3);
  }
  if (fused_update_ok()) u_alt_.alloc(size_t(3 * levels_[0].g.nv));
  IHOM_CUDA(cudaDeviceSynchronize());
  if (slab_.on()) {  // collective, same order on every slab
    if (u_alt_.p) u_alt_l_ = link(u_alt_.p);
    for (size_t l = 0; l < levels_.size(); ++l) {
      Level& L = levels_[l];
      if (L.sharded) {
        L.eul = link(L.eu.p);
        L.erl = link(L.er.p);
      } else if (int(l) == rep0_) {
        L.efpeer = peer_table(slab_.fab->exchange(slab_.rank, L.ef.p));
      }
    }
  }
  inner_ready_ = true;
}

template <typename T>
bool Hierarchy<T>::zero_start_ok(int l) const {
  if (knob("ZERO_START", 1) == 0) return false;
  if (l > 0) return true;  // every stencil GS kernel takes the zero mask
  if constexpr (std::is_same_v<T, float>)
    return l0_gs_zero_start_ok<float, float, float>(levels_[0].g);
  return false;  // level-0 f32 inner fields exist in mixed precision only
}

template <typename T>
void Hierarchy<T>::relax_f32(int l, int sweeps, bool reverse, bool zero_start) {
  Level& L = levels_[size_t(l)];
  if constexpr (std::is_same_v<T, float>) {
    if (zero_start && reverse) throw std::logic_error("zero-start sweeps run the colours forward");
    const bool pair = l == 0 && !reverse && l0_gs_pair_ok(L.g);
    for (int sw = 0; sw < sweeps; ++sw)
      for (int ci = 0; ci < 8; ++ci) {
        const int c = reverse ? 7 - ci : ci;
        if (L.g.size[c] == 0) continue;
        if (L.sharded) sync_halo();
        const bool zs = zero_start && sw == 0;
        if (pair) {  // colours c, c + 1 in one launch (c even)
          ProfScope p(s_, "l0_gs_f32", gs_l0_pair_bytes(L.g, c, zs));
          launch_l0_gs_pair(L.g, coeff_.p, L.ef.p, L.eu.p, c, s_, L.sharded ? coeff_l_ : ZLink<float>{}, L.eul, zs);
          ++launches_;
          ++ci;
          continue;
        }
        if (l == 0) {
          ProfScope p(s_, "l0_gs_f32", zs ? gs_l0_bytes_zs(L.g, c, 4, 4) : gs_l0_bytes(L.g, c, 4, 4));
          launch_l0_gs_color<float, float, float>(L.g, coeff_.p, L.ef.p, L.eu.p, c, s_,
                                                  L.sharded ? coeff_l_ : ZLink<float>{}, L.eul, zs);
        } else {
          ProfScope p(s_, l == 1 ? "l1_gs_f32" : (l == 2 ? "l2_gs_f32" : "coarse_gs_f32"),
                      zs ? gs_coarse_bytes_zs(L.g, c, 4, 4) : gs_coarse_bytes(L.g, c, 4, 4));
          launch_stencil_gs_color<float, float>(L.g, L.st.p, L.ef.p, L.eu.p, c, err_.p, s_, L.eul, zs);
        }
        ++launches_;
      }
  }
}

template <typename T>
void Hierarchy<T>::residual_f32(int l) {
  Level& L = levels_[size_t(l)];
  if constexpr (std::is_same_v<T, float>) {
    if (L.sharded) sync_halo();
    if (l == 0) {
      ProfScope p(s_, "l0_residual_f32", resid_l0_bytes(L.g, 4, 4, true));
      launch_l0_apply<float, float, float>(L.g, coeff_.p, L.eu.p, L.ef.p, L.er.p, s_,
                                           L.sharded ? coeff_l_ : ZLink<float>{}, L.eul);
    } else {
      ProfScope p(s_, l == 1 ? "l1_residual_f32" : (l == 2 ? "l2_residual_f32" : "coarse_residual_f32"), resid_coarse_bytes(L.g, 4, 4, true));
      launch_stencil_apply<float, float>(L.g, L.st.p, L.eu.p, L.ef.p, L.er.p, s_, L.eul);
    }
    ++launches_;
  }
}

template <typename T>
void Hierarchy<T>::coarsest_f32() {
  join_coarsest();
  const int lc = num_levels() - 1;
  Level& L = levels_[size_t(lc)];
  ProfScope p(s_, "coarsest", 0.0);
  launch_coarsest_solve<float>(ndof_c_, L.g.nv, Ainv_.p, A_.p, Q_.p, nnull_, L.ef.p, L.eu.p, 0.0, cwork_.p, err_.p, s_);
  ++launches_;
}

template <typename T>
bool Hierarchy<T>::fused_update_ok() const {
  return !lean_ && std::is_same_v<T, float> && knob("FUSED_UPDATE", 1) != 0 && sweep_ok(levels_[0].g);
}

template <typename T>
void Hierarchy<T>::restore_home() {
  if (!u_home_ || u0_bound_ == u_home_) return;
  const long long n0 = 3 * levels_[0].g.nv;
  IHOM_CUDA(cudaMemcpyAsync(u_home_, u0_bound_, sizeof(double) * n0, cudaMemcpyDeviceToDevice, s_));
  u0_bound_ = u_home_;
  u0l_ = u_home_l_;
}

template <typename T>
double Hierarchy<T>::defect_residual(bool update, double* slot) {
  Level& L0 = levels_[0];
  if constexpr (std::is_same_v<T, float>) {
    if (!npart_.p) npart_.alloc(size_t(L0.g.nv / 32 + 1024));
    long long nb;
    if (L0.sharded) sync_halo();
    if (update) {  // u' = u + e into the other buffer, r = f - K u'; then u' is the bound field
      if (!u_home_ || !u_alt_.p) throw StateError("fused update outside a bound solve");
      const bool home = u0_bound_ == u_home_;
      double* nxt = home ? u_alt_.p : u_home_;
      const ZLink<double> nxtl = home ? u_alt_l_ : u_home_l_;
      {
        ProfScope p(s_, "l0_residual_f64", double(L0.g.nv) * (48.0 + sizeof(T) + 12.0 + 12.0 + 24.0));
        nb = launch_l0_defect_update_sweep(L0.g, coeff_.p, L0.sharded ? coeff_l_ : ZLink<float>{}, u0_bound_,
                                           L0.sharded ? u0l_ : ZLink<double>{}, L0.eu.p,
                                           L0.sharded ? L0.eul : ZLink<float>{}, nxt, L0.f.p, L0.ef.p, npart_.p,
                                           s_);
      }
      u0_bound_ = nxt;
      u0l_ = L0.sharded ? nxtl : resolve(ZLink<double>{}, nxt);
    } else {
      ProfScope p(s_, "l0_residual_f64", double(L0.g.nv) * (48.0 + sizeof(T) + 12.0));
      nb = launch_l0_residual_norm<float>(L0.g, coeff_.p, level_u(0), L0.f.p, L0.ef.p, npart_.p, s_,
                                          L0.sharded ? coeff_l_ : ZLink<float>{}, L0.sharded ? ulink(0) : ZLink<double>{});
    }
    {
      ProfScope p(s_, "reduce", double(nb) * 8.0);
      launch_sum(npart_.p, nb, ws_.partials, slot ? slot : ws_.scalars + 4, s_, ticket_.p);
    }
    launches_ += 2;
    if (slot) return 0.0;  // deferred: ||r||^2 of this slab in *slot (finish_defect_cycles reads them together)
    allreduce(ws_.scalars + 4, 1);
    IHOM_CUDA(cudaMemcpyAsync(h_pinned_, ws_.scalars + 4, sizeof(double), cudaMemcpyDeviceToHost, s_));
    IHOM_CUDA(cudaStreamSynchronize(s_));
    return std::sqrt(h_pinned_[0]);
  } else {
    throw StateError("defect residual exists in mixed precision only");
  }
}

// One V-cycle on K e = ef0 starting from e = 0, entirely on the f32 inner fields.
// symmetric: post-smoothing walks the colours 7..0 (adjoint of the pre-smoother),
// which makes the cycle an SPD preconditioner for PCG.
template <typename T>
void Hierarchy<T>::inner_down(int l, const SolverOptions& opts) {
  // e = 0 on every level before its pre-smoothing: with zero-start sweeps the first sweep never
  // reads a colour it has not written yet, so the clear is skipped (bit-identical)
  const bool zs = opts.pre_sweeps > 0 && zero_start_ok(l);
  if (!zs) {
    IHOM_CUDA(cudaMemsetAsync(levels_[size_t(l)].eu.p, 0, sizeof(float) * 3 * levels_[size_t(l)].g.nv, s_));
    launches_ += l == 0 ? 1 : 0;
  }
  relax_f32(l, opts.pre_sweeps, false, zs);
  residual_f32(l);
  restrict_to_f32(l);
}

template <typename T>
void Hierarchy<T>::inner_coarsest() {
  const int lmax = num_levels() - 1;
  if (lmax > 0) IHOM_CUDA(cudaMemsetAsync(levels_[size_t(lmax)].eu.p, 0, sizeof(float) * 3 * levels_[size_t(lmax)].g.nv, s_));
  coarsest_f32();
}

template <typename T>
void Hierarchy<T>::inner_prolong(int l) {
  Level& F = levels_[size_t(l)];
  Level& C = levels_[size_t(l + 1)];
  if (F.sharded) sync_halo();
  {
    ProfScope p(s_, "prolong", double(F.g.nv) * 25.5);
    if (!(F.sharded && !C.sharded))
      launch_prolong_add<float>(C.g, F.g, C.eu.p, F.eu.p, s_, C.sharded ? C.eul : ZLink<float>{});
    else
      launch_prolong_add<float>(C.g, F.g, C.eu.p, F.eu.p, s_, {}, slab_.rank * (F.g.n[2] / 2));
  }
  ++launches_;
}

template <typename T>
void Hierarchy<T>::inner_vcycle(const SolverOptions& opts, bool symmetric) {
  const int lmax = num_levels() - 1;
  for (int l = 0; l < lmax; ++l) inner_down(l, opts);
  inner_coarsest();
  for (int l = lmax - 1; l >= 0; --l) {
    inner_prolong(l);
    relax_f32(l, opts.post_sweeps, symmetric);
  }
}

template <typename T>
SolveStats Hierarchy<T>::solve_pcg(double* u, const SolverOptions& opts) {
  SolveStats st;
  if (slab_.on()) throw std::invalid_argument("MG-PCG mode is not available on z-slabs (use vcycle or mixed_defect)");
  if constexpr (!std::is_same_v<T, float>) {
    throw std::invalid_argument("MG-PCG mode needs mixed precision (f32 inner preconditioner)");
  } else {
    Level& L0 = levels_[0];
    const long long nv = L0.g.nv, n0 = 3 * nv;
    ensure_inner();
    if (!pcg_p_.p) {
      pcg_p_.alloc(size_t(n0));
      pcg_q_.alloc(size_t(n0));
      pcg_s_.alloc(8);
    }
    double* sc = pcg_s_.p;  // [0] rz [1] pq [2] alpha [3] beta [4] rr [5] rz_new
    auto readback = [&](const double* d) {
      IHOM_CUDA(cudaMemcpyAsync(h_pinned_, d, sizeof(double), cudaMemcpyDeviceToHost, s_));
      IHOM_CUDA(cudaStreamSynchronize(s_));
      return h_pinned_[0];
    };
    auto precondition = [&]() {  // eu0 = M^-1 ef0, rz_new = (r, eu0)
      inner_vcycle(opts, true);
      ProfScope p(s_, "reduce", double(n0) * 12.0);
      launch_dot_df(L0.r.p, L0.eu.p, n0, ws_.partials, sc + 5, s_);
      launches_ += 2;
    };
    compute_residual(0);  // r = f - K u (f64)
    double rn = norm(L0.r.p, n0);
    st.rel_residual = rn / fnorm0_;
    if (st.rel_residual <= opts.tol) {
      st.converged = true;
      return st;
    }
    {
      ProfScope p(s_, "vector", double(n0) * 12.0);
      launch_convert<double, float>(L0.r.p, L0.ef.p, n0, s_);
    }
    precondition();
    launch_pcg_p(pcg_p_.p, L0.eu.p, sc + 3, n0, true, s_);
    IHOM_CUDA(cudaMemcpyAsync(sc, sc + 5, sizeof(double), cudaMemcpyDeviceToDevice, s_));
    launches_ += 1;
    while (st.cycles < opts.max_cycles) {
      {
        ProfScope p(s_, "l0_apply_f64", double(nv) * (48.0 + sizeof(T)));
        launch_l0_apply<T, double, double>(L0.g, coeff_.p, pcg_p_.p, nullptr, pcg_q_.p, s_);  // q = K p
      }
      {
        ProfScope p(s_, "reduce", double(n0) * 16.0);
        launch_dot<double>(pcg_p_.p, pcg_q_.p, n0, ws_.partials, sc + 1, s_);
      }
      launch_ratio(sc, sc + 1, sc + 2, s_);  // alpha = rz / pq
      {
        ProfScope p(s_, "vector", double(n0) * 60.0);
        launch_pcg_ur(u, L0.r.p, pcg_p_.p, pcg_q_.p, sc + 2, L0.ef.p, n0, ws_.partials, sc + 4, s_);
      }
      launches_ += 6;
      ++st.cycles;
      st.rel_residual = std::sqrt(readback(sc + 4)) / fnorm0_;
      check_error("pcg");
      if (st.rel_residual <= opts.tol) break;
      precondition();
      launch_ratio(sc + 5, sc, sc + 3, s_);  // beta = rz_new / rz
      IHOM_CUDA(cudaMemcpyAsync(sc, sc + 5, sizeof(double), cudaMemcpyDeviceToDevice, s_));
      {
        ProfScope p(s_, "vector", double(n0) * 20.0);
        launch_pcg_p(pcg_p_.p, L0.eu.p, sc + 3, n0, false, s_);
      }
      launches_ += 2;
    }
    st.converged = st.rel_residual <= opts.tol;
  }
  return st;
}

template <typename T>
double Hierarchy<T>::v_cycle_defect(const SolverOptions& opts) {
  ensure_inner();
  const int lmax = num_levels() - 1;
  Level& L0 = levels_[0];
  const long long n0 = 3 * L0.g.nv;
  // inner right-hand side ef0 = float(f - K u): inside solve() it is left current
  // by the fused residual at the end of the previous cycle (or before the loop).
  const bool fast = fast_ok(L0.g);
  if (!u0_bound_ || !fast) {
    if (fast) {
      defect_residual();
    } else {
      compute_residual(0);
      ProfScope p(s_, "vector", double(n0) * 12.0);
      launch_convert<double, float>(L0.r.p, L0.ef.p, n0, s_);
    }
  }
  inner_vcycle(opts, false);
  const double rn = finish_defect_cycle();
  const double fn = (u0_bound_ && lmax > 0) ? fnorm0_ : norm(L0.f.p, n0);
  check_error("v_cycle");
  return fn > 0.0 ? rn / fn : 0.0;
}

template <typename T>
double Hierarchy<T>::finish_defect_cycle(double* slot) {
  Level& L0 = levels_[0];
  const long long n0 = 3 * L0.g.nv;
  const bool fast = fast_ok(L0.g);
  const bool fused = fast && u0_bound_ && u_alt_.p && fused_update_ok();
  if (!fused) {
    ProfScope p(s_, "vector", double(n0) * 20.0);
    launch_axpy_update<float>(level_u(0), L0.eu.p, n0, s_);
    ++launches_;
  }
  if (fast) return defect_residual(fused, slot);  // also leaves ef0 ready for the next cycle
  if (slot) throw std::logic_error("deferred defect norms need an even level-0 grid");
  compute_residual(0);
  return norm(L0.r.p, n0);
}

// ---------------------------------------------------------------- lockstep RHS groups
template <typename T>
bool Hierarchy<T>::pair_ok(const SolverOptions& opts) const {
  return !lean_ && std::is_same_v<T, float> && opts.mode == kMixedDefect && knob("RHS_PAIRS", 1) != 0 &&
         fast_ok(levels_[0].g) && num_levels() > 1;
}

// RHS_GROUP = 2, 3 or 6 forces the group size; 0 (default) picks the largest of 6, 3, 2 (else 1) whose extra
// per-RHS fields fit in this rank's share of the free HBM next to a reserve for the energy cache and
// workspace. z-slabs decide collectively (every slab allocates the same slots, with links): the free
// memory is split between the slabs that share a device, and all slabs take the smallest choice.
// Decided once per hierarchy (later calls return the cached size).
template <typename T>
int Hierarchy<T>::group_size(const SolverOptions& opts) {
  if (!pair_ok(opts)) return 1;
  const int forced = knob("RHS_GROUP", 0);
  if (forced == 2 || forced == 3 || forced == 6) return forced;
  if (group_auto_) return group_auto_;
  int dev = 0;
  IHOM_CUDA(cudaGetDevice(&dev));
  double share = 1.0;
  if (slab_.on()) {  // slabs on this device: one-hot by device ordinal, summed over the slabs
    double h[16] = {};
    h[dev & 15] = 1.0;
    IHOM_CUDA(cudaMemcpyAsync(ws_.scalars + 32, h, sizeof(h), cudaMemcpyHostToDevice, s_));
    allreduce(ws_.scalars + 32, 16, false);
    IHOM_CUDA(cudaMemcpyAsync(h, ws_.scalars + 32, sizeof(h), cudaMemcpyDeviceToHost, s_));
    IHOM_CUDA(cudaStreamSynchronize(s_));
    share = std::max(1.0, h[dev & 15]);
  }
  double per_slot = 2.0 * 3.0 * 8.0 * double(levels_[0].g.nv);  // f64 f and ping-pong u at level 0
  for (const Level& L : levels_) per_slot += 3.0 * 3.0 * 4.0 * double(L.g.nv);  // f32 e, f, r per level
  size_t free_b = 0, total_b = 0;
  IHOM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  free_b = hbm_free_limit(free_b);
  const double budget = double(free_b) / share;
  const double reserve = 21.0 * 8.0 * double(levels_[0].g.nv) + 8e9 / share;  // energy cache (f64 worst case)
  int g = 1;  // memory lever: no lockstep grouping when even a pair's extra fields do not fit
  for (int c : {6, 3, 2}) {
    const double extra = double(std::max(0, c - 1 - int(slots_.size()))) * per_slot;
    if (extra + reserve <= budget) {
      g = c;
      break;
    }
  }
  if (slab_.on()) {  // the smallest choice of all slabs: max of -g
    double v = -double(g);
    IHOM_CUDA(cudaMemcpyAsync(ws_.scalars + 48, &v, sizeof(v), cudaMemcpyHostToDevice, s_));
    allreduce(ws_.scalars + 48, 1, true);
    IHOM_CUDA(cudaMemcpyAsync(&v, ws_.scalars + 48, sizeof(v), cudaMemcpyDeviceToHost, s_));
    IHOM_CUDA(cudaStreamSynchronize(s_));
    g = int(-v);
  }
  group_auto_ = g;
  return g;
}

template <typename T>
void Hierarchy<T>::ensure_group(int G) {
  ensure_inner();
  const size_t nl = levels_.size();
  while (slots_.size() + 1 < size_t(G)) {
    slots_.emplace_back();
    RhsSlot& o = slots_.back();
    o.eu.resize(nl);
    o.ef.resize(nl);
    o.er.resize(nl);
    o.eul.assign(nl, ZLink<float>{});
    o.erl.assign(nl, ZLink<float>{});
    o.efpeer.assign(nl, PeerTable{});
    for (size_t l = 0; l < nl; ++l) {
      const size_t n3 = size_t(3 * levels_[l].g.nv);
      o.eu[l].alloc(n3);
      o.ef[l].alloc(n3);
      o.er[l].alloc(n3);
    }
    o.f0.alloc(size_t(3 * levels_[0].g.nv));
    if (u_alt_.p) o.ualt.alloc(size_t(3 * levels_[0].g.nv));
    IHOM_CUDA(cudaDeviceSynchronize());
    if (slab_.on()) {  // collective, same order on every slab (mirrors ensure_inner)
      if (o.ualt.p) o.ualtl = link(o.ualt.p);
      for (size_t l = 0; l < nl; ++l) {
        Level& L = levels_[l];
        if (L.sharded) {
          o.eul[l] = link(o.eu[l].p);
          o.erl[l] = link(o.er[l].p);
        } else if (int(l) == rep0_) {
          o.efpeer[l] = peer_table(slab_.fab->exchange(slab_.rank, o.ef[l].p));
        }
      }
    }
    o.ready = true;
  }
}

template <typename T>
void Hierarchy<T>::swap_live(RhsSlot& o) {
  for (size_t l = 0; l < levels_.size(); ++l) {
    Level& L = levels_[l];
    std::swap(L.eu, o.eu[l]);
    std::swap(L.ef, o.ef[l]);
    std::swap(L.er, o.er[l]);
    std::swap(L.eul, o.eul[l]);
    std::swap(L.erl, o.erl[l]);
    std::swap(L.efpeer, o.efpeer[l]);
  }
  std::swap(levels_[0].f, o.f0);
  std::swap(u_alt_, o.ualt);
  std::swap(u_alt_l_, o.ualtl);
  std::swap(u0_bound_, o.u0_bound);
  std::swap(u_home_, o.u_home);
  std::swap(u0l_, o.u0l);
  std::swap(u_home_l_, o.u_home_l);
  std::swap(fnorm0_, o.fnorm0);
}

// RHS k's fields become the live level fields; the previous live RHS takes k's slot.
template <typename T>
void Hierarchy<T>::select_rhs(int k) {
  if (k == cur_rhs_) return;
  if (k < 0 || k >= kMaxRhsGroup) throw std::logic_error("right-hand side index out of range");
  ensure_group(k + 1);
  const int j = where_[k];
  swap_live(slots_[size_t(j)]);
  where_[cur_rhs_] = j;
  where_[k] = -1;
  cur_rhs_ = k;
}

template <typename T>
void Hierarchy<T>::relax_f32_group(int G, int l, int sweeps, bool zero_start) {
  Level& L = levels_[size_t(l)];
  if (l == 0) throw std::logic_error("grouped sweeps run on the stencil levels");
  float* u[kMaxRhsGroup];
  const float* f[kMaxRhsGroup];
  ZLink<float> ul[kMaxRhsGroup];
  for (int k = 0; k < G; ++k) {
    RhsSlot* o = slot_of(k);
    u[k] = o ? o->eu[size_t(l)].p : L.eu.p;
    f[k] = o ? o->ef[size_t(l)].p : L.ef.p;
    ul[k] = o ? o->eul[size_t(l)] : L.eul;
  }
  for (int sw = 0; sw < sweeps; ++sw)
    for (int c = 0; c < 8; ++c) {
      if (L.g.size[c] == 0) continue;
      if (L.sharded) sync_halo();
      const bool zs = zero_start && sw == 0;
      if constexpr (std::is_same_v<T, float>) {
        ProfScope p(s_, l == 1 ? "l1_gs_f32" : (l == 2 ? "l2_gs_f32" : "coarse_gs_f32"),
                    (zs ? gs_coarse_bytes_zs(L.g, c, 4.0 * G, 4) : gs_coarse_bytes(L.g, c, 4.0 * G, 4)));
        launch_stencil_gs_color_group<float, float>(L.g, L.st.p, G, f, u, c, err_.p, s_, ul, zs);
      }
      ++launches_;
    }
}

template <typename T>
void Hierarchy<T>::residual_f32_group(int G, int l) {
  Level& L = levels_[size_t(l)];
  if (L.sharded) sync_halo();
  const float* x[kMaxRhsGroup];
  const float* f[kMaxRhsGroup];
  float* y[kMaxRhsGroup];
  ZLink<float> xl[kMaxRhsGroup];
  for (int k = 0; k < G; ++k) {
    RhsSlot* o = slot_of(k);
    x[k] = o ? o->eu[size_t(l)].p : L.eu.p;
    f[k] = o ? o->ef[size_t(l)].p : L.ef.p;
    y[k] = o ? o->er[size_t(l)].p : L.er.p;
    xl[k] = o ? o->eul[size_t(l)] : L.eul;
  }
  if constexpr (std::is_same_v<T, float>) {
    ProfScope p(s_, l == 1 ? "l1_residual_f32" : (l == 2 ? "l2_residual_f32" : "coarse_residual_f32"),
                resid_coarse_bytes(L.g, 4.0 * G, 4, true));
    launch_stencil_apply_group<float, float>(L.g, L.st.p, G, x, f, y, s_, xl);
  }
  ++launches_;
}

// One inner V-cycle for each active RHS, the stencil levels in lockstep. An inactive RHS (already
// converged) skips every level-0 and transfer step; the grouped coarse kernels still compute its lane
// on stale (finite) data, which nothing reads.
// Restriction l -> l+1 (down) or prolongation l+1 -> l (up) of every RHS lane of a lockstep group in one
// launch (levels >= 1, where the group's lanes run together anyway; an inactive lane transfers stale data
// nothing reads). False when the level pair needs the per-lane path (slab transition, odd grids).
template <typename T>
bool Hierarchy<T>::transfer_group(int G, int l, bool down) {
  if constexpr (!std::is_same_v<T, float>) {
    return false;
  } else {
    Level& F = levels_[size_t(l)];
    Level& C = levels_[size_t(l + 1)];
    if (l < 1 || G < 2 || (F.sharded && !C.sharded) || !transfer_group_ok(F.g, C.g)) return false;
    const float* src[kMaxRhsGroup];
    float* dst[kMaxRhsGroup];
    ZLink<float> lk[kMaxRhsGroup];
    for (int k = 0; k < G; ++k) {
      RhsSlot* o = slot_of(k);
      if (down) {
        src[k] = o ? o->er[size_t(l)].p : F.er.p;
        lk[k] = F.sharded ? (o ? o->erl[size_t(l)] : F.erl) : ZLink<float>{};
        dst[k] = o ? o->ef[size_t(l + 1)].p : C.ef.p;
      } else {
        src[k] = o ? o->eu[size_t(l + 1)].p : C.eu.p;
        lk[k] = C.sharded ? (o ? o->eul[size_t(l + 1)] : C.eul) : ZLink<float>{};
        dst[k] = o ? o->eu[size_t(l)].p : F.eu.p;
      }
    }
    if (F.sharded) sync_halo();
    {
      ProfScope p(s_, down ? "restrict" : "prolong", double(F.g.nv) * (down ? 13.5 : 25.5) * G);
      if (down) launch_restrict_group(F.g, C.g, G, src, lk, dst, s_);
      else launch_prolong_add_group(C.g, F.g, G, src, lk, dst, s_);
    }
    ++launches_;
    return true;
  }
}

// First level of the bottom cycle (one cooperative launch for the small levels and the coarsest,
// knob BOTTOM_CYCLE): the smallest l >= 1 from which every level down to the coarsest is replicated
// (not split into z-slabs) and small enough for the warp-per-vertex kernels; lmax: none.
template <typename T>
int Hierarchy<T>::bottom_start(int G) const {
  const int lmax = num_levels() - 1;
  if (!std::is_same_v<T, float> || (G != 2 && G != 3 && G != 6) || !bottom_ok_ || knob("BOTTOM_CYCLE", 1) == 0)
    return lmax;
  int lb = lmax;
  for (int l = lmax - 1; l >= 1; --l) {
    const Level& L = levels_[size_t(l)];
    if (L.sharded || !bottom_level_ok(L.g, levels_[size_t(l + 1)].g) || lmax - l + 1 > kMaxBottom) break;
    lb = l;
  }
  return lb;
}

template <typename T>
bool Hierarchy<T>::bottom_cycle(int G, int lb, const SolverOptions& opts) {
  const int lmax = num_levels() - 1;
  join_coarsest();
  BottomCycle bc{};
  bc.nlev = lmax - lb + 1;
  for (int l = lb; l <= lmax; ++l) {
    Level& L = levels_[size_t(l)];
    BottomLevel& B = bc.L[l - lb];
    B.g = L.g;
    B.st = reinterpret_cast<const float*>(L.st.p);
    B.zs = opts.pre_sweeps > 0 && zero_start_ok(l) ? 1 : 0;
    for (int k = 0; k < G; ++k) {
      RhsSlot* o = slot_of(k);
      B.eu[k] = o ? o->eu[size_t(l)].p : L.eu.p;
      B.ef[k] = o ? o->ef[size_t(l)].p : L.ef.p;
      B.er[k] = o ? o->er[size_t(l)].p : L.er.p;
    }
  }
  bc.pre = opts.pre_sweeps;
  bc.post = opts.post_sweeps;
  bc.N = ndof_c_;
  bc.nvc = levels_[size_t(lmax)].g.nv;
  bc.Ainv = Ainv_.p;
  bc.A = A_.p;
  bc.Q = Q_.p;
  bc.nq = nnull_;
  if (cwork_.n < size_t(3 * ndof_c_ * G)) cwork_.alloc(size_t(3 * ndof_c_ * kMaxRhsGroup));
  bc.work = cwork_.p;
  bc.err = err_.p;
  {
    ProfScope p(s_, "bottom_cycle", 0.0);
    if (!launch_bottom_cycle(bc, G, s_)) {  // not every block can be co-resident here (e.g. a partitioned GPU)
      bottom_ok_ = false;
      return false;
    }
  }
  ++launches_;
  return true;
}

template <typename T>
void Hierarchy<T>::inner_vcycle_group(int G, const SolverOptions& opts, const bool* act) {
  const int lmax = num_levels() - 1;
  const int lb = bottom_start(G);  // levels lb .. lmax in one launch (lmax: none)
  auto down = [&](int l) {  // pre-smooth, residual, restrict of level l >= 1 (all lanes)
    const bool zs = opts.pre_sweeps > 0 && zero_start_ok(l);
    if (!zs)
      for (int k = 0; k < G; ++k) {
        select_rhs(k);
        IHOM_CUDA(cudaMemsetAsync(levels_[size_t(l)].eu.p, 0, sizeof(float) * 3 * levels_[size_t(l)].g.nv, s_));
      }
    relax_f32_group(G, l, opts.pre_sweeps, zs);
    residual_f32_group(G, l);
    if (!transfer_group(G, l, true))
      for (int k = 0; k < G; ++k)
        if (act[k]) {
          select_rhs(k);
          restrict_to_f32(l);
        }
  };
  auto up = [&](int l) {  // prolong-add from l + 1, post-smooth level l >= 1
    if (!transfer_group(G, l, false))
      for (int k = 0; k < G; ++k)
        if (act[k]) {
          select_rhs(k);
          inner_prolong(l);
        }
    relax_f32_group(G, l, opts.post_sweeps, false);
  };
  auto coarsest = [&] {
    if (lmax > 0 && G > 1) {  // the coarsest solves of all lanes in one launch (block per lane)
      join_coarsest();
      const Level& L = levels_[size_t(lmax)];
      float* f[kMaxRhsGroup];
      float* u[kMaxRhsGroup];
      for (int k = 0; k < G; ++k) {
        RhsSlot* o = slot_of(k);
        f[k] = o ? o->ef[size_t(lmax)].p : L.ef.p;
        u[k] = o ? o->eu[size_t(lmax)].p : L.eu.p;
      }
      if (cwork_.n < size_t(3 * ndof_c_ * G)) cwork_.alloc(size_t(3 * ndof_c_ * kMaxRhsGroup));
      ProfScope p(s_, "coarsest", 0.0);
      launch_coarsest_solve_group(ndof_c_, L.g.nv, Ainv_.p, A_.p, Q_.p, nnull_, G, f, u, cwork_.p, err_.p, s_);
      ++launches_;
    } else {
      for (int k = 0; k < G; ++k)
        if (act[k]) {
          select_rhs(k);
          inner_coarsest();
        }
    }
  };
  for (int k = 0; k < G; ++k)  // level 0 down, per RHS
    if (act[k]) {
      select_rhs(k);
      inner_down(0, opts);
    }
  for (int l = 1; l < lb; ++l) down(l);
  if (!(lb < lmax && bottom_cycle(G, lb, opts))) {  // level by level (also if the cooperative launch is refused)
    for (int l = lb; l < lmax; ++l) down(l);
    coarsest();
    for (int l = lmax - 1; l >= lb; --l) up(l);
  }
  for (int l = std::min(lb, lmax) - 1; l >= 1; --l) up(l);
  for (int k = 0; k < G; ++k)
    if (act[k]) {
      select_rhs(k);
      inner_prolong(0);
      relax_f32(0, opts.post_sweeps, false);
    }
}

// The outer defect-correction step (u += e, r = f - K u, ||r||) of every active RHS of a lockstep group,
// enqueued back to back; the squared norms and the error flag come back in one read (one host round trip
// per round of the group instead of two per RHS). Slabs: one allreduce of the norms, one of the flag.
template <typename T>
void Hierarchy<T>::finish_defect_cycles(int G, const bool* act, double* rn) {
  double* slots = ws_.scalars + 52;  // [0, G): ||r||^2 per RHS, [6]: error flag
  for (int k = 0; k < G; ++k)
    if (act[k]) {
      select_rhs(k);
      finish_defect_cycle(slots + k);
    }
  launch_int_to_double(err_.p, slots + 6, s_);
  if (slab_.on()) {
    slab_.fab->check(slab_.rank);
    allreduce(slots, G);
    allreduce(slots + 6, 1, true);
  }
  IHOM_CUDA(cudaMemcpyAsync(h_pinned_, slots, sizeof(double) * 7, cudaMemcpyDeviceToHost, s_));
  IHOM_CUDA(cudaStreamSynchronize(s_));
  const int e = int(h_pinned_[6]);
  if (e) {
    IHOM_CUDA(cudaMemsetAsync(err_.p, 0, sizeof(int), s_));
    if (e == 1) throw NumericError("non-invertible coarse stencil diagonal (v_cycle)");
    throw NumericError("coarsest operator is singular beyond translations (v_cycle)");
  }
  for (int k = 0; k < G; ++k) rn[k] = act[k] ? std::sqrt(h_pinned_[k]) : 0.0;
}

template <typename T>
void Hierarchy<T>::solve_bound_group(int G, double* const* u, const SolverOptions& opts, const ZLink<double>* ul,
                                     SolveStats* st) {
  if (!density_set_) throw StateError("set_density before solve");
  if (!pair_ok(opts)) throw std::logic_error("lockstep group solve needs mixed precision, mixed_defect and an even grid");
  if (G < 1 || G > kMaxRhsGroup) throw std::invalid_argument("right-hand-side group size must be in [1, 6]");
  ensure_group(G);
  Level& L0 = levels_[0];
  const long long n0 = 3 * L0.g.nv;
  bool act[kMaxRhsGroup] = {}, negligible[kMaxRhsGroup] = {};
  auto any = [&] {
    for (int k = 0; k < G; ++k)
      if (act[k]) return true;
    return false;
  };
  try {
    for (int k = 0; k < G; ++k) {  // src/multigrid.cpp:474-501 prologue, per RHS
      select_rhs(k);
      if (slab_.on() && is_self(ul[k], u[k])) throw std::invalid_argument("z-slab solve needs the links of the bound field");
      st[k] = SolveStats{};
      u0_bound_ = u[k];
      u0l_ = resolve(ul[k], u[k]);
      u_home_ = u[k];
      u_home_l_ = u0l_;
      fnorm0_ = project_norm0(L0.f.p);
      if (fnorm0_ <= negligible_load(n0)) {
        IHOM_CUDA(cudaMemsetAsync(u[k], 0, sizeof(double) * n0, s_));
        st[k].converged = true;
        negligible[k] = true;
        continue;
      }
      st[k].rel_residual = defect_residual() / fnorm0_;
      act[k] = st[k].rel_residual > opts.tol && st[k].cycles < opts.max_cycles;
    }
    const bool deferred = fast_ok(L0.g);  // the group's outer steps back to back, one read-back per round
    while (any()) {
      inner_vcycle_group(G, opts, act);
      double rn[kMaxRhsGroup] = {};
      if (deferred) {
        finish_defect_cycles(G, act, rn);
      } else {
        for (int k = 0; k < G; ++k)
          if (act[k]) {
            select_rhs(k);
            rn[k] = finish_defect_cycle();
            check_error("v_cycle");
          }
      }
      for (int k = 0; k < G; ++k)
        if (act[k]) {
          select_rhs(k);
          st[k].rel_residual = fnorm0_ > 0.0 ? rn[k] / fnorm0_ : 0.0;
          ++st[k].cycles;
          act[k] = st[k].rel_residual > opts.tol && st[k].cycles < opts.max_cycles;
        }
    }
    for (int k = 0; k < G; ++k) {  // epilogue per RHS, as solve_bound
      if (negligible[k]) continue;
      select_rhs(k);
      st[k].converged = st[k].rel_residual <= opts.tol;
      if (u0_bound_ != u[k]) {  // the fused update left the result in the other buffer
        remove_translations_to(u0_bound_, u[k], 0);
        u0_bound_ = u[k];
        u0l_ = u_home_l_;
      } else {
        remove_translations(u[k], 0);
      }
    }
  } catch (...) {
    for (int k = 0; k < G; ++k) {
      try {
        select_rhs(k);
        restore_home();
      } catch (...) {
      }
      u0_bound_ = nullptr;
      u_home_ = nullptr;
    }
    select_rhs(0);
    throw;
  }
  for (int k = 0; k < G; ++k) {
    select_rhs(k);
    u0_bound_ = nullptr;
    u_home_ = nullptr;
  }
  select_rhs(0);
}

template <typename T>
SolveStats Hierarchy<T>::solve_bound(double* u, const SolverOptions& opts, ZLink<double> ul) {  // src/multigrid.cpp:474-501
  if (!density_set_) throw StateError("set_density before solve");
  if (slab_.on() && is_self(ul, u)) throw std::invalid_argument("z-slab solve needs the links of the bound field");
  u0_bound_ = u;
  u0l_ = resolve(ul, u);
  u_home_ = u;
  u_home_l_ = u0l_;
  Level& L0 = levels_[0];
  const long long n0 = 3 * L0.g.nv;
  SolveStats st;
  try {
    fnorm0_ = project_norm0(L0.f.p);
    if (fnorm0_ <= negligible_load(n0)) {
      IHOM_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * n0, s_));
      st.converged = true;
      u0_bound_ = nullptr;
      return st;
    }
    if (opts.mode == kPCG) {
      st = solve_pcg(u, opts);
      remove_translations(u, 0);
      u0_bound_ = nullptr;
      return st;
    }
    if (opts.mode == kMixedDefect && std::is_same_v<T, float> && fast_ok(L0.g)) {
      ensure_inner();
      st.rel_residual = defect_residual() / fnorm0_;  // ef0 now holds the inner right-hand side
    } else {
      compute_residual(0);
      st.rel_residual = norm(L0.r.p, n0) / fnorm0_;
      if (opts.mode == kMixedDefect && std::is_same_v<T, float>) {
        ensure_inner();
        launch_convert<double, float>(L0.r.p, L0.ef.p, n0, s_);
      }
    }
    while (st.rel_residual > opts.tol && st.cycles < opts.max_cycles) {
      st.rel_residual = v_cycle(opts);
      ++st.cycles;
    }
    st.converged = st.rel_residual <= opts.tol;
    if (u0_bound_ != u) {  // the fused update left the result in the other buffer
      remove_translations_to(u0_bound_, u, 0);
      u0_bound_ = u;
      u0l_ = u_home_l_;
    } else {
      remove_translations(u, 0);
    }
  } catch (...) {
    try {
      restore_home();
    } catch (...) {
    }
    u0_bound_ = nullptr;
    u_home_ = nullptr;
    throw;
  }
  u0_bound_ = nullptr;
  u_home_ = nullptr;
  return st;
}

template <typename T>
void Hierarchy<T>::bench_op(const std::string& op, int reps) {
  if (!density_set_) throw StateError("set_density before bench_op");
  const bool f32 = op.find("_f32") != std::string::npos;
  if (f32 && !std::is_same_v<T, float>) throw std::invalid_argument("f32 inner kernels exist in mixed precision only");
  if (f32) ensure_inner();
  const int lmax = num_levels() - 1;
  for (int r = 0; r < reps; ++r) {
    if (op == "l0_gs_f64") relax(0, 1);
    else if (op == "l0_gs_f32") relax_f32(0, 1);
    else if (op == "l0_residual_f64") compute_residual(0);
    else if (op == "l0_residual_f32") residual_f32(0);
    else if (op == "l0_defect_f64") {  // fused f64 defect residual + f32 rhs + norm (mixed_defect outer step)
      ensure_inner();
      defect_residual();
    }
    else if (op == "l1_gs_f64" && lmax >= 1) relax(1, 1);
    else if (op == "l1_gs_f32" && lmax >= 1) relax_f32(1, 1);
    else if (op == "l1_residual_f64" && lmax >= 1) compute_residual(1);
    else if (op == "l1_residual_f32" && lmax >= 1) residual_f32(1);
    else if (op == "vcycle_f64" || op == "vcycle_f32") {
      SolverOptions o;
      o.mode = f32 ? kMixedDefect : kVCycle;
      v_cycle(o);
    } else if (op == "set_density") {
      // Galerkin rebuild from the current coefficients (coeff kernel skipped)
      if (levels_.size() > 1) {
        {
          ProfScope p(s_, "galerkin_l1", double(levels_[0].g.nv) * sizeof(T) + double(levels_[1].g.nv) * 243.0 * sizeof(T));
          launch_galerkin_from_elements<T>(levels_[0].g, levels_[1].g, coeff_.p, levels_[1].st.p, s_);
        }
        for (size_t l = 2; l < levels_.size(); ++l) {
          ProfScope p(s_, "galerkin_coarse", double(levels_[l - 1].g.nv + levels_[l].g.nv) * 243.0 * sizeof(T));
          launch_galerkin_from_stencil<T>(levels_[l - 1].g, levels_[l].g, levels_[l - 1].st.p, levels_[l].st.p, s_);
        }
      }
    } else {
      throw std::invalid_argument("unknown bench op: " + op);
    }
  }
  IHOM_CUDA(cudaStreamSynchronize(s_));
}

// ============================================================== Homogenizer
namespace {
int lean_request(const SolverOptions& opts) {  // Hierarchy lean argument from the U_HOST knob
  const int k = knob("U_HOST", 0);
  if (k < 0 || opts.mode != kMixedDefect) return 0;
  return k == 0 ? 1 : 2;
}
}  // namespace

template <typename T>
Homogenizer<T>::Homogenizer(const int n[3], const Material& mat, double penal, const SolverOptions& opts,
                            cudaStream_t s, Slab slab)
    : hier_(n, mat, penal, s, slab, lean_request(opts)), opts_(opts), penal_(penal) {
  const long long nv = hier_.geo(0).nv;
  rho_.alloc(size_t(nv));
  seed_.alloc(36);
  if (hier_.lean()) {
    host_u_ = knob("U_HOST", 0) == 1 ? 1 : 2;
    const size_t n3 = size_t(3 * nv);
    for (int i = 0; i < 6; ++i) {
      IHOM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hu32_[size_t(i)]), sizeof(float) * n3));
      std::memset(hu32_[size_t(i)], 0, sizeof(float) * n3);
      if (host_u_ == 2) {
        IHOM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hu64_[size_t(i)]), sizeof(double) * n3));
        std::memset(hu64_[size_t(i)], 0, sizeof(double) * n3);
      }
    }
    hier_.ensure_inner();
    IHOM_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
    IHOM_CUDA(cudaEventCreateWithFlags(&ev_solved_, cudaEventDisableTiming));
    IHOM_CUDA(cudaEventCreateWithFlags(&ev_staged_out_, cudaEventDisableTiming));
    IHOM_CUDA(cudaEventRecord(ev_staged_out_, cs_));
    for (auto& e : ev_back_) IHOM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    float* u0 = reinterpret_cast<float*>(hier_.level_u(0));
    float* f0 = reinterpret_cast<float*>(hier_.level_f(0));
    // snapshots 4 and 5 go last, into f0: the last solve's write-back still reads f0 (ensure_snapshots)
    snap_ = {u0, u0 + n3, hier_.inner_e(0), hier_.inner_f(0), f0, f0 + n3};
    for (int i = 0; i < 6; ++i) snapl_[size_t(i)] = hier_.link(snap_[size_t(i)]);  // collective on z-slabs
    IHOM_CUDA(cudaStreamSynchronize(s));
    return;
  }
  for (auto& u : u_) {
    u.alloc(size_t(3 * nv));
    IHOM_CUDA(cudaMemsetAsync(u.p, 0, sizeof(double) * 3 * nv, s));
  }
  IHOM_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < 6; ++i) ul_[size_t(i)] = hier_.link(u_[size_t(i)].p);  // collective on z-slabs
}

template <typename T>
Homogenizer<T>::~Homogenizer() {
  hier_.quiesce();
  try {
    join_conversions();
  } catch (...) {
  }
  for (cudaEvent_t e : ev_back_)
    if (e) cudaEventDestroy(e);
  if (cs_) {
    cudaStreamSynchronize(cs_);
    cudaStreamDestroy(cs_);
  }
  if (ev_solved_) cudaEventDestroy(ev_solved_);
  if (ev_staged_out_) cudaEventDestroy(ev_staged_out_);
  for (float* p : hu32_)
    if (p) cudaFreeHost(p);
  for (double* p : hu64_)
    if (p) cudaFreeHost(p);
}

template <typename T>
void Homogenizer<T>::join_conversions() {
  for (auto& c : conv_)
    if (c.valid()) c.get();
}

// f32 snapshot of field i from its f64 host copy once the write-back (ev) has landed; round to nearest
// like the device conversion. Eight host threads.
static void convert_snapshot(cudaEvent_t ev, int dev, const double* src, float* dst, long long n) {
  IHOM_CUDA(cudaSetDevice(dev));
  IHOM_CUDA(cudaEventSynchronize(ev));
  constexpr int kThreads = 8;
  std::vector<std::thread> pool;
  for (int t = 0; t < kThreads; ++t)
    pool.emplace_back([=] {
      const long long a = n * t / kThreads, b = n * (t + 1) / kThreads;
      for (long long k = a; k < b; ++k) dst[k] = float(src[k]);
    });
  for (auto& th : pool) th.join();
}

template <typename T>
void Homogenizer<T>::read_displacement(int i, double* dst) {
  const long long n3 = 3 * hier_.geo(0).nv;
  cudaStream_t s = hier_.stream();
  if (cs_) IHOM_CUDA(cudaStreamSynchronize(cs_));  // the last write-back has landed
  if (host_u_ == 2) {
    IHOM_CUDA(cudaMemcpyAsync(dst, hu64_[size_t(i)], sizeof(double) * n3, cudaMemcpyHostToDevice, s));
  } else if (host_u_ == 1) {
    std::vector<double> w(static_cast<size_t>(n3));
    for (long long k = 0; k < n3; ++k) w[size_t(k)] = double(hu32_[size_t(i)][k]);
    IHOM_CUDA(cudaMemcpyAsync(dst, w.data(), sizeof(double) * n3, cudaMemcpyHostToDevice, s));
  } else {
    IHOM_CUDA(cudaMemcpyAsync(dst, u_[size_t(i)].p, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s));
  }
  IHOM_CUDA(cudaStreamSynchronize(s));
}

template <typename T>
void Homogenizer<T>::write_displacement(int i, const double* src) {
  const long long n3 = 3 * hier_.geo(0).nv;
  cudaStream_t s = hier_.stream();
  ecache_valid_ = false;  // cached energies no longer describe the fields
  if (!host_u_) {
    IHOM_CUDA(cudaMemcpyAsync(u_[size_t(i)].p, src, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    return;
  }
  IHOM_CUDA(cudaStreamSynchronize(cs_));
  join_conversions();
  std::vector<double> w;
  double* h = hu64_[size_t(i)];
  if (!h) {
    w.resize(static_cast<size_t>(n3));
    h = w.data();
  }
  IHOM_CUDA(cudaMemcpyAsync(h, src, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
  IHOM_CUDA(cudaStreamSynchronize(s));
  for (long long k = 0; k < n3; ++k) hu32_[size_t(i)][k] = float(h[k]);  // round to nearest, as the device cast
  snaps_ready_ = false;
}

// The six cell problems with host-staged displacements: one device working field (level-0 u), the warm
// start staged in and the result (and its f32 snapshot) staged out around each solve; then the snapshots
// are placed in the level-0 buffers for the C^H / sensitivity passes. Same solves, same order, same
// arithmetic as the device-resident loop with group size 1 (bitwise equal displacements in mode 2).
// PCIe duplex: solve i's write-back (from the inner residual e_r0 and, mode 2, an f64 copy in f0, both
// free until the next macro force) runs on the copy stream while solve i+1's warm start comes in.
template <typename T>
CellSolveStats Homogenizer<T>::solve_host_staged() {
  if (comm_ && comm_->size() > 1) throw std::invalid_argument("host-staged displacements and the load-case split are exclusive");
  if (opts_.mode != kMixedDefect) throw StateError("host-staged displacements need the mixed_defect solver");
  const long long nv = hier_.geo(0).nv, n3 = 3 * nv;
  cudaStream_t s = hier_.stream();
  snaps_ready_ = false;
  ecache_valid_ = false;
  double* u = hier_.level_u(0);
  double* f = hier_.level_f(0);
  const ZLink<double> ul = hier_.ulink(0);
  float* out32 = hier_.inner_r(0);  // f32 write-back staging (mode 1)
  float* in32 = hier_.inner_f(0);   // f32 warm-start staging (mode 1)
  int dev = 0;
  IHOM_CUDA(cudaGetDevice(&dev));
  join_conversions();  // the host copies are not being read any more
  CellSolveStats out;
  for (int i = 0; i < 6; ++i) {
    hier_.sync();  // coefficients of the neighbouring slabs are current; nobody still reads u / e_r
    {
      ProfScope p(s, "host_stage", double(n3) * (host_u_ == 2 ? 8.0 : 4.0));
      if (host_u_ == 2) {
        IHOM_CUDA(cudaMemcpyAsync(u, hu64_[size_t(i)], sizeof(double) * n3, cudaMemcpyHostToDevice, s));
      } else {
        IHOM_CUDA(cudaMemcpyAsync(in32, hu32_[size_t(i)], sizeof(float) * n3, cudaMemcpyHostToDevice, s));
        launch_convert<float, double>(in32, u, n3, s);
      }
    }
    IHOM_CUDA(cudaStreamWaitEvent(s, ev_staged_out_, 0));  // f0 and e_r0 are read out
    hier_.macro_force(i);
    const SolveStats st = hier_.solve_bound(u, opts_, ul);
    hier_.sync();  // the neighbours' last halo reads of e_r0 are done
    {
      ProfScope p(s, "vector", double(n3) * (host_u_ == 2 ? 48.0 : 12.0));
      if (host_u_ == 2) IHOM_CUDA(cudaMemcpyAsync(f, u, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s));
      else launch_convert<double, float>(u, out32, n3, s);
    }
    IHOM_CUDA(cudaEventRecord(ev_solved_, s));
    IHOM_CUDA(cudaStreamWaitEvent(cs_, ev_solved_, 0));
    if (host_u_ == 2) {
      IHOM_CUDA(cudaMemcpyAsync(hu64_[size_t(i)], f, sizeof(double) * n3, cudaMemcpyDeviceToHost, cs_));
      IHOM_CUDA(cudaEventRecord(ev_back_[size_t(i)], cs_));
      conv_[size_t(i)] = std::async(std::launch::async, convert_snapshot, ev_back_[size_t(i)], dev,
                                    hu64_[size_t(i)], hu32_[size_t(i)], n3);
    } else {
      IHOM_CUDA(cudaMemcpyAsync(hu32_[size_t(i)], out32, sizeof(float) * n3, cudaMemcpyDeviceToHost, cs_));
    }
    IHOM_CUDA(cudaEventRecord(ev_staged_out_, cs_));
    out.total_cycles += st.cycles;  // combined in load order, exactly as the reference loop does
    if (st.rel_residual >= out.worst_residual) {
      out.worst_residual = st.rel_residual;
      out.worst_load = i;
    }
    if (!st.converged) out.converged = false;
  }
  ensure_snapshots();
  return out;
}

template <typename T>
void Homogenizer<T>::ensure_snapshots() {
  if (snaps_ready_) return;
  const long long n3 = 3 * hier_.geo(0).nv;
  cudaStream_t s = hier_.stream();
  hier_.sync();  // no slab still reads the level-0 buffers the snapshots overwrite
  {
    ProfScope p(s, "host_stage", double(n3) * 4.0 * 6.0);
    // snapshots 0-3 (written back before the last solve began) into u0 / e0 / f0-inner while the last
    // write-back (from f0 and e_r0 into hu32_[5]) may still run on the copy stream
    for (int i = 0; i < 6; ++i) {
      if (i == 4) IHOM_CUDA(cudaStreamWaitEvent(s, ev_staged_out_, 0));
      if (conv_[size_t(i)].valid()) conv_[size_t(i)].get();  // mode 2: the host-made snapshot is complete
      IHOM_CUDA(cudaMemcpyAsync(snap_[size_t(i)], hu32_[size_t(i)], sizeof(float) * n3, cudaMemcpyHostToDevice, s));
    }
  }
  hier_.sync();  // every slab's snapshots are in place before any reads a neighbour's top plane
  snaps_ready_ = true;
}

template <typename T>
void Homogenizer<T>::set_density(const double* rho) {  // src/homogenization.cpp:16-21
  IHOM_CUDA(cudaMemcpyAsync(rho_.p, rho, sizeof(double) * rho_.n, cudaMemcpyDeviceToDevice, hier_.stream()));
  hier_.set_density(rho_.p);
  density_set_ = true;
}

template <typename T>
CellSolveStats Homogenizer<T>::solve_cell_problems() {  // src/homogenization.cpp:23-40
  if (!density_set_) throw StateError("set_density before solve_cell_problems");
  if (host_u_) return solve_host_staged();
  const GridGeo& g = hier_.geo(0);
  const bool multi = comm_ && comm_->size() > 1;
  const bool slabs = hier_.slab().on();
  if (multi && slabs) throw std::invalid_argument("load-case split and z-slabs are exclusive");
  ecache_valid_ = false;
  double per[18] = {};  // per load: cycles, rel_residual, converged
  const int G = multi ? 1 : hier_.group_size(opts_);
  if (G > 1) {
    // loads in lockstep groups of G ((0,1), (2,3), (4,5) for pairs): each group streams the coarse
    // stencils once
    for (int i = 0; i < 6; i += G) {
      for (int k = 0; k < G; ++k) {
        hier_.select_rhs(k);
        hier_.sync();  // coefficients of the neighbouring slabs are current
        hier_.macro_force(i + k);
      }
      hier_.select_rhs(0);
      double* uu[kMaxRhsGroup];
      ZLink<double> ll[kMaxRhsGroup];
      for (int k = 0; k < G; ++k) uu[k] = u_[size_t(i + k)].p, ll[k] = ul_[size_t(i + k)];
      SolveStats st[kMaxRhsGroup];
      hier_.solve_bound_group(G, uu, opts_, ll, st);
      for (int k = 0; k < G; ++k) {
        per[3 * (i + k)] = st[k].cycles;
        per[3 * (i + k) + 1] = st[k].rel_residual;
        per[3 * (i + k) + 2] = st[k].converged ? 1.0 : 0.0;
      }
    }
  }
  for (int i = 0; i < 6 && G == 1; ++i) {
    if (multi && owner_[i] != comm_->rank()) continue;
    hier_.sync();  // coefficients of the neighbouring slabs are current
    hier_.macro_force(i);
    const SolveStats s = hier_.solve_bound(u_[size_t(i)].p, opts_, ul_[size_t(i)]);
    per[3 * i] = s.cycles;
    per[3 * i + 1] = s.rel_residual;
    per[3 * i + 2] = s.converged ? 1.0 : 0.0;
  }
  if (multi) {
    // every solved field from its owner to all ranks (NVLink), then one allreduce of the stats
    cudaStream_t s = hier_.stream();
    {
      ProfScope p(s, "nccl_broadcast", double(6 * 3 * g.nv * 8));
      comm_->group_start();
      for (int i = 0; i < 6; ++i) comm_->broadcast(u_[size_t(i)].p, size_t(3 * g.nv), owner_[i], s);
      comm_->group_end();
    }
    if (!stats_.p) stats_.alloc(18);
    IHOM_CUDA(cudaMemcpyAsync(stats_.p, per, sizeof(per), cudaMemcpyHostToDevice, s));
    comm_->allreduce_sum(stats_.p, 18, s);
    IHOM_CUDA(cudaMemcpyAsync(per, stats_.p, sizeof(per), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
  }
  CellSolveStats out;  // combined in load order, exactly as the reference loop does
  for (int i = 0; i < 6; ++i) {
    out.total_cycles += int(per[3 * i]);
    if (per[3 * i + 1] >= out.worst_residual) {
      out.worst_residual = per[3 * i + 1];
      out.worst_load = i;
    }
    if (per[3 * i + 2] == 0.0) out.converged = false;
  }
  return out;
}

template <typename T>
void Homogenizer<T>::effective_tensor(double C[36]) {  // src/homogenization.cpp:58-111
  Workspace& ws = hier_.workspace();
  const Material& m = hier_.material();
  const long long nv = hier_.geo(0).nv;
  if (host_u_) {  // f32 snapshots: the values the mixed mode rounds the f64 fields to (f64 energies)
    ensure_snapshots();
    const float* u[6];
    const float* uhi[6];
    for (int i = 0; i < 6; ++i) {
      u[i] = snap_[size_t(i)];
      uhi[i] = snapl_[size_t(i)].hi ? snapl_[size_t(i)].hi : u[i];
    }
    ProfScope p(hier_.stream(), "tensor", double(nv) * 80.0);
    launch_effective_tensor<float>(hier_.geo(0), u, rho_.p, penal_, true, m.lambda(), m.mu(), ws.partials,
                                   ws.scalars + 16, hier_.stream(), uhi, nullptr);
    ecache_valid_ = false;
  } else {
  const double* u[6];
  const double* uhi[6];
  for (int i = 0; i < 6; ++i) {
    u[i] = u_[size_t(i)].p;
    uhi[i] = ul_[size_t(i)].hi ? ul_[size_t(i)].hi : u[i];
  }
  hier_.sync();  // the six fields of the slab above are final
  const size_t esz = energy_f32(std::is_same_v<T, float>) ? sizeof(float) : sizeof(double);
  void* ec = nullptr;
  if (knob("ENERGY_CACHE", 1)) {
    if (!ecache_.p && !ecache_skip_) {
      // memory lever: the cache (21 energies per element) is an optimisation -- skip it when it would
      // leave less than 4 GB of HBM (the sensitivity pass then recomputes the energies)
      size_t free_b = 0, total_b = 0;
      IHOM_CUDA(cudaMemGetInfo(&free_b, &total_b));
      free_b = hbm_free_limit(free_b);
      if (double(free_b) >= double(21 * nv) * double(esz) + 4e9) ecache_.alloc(size_t(21 * nv) * esz);
      else ecache_skip_ = true;
    }
    ec = ecache_.p;
  }
  {
    ProfScope p(hier_.stream(), "tensor", double(nv) * (152.0 + (ec ? 21.0 * double(esz) : 0.0)));
    launch_effective_tensor<double>(hier_.geo(0), u, rho_.p, penal_, std::is_same_v<T, float>, m.lambda(), m.mu(),
                                    ws.partials, ws.scalars + 16, hier_.stream(), uhi, ec);
  }
  ecache_valid_ = ec != nullptr;
  }
  hier_.allreduce(ws.scalars + 16, 21);  // element sums over all slabs
  double c21[21];
  IHOM_CUDA(cudaMemcpyAsync(c21, ws.scalars + 16, sizeof(c21), cudaMemcpyDeviceToHost, hier_.stream()));
  IHOM_CUDA(cudaStreamSynchronize(hier_.stream()));
  const double M = double(hier_.global_nv(0));
  int q = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j, ++q) {
      C[i * 6 + j] = c21[q] / M;
      C[j * 6 + i] = C[i * 6 + j];
    }
}

template <typename T>
void Homogenizer<T>::tensor_sensitivity(const double seed[36], double* out) {  // src/homogenization.cpp:113-144
  double s[36];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) s[i * 6 + j] = 0.5 * (seed[i * 6 + j] + seed[j * 6 + i]);
  IHOM_CUDA(cudaMemcpyAsync(seed_.p, s, sizeof(s), cudaMemcpyHostToDevice, hier_.stream()));
  if (host_u_) {
    ensure_snapshots();
    const float* u[6];
    const float* uhi[6];
    for (int i = 0; i < 6; ++i) {
      u[i] = snap_[size_t(i)];
      uhi[i] = snapl_[size_t(i)].hi ? snapl_[size_t(i)].hi : u[i];
    }
    const Material& m = hier_.material();
    ProfScope p(hier_.stream(), "sensitivity", double(hier_.geo(0).nv) * 88.0);
    launch_tensor_sensitivity<float>(hier_.geo(0), u, rho_.p, penal_, true, m.lambda(), m.mu(), seed_.p, out,
                                     hier_.stream(), uhi, hier_.global_nv(0));
    IHOM_CUDA(cudaStreamSynchronize(hier_.stream()));
    return;
  }
  const double* u[6];
  const double* uhi[6];
  for (int i = 0; i < 6; ++i) {
    u[i] = u_[size_t(i)].p;
    uhi[i] = ul_[size_t(i)].hi ? ul_[size_t(i)].hi : u[i];
  }
  const Material& m = hier_.material();
  hier_.sync();
  if (ecache_valid_) {  // energies of the current displacements from effective_tensor()
    const long long nv = hier_.geo(0).nv;
    const bool f32 = energy_f32(std::is_same_v<T, float>);
    ProfScope p(hier_.stream(), "sensitivity", double(nv) * (21.0 * (f32 ? 4.0 : 8.0) + 16.0));
    launch_sensitivity_cached(nv, ecache_.p, f32, rho_.p, penal_, seed_.p, out, hier_.stream(), hier_.global_nv(0));
  } else {
    ProfScope p(hier_.stream(), "sensitivity", double(hier_.geo(0).nv) * 160.0);
    launch_tensor_sensitivity<double>(hier_.geo(0), u, rho_.p, penal_, std::is_same_v<T, float>, m.lambda(), m.mu(),
                                      seed_.p, out, hier_.stream(), uhi, hier_.global_nv(0));
  }
  IHOM_CUDA(cudaStreamSynchronize(hier_.stream()));
}

template class Hierarchy<float>;
template class Hierarchy<double>;
template class Homogenizer<float>;
template class Homogenizer<double>;

}  // namespace ihomgpu
