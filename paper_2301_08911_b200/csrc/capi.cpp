// capi.cpp -- the C ABI (include/ihom_b200.h) over the device hierarchy,
// homogenizer, design pipeline and the optimisation loop
// (src/runner.cpp:51-136). Exceptions map to status codes at this boundary.
#include "../../include/ihom_b200.h"

#include <chrono>
#include <cstdio>
#include <iterator>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "density.hpp"
#include "hierarchy.hpp"
#include "objective.hpp"
#include "profiler.hpp"

using namespace ihomgpu;

namespace {

thread_local std::string g_err;
// context whose constant tables this thread bound last (z-slab threads each bind
// their own context; the tables are per material, identical across slabs)
thread_local const void* g_bound = nullptr;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return IHOM_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return IHOM_E_INVALID;
  } catch (const NumericError& e) {
    g_err = e.what();
    return IHOM_E_NUMERIC;
  } catch (const EvalError& e) {
    g_err = e.what();
    return IHOM_E_EVAL;
  } catch (const CudaError& e) {
    g_err = e.what();
    return IHOM_E_CUDA;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return IHOM_E_STATE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return IHOM_E_INTERNAL;
  }
}

// Library stream for the context-free design-pipeline entry points.
cudaStream_t lib_stream() {
  static thread_local cudaStream_t s = nullptr;
  static thread_local int dev = -1;
  int cur = 0;
  IHOM_CUDA(cudaGetDevice(&cur));
  if (!s || dev != cur) {
    IHOM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    dev = cur;
  }
  return s;
}

struct Scratch {  // reduction workspace for context-free calls
  DevBuf<double> red;
  DevBuf<int> flag;
  Workspace ws;
  Scratch() : red(21 * kReducePartials + 128), flag(1) {
    ws.partials = red.p;
    ws.scalar = red.p + 21 * kReducePartials;
    ws.scalar2 = ws.scalar + 1;
    ws.scalars = ws.scalar + 8;
    ws.flag = flag.p;
  }
};

Scratch& scratch() {
  static thread_local std::unique_ptr<Scratch> s;
  if (!s) s = std::make_unique<Scratch>();
  return *s;
}

long long count(const int n[3]) {
  for (int k = 0; k < 3; ++k)
    if (n[k] < 1) throw std::invalid_argument("grid resolution must be positive");
  return (long long)n[0] * n[1] * n[2];
}

// Stages a host or device input array into device memory.
struct DevIn {
  DevBuf<double> own;
  const double* p = nullptr;
  DevIn(const double* src, size_t n, int where, cudaStream_t s) {
    if (where == IHOM_DEVICE) {
      p = src;
    } else {
      own.alloc(n);
      IHOM_CUDA(cudaMemcpyAsync(own.p, src, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      p = own.p;
    }
  }
};

// Device output: either the caller's device pointer or a staging buffer copied back on finish().
struct DevOut {
  DevBuf<double> own;
  double* p = nullptr;
  double* dst;
  size_t n;
  int where;
  DevOut(double* d, size_t count, int w) : dst(d), n(count), where(w) {
    if (w == IHOM_DEVICE) p = d;
    else {
      own.alloc(count);
      p = own.p;
    }
  }
  void finish(cudaStream_t s) {
    if (where != IHOM_DEVICE) IHOM_CUDA(cudaMemcpyAsync(dst, own.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
  }
};

}  // namespace

struct ihom_fabric {
  std::unique_ptr<Fabric> f;
};

struct ihom_ctx {
  std::unique_ptr<Comm> comm;
  int device = 0;
  cudaStream_t s = nullptr;
  int precision = IHOM_MIXED;
  int n[3] = {0, 0, 0};
  std::unique_ptr<Homogenizer<float>> hf;
  std::unique_ptr<Homogenizer<double>> hd;

  template <class F>
  void with(F&& f) {
    IHOM_CUDA(cudaSetDevice(device));
    if (g_bound != this) {
      if (hf) hf->hierarchy().bind_tables();
      else hd->hierarchy().bind_tables();
      g_bound = this;
    }
    if (hf) f(*hf);
    else f(*hd);
  }
  // vertices stored by this context (its z-slab's share of the grid)
  long long nv() const { return hf ? hf->nv() : hd->nv(); }
};

extern "C" {

const char* ihom_last_error(void) { return g_err.c_str(); }
const char* ihom_version(void) { return "ihom-b200 0.1 (sm_100a)"; }

static ihom_ctx* create_ctx(const ihom_desc* d, const ihom_solver_opts* o, Slab slab) {
  ihom_ctx* ctx = nullptr;
  const int rc = guarded([&] {
    if (!d) throw std::invalid_argument("null descriptor");
    auto c = std::make_unique<ihom_ctx>();
    c->device = d->device;
    IHOM_CUDA(cudaSetDevice(c->device));
    IHOM_CUDA(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
    c->precision = d->precision;
    for (int k = 0; k < 3; ++k) c->n[k] = d->n[k];
    Material m{d->youngs, d->poisson};
    validate_material(m);
    SolverOptions so;
    if (o) {
      so.tol = o->tol;
      so.max_cycles = o->max_cycles;
      so.pre_sweeps = o->pre_sweeps;
      so.post_sweeps = o->post_sweeps;
      so.mode = o->mode;
    }
    if (d->precision == IHOM_ALL_DOUBLE)
      c->hd = std::make_unique<Homogenizer<double>>(d->n, m, d->penal, so, c->s, slab);
    else if (d->precision == IHOM_MIXED)
      c->hf = std::make_unique<Homogenizer<float>>(d->n, m, d->penal, so, c->s, slab);
    else throw std::invalid_argument("precision must be IHOM_MIXED or IHOM_ALL_DOUBLE");
    g_bound = c.get();
    ctx = c.release();
  });
  return rc == IHOM_OK ? ctx : nullptr;
}

ihom_ctx* ihom_create(const ihom_desc* d, const ihom_solver_opts* o) { return create_ctx(d, o, Slab{}); }

ihom_ctx* ihom_create_slab(const ihom_desc* d, const ihom_solver_opts* o, ihom_fabric* f, int rank) {
  if (!f) {
    g_err = "null fabric";
    return nullptr;
  }
  return create_ctx(d, o, Slab{f->f.get(), rank, f->f->size()});
}

ihom_fabric* ihom_fabric_local(int nranks, int device) {
  ihom_fabric* out = nullptr;
  guarded([&] {
    auto f = std::make_unique<ihom_fabric>();
    f->f = std::make_unique<LocalFabric>(nranks, device);
    out = f.release();
  });
  return out;
}

ihom_fabric* ihom_fabric_ipc(int rank, int nranks, int device, ihom_allgather_fn ag, void* user) {
  ihom_fabric* out = nullptr;
  guarded([&] {
    auto f = std::make_unique<ihom_fabric>();
    f->f = std::make_unique<IpcFabric>(rank, nranks, device, reinterpret_cast<HostAllgather>(ag), user);
    out = f.release();
  });
  return out;
}

void ihom_fabric_destroy(ihom_fabric* f) { delete f; }

int ihom_slab_info(ihom_ctx* ctx, int* z0, int* planes, int* nranks) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      const Slab& sl = h.hierarchy().slab();
      const int t = h.hierarchy().geo(0).n[2];
      if (z0) *z0 = sl.rank * t;
      if (planes) *planes = t;
      if (nranks) *nranks = sl.nranks;
    });
  });
}

void ihom_destroy(ihom_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->s);
  if (g_bound == ctx) g_bound = nullptr;
  cudaStream_t s = ctx->s;
  delete ctx;
  cudaStreamDestroy(s);
}

int ihom_set_solver(ihom_ctx* ctx, const ihom_solver_opts* o) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      SolverOptions& so = h.options();
      so.tol = o->tol;
      so.max_cycles = o->max_cycles;
      so.pre_sweeps = o->pre_sweeps;
      so.post_sweeps = o->post_sweeps;
      so.mode = o->mode;
    });
  });
}

int ihom_set_comm(ihom_ctx* ctx, const void* uid128, int rank, int nranks, const int* owner6) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      if (nranks <= 1) {
        h.set_comm(nullptr, nullptr);
        ctx->comm.reset();
        return;
      }
      NcclUid id;
      std::memcpy(id.internal, uid128, sizeof(id.internal));
      ctx->comm = std::make_unique<Comm>(id, rank, nranks, ctx->device);
      h.set_comm(ctx->comm.get(), owner6);
    });
  });
}

int ihom_set_density(ihom_ctx* ctx, const double* rho, int where) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      DevIn in(rho, size_t(ctx->nv()), where, ctx->s);
      h.set_density(in.p);
      IHOM_CUDA(cudaStreamSynchronize(ctx->s));
    });
  });
}

int ihom_solve_cell_problems(ihom_ctx* ctx, ihom_cell_stats* st) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      const CellSolveStats s = h.solve_cell_problems();
      if (st) {
        st->total_cycles = s.total_cycles;
        st->worst_residual = s.worst_residual;
        st->worst_load = s.worst_load;
        st->converged = s.converged ? 1 : 0;
      }
    });
  });
}

int ihom_effective_tensor(ihom_ctx* ctx, double C[36]) {
  return guarded([&] { ctx->with([&](auto& h) { h.effective_tensor(C); }); });
}

int ihom_tensor_sensitivity(ihom_ctx* ctx, const double seed[36], double* out, int where) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      DevOut o(out, size_t(ctx->nv()), where);
      h.tensor_sensitivity(seed, o.p);
      o.finish(ctx->s);
    });
  });
}

int ihom_get_displacement(ihom_ctx* ctx, int load, double* u, int where) {
  return guarded([&] {
    if (load < 0 || load > 5) throw std::invalid_argument("load case must be in [0, 6)");
    ctx->with([&](auto& h) {
      DevOut o(u, size_t(3 * ctx->nv()), where);
      h.read_displacement(load, o.p);
      o.finish(ctx->s);
    });
  });
}

int ihom_set_displacement(ihom_ctx* ctx, int load, const double* u, int where) {
  return guarded([&] {
    if (load < 0 || load > 5) throw std::invalid_argument("load case must be in [0, 6)");
    ctx->with([&](auto& h) {
      DevIn in(u, size_t(3 * ctx->nv()), where, ctx->s);
      h.write_displacement(load, in.p);
    });
  });
}

int ihom_host_staged(ihom_ctx* ctx) {
  int v = -1;
  if (guarded([&] { ctx->with([&](auto& h) { v = h.host_staged(); }); }) != IHOM_OK) return -1;
  return v;
}

int ihom_num_levels(ihom_ctx* ctx) {
  int n = 0;
  if (guarded([&] { ctx->with([&](auto& h) { n = h.hierarchy().num_levels(); }); }) != IHOM_OK) return -1;
  return n;
}

int ihom_level_dims(ihom_ctx* ctx, int l, int n[3]) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      if (l < 0 || l >= h.hierarchy().num_levels()) throw std::invalid_argument("level out of range");
      for (int k = 0; k < 3; ++k) n[k] = h.hierarchy().geo(l).n[k];
    });
  });
}

int ihom_level_field(ihom_ctx* ctx, int l, int which, int write, double* buf) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      auto& H = h.hierarchy();
      if (l < 0 || l >= H.num_levels()) throw std::invalid_argument("level out of range");
      double* f = which == 0 ? H.level_u(l) : which == 1 ? H.level_f(l) : H.level_r(l);
      if (!f) throw StateError("this f64 level field is not allocated (lean layout)");
      const long long nv = H.geo(l).nv;
      if (write) {
        DevIn in(buf, size_t(3 * nv), IHOM_HOST, ctx->s);
        copy_nodal(in.p, f, nv, ctx->s);
        IHOM_CUDA(cudaStreamSynchronize(ctx->s));
      } else {
        DevOut o(buf, size_t(3 * nv), IHOM_HOST);
        copy_nodal(f, o.p, nv, ctx->s);
        o.finish(ctx->s);
      }
    });
  });
}

int ihom_apply(ihom_ctx* ctx, int l, const double* x, double* y) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      auto& H = h.hierarchy();
      if (l < 0 || l >= H.num_levels()) throw std::invalid_argument("level out of range");
      const long long nv = H.geo(l).nv;
      DevIn in(x, size_t(3 * nv), IHOM_HOST, ctx->s);
      DevBuf<double> xs(static_cast<size_t>(3 * nv)), ys(static_cast<size_t>(3 * nv));
      copy_nodal(in.p, xs.p, nv, ctx->s);
      H.apply(l, xs.p, ys.p);
      DevOut o(y, size_t(3 * nv), IHOM_HOST);
      copy_nodal(ys.p, o.p, nv, ctx->s);
      o.finish(ctx->s);
    });
  });
}

int ihom_relax(ihom_ctx* ctx, int l, int sweeps) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      h.hierarchy().relax(l, sweeps);
      IHOM_CUDA(cudaStreamSynchronize(ctx->s));
    });
  });
}

int ihom_compute_residual(ihom_ctx* ctx, int l) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      h.hierarchy().compute_residual(l);
      IHOM_CUDA(cudaStreamSynchronize(ctx->s));
    });
  });
}

int ihom_coarsest_solve(ihom_ctx* ctx) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      h.hierarchy().coarsest_solve();
      IHOM_CUDA(cudaStreamSynchronize(ctx->s));
    });
  });
}

int ihom_coarse_dense_solve(long long nv, const double* raw, const double* f, double* x, double* rel) {
  return guarded([&] {
    if (nv <= 0 || !raw || !f || !x) throw std::invalid_argument("coarse_dense_solve: null or empty input");
    const long long N = 3 * nv;
    std::vector<double> a(raw, raw + N * N), inv, q;
    int nq = 0;
    const double op_scale = factor_coarse_dense(a, nv, inv, &q, &nq);
    cudaStream_t s = nullptr;
    IHOM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DevBuf<double> dA, dInv, df, du, work, dQ;
    DevBuf<int> err;
    dA.alloc(a.size());
    dInv.alloc(inv.size());
    df.alloc(size_t(N));
    du.alloc(size_t(N));
    work.alloc(size_t(3 * N));
    err.alloc(1);
    IHOM_CUDA(cudaMemcpyAsync(dA.p, a.data(), sizeof(double) * a.size(), cudaMemcpyHostToDevice, s));
    IHOM_CUDA(cudaMemcpyAsync(dInv.p, inv.data(), sizeof(double) * inv.size(), cudaMemcpyHostToDevice, s));
    IHOM_CUDA(cudaMemcpyAsync(df.p, f, sizeof(double) * size_t(N), cudaMemcpyHostToDevice, s));
    IHOM_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), s));
    if (nq > 0) {
      dQ.alloc(q.size());
      IHOM_CUDA(cudaMemcpyAsync(dQ.p, q.data(), sizeof(double) * q.size(), cudaMemcpyHostToDevice, s));
    }
    launch_coarsest_solve<double>(int(N), nv, dInv.p, dA.p, dQ.p, nq, df.p, du.p,
                                  1e-12 * op_scale * std::sqrt(double(N)), work.p, err.p, s);
    int e = 0;
    std::vector<double> fp(static_cast<size_t>(N));
    IHOM_CUDA(cudaMemcpyAsync(x, du.p, sizeof(double) * size_t(N), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaMemcpyAsync(fp.data(), df.p, sizeof(double) * size_t(N), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaMemcpyAsync(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    IHOM_CUDA(cudaStreamDestroy(s));
    if (rel) {  // ||A x - f|| / ||f|| against the operator the solve used, f translation-free
      double rn = 0.0, fn = 0.0;
      for (long long i = 0; i < N; ++i) {
        double y = 0.0;
        for (long long j = 0; j < N; ++j) y += a[size_t(i * N + j)] * x[j];
        rn += (y - fp[size_t(i)]) * (y - fp[size_t(i)]);
        fn += fp[size_t(i)] * fp[size_t(i)];
      }
      *rel = fn > 0.0 ? std::sqrt(rn / fn) : 0.0;
    }
    if (e) throw NumericError("coarsest operator is singular beyond translations");
  });
}

int ihom_v_cycle(ihom_ctx* ctx, double* rel) {
  return guarded([&] { ctx->with([&](auto& h) { *rel = h.hierarchy().v_cycle(h.options()); }); });
}

int ihom_solve(ihom_ctx* ctx, const double* f, double* u, ihom_solve_stats* st) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      auto& H = h.hierarchy();
      const long long nv = H.geo(0).nv;
      DevIn fin(f, size_t(3 * nv), IHOM_HOST, ctx->s);
      copy_nodal(fin.p, H.level_f(0), nv, ctx->s);
      DevIn uin(u, size_t(3 * nv), IHOM_HOST, ctx->s);
      DevBuf<double> us(static_cast<size_t>(3 * nv));
      copy_nodal(uin.p, us.p, nv, ctx->s);
      const SolveStats s = H.solve_bound(us.p, h.options());
      DevOut o(u, size_t(3 * nv), IHOM_HOST);
      copy_nodal(us.p, o.p, nv, ctx->s);
      o.finish(ctx->s);
      if (st) {
        st->cycles = s.cycles;
        st->rel_residual = s.rel_residual;
        st->converged = s.converged ? 1 : 0;
      }
    });
  });
}

int ihom_get_stencil(ihom_ctx* ctx, int l, double* out) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      using T = typename std::remove_reference_t<decltype(h.hierarchy())>::value_type;
      auto& H = h.hierarchy();
      if (l < 1 || l >= H.num_levels()) throw std::invalid_argument("level has no assembled stencil");
      const long long nv = H.geo(l).nv;
      std::vector<T> st(stencil_alloc(nv));
      IHOM_CUDA(cudaMemcpyAsync(st.data(), H.stencil(l), sizeof(T) * st.size(), cudaMemcpyDeviceToHost, ctx->s));
      IHOM_CUDA(cudaStreamSynchronize(ctx->s));
      for (long long v = 0; v < nv; ++v)
        for (int k = 0; k < 243; ++k) out[v * 243 + k] = double(st[st_index(k, (unsigned)v)]);
    });
  });
}

int ihom_get_coeff(ihom_ctx* ctx, double* out) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      using T = typename std::remove_reference_t<decltype(h.hierarchy())>::value_type;
      std::vector<T> c(size_t(ctx->nv()));
      IHOM_CUDA(cudaMemcpyAsync(c.data(), h.hierarchy().coeff(), sizeof(T) * c.size(), cudaMemcpyDeviceToHost, ctx->s));
      IHOM_CUDA(cudaStreamSynchronize(ctx->s));
      for (size_t i = 0; i < c.size(); ++i) out[i] = double(c[i]);
    });
  });
}

int ihom_macro_force(ihom_ctx* ctx, int load, double* f) {
  return guarded([&] {
    if (load < 0 || load > 5) throw std::invalid_argument("macro strain index must be in [0, 6)");
    ctx->with([&](auto& h) {
      auto& H = h.hierarchy();
      const long long nv = H.geo(0).nv;
      DevBuf<double> fs(static_cast<size_t>(3 * nv));
      launch_macro_force(H.geo(0), H.coeff(), load, fs.p, ctx->s);
      DevOut o(f, size_t(3 * nv), IHOM_HOST);
      copy_nodal(fs.p, o.p, nv, ctx->s);
      o.finish(ctx->s);
    });
  });
}

double ihom_op_scale(ihom_ctx* ctx) {
  double v = 0.0;
  guarded([&] { ctx->with([&](auto& h) { v = h.hierarchy().op_scale(); }); });
  return v;
}

long long ihom_kernel_launches(ihom_ctx* ctx) {
  long long v = 0;
  guarded([&] { ctx->with([&](auto& h) { v = h.hierarchy().launches(); }); });
  return v;
}

int ihom_grid_locs(const int n[3], long long* locs, long long* nbr27) {
  return guarded([&] {
    const long long m = count(n);
    if (m >= (1LL << 31)) throw std::invalid_argument("grid too large");
    const GridGeo g = make_geo(n[0], n[1], n[2]);
    cudaStream_t s = lib_stream();
    DevBuf<long long> d(static_cast<size_t>(m)), d27(nbr27 ? size_t(27 * m) : 0);
    launch_grid_locs(g, d.p, nbr27 ? d27.p : nullptr, s);
    IHOM_CUDA(cudaMemcpyAsync(locs, d.p, sizeof(long long) * m, cudaMemcpyDeviceToHost, s));
    if (nbr27) IHOM_CUDA(cudaMemcpyAsync(nbr27, d27.p, sizeof(long long) * 27 * m, cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"

namespace {
template <typename TN>
void transfer_typed(const GridGeo& gf, const GridGeo& gc, int dir, const double* in, double* out, cudaStream_t s) {
  const long long nf = 3 * gf.nv, nc = 3 * gc.nv;
  const long long nin = dir == 0 ? nf : nc, nout = dir == 0 ? nc : nf;
  std::vector<TN> hin(in, in + nin), hout(out, out + nout);
  DevBuf<TN> din(static_cast<size_t>(nin)), dout(static_cast<size_t>(nout));
  IHOM_CUDA(cudaMemcpyAsync(din.p, hin.data(), sizeof(TN) * nin, cudaMemcpyHostToDevice, s));
  IHOM_CUDA(cudaMemcpyAsync(dout.p, hout.data(), sizeof(TN) * nout, cudaMemcpyHostToDevice, s));
  if (dir == 0) launch_restrict<TN>(gf, gc, din.p, dout.p, s);
  else launch_prolong_add<TN>(gc, gf, din.p, dout.p, s);
  IHOM_CUDA(cudaMemcpyAsync(hout.data(), dout.p, sizeof(TN) * nout, cudaMemcpyDeviceToHost, s));
  IHOM_CUDA(cudaStreamSynchronize(s));
  for (long long i = 0; i < nout; ++i) out[i] = double(hout[size_t(i)]);
}
}  // namespace

extern "C" {

int ihom_transfer(const int nf[3], int dir, int f32, const double* in, double* out) {
  return guarded([&] {
    if (nf[0] % 2 || nf[1] % 2 || nf[2] % 2) throw std::invalid_argument("transfer needs an even fine grid");
    if (dir != 0 && dir != 1) throw std::invalid_argument("transfer direction must be 0 (restrict) or 1 (prolong)");
    const GridGeo gf = make_geo(nf[0], nf[1], nf[2]), gc = make_geo(nf[0] / 2, nf[1] / 2, nf[2] / 2);
    if (f32) transfer_typed<float>(gf, gc, dir, in, out, lib_stream());
    else transfer_typed<double>(gf, gc, dir, in, out, lib_stream());
  });
}

// ------------------------------------------------------------------ design pipeline
int ihom_radial_filter(const int n[3], const double* f, double radius, int kernel, double* out, int where) {
  return guarded([&] {
    const long long m = count(n);
    cudaStream_t s = lib_stream();
    DevIn in(f, size_t(m), where, s);
    DevOut o(out, size_t(m), where);
    radial_filter(n, in.p, radius, kernel, o.p, s);
    o.finish(s);
  });
}

int ihom_density_expr_eval(const int n[3], double radius, int kernel, double exponent, const double* design,
                           double* phys, double* pre_out, int where) {
  return guarded([&] {
    const long long m = count(n);
    cudaStream_t s = lib_stream();
    DevIn in(design, size_t(m), where, s);
    DevOut pre(pre_out, size_t(m), pre_out ? where : IHOM_HOST);
    if (!pre_out) pre.dst = nullptr;
    radial_filter(n, in.p, radius >= 1.0 ? radius : 0.0, kernel, pre.p, s);  // src/density.cpp:65-72
    DevOut o(phys, size_t(m), where);
    pow_field(pre.p, exponent, m, o.p, s);
    o.finish(s);
    if (pre_out) pre.finish(s);
  });
}

int ihom_density_expr_backward(const int n[3], double radius, int kernel, double exponent, const double* pre,
                               const double* g_phys, double* g_design, int where) {
  return guarded([&] {
    const long long m = count(n);
    cudaStream_t s = lib_stream();
    DevIn p(pre, size_t(m), where, s);
    DevIn g(g_phys, size_t(m), where, s);
    DevBuf<double> tmp(static_cast<size_t>(m));
    pow_backward(p.p, g.p, exponent, m, tmp.p, s);  // src/density.cpp:74-83
    DevOut o(g_design, size_t(m), where);
    radial_filter(n, tmp.p, radius >= 1.0 ? radius : 0.0, kernel, o.p, s);
    o.finish(s);
  });
}

int ihom_symmetrize(const int n[3], double* field, int sym, int where) {
  return guarded([&] {
    const long long m = count(n);
    cudaStream_t s = lib_stream();
    DevOut o(field, size_t(m), where);
    if (where != IHOM_DEVICE) IHOM_CUDA(cudaMemcpyAsync(o.p, field, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    DevBuf<double> tmp(static_cast<size_t>(m));
    symmetrize(n, o.p, sym, tmp.p, s);
    o.finish(s);
  });
}

int ihom_field_mean(const double* f, long long m, double* mean, int where) {
  return guarded([&] {
    if (m <= 0) {
      *mean = 0.0;
      return;
    }
    cudaStream_t s = lib_stream();
    DevIn in(f, size_t(m), where, s);
    Scratch& sc = scratch();
    field_sum(in.p, m, sc.ws.partials, sc.ws.scalar, s);
    double sum = 0.0;
    IHOM_CUDA(cudaMemcpyAsync(&sum, sc.ws.scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    *mean = sum / double(m);
  });
}

int ihom_oc_update(long long m, const double* rho, const double* sens, const ihom_oc_config* cfg, double* out,
                   double* lambda, int* ok, int where) {
  return guarded([&] {
    if (m <= 0) throw std::invalid_argument("empty density field");
    if (out == rho || out == sens) throw std::invalid_argument("oc_update: out must not alias rho or sens");
    cudaStream_t s = lib_stream();
    DevIn r(rho, size_t(m), where, s);
    DevIn g(sens, size_t(m), where, s);
    DevOut o(out, size_t(m), where);
    OCConfig c;
    if (cfg) {
      c.min_density = cfg->min_density;
      c.step_limit = cfg->step_limit;
      c.damp = cfg->damp;
      c.volume = cfg->volume;
      c.bisect_tol = cfg->bisect_tol;
    }
    const OCResult res = oc_update(m, r.p, g.p, c, o.p, scratch().ws, s);
    o.finish(s);
    if (lambda) *lambda = res.lambda;
    if (ok) *ok = res.bisection_ok ? 1 : 0;
  });
}

int ihom_sensitivity_filter(const int n[3], const double* sens, const double* rho, double radius, double* out,
                            int where) {
  return guarded([&] {
    const long long m = count(n);
    cudaStream_t s = lib_stream();
    DevIn g(sens, size_t(m), where, s);
    DevIn r(rho, size_t(m), where, s);
    DevOut o(out, size_t(m), where);
    sensitivity_filter(n, g.p, r.p, radius, o.p, s);
    o.finish(s);
  });
}

int ihom_init_trig(const int n[3], int basis_n, uint64_t seed, double volume, double sigmoid_k, double* rho,
                   int* fallback) {
  return guarded([&] {
    const long long m = count(n);
    cudaStream_t s = lib_stream();
    DevBuf<double> d(static_cast<size_t>(m)), y(static_cast<size_t>(m));
    const bool fb = init_trig(n, basis_n, seed, volume, sigmoid_k, d.p, y.p, scratch().ws, s);
    IHOM_CUDA(cudaMemcpyAsync(rho, d.p, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    if (fallback) *fallback = fb ? 1 : 0;
  });
}

int ihom_objective(int obj, double beta, double eta, double tau, double gamma, int iter, const double C[36],
                   double* value, double grad[36]) {
  return guarded([&] {
    const Objective e = obj == IHOM_OBJ_BULK    ? bulk_objective()
             : obj == IHOM_OBJ_SHEAR ? shear_objective()
             : obj == IHOM_OBJ_NPR_RELAXED ? npr_relaxed(beta, iter)
             : obj == IHOM_OBJ_NPR_LOG     ? npr_log(eta, tau, gamma)
                                           : throw std::invalid_argument("unknown objective");
    *value = e.eval(C);
    if (grad) e.grad(1.0, C, grad);
  });
}

}  // extern "C"

// ------------------------------------------------------------------ optimisation loop
namespace {

Objective make_objective(const ihom_run_config& c, int iter) {  // src/runner.cpp:13-21
  switch (c.obj) {
    case IHOM_OBJ_BULK: return bulk_objective();
    case IHOM_OBJ_SHEAR: return shear_objective();
    case IHOM_OBJ_NPR_RELAXED: return npr_relaxed(c.beta, iter);
    case IHOM_OBJ_NPR_LOG: return npr_log(c.eta, c.tau, c.gamma);
    default: throw std::invalid_argument("unknown objective");
  }
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

struct OptBase {
  virtual ~OptBase() = default;
  // status: 0 updated, 1 solver failed, 2 converged (no update), 3 last iteration (no update)
  virtual int step(ihom_iter_record* rec) = 0;
  virtual double* design() = 0;
  virtual double* prev_design() = 0;
  virtual long long count() const = 0;
  virtual long long launches() = 0;
  virtual cudaStream_t stream() const = 0;
  virtual void bind() = 0;
  virtual void set_comm(Comm* c, const int* owner) = 0;
  std::unique_ptr<Comm> comm;
  int flags = 0;
  int iter = 0;
  bool done = false;
};

// One optimisation iteration per step(), exactly the loop body of
// src/runner.cpp:83-131 (the loop itself is ihom_run_optimization or the
// caller driving ihom_opt_step).
template <typename T>
struct Optimizer : OptBase {
  ihom_run_config cfg;
  int n[3];
  int nl[3];            // this slab's dims (n0, n1, t); == n on one domain
  long long m;          // elements held here
  long long m_total;    // elements of the whole grid
  Slab slab;
  std::map<const double*, ZLink<double>> zlinks;  // z-slab: design buffers on the slabs below / above
  std::map<const double*, PeerTable> peers;       //         and on every slab
  cudaStream_t s = nullptr;
  std::unique_ptr<Homogenizer<T>> hom;
  DevBuf<double> rho, next, pre, phys, grad, tmp, gd;
  bool dfilt = false;
  OCConfig oc;
  ConvergeChecker conv;

  Optimizer(const ihom_run_config& c, const double* init_rho, Slab sl = {}) : cfg(c), slab(sl) {
    IHOM_CUDA(cudaSetDevice(cfg.device));
    if (cfg.reso < 4) throw std::invalid_argument("grid resolution must be >= 4 per axis");
    if (!(cfg.vol > 0.0 && cfg.vol <= 1.0)) throw std::invalid_argument("volume fraction out of range");
    n[0] = n[1] = n[2] = cfg.reso;
    m_total = (long long)cfg.reso * cfg.reso * cfg.reso;
    nl[0] = n[0];
    nl[1] = n[1];
    nl[2] = slab.on() ? n[2] / slab.nranks : n[2];
    m = (long long)nl[0] * nl[1] * nl[2];
    IHOM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SolverOptions so;
    so.tol = cfg.tol;
    so.max_cycles = cfg.max_cycles;
    so.mode = cfg.solver_mode;
    // homogenizer penal = 1: the SIMP power lives in DensityExpr (src/runner.cpp:59-62)
    hom = std::make_unique<Homogenizer<T>>(n, Material{cfg.youngs, cfg.poisson}, 1.0, so, s, slab);
    g_bound = this;
    for (DevBuf<double>* b : {&rho, &next, &pre, &phys, &grad, &tmp, &gd}) b->alloc(size_t(m));
    IHOM_CUDA(cudaDeviceSynchronize());
    if (slab.on())  // collective, same order on every slab
      for (DevBuf<double>* b : {&rho, &next, &pre, &phys, &grad, &tmp, &gd}) {
        const std::vector<void*> all = slab.fab->exchange(slab.rank, b->p);
        zlinks[b->p] = neighbours<double>(all, slab.rank);
        peers[b->p] = peer_table(all);
      }
    Workspace& ws = hom->hierarchy().workspace();
    if (cfg.init == 0) {  // init_constant (src/density.cpp:261-265)
      std::vector<double> v(size_t(m), cfg.vol);
      IHOM_CUDA(cudaMemcpyAsync(rho.p, v.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s));
      IHOM_CUDA(cudaStreamSynchronize(s));
    } else if (cfg.init == 1) {
      if (init_trig(n, cfg.basis_n, cfg.seed, cfg.vol, 15.0, rho.p, tmp.p, ws, s, slab)) flags |= 4;
    } else {
      if (!init_rho) throw std::invalid_argument("init from file requires init_rho");
      IHOM_CUDA(cudaMemcpyAsync(rho.p, init_rho, sizeof(double) * m, cudaMemcpyHostToDevice, s));
      clamp_field(rho.p, m, kRhoMin, 1.0, s);  // src/runner.cpp:38-42
    }
    if (cfg.sym != IHOM_SYM_NONE) {  // src/runner.cpp:66-69
      sym(rho.p, tmp.p);
      clamp_field(rho.p, m, kRhoMin, 1.0, s);
    }
    IHOM_CUDA(cudaMemcpyAsync(next.p, rho.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    dfilt = cfg.filter_placement == 0 && cfg.filter_radius >= 1.0;
    oc.volume = cfg.vol;
    oc.step_limit = cfg.step;
    oc.damp = cfg.damp;
  }
  ~Optimizer() override {
    hom.reset();
    if (g_bound == this) g_bound = nullptr;
    if (s) cudaStreamDestroy(s);
  }
  void bind() override {
    IHOM_CUDA(cudaSetDevice(cfg.device));
    if (g_bound != this) {
      hom->hierarchy().bind_tables();
      g_bound = this;
    }
  }
  double* design() override { return rho.p; }
  double* prev_design() override { return next.p; }
  long long count() const override { return m; }
  long long launches() override { return hom->hierarchy().launches(); }
  cudaStream_t stream() const override { return s; }
  void set_comm(Comm* c, const int* owner) override { hom->set_comm(c, owner); }

  double mean_of(const double* f) {
    Workspace& ws = hom->hierarchy().workspace();
    field_sum(f, m, ws.partials, ws.scalar, s, slab);
    double sum = 0.0;
    IHOM_CUDA(cudaMemcpyAsync(&sum, ws.scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
    IHOM_CUDA(cudaStreamSynchronize(s));
    return sum / double(m_total);
  }
  ZLink<double> zl(const double* p) const {
    auto it = zlinks.find(p);
    return it == zlinks.end() ? ZLink<double>{} : it->second;
  }
  void sym(double* field, double* scratch) {
    if (slab.on()) symmetrize_slab(n, slab, field, peers.at(field), scratch, peers.at(scratch), cfg.sym, s);
    else symmetrize(n, field, cfg.sym, scratch, s);
  }

  int step(ihom_iter_record* out) override {
    if (done) throw StateError("optimisation already finished");
    const auto t0 = std::chrono::steady_clock::now();
    Workspace& ws = hom->hierarchy().workspace();
    // DensityExpr::eval (src/density.cpp:65-72)
    // knob PHASE_PROF: whole-phase event pairs ("phase:*" families, overlapping the kernel families) to
    // locate host-side gaps; off in the bench
    const bool ph = knob("PHASE_PROF", 0) != 0;
    auto phase = [&](const char* name) { return ProfScope(s, ph ? name : nullptr, 0.0); };
    slab.sync(s);  // neighbours' designs are current
    CellSolveStats st;
    ihom_iter_record rec{};
    {
      auto p0 = phase("phase:density_eval");
      radial_filter(nl, rho.p, dfilt ? cfg.filter_radius : 0.0, cfg.kernel, pre.p, s, zl(rho.p));
      pow_field(pre.p, cfg.penal, m, phys.p, s);
    }
    {
      auto p1 = phase("phase:set_density");
      hom->set_density(phys.p);
    }
    {
      auto p2 = phase("phase:solve");
      st = hom->solve_cell_problems();
    }
    {
      auto p3 = phase("phase:tensor");
      hom->effective_tensor(rec.C);
    }
    const Objective objective = make_objective(cfg, iter);
    const double fval = objective.eval(rec.C);
    rec.iter = iter;
    rec.objective = fval;
    rec.volume = mean_of(rho.p);
    rec.cycles = st.total_cycles;
    rec.residual = st.worst_residual;
    rec.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    int status = 0;
    if (!st.converged) {  // src/runner.cpp:105-113
      flags |= 1;
      status = 1;
    } else if (conv.update(fval)) {
      flags |= 2;
      status = 2;
    } else if (iter + 1 == cfg.max_iter) {
      status = 3;
    }
    if (status == 0) {
      auto p4 = phase("phase:sens_filter_oc");
      double seed[36];
      objective.grad(1.0, rec.C, seed);
      hom->tensor_sensitivity(seed, grad.p);
      pow_backward(pre.p, grad.p, cfg.penal, m, tmp.p, s);  // DensityExpr::backward
      slab.sync(s);
      radial_filter(nl, tmp.p, dfilt ? cfg.filter_radius : 0.0, cfg.kernel, gd.p, s, zl(tmp.p));
      if (cfg.filter_placement == 1 && cfg.filter_radius >= 1.0) {
        slab.sync(s);
        sensitivity_filter(nl, gd.p, rho.p, cfg.filter_radius, tmp.p, s, zl(gd.p), zl(rho.p));
        slab.sync(s);
        IHOM_CUDA(cudaMemcpyAsync(gd.p, tmp.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
      }
      if (cfg.sym != IHOM_SYM_NONE) sym(gd.p, tmp.p);
      const OCResult res = oc_update(m, rho.p, gd.p, oc, next.p, ws, s, slab, m_total);
      if (!res.bisection_ok) flags |= 8;
      std::swap(rho.p, next.p);  // previous design now in next.p
      if (cfg.sym != IHOM_SYM_NONE) {
        sym(rho.p, tmp.p);
        clamp_field(rho.p, m, kRhoMin, 1.0, s);
      }
      rec.lambda = res.lambda;
      rec.oc_trials = res.trials;
      IHOM_CUDA(cudaStreamSynchronize(s));
    } else {
      done = true;
    }
    ++iter;
    if (out) *out = rec;
    return status;
  }
};

}  // namespace

extern "C" {

int ihom_run_optimization(const ihom_run_config* cfg, const double* init_rho, ihom_iter_record* records, int capacity,
                          int* nrec, double* rho_out, int* flags, ihom_observer obs, void* user) {
  return guarded([&] {
    if (!cfg) throw std::invalid_argument("null config");
    std::unique_ptr<OptBase> o;
    if (cfg->precision == IHOM_ALL_DOUBLE) o = std::make_unique<Optimizer<double>>(*cfg, init_rho);
    else o = std::make_unique<Optimizer<float>>(*cfg, init_rho);
    *nrec = 0;
    std::vector<double> h_prev, h_next;
    const long long m = o->count();
    for (int it = 0; it < cfg->max_iter; ++it) {  // src/runner.cpp:83-132
      ihom_iter_record rec{};
      const int status = o->step(&rec);
      if (*nrec < capacity) records[(*nrec)++] = rec;
      if (status != 0) break;
      if (obs) {
        h_prev.resize(size_t(m));
        h_next.resize(size_t(m));
        IHOM_CUDA(cudaMemcpyAsync(h_prev.data(), o->prev_design(), sizeof(double) * m, cudaMemcpyDeviceToHost, o->stream()));
        IHOM_CUDA(cudaMemcpyAsync(h_next.data(), o->design(), sizeof(double) * m, cudaMemcpyDeviceToHost, o->stream()));
        IHOM_CUDA(cudaStreamSynchronize(o->stream()));
        if (!obs(it, h_prev.data(), h_next.data(), &rec, user)) break;
      }
    }
    if (rho_out) {
      IHOM_CUDA(cudaMemcpyAsync(rho_out, o->design(), sizeof(double) * m, cudaMemcpyDeviceToHost, o->stream()));
      IHOM_CUDA(cudaStreamSynchronize(o->stream()));
    }
    *flags = o->flags;
  });
}

struct ihom_opt {
  std::unique_ptr<OptBase> o;
};

ihom_opt* ihom_opt_create_slab(const ihom_run_config* cfg, const double* init_rho, ihom_fabric* f, int rank) {
  ihom_opt* out = nullptr;
  guarded([&] {
    if (!cfg) throw std::invalid_argument("null config");
    if (!f) throw std::invalid_argument("null fabric");
    const Slab sl{f->f.get(), rank, f->f->size()};
    auto h = std::make_unique<ihom_opt>();
    if (cfg->precision == IHOM_ALL_DOUBLE) h->o = std::make_unique<Optimizer<double>>(*cfg, init_rho, sl);
    else h->o = std::make_unique<Optimizer<float>>(*cfg, init_rho, sl);
    out = h.release();
  });
  return out;
}

ihom_opt* ihom_opt_create(const ihom_run_config* cfg, const double* init_rho) {
  ihom_opt* out = nullptr;
  const int rc = guarded([&] {
    if (!cfg) throw std::invalid_argument("null config");
    auto h = std::make_unique<ihom_opt>();
    if (cfg->precision == IHOM_ALL_DOUBLE) h->o = std::make_unique<Optimizer<double>>(*cfg, init_rho);
    else h->o = std::make_unique<Optimizer<float>>(*cfg, init_rho);
    out = h.release();
  });
  return rc == IHOM_OK ? out : nullptr;
}

void ihom_opt_destroy(ihom_opt* h) { delete h; }

int ihom_opt_step(ihom_opt* h, const double* rho_in, double* rho_out, int where, ihom_iter_record* rec, int* status) {
  return guarded([&] {
    OptBase& o = *h->o;
    o.bind();
    const long long m = o.count();
    const cudaMemcpyKind kin = where == IHOM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (rho_in) IHOM_CUDA(cudaMemcpyAsync(o.design(), rho_in, sizeof(double) * m, kin, o.stream()));
    const int st = o.step(rec);
    if (status) *status = st;
    if (rho_out) {
      const cudaMemcpyKind kout = where == IHOM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
      IHOM_CUDA(cudaMemcpyAsync(rho_out, o.design(), sizeof(double) * m, kout, o.stream()));
    }
    IHOM_CUDA(cudaStreamSynchronize(o.stream()));
  });
}

int ihom_opt_design(ihom_opt* h, double* out, int where) {
  return guarded([&] {
    OptBase& o = *h->o;
    const cudaMemcpyKind k = where == IHOM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    IHOM_CUDA(cudaMemcpyAsync(out, o.design(), sizeof(double) * o.count(), k, o.stream()));
    IHOM_CUDA(cudaStreamSynchronize(o.stream()));
  });
}

int ihom_nccl_unique_id(void* out128) {
  return guarded([&] {
    const NcclUid id = Comm::unique_id();
    std::memcpy(out128, id.internal, sizeof(id.internal));
  });
}

int ihom_opt_set_comm(ihom_opt* h, const void* uid128, int rank, int nranks, const int* owner6) {
  return guarded([&] {
    OptBase& o = *h->o;
    o.bind();
    if (nranks <= 1) {
      o.set_comm(nullptr, nullptr);
      o.comm.reset();
      return;
    }
    NcclUid id;
    std::memcpy(id.internal, uid128, sizeof(id.internal));
    int dev = 0;
    IHOM_CUDA(cudaGetDevice(&dev));
    o.comm = std::make_unique<Comm>(id, rank, nranks, dev);
    o.set_comm(o.comm.get(), owner6);
  });
}

int ihom_opt_flags(ihom_opt* h) { return h->o->flags; }
long long ihom_opt_launches(ihom_opt* h) { return h->o->launches(); }
void* ihom_opt_stream(ihom_opt* h) { return (void*)h->o->stream(); }

int ihom_set_knob(const char* name, int value) {
  return guarded([&] {
    if (!name) throw std::invalid_argument("knob name");
    set_knob(name, value);
  });
}
int ihom_get_knob(const char* name, int dflt) { return name ? knob(name, dflt) : dflt; }

int ihom_profile_enable(int on) {
  return guarded([&] {
    Profiler::get().enable(on != 0);
    if (on) Profiler::get().reset();
  });
}

int ihom_profile_get(int index, char* family, int cap, long long* launches, double* ms, double* bytes) {
  int rc = guarded([&] {
    const auto& t = Profiler::get().totals();
    if (index < 0 || index >= (int)t.size()) throw std::invalid_argument("profile index out of range");
    auto it = t.begin();
    std::advance(it, index);
    std::snprintf(family, size_t(cap), "%s", it->first.c_str());
    *launches = it->second.launches;
    *ms = it->second.ms;
    *bytes = it->second.bytes;
  });
  return rc;
}

long long ihom_launch_count(void) { return launch_counter(); }

int ihom_bench_op(ihom_ctx* ctx, const char* op, int reps) {
  return guarded([&] {
    ctx->with([&](auto& h) {
      const std::string o(op);
      if (o == "tensor" || o == "sensitivity") {
        for (int r = 0; r < reps; ++r) {
          if (o == "tensor") {
            double C[36];
            h.effective_tensor(C);
          } else {
            double seed[36] = {};
            for (int i = 0; i < 6; ++i) seed[i * 6 + i] = 1.0;
            DevBuf<double> out(static_cast<size_t>(ctx->nv()));
            h.tensor_sensitivity(seed, out.p);
          }
        }
      } else {
        h.hierarchy().bench_op(o, reps);
      }
    });
  });
}

int ihom_profile_count(void) {
  int n = 0;
  guarded([&] { n = (int)Profiler::get().totals().size(); });
  return n;
}

}  // extern "C"
