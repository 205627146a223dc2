"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for
  * ``libihom_oracle.so``: the Eigen-free C++ restatement of the reference hot
    path (``oracle/ihom_oracle.cpp``, every function cites the reference
    file:line it follows), and
  * ``_ref/libihom_ref.so``: the reference's own ``src/density.cpp`` +
    ``src/oc.cpp`` compiled unmodified from ``/root/reference`` (present only
    where that tree exists; the GPU box gets the prebuilt copy).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package, and only as the checker/baseline.
The product path (``paper_2301_08911_b200``) never touches it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libihom_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libihom_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_longlong)


def build() -> None:
    """Compile the oracle (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a: np.ndarray):
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.int32:
        return a.ctypes.data_as(_ip)
    if a.dtype == np.int64:
        return a.ctypes.data_as(_lp)
    raise TypeError(a.dtype)


class OracleError(RuntimeError):
    pass


class OrcRunConfig(C.Structure):
    _fields_ = [
        ("reso", C.c_int), ("vol", C.c_double), ("youngs", C.c_double), ("poisson", C.c_double),
        ("obj", C.c_int), ("beta", C.c_double), ("eta", C.c_double), ("tau", C.c_double),
        ("gamma", C.c_double), ("penal", C.c_double), ("filter_radius", C.c_double),
        ("filter_placement", C.c_int), ("kernel", C.c_int), ("sym", C.c_int), ("init", C.c_int),
        ("basis_n", C.c_int), ("seed", C.c_ulonglong), ("max_iter", C.c_int), ("step", C.c_double),
        ("damp", C.c_double), ("tol", C.c_double), ("max_cycles", C.c_int), ("mixed", C.c_int),
    ]


class OrcIterRecord(C.Structure):
    _fields_ = [("iter", C.c_int), ("objective", C.c_double), ("volume", C.c_double),
                ("cycles", C.c_int), ("residual", C.c_double), ("ms", C.c_double),
                ("C", C.c_double * 36)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_hom_create.restype = C.c_void_p
        L.orc_hom_create.argtypes = [C.c_int] * 3 + [C.c_double] * 3 + [C.c_int, C.c_double, C.c_int]
        for name in ("orc_hom_destroy",):
            getattr(L, name).argtypes = [C.c_void_p]
        for name in ("orc_hom_set_density", "orc_hom_solve", "orc_hom_tensor", "orc_hom_sensitivity",
                     "orc_hom_get_u", "orc_hom_set_u", "orc_hom_num_levels", "orc_hom_get_stencil",
                     "orc_hom_level_field", "orc_hom_vcycle", "orc_hom_relax", "orc_hom_residual",
                     "orc_hom_coarsest_solve", "orc_hom_hsolve"):
            getattr(L, name).restype = C.c_int
        L.orc_hom_op_scale.restype = C.c_double
        L.orc_hom_op_scale.argtypes = [C.c_void_p]
        L.orc_field_mean.restype = C.c_double
        L.orc_field_mean.argtypes = [_dp, C.c_longlong]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The reference's own density/OC code (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise OracleError("oracle/_ref/libihom_ref.so not built (reference tree absent)")
        R = C.CDLL(REF_PATH)
        R.ref_field_mean.restype = C.c_double
        _ref = R
    return _ref


def _check(rc: int):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise OracleError(msg)


def set_threads(n: int) -> int:
    return lib().orc_set_threads(int(n))


def set_coarse_project(on: bool) -> None:
    """Coarsest-operator translation projection (the one documented deviation; default on).
    False restores the reference's raw operator and its throw (src/multigrid.cpp:446-447)."""
    lib().orc_set_coarse_project(int(bool(on)))


def set_coarse_dump(path) -> None:
    """Write (raw operator, load) of the next failing coarsest solve to `path` (fixture generation)."""
    lib().orc_set_coarse_dump(None if path is None else str(path).encode())


def coarse_dense_solve(raw, f):
    """Coarsest-level dense solve of an assembled operator (dof order 3*loc+c): the hierarchy's
    factor_coarsest + coarsest_solve (src/multigrid.cpp:368-451) on a given matrix. Returns (x, rel)."""
    raw = np.ascontiguousarray(raw, np.float64)
    N = raw.shape[0]
    f = np.ascontiguousarray(f, np.float64).ravel()
    x = np.zeros(N)
    rel = C.c_double()
    _check(lib().orc_coarse_dense_solve(C.c_longlong(N // 3), _ptr(raw), _ptr(f), _ptr(x), C.byref(rel)))
    return x, rel.value


# ---------------------------------------------------------------- basics
def k0(E=1.0, nu=0.3) -> np.ndarray:
    out = np.zeros(576)
    _check(lib().orc_k0(C.c_double(E), C.c_double(nu), _ptr(out)))
    return out.reshape(24, 24)


def grid_info(n):
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    base = np.zeros(8, np.int64)
    dim = np.zeros(24, np.int32)
    _check(lib().orc_grid_info(nx, ny, nz, _ptr(base), _ptr(dim)))
    return base, dim.reshape(8, 3)


def grid_locs(n) -> np.ndarray:
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    out = np.zeros(nx * ny * nz, np.int64)
    _check(lib().orc_grid_locs(nx, ny, nz, _ptr(out)))
    return out


def fem_tables(E=1.0, nu=0.3):
    fm = np.zeros(144)
    ngb = np.zeros(64, np.int32)
    _check(lib().orc_fem_tables(C.c_double(E), C.c_double(nu), _ptr(fm), _ptr(ngb)))
    return fm.reshape(8, 6, 3), ngb.reshape(8, 8)


def _n3(n):
    return (int(n),) * 3 if np.isscalar(n) else tuple(int(v) for v in n)


def fem(n, which, coeff, u=None, f=None, E=1e6, nu=0.3, mixed=False, load=0):
    """which: 'apply' | 'residual' | 'gs' | 'macro'. Nodal AoS [nv,3] arrays."""
    nx, ny, nz = _n3(n)
    nv = nx * ny * nz
    code = {"apply": 0, "residual": 1, "gs": 2, "macro": 3}[which]
    coeff = np.ascontiguousarray(coeff, np.float64).ravel()
    u = np.zeros(3 * nv) if u is None else np.array(u, np.float64).ravel()
    f = np.zeros(3 * nv) if f is None else np.ascontiguousarray(f, np.float64).ravel()
    out = np.zeros(3 * nv)
    _check(lib().orc_fem(nx, ny, nz, C.c_double(E), C.c_double(nu), int(mixed), code, int(load),
                         _ptr(coeff), _ptr(u), _ptr(f), _ptr(out)))
    return (u if which == "gs" else out).reshape(nv, 3)


def restrict(n, fine):
    nx, ny, nz = _n3(n)
    fine = np.ascontiguousarray(fine, np.float64).ravel()
    out = np.zeros(3 * (nx // 2) * (ny // 2) * (nz // 2))
    _check(lib().orc_restrict(nx, ny, nz, _ptr(fine), _ptr(out)))
    return out.reshape(-1, 3)


def prolong_add(n, coarse, fine):
    nx, ny, nz = _n3(n)
    coarse = np.ascontiguousarray(coarse, np.float64).ravel()
    fine = np.array(fine, np.float64).ravel()
    _check(lib().orc_prolong_add(nx, ny, nz, _ptr(coarse), _ptr(fine)))
    return fine.reshape(-1, 3)


class Homogenizer:
    """Oracle twin of ihom::Homogenizer<T> (inc/homogenization.hpp:26-51)."""

    def __init__(self, n, E=1e6, nu=0.3, penal=3.0, mixed=False, tol=1e-2, max_cycles=50):
        self.n = _n3(n)
        self.nv = int(np.prod(self.n))
        self.h = lib().orc_hom_create(*self.n, C.c_double(E), C.c_double(nu), C.c_double(penal),
                                      int(mixed), C.c_double(tol), int(max_cycles))
        if not self.h:
            raise ValueError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_hom_destroy(C.c_void_p(self.h))
            self.h = None

    def _h(self):
        return C.c_void_p(self.h)

    def set_density(self, rho):
        rho = np.ascontiguousarray(rho, np.float64).ravel()
        _check(lib().orc_hom_set_density(self._h(), _ptr(rho), C.c_longlong(rho.size)))

    def solve_cell_problems(self):
        tc, wl, cv = C.c_int(), C.c_int(), C.c_int()
        wr = C.c_double()
        _check(lib().orc_hom_solve(self._h(), C.byref(tc), C.byref(wr), C.byref(wl), C.byref(cv)))
        return dict(total_cycles=tc.value, worst_residual=wr.value, worst_load=wl.value,
                    converged=bool(cv.value))

    def effective_tensor(self):
        out = np.zeros(36)
        _check(lib().orc_hom_tensor(self._h(), _ptr(out)))
        return out.reshape(6, 6)

    def tensor_sensitivity(self, seed):
        seed = np.ascontiguousarray(seed, np.float64).ravel()
        out = np.zeros(self.nv)
        _check(lib().orc_hom_sensitivity(self._h(), _ptr(seed), _ptr(out)))
        return out

    def displacement(self, i):
        out = np.zeros(3 * self.nv)
        _check(lib().orc_hom_get_u(self._h(), int(i), _ptr(out)))
        return out.reshape(-1, 3)

    def set_displacement(self, i, u):
        u = np.ascontiguousarray(u, np.float64).ravel()
        _check(lib().orc_hom_set_u(self._h(), int(i), _ptr(u)))

    def num_levels(self):
        return lib().orc_hom_num_levels(self._h())

    def stencil(self, l):
        nl = tuple(x >> l for x in self.n)
        out = np.zeros(243 * int(np.prod(nl)))
        _check(lib().orc_hom_get_stencil(self._h(), int(l), _ptr(out)))
        return out.reshape(-1, 27, 3, 3)

    def level_field(self, l, which, value=None):
        """which: 'u' | 'f' | 'r'; read (value None) or write."""
        nl = tuple(x >> l for x in self.n)
        w = {"u": 0, "f": 1, "r": 2}[which]
        if value is None:
            out = np.zeros(3 * int(np.prod(nl)))
            _check(lib().orc_hom_level_field(self._h(), int(l), w, 0, _ptr(out)))
            return out.reshape(-1, 3)
        buf = np.ascontiguousarray(value, np.float64).ravel().copy()
        _check(lib().orc_hom_level_field(self._h(), int(l), w, 1, _ptr(buf)))

    def v_cycle(self):
        rel = C.c_double()
        _check(lib().orc_hom_vcycle(self._h(), C.byref(rel)))
        return rel.value

    def relax(self, l, sweeps=1):
        _check(lib().orc_hom_relax(self._h(), int(l), int(sweeps)))

    def compute_residual(self, l):
        _check(lib().orc_hom_residual(self._h(), int(l)))

    def coarsest_solve(self):
        _check(lib().orc_hom_coarsest_solve(self._h()))

    def solve(self, f, u):
        f = np.ascontiguousarray(f, np.float64).ravel()
        u = np.array(u, np.float64).ravel()
        cyc, cv = C.c_int(), C.c_int()
        rel = C.c_double()
        _check(lib().orc_hom_hsolve(self._h(), _ptr(f), _ptr(u), C.byref(cyc), C.byref(rel), C.byref(cv)))
        return u.reshape(-1, 3), dict(cycles=cyc.value, rel_residual=rel.value, converged=bool(cv.value))

    def op_scale(self):
        return lib().orc_hom_op_scale(self._h())


# ---------------------------------------------------------------- density
def field_mean(f):
    f = np.ascontiguousarray(f, np.float64).ravel()
    return lib().orc_field_mean(_ptr(f), C.c_longlong(f.size))


def radial_filter(n, f, radius=2.0, kernel="spline4"):
    nx, ny, nz = _n3(n)
    f = np.ascontiguousarray(f, np.float64).ravel()
    out = np.zeros_like(f)
    _check(lib().orc_radial_filter(nx, ny, nz, _ptr(f), C.c_double(radius),
                                   0 if kernel == "linear" else 1, _ptr(out)))
    return out


SYM = {"none": 0, "reflect3": 1, "reflect6": 2, "rotate3": 3}
OBJ = {"bulk": 0, "shear": 1, "npr-relaxed": 2, "npr_relaxed": 2, "npr-log": 3, "npr_log": 3}


def symmetrize(n, f, sym="reflect6"):
    nx, ny, nz = _n3(n)
    f = np.array(f, np.float64).ravel()
    _check(lib().orc_symmetrize(nx, ny, nz, _ptr(f), SYM[sym]))
    return f


def init_trig(n, basis_n=2, seed=0, volume=0.3, sigmoid_k=15.0):
    nx, ny, nz = _n3(n)
    rho = np.zeros(nx * ny * nz)
    fb = C.c_int()
    _check(lib().orc_init_trig(nx, ny, nz, int(basis_n), C.c_ulonglong(seed), C.c_double(volume),
                               C.c_double(sigmoid_k), _ptr(rho), C.byref(fb)))
    return rho, bool(fb.value)


def oc_update(rho, sens, volume=0.3, step=0.05, damp=0.5, min_density=1e-3, bisect_tol=1e-6):
    rho = np.ascontiguousarray(rho, np.float64).ravel()
    sens = np.ascontiguousarray(sens, np.float64).ravel()
    out = np.zeros_like(rho)
    lam = C.c_double()
    ok = C.c_int()
    _check(lib().orc_oc_update(C.c_longlong(rho.size), _ptr(rho), _ptr(sens), C.c_double(volume),
                               C.c_double(step), C.c_double(damp), C.c_double(min_density),
                               C.c_double(bisect_tol), _ptr(out), C.byref(lam), C.byref(ok)))
    return out, lam.value, bool(ok.value)


def sensitivity_filter(n, sens, rho, radius):
    nx, ny, nz = _n3(n)
    sens = np.ascontiguousarray(sens, np.float64).ravel()
    rho = np.ascontiguousarray(rho, np.float64).ravel()
    out = np.zeros_like(sens)
    _check(lib().orc_sensitivity_filter(nx, ny, nz, _ptr(sens), _ptr(rho), C.c_double(radius), _ptr(out)))
    return out


def objective(obj, C6, iter=0, beta=0.8, eta=0.6, tau=-1e-3, gamma=0.5):
    C6 = np.ascontiguousarray(C6, np.float64).ravel()
    val = C.c_double()
    g = np.zeros(36)
    _check(lib().orc_objective(OBJ[obj], C.c_double(beta), C.c_double(eta), C.c_double(tau),
                               C.c_double(gamma), int(iter), _ptr(C6), C.byref(val), _ptr(g)))
    return val.value, g.reshape(6, 6)


def run(reso=32, vol=0.2, obj="bulk", max_iter=5, mixed=True, tol=1e-2, max_cycles=50, init="trig",
        sym="reflect6", seed=0, basis_n=2, youngs=1e6, poisson=0.3, beta=0.8, eta=0.6, tau=-1e-3,
        gamma=0.5, penal=3.0, filter_radius=2.0, filter_placement="density", kernel="spline4",
        step=0.05, damp=0.5):
    """src/runner.cpp:51-136 restated. Returns (records list of dicts, final rho, flags dict)."""
    cfg = OrcRunConfig(reso, vol, youngs, poisson, OBJ[obj], beta, eta, tau, gamma, penal,
                       filter_radius, 0 if filter_placement == "density" else 1,
                       0 if kernel == "linear" else 1, SYM[sym], 0 if init == "constant" else 1,
                       basis_n, seed, max_iter, step, damp, tol, max_cycles, int(mixed))
    recs = (OrcIterRecord * max(1, max_iter))()
    nrec = C.c_int()
    rho = np.zeros(reso ** 3)
    flags = C.c_int()
    _check(lib().orc_run(C.byref(cfg), recs, C.byref(nrec), _ptr(rho), C.byref(flags)))
    out = []
    for r in recs[: nrec.value]:
        out.append(dict(iter=r.iter, objective=r.objective, volume=r.volume, cycles=r.cycles,
                        residual=r.residual, ms=r.ms, C=np.array(r.C[:]).reshape(6, 6)))
    fl = flags.value
    return out, rho, dict(solver_failed=bool(fl & 1), converged=bool(fl & 2),
                          init_fallback=bool(fl & 4), oc_warning=bool(fl & 8))
