"""paper_2301_08911_b200 -- B200-native inverse-homogenization hot path.

Python mirror of the reference C++ API (``/root/reference/proj/include/ihom``)
over the C ABI in ``include/ihom_b200.h``. Every heavy operation runs in
``libihom_b200.so`` (hand-written sm_100a CUDA kernels + C++ host
orchestration). There is no CPU fallback: importing works without a GPU, but
any compute call raises if the library or a CUDA device is missing.

Names follow the reference:
  Homogenizer(reso, mat, penal, opts)       inc/homogenization.hpp:26-51
  Homogenizer.hierarchy() -> Hierarchy       inc/multigrid.hpp:53-93
  radial_filter / DensityExpr / symmetrize   inc/density.hpp:36-69
  oc_update / sensitivity_filter / ConvergeChecker  inc/oc.hpp:10-61
  Expr + bulk/shear/npr objectives          inc/objective.hpp:19-66
  run_optimization(RunConfig, observer)      inc/runner.hpp:36-40
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
from typing import Callable, Optional

import numpy as np

from .expr import (ConvergeChecker, EvalError, Expr, bulk_objective, npr_log, npr_relaxed,  # noqa: F401
                   poisson_ratio_report, shear_objective)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libihom_b200.so")
kRhoMin = 0.001
kNumLoadCases = 6

IHOM_HOST, IHOM_DEVICE = 0, 1
PRECISION = {"mixed": 0, "double": 1, "all_double": 1}
SOLVER_MODE = {"vcycle": 0, "mixed_defect": 1, "pcg": 2}
SYMMETRY = {"none": 0, "reflect3": 1, "reflect6": 2, "rotate3": 3}
KERNEL = {"linear": 0, "spline4": 1}
OBJECTIVE = {"bulk": 0, "shear": 1, "npr-relaxed": 2, "npr_relaxed": 2, "npr-log": 3, "npr_log": 3}


class IhomError(RuntimeError):
    """Numerical failure (reference std::runtime_error)."""


class CudaError(RuntimeError):
    pass


def build() -> None:
    """Compile libihom_b200.so for sm_100a (nvcc) in-tree."""
    subprocess.run(["make", "-s", "-j8", "-C", HERE], check=True)


_dp = C.POINTER(C.c_double)
_lib = None


class _Desc(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("youngs", C.c_double), ("poisson", C.c_double), ("penal", C.c_double),
                ("precision", C.c_int), ("device", C.c_int)]


class _SolverOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_cycles", C.c_int), ("pre_sweeps", C.c_int),
                ("post_sweeps", C.c_int), ("mode", C.c_int)]


class _CellStats(C.Structure):
    _fields_ = [("total_cycles", C.c_int), ("worst_residual", C.c_double), ("worst_load", C.c_int),
                ("converged", C.c_int)]


class _SolveStats(C.Structure):
    _fields_ = [("cycles", C.c_int), ("rel_residual", C.c_double), ("converged", C.c_int)]


class _OCConfig(C.Structure):
    _fields_ = [("min_density", C.c_double), ("step_limit", C.c_double), ("damp", C.c_double),
                ("volume", C.c_double), ("bisect_tol", C.c_double)]


class _RunConfig(C.Structure):
    _fields_ = [("reso", C.c_int), ("vol", C.c_double), ("youngs", C.c_double), ("poisson", C.c_double),
                ("obj", C.c_int), ("beta", C.c_double), ("eta", C.c_double), ("tau", C.c_double),
                ("gamma", C.c_double), ("penal", C.c_double), ("filter_radius", C.c_double),
                ("filter_placement", C.c_int), ("kernel", C.c_int), ("sym", C.c_int), ("init", C.c_int),
                ("basis_n", C.c_int), ("seed", C.c_uint64), ("max_iter", C.c_int), ("step", C.c_double),
                ("damp", C.c_double), ("tol", C.c_double), ("max_cycles", C.c_int), ("precision", C.c_int),
                ("solver_mode", C.c_int), ("device", C.c_int)]


class _IterRecord(C.Structure):
    _fields_ = [("iter", C.c_int), ("objective", C.c_double), ("volume", C.c_double), ("cycles", C.c_int),
                ("residual", C.c_double), ("ms", C.c_double), ("C", C.c_double * 36), ("lambda_", C.c_double),
                ("oc_trials", C.c_int)]


_OBSERVER = C.CFUNCTYPE(C.c_int, C.c_int, _dp, _dp, C.POINTER(_IterRecord), C.c_void_p)


def lib():
    """Load the CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2301_08911_b200.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        L.ihom_last_error.restype = C.c_char_p
        L.ihom_version.restype = C.c_char_p
        L.ihom_create.restype = C.c_void_p
        L.ihom_create.argtypes = [C.POINTER(_Desc), C.POINTER(_SolverOpts)]
        L.ihom_destroy.argtypes = [C.c_void_p]
        L.ihom_op_scale.restype = C.c_double
        L.ihom_op_scale.argtypes = [C.c_void_p]
        L.ihom_kernel_launches.restype = C.c_longlong
        L.ihom_kernel_launches.argtypes = [C.c_void_p]
        L.ihom_num_levels.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def version() -> str:
    return lib().ihom_version().decode()


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ihom_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise IhomError(msg)
    if rc == 3:
        raise RuntimeError(msg)  # logic_error (call order)
    if rc == 5:
        raise EvalError(msg)
    if rc == 4:
        raise CudaError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------- buffers
def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _in(x, n=None):
    """Returns (pointer, where, keepalive) for a read-only f64 input."""
    if _is_torch_cuda(x):
        import torch
        assert x.dtype == torch.float64 and x.is_contiguous(), "device inputs must be contiguous float64"
        return C.cast(C.c_void_p(x.data_ptr()), _dp), IHOM_DEVICE, x
    a = np.ascontiguousarray(x, dtype=np.float64).ravel()
    if n is not None and a.size != n:
        raise ValueError(f"expected {n} values, got {a.size}")
    return a.ctypes.data_as(_dp), IHOM_HOST, a


def _out_like(x, n):
    if _is_torch_cuda(x):
        import torch
        out = torch.empty(n, dtype=torch.float64, device=x.device)
        return out, C.cast(C.c_void_p(out.data_ptr()), _dp), IHOM_DEVICE
    out = np.zeros(n)
    return out, out.ctypes.data_as(_dp), IHOM_HOST


def _n3(n):
    if np.isscalar(n):
        return (int(n),) * 3
    return tuple(int(v) for v in n)


# ---------------------------------------------------------------- material / options
@dataclasses.dataclass
class BaseMaterial:  # inc/material.hpp:17-35
    youngs: float = 1.0
    poisson: float = 0.3

    def __post_init__(self):
        if not self.youngs > 0.0:
            raise ValueError("Young's modulus must be positive")
        if not (-1.0 < self.poisson < 0.5):
            raise ValueError("Poisson's ratio must lie in (-1, 0.5)")

    def lam(self):
        return self.youngs * self.poisson / ((1.0 + self.poisson) * (1.0 - 2.0 * self.poisson))

    def mu(self):
        return self.youngs / (2.0 * (1.0 + self.poisson))

    def elasticity(self):
        l, m = self.lam(), self.mu()
        c = np.zeros((6, 6))
        c[:3, :3] = l
        for i in range(3):
            c[i, i] = l + 2 * m
            c[3 + i, 3 + i] = m
        return c


@dataclasses.dataclass
class SolverOptions:  # inc/multigrid.hpp:22-27
    tol: float = 1e-2
    max_cycles: int = 50
    pre_sweeps: int = 1
    post_sweeps: int = 1
    mode: str = "vcycle"

    def _c(self):
        return _SolverOpts(self.tol, self.max_cycles, self.pre_sweeps, self.post_sweeps, SOLVER_MODE[self.mode])


# ---------------------------------------------------------------- homogenizer
class Hierarchy:
    """View of the device hierarchy owned by a Homogenizer (inc/multigrid.hpp:53-93)."""

    def __init__(self, hom: "Homogenizer"):
        self._h = hom

    def _ctx(self):
        return self._h._ctx()

    def num_levels(self) -> int:
        return lib().ihom_num_levels(self._ctx())

    def level_dims(self, l):
        n = (C.c_int * 3)()
        _check(lib().ihom_level_dims(self._ctx(), int(l), n))
        return tuple(n)

    def _nv(self, l):
        return int(np.prod(self.level_dims(l)))

    def field(self, l, which):
        """Download level-l u/f/r as AoS [nv, 3] (reference NodalField layout)."""
        out = np.zeros(3 * self._nv(l))
        _check(lib().ihom_level_field(self._ctx(), int(l), {"u": 0, "f": 1, "r": 2}[which], 0,
                                      out.ctypes.data_as(_dp)))
        return out.reshape(-1, 3)

    def set_field(self, l, which, value):
        buf = np.ascontiguousarray(value, dtype=np.float64).ravel().copy()
        if buf.size != 3 * self._nv(l):
            raise ValueError("field size mismatch")
        _check(lib().ihom_level_field(self._ctx(), int(l), {"u": 0, "f": 1, "r": 2}[which], 1,
                                      buf.ctypes.data_as(_dp)))

    def apply(self, l, x):
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        y = np.zeros_like(x)
        _check(lib().ihom_apply(self._ctx(), int(l), x.ctypes.data_as(_dp), y.ctypes.data_as(_dp)))
        return y.reshape(-1, 3)

    def relax(self, l, sweeps=1):
        _check(lib().ihom_relax(self._ctx(), int(l), int(sweeps)))

    def compute_residual(self, l):
        _check(lib().ihom_compute_residual(self._ctx(), int(l)))

    def coarsest_solve(self):
        _check(lib().ihom_coarsest_solve(self._ctx()))

    def v_cycle(self) -> float:
        rel = C.c_double()
        _check(lib().ihom_v_cycle(self._ctx(), C.byref(rel)))
        return rel.value

    def solve(self, f, u):
        f = np.ascontiguousarray(f, dtype=np.float64).ravel()
        u = np.array(u, dtype=np.float64).ravel()
        st = _SolveStats()
        _check(lib().ihom_solve(self._ctx(), f.ctypes.data_as(_dp), u.ctypes.data_as(_dp), C.byref(st)))
        return u.reshape(-1, 3), dict(cycles=st.cycles, rel_residual=st.rel_residual, converged=bool(st.converged))

    def stencil(self, l):
        out = np.zeros(243 * self._nv(l))
        _check(lib().ihom_get_stencil(self._ctx(), int(l), out.ctypes.data_as(_dp)))
        return out.reshape(-1, 27, 3, 3)

    def coeff(self):
        out = np.zeros(self._nv(0))
        _check(lib().ihom_get_coeff(self._ctx(), out.ctypes.data_as(_dp)))
        return out

    def macro_force(self, load):
        out = np.zeros(3 * self._nv(0))
        _check(lib().ihom_macro_force(self._ctx(), int(load), out.ctypes.data_as(_dp)))
        return out.reshape(-1, 3)

    def op_scale(self) -> float:
        return lib().ihom_op_scale(self._ctx())

    def kernel_launches(self) -> int:
        return lib().ihom_kernel_launches(self._ctx())

    def bench_op(self, op: str, reps: int = 1):
        """Runs one kernel family reps times (see ihom_bench_op); time it with profile_enable/profile_totals."""
        _check(lib().ihom_bench_op(self._ctx(), op.encode(), int(reps)))


_ALLGATHER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class Fabric:
    """How the z-slabs of one grid reach each other (include/ihom_b200.h).

    Fabric.local(P): all P slabs in this process on one device, one host thread
    per slab (every slab call is collective: drive the slabs from P threads, see
    run_slabs). Fabric.ipc(rank, P, allgather): one slab per process; CUDA IPC
    handles travel through ``allgather(bytes) -> list[bytes]`` (e.g. built on
    torch.distributed), peers are read over NVLink.
    """

    def __init__(self, ptr, nranks, keep=None):
        if not ptr:
            _raise_last()
        self._p, self.nranks, self._keep = ptr, int(nranks), keep

    @staticmethod
    def local(nranks: int, device: int = 0) -> "Fabric":
        L = lib()
        L.ihom_fabric_local.restype = C.c_void_p
        L.ihom_fabric_local.argtypes = [C.c_int, C.c_int]
        return Fabric(L.ihom_fabric_local(int(nranks), int(device)), nranks)

    @staticmethod
    def ipc(rank: int, nranks: int, allgather: Callable, device: int = 0) -> "Fabric":
        def _cb(send, recv, nbytes, user):
            parts = allgather(C.string_at(send, nbytes))
            blob = b"".join(parts)
            C.memmove(recv, blob, len(blob))
        cb = _ALLGATHER_FN(_cb)
        L = lib()
        L.ihom_fabric_ipc.restype = C.c_void_p
        L.ihom_fabric_ipc.argtypes = [C.c_int, C.c_int, C.c_int, _ALLGATHER_FN, C.c_void_p]
        return Fabric(L.ihom_fabric_ipc(int(rank), int(nranks), int(device), cb, None), nranks, keep=cb)

    def close(self):
        if getattr(self, "_p", None):
            L = lib()
            L.ihom_fabric_destroy.argtypes = [C.c_void_p]
            L.ihom_fabric_destroy(C.c_void_p(self._p))
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_slabs(nranks: int, fn: Callable[[int], object]) -> list:
    """Runs fn(rank) for every slab of a local fabric in its own thread; returns the results by rank
    (re-raises the first exception). ctypes releases the GIL inside library calls."""
    import threading
    out, err = [None] * nranks, [None] * nranks

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


class Homogenizer:
    """Device twin of ihom::Homogenizer<T> (inc/homogenization.hpp:26-51).

    precision 'mixed' = Homogenizer<float> (f32 coefficients/stencils, f64 nodal);
    'double' = Homogenizer<double>. With ``fabric`` the context holds z-slab
    ``rank`` of the grid (planes [z0, z0 + planes)); densities and sensitivities
    are then that slab's elements and every call is collective over the slabs.
    """

    def __init__(self, reso, mat: BaseMaterial = None, penal: float = 3.0, opts: SolverOptions = None,
                 precision: str = "mixed", device: int = 0, fabric: Optional[Fabric] = None, rank: int = 0):
        mat = mat or BaseMaterial()
        opts = opts or SolverOptions()
        self.n = _n3(reso)
        self.mat, self.penal, self.precision, self._opts = mat, penal, precision, opts
        d = _Desc((C.c_int * 3)(*self.n), mat.youngs, mat.poisson, penal, PRECISION[precision], device)
        o = opts._c()
        if fabric is None:
            self._p = lib().ihom_create(C.byref(d), C.byref(o))
        else:
            L = lib()
            L.ihom_create_slab.restype = C.c_void_p
            L.ihom_create_slab.argtypes = [C.POINTER(_Desc), C.POINTER(_SolverOpts), C.c_void_p, C.c_int]
            self._p = L.ihom_create_slab(C.byref(d), C.byref(o), C.c_void_p(fabric._p), int(rank))
        if not self._p:
            _raise_last()
        self.fabric = fabric
        z0, t, P = C.c_int(), C.c_int(), C.c_int()
        L = lib()
        L.ihom_slab_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        _check(L.ihom_slab_info(self._ctx(), C.byref(z0), C.byref(t), C.byref(P)))
        self.z0, self.planes, self.nranks = z0.value, t.value, P.value
        self.nv = self.n[0] * self.n[1] * self.planes  # vertices / elements held by this context

    def _ctx(self):
        if not self._p:
            raise RuntimeError("homogenizer destroyed")
        return C.c_void_p(self._p)

    def close(self):
        if getattr(self, "_p", None):
            lib().ihom_destroy(C.c_void_p(self._p))
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def options(self) -> SolverOptions:
        return self._opts

    def set_options(self, opts: SolverOptions):
        self._opts = opts
        o = opts._c()
        _check(lib().ihom_set_solver(self._ctx(), C.byref(o)))

    def set_density(self, rho_phys):
        p, where, keep = _in(rho_phys, self.nv)
        _check(lib().ihom_set_density(self._ctx(), p, where))

    def solve_cell_problems(self):
        st = _CellStats()
        _check(lib().ihom_solve_cell_problems(self._ctx(), C.byref(st)))
        return dict(total_cycles=st.total_cycles, worst_residual=st.worst_residual, worst_load=st.worst_load,
                    converged=bool(st.converged))

    def effective_tensor(self) -> np.ndarray:
        c = (C.c_double * 36)()
        _check(lib().ihom_effective_tensor(self._ctx(), c))
        return np.array(c[:]).reshape(6, 6)

    def tensor_sensitivity(self, seed, out=None):
        seed = np.ascontiguousarray(seed, dtype=np.float64).ravel()
        if out is not None and _is_torch_cuda(out):
            ptr, where = C.cast(C.c_void_p(out.data_ptr()), _dp), IHOM_DEVICE
            res = out
        else:
            res = np.zeros(self.nv)
            ptr, where = res.ctypes.data_as(_dp), IHOM_HOST
        _check(lib().ihom_tensor_sensitivity(self._ctx(), seed.ctypes.data_as(_dp), ptr, where))
        return res

    def displacement(self, i) -> np.ndarray:
        out = np.zeros(3 * self.nv)
        _check(lib().ihom_get_displacement(self._ctx(), int(i), out.ctypes.data_as(_dp), IHOM_HOST))
        return out.reshape(-1, 3)

    def set_displacement(self, i, u):
        p, where, keep = _in(u, 3 * self.nv)
        _check(lib().ihom_set_displacement(self._ctx(), int(i), p, where))

    @property
    def host_staged(self) -> int:
        """Displacement storage: 0 device-resident f64, 2 pinned-host f64 + f32 evaluation snapshots,
        1 pinned-host f32 snapshots only (memory lever; knob U_HOST)."""
        v = lib().ihom_host_staged(self._ctx())
        if v < 0:
            raise IhomError(lib().ihom_last_error().decode())
        return v

    def hierarchy(self) -> Hierarchy:
        return Hierarchy(self)

    def set_comm(self, uid: bytes, rank: int, nranks: int, owners=None):
        """Split solve_cell_problems over nranks GPUs (load i on owners[i]; see distributed.py)."""
        L = lib()
        L.ihom_set_comm.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int)]
        own = (C.c_int * 6)(*owners) if owners is not None else None
        _check(L.ihom_set_comm(self._ctx(), uid, int(rank), int(nranks), own))


def _raise_last():
    msg = lib().ihom_last_error().decode()
    if "resolution" in msg or "must" in msg or "range" in msg or "supported" in msg:
        raise ValueError(msg)
    raise RuntimeError(msg)


def transfer(n, x, direction="restrict", f32=False, out=None):
    """restrict_residual_field / prolong_add_field (src/multigrid.cpp:19-79) on the device. restrict:
    returns R x (coarse, AoS). prolong: returns out + P x (fine, AoS; out defaults to zeros)."""
    nf = _n3(n)
    nvf = int(np.prod(nf))
    nvc = nvf // 8
    x = np.ascontiguousarray(x, np.float64).ravel()
    d = 0 if direction == "restrict" else 1
    o = np.zeros(3 * (nvc if d == 0 else nvf)) if out is None else np.array(out, np.float64).ravel()
    _check(lib().ihom_transfer((C.c_int * 3)(*nf), d, int(bool(f32)), x.ctypes.data_as(_dp), o.ctypes.data_as(_dp)))
    return o.reshape(-1, 3)


def coarse_dense_solve(raw, f):
    """Coarsest-level dense solve of an assembled operator (dof order 3*loc+c) on the device:
    factor_coarsest + coarsest_solve (src/multigrid.cpp:368-451). Returns (x, rel) with rel the
    relative residual against the operator the solve used. Raises on the singularity gate."""
    raw = np.ascontiguousarray(raw, np.float64)
    n = raw.shape[0]
    f = np.ascontiguousarray(f, np.float64).ravel().copy()
    x = np.zeros(n)
    rel = C.c_double()
    _check(lib().ihom_coarse_dense_solve(C.c_longlong(n // 3), raw.ctypes.data_as(_dp), f.ctypes.data_as(_dp),
                                         x.ctypes.data_as(_dp), C.byref(rel)))
    return x, rel.value


# ---------------------------------------------------------------- design pipeline
def grid_locs(n, neighbors=False):
    """Device-computed colour-block location of every vertex (x-fastest) [+ 27-neighbour table]."""
    m = int(np.prod(_n3(n)))
    locs = np.zeros(m, np.int64)
    nb = np.zeros(27 * m, np.int64) if neighbors else None
    _check(lib().ihom_grid_locs((C.c_int * 3)(*_n3(n)), locs.ctypes.data_as(C.POINTER(C.c_longlong)),
                                nb.ctypes.data_as(C.POINTER(C.c_longlong)) if neighbors else None))
    return (locs, nb.reshape(m, 27)) if neighbors else locs


def radial_filter(n, f, radius=2.0, kernel="spline4"):
    """Normalised periodic radial convolution (src/density.cpp:48-63)."""
    n3 = (C.c_int * 3)(*_n3(n))
    p, where, keep = _in(f, int(np.prod(_n3(n))))
    out, op, _ = _out_like(f, int(np.prod(_n3(n))))
    _check(lib().ihom_radial_filter(n3, p, C.c_double(radius), KERNEL[kernel], op, where))
    return out


class DensityExpr:
    """rho_design -> [conv] -> pow(p) with its adjoint (inc/density.hpp:45-66)."""

    def __init__(self, filter_radius: Optional[float], kernel: str = "spline4", exponent: float = 3.0):
        self.radius = filter_radius if filter_radius is not None else -1.0
        self.kernel, self.p = kernel, exponent
        self._pre = None
        self._n = None

    @staticmethod
    def pow_only(exponent):
        return DensityExpr(None, "linear", exponent)

    def exponent(self):
        return self.p

    def has_filter(self):
        return self.radius >= 0

    def eval(self, n, design):
        m = int(np.prod(_n3(n)))
        p, where, keep = _in(design, m)
        out, op, _ = _out_like(design, m)
        pre, pp, _ = _out_like(design, m)
        _check(lib().ihom_density_expr_eval((C.c_int * 3)(*_n3(n)), C.c_double(self.radius), KERNEL[self.kernel],
                                            C.c_double(self.p), p, op, pp, where))
        self._pre, self._n = pre, _n3(n)
        return out

    def backward(self, g_phys):
        if self._pre is None:
            raise RuntimeError("DensityExpr::backward before eval")
        m = int(np.prod(self._n))
        pp, where, k1 = _in(self._pre, m)
        gp, where2, k2 = _in(g_phys, m)
        if where != where2:
            raise ValueError("pre and gradient must live in the same memory space")
        out, op, _ = _out_like(g_phys, m)
        _check(lib().ihom_density_expr_backward((C.c_int * 3)(*self._n), C.c_double(self.radius),
                                                KERNEL[self.kernel], C.c_double(self.p), pp, gp, op, where))
        return out


def symmetrize(n, f, sym="reflect6"):
    """Orbit average under the cube symmetry group (src/density.cpp:131-150); returns a new array."""
    m = int(np.prod(_n3(n)))
    if _is_torch_cuda(f):
        out = f.clone()
        ptr, where = C.cast(C.c_void_p(out.data_ptr()), _dp), IHOM_DEVICE
    else:
        out = np.array(f, dtype=np.float64).ravel().copy()
        if out.size != m:
            raise ValueError("field size mismatch")
        ptr, where = out.ctypes.data_as(_dp), IHOM_HOST
    _check(lib().ihom_symmetrize((C.c_int * 3)(*_n3(n)), ptr, SYMMETRY[sym], where))
    return out


def field_mean(f) -> float:
    p, where, keep = _in(f)
    m = keep.numel() if _is_torch_cuda(keep) else keep.size
    v = C.c_double()
    _check(lib().ihom_field_mean(p, C.c_longlong(m), C.byref(v), where))
    return v.value


@dataclasses.dataclass
class OCConfig:  # inc/oc.hpp:10-16
    min_density: float = kRhoMin
    step_limit: float = 0.05
    damp: float = 0.5
    volume: float = 0.3
    bisect_tol: float = 1e-6


def oc_update(rho, sens, cfg: OCConfig = None):
    """Returns (rho', lambda, bisection_ok) (src/oc.cpp:27-77)."""
    cfg = cfg or OCConfig()
    p, where, k1 = _in(rho)
    g, where2, k2 = _in(sens)
    m = k1.numel() if _is_torch_cuda(k1) else k1.size
    out, op, _ = _out_like(rho, m)
    c = _OCConfig(cfg.min_density, cfg.step_limit, cfg.damp, cfg.volume, cfg.bisect_tol)
    lam, ok = C.c_double(), C.c_int()
    _check(lib().ihom_oc_update(C.c_longlong(m), p, g, C.byref(c), op, C.byref(lam), C.byref(ok), where))
    return out, lam.value, bool(ok.value)


def sensitivity_filter(n, sens, rho, radius):
    m = int(np.prod(_n3(n)))
    g, where, k1 = _in(sens, m)
    r, where2, k2 = _in(rho, m)
    out, op, _ = _out_like(sens, m)
    _check(lib().ihom_sensitivity_filter((C.c_int * 3)(*_n3(n)), g, r, C.c_double(radius), op, where))
    return out


def init_trig(n, basis_n=2, seed=0, volume=0.3, sigmoid_k=15.0):
    """Random trigonometric initial density (src/density.cpp:169-259). Returns (rho, fallback)."""
    m = int(np.prod(_n3(n)))
    out = np.zeros(m)
    fb = C.c_int()
    _check(lib().ihom_init_trig((C.c_int * 3)(*_n3(n)), int(basis_n), C.c_uint64(seed), C.c_double(volume),
                                C.c_double(sigmoid_k), out.ctypes.data_as(_dp), C.byref(fb)))
    return out, bool(fb.value)


def objective_native(obj, Cmat, iter=0, beta=0.8, eta=0.6, tau=-1e-3, gamma=0.5):
    """The predefined objectives evaluated by the native C++ Expr (value, dC)."""
    c = np.ascontiguousarray(Cmat, dtype=np.float64).ravel()
    v = C.c_double()
    g = (C.c_double * 36)()
    _check(lib().ihom_objective(OBJECTIVE[obj], C.c_double(beta), C.c_double(eta), C.c_double(tau),
                                C.c_double(gamma), int(iter), c.ctypes.data_as(_dp), C.byref(v), g))
    return v.value, np.array(g[:]).reshape(6, 6)


# ---------------------------------------------------------------- runner
@dataclasses.dataclass
class RunConfig:  # inc/config.hpp:15-42
    reso: int = 64
    vol: float = 0.3
    youngs: float = 1e6
    poisson: float = 0.3
    obj: str = "bulk"
    beta: float = 0.8
    eta: float = 0.6
    tau: float = -1e-3
    gamma: float = 0.5
    penal: float = 3.0
    filter_radius: float = 2.0
    filter_placement: str = "density"
    kernel: str = "spline4"
    sym: str = "reflect6"
    init: str = "trig"
    basis_n: int = 2
    seed: int = 0
    max_iter: int = 300
    step: float = 0.05
    damp: float = 0.5
    tol: float = 1e-2
    max_cycles: int = 50
    precision: str = "mixed"
    solver_mode: str = "vcycle"
    device: int = 0

    def _c(self):
        return _RunConfig(self.reso, self.vol, self.youngs, self.poisson, OBJECTIVE[self.obj], self.beta, self.eta,
                          self.tau, self.gamma, self.penal, self.filter_radius,
                          0 if self.filter_placement == "density" else 1, KERNEL[self.kernel], SYMMETRY[self.sym],
                          {"constant": 0, "trig": 1, "file": 2}[self.init], self.basis_n, self.seed, self.max_iter,
                          self.step, self.damp, self.tol, self.max_cycles, PRECISION[self.precision],
                          SOLVER_MODE[self.solver_mode], self.device)


@dataclasses.dataclass
class OptimizationReport:  # inc/runner.hpp:21-31
    records: list
    tensors: list
    tensor: np.ndarray
    density: np.ndarray
    poisson_est: float
    converged: bool
    solver_failed: bool
    init_fallback: bool
    oc_warning: bool


def run_optimization(cfg: RunConfig, observer: Optional[Callable] = None, init_rho=None) -> OptimizationReport:
    """The native optimisation loop (src/runner.cpp:51-136); observer(iter, prev, next, C, rec) -> bool."""
    c = cfg._c()
    recs = (_IterRecord * max(1, cfg.max_iter))()
    nrec, flags = C.c_int(), C.c_int()
    m = cfg.reso ** 3
    rho = np.zeros(m)
    init = None
    if init_rho is not None:
        init = np.ascontiguousarray(init_rho, dtype=np.float64).ravel()
    cb = None
    if observer is not None:
        def _cb(it, prev, nxt, rec, user):
            pv = np.ctypeslib.as_array(prev, shape=(m,)).copy()
            nx = np.ctypeslib.as_array(nxt, shape=(m,)).copy()
            r = rec.contents
            return 1 if observer(it, pv, nx, np.array(r.C[:]).reshape(6, 6), _rec_dict(r)) else 0
        cb = _OBSERVER(_cb)
    _check(lib().ihom_run_optimization(C.byref(c), init.ctypes.data_as(_dp) if init is not None else None, recs,
                                       cfg.max_iter, C.byref(nrec), rho.ctypes.data_as(_dp), C.byref(flags),
                                       cb if cb is not None else _OBSERVER(0), None))
    records = [_rec_dict(r) for r in recs[: nrec.value]]
    tensors = [r["C"] for r in records]
    fl = flags.value
    tensor = tensors[-1] if tensors else np.zeros((6, 6))
    return OptimizationReport(records, tensors, tensor, rho, poisson_ratio_report(tensor), bool(fl & 2),
                              bool(fl & 1), bool(fl & 4), bool(fl & 8))


def _rec_dict(r):
    return dict(iter=r.iter, objective=r.objective, volume=r.volume, cycles=r.cycles, residual=r.residual, ms=r.ms,
                C=np.array(r.C[:]).reshape(6, 6), **{"lambda": r.lambda_}, oc_trials=r.oc_trials)


def hs_bulk_bound(youngs, poisson, f):  # src/runner.cpp:168-173
    k = youngs / (3.0 * (1.0 - 2.0 * poisson))
    g = youngs / (2.0 * (1.0 + poisson))
    return 4.0 * f * g * k / (4.0 * g + 3.0 * (1.0 - f) * k)


def hs_shear_bound(youngs, poisson, f):  # src/runner.cpp:175-179
    k = youngs / (3.0 * (1.0 - 2.0 * poisson))
    g = youngs / (2.0 * (1.0 + poisson))
    q = (1.0 - f) * 6.0 * (k + 2.0 * g) / (5.0 * (3.0 * k + 4.0 * g))
    return f * g / (1.0 + q)


# ---------------------------------------------------------------- stepping optimiser + profiler
class Optimizer:
    """One optimisation iteration per step() (the loop body of src/runner.cpp:83-131).

    With ``fabric`` this is z-slab ``rank`` of the run: designs in and out are the
    slab's elements (x-fastest, planes [z0, z0 + planes)) and every call is
    collective over the slabs (drive them from one thread each, see run_slabs).
    """

    STATUS = {0: "updated", 1: "solver_failed", 2: "converged", 3: "last_iteration"}

    def __init__(self, cfg: RunConfig, init_rho=None, fabric: Optional[Fabric] = None, rank: int = 0):
        L = lib()
        L.ihom_opt_create.restype = C.c_void_p
        L.ihom_opt_create.argtypes = [C.POINTER(_RunConfig), _dp]
        L.ihom_opt_destroy.argtypes = [C.c_void_p]
        L.ihom_opt_step.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.POINTER(_IterRecord), C.POINTER(C.c_int)]
        L.ihom_opt_design.argtypes = [C.c_void_p, _dp, C.c_int]
        L.ihom_opt_flags.argtypes = [C.c_void_p]
        L.ihom_opt_launches.argtypes = [C.c_void_p]
        L.ihom_opt_launches.restype = C.c_longlong
        L.ihom_opt_stream.argtypes = [C.c_void_p]
        L.ihom_opt_stream.restype = C.c_void_p
        self.cfg = cfg
        self.fabric = fabric
        P = fabric.nranks if fabric is not None else 1
        self.planes = cfg.reso // P
        self.z0 = rank * self.planes
        self.m = cfg.reso * cfg.reso * self.planes
        self._c = cfg._c()
        init = None if init_rho is None else np.ascontiguousarray(init_rho, dtype=np.float64).ravel()
        iptr = init.ctypes.data_as(_dp) if init is not None else None
        if fabric is None:
            self._p = L.ihom_opt_create(C.byref(self._c), iptr)
        else:
            L.ihom_opt_create_slab.restype = C.c_void_p
            L.ihom_opt_create_slab.argtypes = [C.POINTER(_RunConfig), _dp, C.c_void_p, C.c_int]
            self._p = L.ihom_opt_create_slab(C.byref(self._c), iptr, C.c_void_p(fabric._p), int(rank))
        if not self._p:
            _raise_last()

    def close(self):
        if getattr(self, "_p", None):
            lib().ihom_opt_destroy(C.c_void_p(self._p))
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, rho_in=None, rho_out=None):
        """Returns (status, record). rho_in/rho_out: numpy (host) or torch CUDA float64 tensors."""
        where = IHOM_HOST
        pin = pout = None
        keep = []
        for buf in (rho_in, rho_out):
            if buf is not None and _is_torch_cuda(buf):
                where = IHOM_DEVICE
        if rho_in is not None:
            if where == IHOM_DEVICE:
                pin = C.cast(C.c_void_p(rho_in.data_ptr()), _dp)
            else:
                a = rho_in if isinstance(rho_in, np.ndarray) and rho_in.flags.c_contiguous else \
                    np.ascontiguousarray(rho_in, dtype=np.float64)
                keep.append(a)
                pin = a.ctypes.data_as(_dp)
        if rho_out is not None:
            if where == IHOM_DEVICE:
                pout = C.cast(C.c_void_p(rho_out.data_ptr()), _dp)
            else:
                if not (isinstance(rho_out, np.ndarray) and rho_out.dtype == np.float64 and rho_out.flags.c_contiguous):
                    raise ValueError("rho_out must be a contiguous float64 numpy array")
                pout = rho_out.ctypes.data_as(_dp)
        rec = _IterRecord()
        st = C.c_int()
        _check(lib().ihom_opt_step(C.c_void_p(self._p), pin, pout, where, C.byref(rec), C.byref(st)))
        return st.value, _rec_dict(rec)

    def design(self):
        out = np.zeros(self.m)
        _check(lib().ihom_opt_design(C.c_void_p(self._p), out.ctypes.data_as(_dp), IHOM_HOST))
        return out

    def flags(self):
        fl = lib().ihom_opt_flags(C.c_void_p(self._p))
        return dict(solver_failed=bool(fl & 1), converged=bool(fl & 2), init_fallback=bool(fl & 4),
                    oc_warning=bool(fl & 8))

    def kernel_launches(self) -> int:
        return lib().ihom_opt_launches(C.c_void_p(self._p))

    def set_comm(self, uid: bytes, rank: int, nranks: int, owners=None):
        """Split the 6 cell problems over nranks GPUs (see distributed.py)."""
        L = lib()
        L.ihom_opt_set_comm.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int)]
        own = (C.c_int * 6)(*owners) if owners is not None else None
        _check(L.ihom_opt_set_comm(C.c_void_p(self._p), uid, int(rank), int(nranks), own))

    def stream(self) -> int:
        return lib().ihom_opt_stream(C.c_void_p(self._p)) or 0


def set_knob(name: str, value: int):
    """Kernel-variant switch (include/ihom_b200.h ihom_set_knob); variants are bit-identical."""
    _check(lib().ihom_set_knob(name.encode(), int(value)))


def get_knob(name: str, default: int = 0) -> int:
    return int(lib().ihom_get_knob(name.encode(), int(default)))


def profile_enable(on: bool = True):
    _check(lib().ihom_profile_enable(1 if on else 0))


def launch_count() -> int:
    """Kernels launched by libihom_b200.so since it was loaded."""
    L = lib()
    L.ihom_launch_count.restype = C.c_longlong
    return L.ihom_launch_count()


def profile_totals() -> dict:
    """{family: {"launches", "ms", "bytes"}} of device time per kernel family since profile_enable(True)."""
    L = lib()
    L.ihom_profile_get.argtypes = [C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_longlong), _dp, _dp]
    n = L.ihom_profile_count()
    out = {}
    for i in range(n):
        buf = C.create_string_buffer(64)
        cnt, ms, by = C.c_longlong(), C.c_double(), C.c_double()
        _check(L.ihom_profile_get(i, buf, 64, C.byref(cnt), C.byref(ms), C.byref(by)))
        out[buf.value.decode()] = dict(launches=cnt.value, ms=ms.value, bytes=by.value)
    return out
