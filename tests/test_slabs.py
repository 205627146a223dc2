"""z-slab decomposition on one device.

P slabs of one grid live in this process (Fabric.local), one host thread per
slab; every cross-slab read goes through the same peer-pointer links the
multi-GPU (IPC / NVLink) fabric uses. The per-vertex arithmetic of a slab is
exactly the single-domain arithmetic, so the solve takes the same number of
cycles and C^H / sensitivities agree with the one-domain run up to the order
of the cross-slab sums.
"""
import numpy as np
import pytest

import paper_2301_08911_b200 as ih

pytestmark = pytest.mark.gpu


def _design(n, seed=0):
    rho, _ = ih.init_trig(n, 2, seed, 0.3)
    return ih.radial_filter(n, rho, 2.0, "spline4") ** 3


def _seed():
    s = np.zeros((6, 6))
    s[:3, :3] = 1.0 / 9.0
    s[3, 3] = s[4, 4] = s[5, 5] = 0.25
    return s


def _single(n, phys, precision, mode, tol):
    hom = ih.Homogenizer(n, penal=1.0, precision=precision, opts=ih.SolverOptions(tol=tol, mode=mode))
    hom.set_density(phys)
    st = hom.solve_cell_problems()
    C = hom.effective_tensor()
    sens = hom.tensor_sensitivity(_seed())
    hom.close()
    return st, C, sens


def _slabs(P, n, phys, precision, mode, tol):
    fab = ih.Fabric.local(P)

    def body(r):
        hom = ih.Homogenizer(n, penal=1.0, precision=precision, opts=ih.SolverOptions(tol=tol, mode=mode),
                             fabric=fab, rank=r)
        m = n * n * hom.planes
        hom.set_density(np.ascontiguousarray(phys[hom.z0 * n * n: hom.z0 * n * n + m]))
        st = hom.solve_cell_problems()
        C = hom.effective_tensor()
        sens = hom.tensor_sensitivity(_seed())
        hom.close()
        return st, C, sens

    out = ih.run_slabs(P, body)
    fab.close()
    return out


@pytest.mark.parametrize("P,n,precision,mode", [
    (2, 32, "double", "vcycle"),
    (4, 32, "mixed", "vcycle"),
    (4, 32, "mixed", "mixed_defect"),
    (2, 64, "mixed", "mixed_defect"),
    (8, 32, "mixed", "mixed_defect"),
])
def test_slabs_match_single_domain(P, n, precision, mode):
    phys = _design(n)
    st1, C1, s1 = _single(n, phys, precision, mode, 1e-2)
    res = _slabs(P, n, phys, precision, mode, 1e-2)
    for st, C, _ in res:
        assert st["total_cycles"] == st1["total_cycles"]
        assert st["converged"]
        np.testing.assert_array_equal(C, res[0][1])  # every slab holds the same tensor (rank-order sums)
        assert np.max(np.abs(C - C1)) <= 1e-9 * np.max(np.abs(C1))
    sens = np.concatenate([r[2] for r in res])
    # mixed: sensitivities read the f32 snapshot of u (src/homogenization.cpp:84-85); u differs from the
    # one-domain u by the order of the cross-slab sums, which can flip an f32 rounding of an element's u
    tol = 1e-9 if precision == "double" else 1e-6
    assert np.max(np.abs(sens - s1)) <= tol * np.max(np.abs(s1))


def test_slabs_tight_tolerance():
    n, P = 32, 4
    phys = _design(n, seed=3)
    _, C1, _ = _single(n, phys, "double", "vcycle", 1e-9)
    res = _slabs(P, n, phys, "double", "vcycle", 1e-9)
    assert np.max(np.abs(res[0][1] - C1)) <= 1e-11 * np.max(np.abs(C1))


def test_slab_geometry_rules():
    fab = ih.Fabric.local(3)
    with pytest.raises((ValueError, RuntimeError)):
        ih.run_slabs(3, lambda r: ih.Homogenizer(32, fabric=fab, rank=r))  # 32 planes do not split in 3
    fab.close()


def _run_single(cfg, iters):
    opt = ih.Optimizer(cfg)
    recs = []
    for _ in range(iters):
        st, rec = opt.step()
        recs.append(rec)
    d = opt.design()
    opt.close()
    return recs, d


def _run_slabs(cfg, iters, P):
    fab = ih.Fabric.local(P)

    def body(r):
        opt = ih.Optimizer(cfg, fabric=fab, rank=r)
        recs = []
        for _ in range(iters):
            st, rec = opt.step()
            recs.append(rec)
        d = opt.design()
        opt.close()
        return recs, d

    out = ih.run_slabs(P, body)
    fab.close()
    return out


@pytest.mark.parametrize("P,obj,sym,precision,mode", [
    (2, "bulk", "reflect6", "mixed", "mixed_defect"),
    (4, "npr-relaxed", "reflect6", "mixed", "mixed_defect"),
    (4, "shear", "reflect3", "double", "vcycle"),
    (2, "bulk", "rotate3", "mixed", "vcycle"),
])
def test_slab_optimizer_matches_single_domain(P, obj, sym, precision, mode):
    cfg = ih.RunConfig(reso=32, vol=0.3, obj=obj, sym=sym, max_iter=10, precision=precision, solver_mode=mode)
    recs1, d1 = _run_single(cfg, 3)
    res = _run_slabs(cfg, 3, P)
    for recs, _ in res:
        for a, b in zip(recs, recs1):
            assert a["cycles"] == b["cycles"]
            assert abs(a["objective"] - b["objective"]) <= 1e-9 * abs(b["objective"])
            assert abs(a["volume"] - b["volume"]) <= 1e-12
    d = np.concatenate([r[1] for r in res])
    assert np.max(np.abs(d - d1)) <= 1e-9


@pytest.mark.parametrize("P", [2, 4])
def test_slab_optimizer_256_bulk(P):
    """BASELINE configs[2]: bulk modulus 256^3, vol 0.3, 1 vs 2/4 z-slabs (slabs share one GPU here)."""
    cfg = ih.RunConfig(reso=256, vol=0.3, obj="bulk", sym="reflect6", max_iter=10, precision="mixed",
                       solver_mode="mixed_defect")
    recs1, d1 = _run_single(cfg, 2)
    res = _run_slabs(cfg, 2, P)
    for recs, _ in res:
        for a, b in zip(recs, recs1):
            assert a["cycles"] == b["cycles"]
            # 1e-8: the inner cycle's stencil levels accumulate in f32 (STENCIL_F32) and a slab's small
            # levels may take the warp-per-vertex (f64) kernel where one domain takes the thread-per-
            # vertex one, so the coarse corrections differ at f32 rounding (observed 1.2e-9 at P = 4)
            assert abs(a["objective"] - b["objective"]) <= 1e-8 * abs(b["objective"])
    d = np.concatenate([r[1] for r in res])
    # the cross-slab sums (norms, C^H, OC means) fold in another order: the OC multiplier, and with it
    # every density, moves at the 1e-9 level per iteration on 16.7M elements
    assert np.max(np.abs(d - d1)) <= 1e-7
