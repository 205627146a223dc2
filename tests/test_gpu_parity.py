"""GPU parity: every kernel of the hot path against the CPU oracle (oracle/),
through the C ABI. Tolerances: integer/index work bit-exact; all-double
arithmetic <= 1e-12 relative; mixed (f32 coefficients) <= 1e-6 relative on
single operator applications. Mirrors proj/tests/test_fem.cpp,
test_multigrid.cpp, test_homogenization.cpp, test_density.cpp, test_oc.cpp.
"""
import numpy as np
import pytest

from conftest import mt_uniform

pytestmark = pytest.mark.gpu

E, NU = 1e6, 0.3


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- grid (bit-exact)
@pytest.mark.parametrize("n", [(4, 4, 4), (8, 8, 8), (6, 10, 8), (5, 7, 9), (16, 16, 16)])
def test_grid_locations_bit_exact(ih, orc, n):
    locs = ih.grid_locs(n)
    assert np.array_equal(locs, orc.grid_locs(n))
    assert np.array_equal(np.sort(locs), np.arange(np.prod(n)))  # bijection (tests/test_grid.cpp:33-45)


@pytest.mark.parametrize("n", [(8, 8, 8), (6, 4, 10)])
def test_neighbour_tables_bit_exact(ih, orc, n):
    locs, nb = ih.grid_locs(n, neighbors=True)
    nx, ny, nz = n
    # brute force: neighbour t of vertex v is loc(wrap(v + t)) (src/fem.cpp:37-68)
    loc3 = locs.reshape(nz, ny, nx)
    inv = np.empty((np.prod(n), 3), int)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                inv[loc3[z, y, x]] = (x, y, z)
    for t in range(27):
        dx, dy, dz = t % 3 - 1, (t // 3) % 3 - 1, t // 9 - 1
        exp = loc3[(inv[:, 2] + dz) % nz, (inv[:, 1] + dy) % ny, (inv[:, 0] + dx) % nx]
        assert np.array_equal(nb[:, t], exp)


# ---------------------------------------------------------------- level-0 operators
def make_hom(ih, n, precision, penal=3.0, tol=1e-2, max_cycles=50, mode="vcycle"):
    return ih.Homogenizer(n, ih.BaseMaterial(E, NU), penal,
                          ih.SolverOptions(tol=tol, max_cycles=max_cycles, mode=mode), precision=precision)


@pytest.mark.parametrize("precision,tol", [("double", 1e-12), ("mixed", 2e-6)])
@pytest.mark.parametrize("n", [8, 16, (10, 8, 12), (5, 7, 9), 64, (64, 32, 32), (64, 48, 32)])
def test_level0_apply_residual(ih, orc, precision, tol, n):
    nv = int(np.prod(n)) if not np.isscalar(n) else n ** 3
    rho = mt_uniform(nv, 1, 1e-3, 1.0)
    hom = make_hom(ih, n, precision, penal=3.0)
    hom.set_density(rho)
    coeff = hom.hierarchy().coeff()
    u = mt_uniform(3 * nv, 7, -1, 1).reshape(nv, 3)
    f = mt_uniform(3 * nv, 8, -1, 1).reshape(nv, 3)
    y = hom.hierarchy().apply(0, u)
    yo = orc.fem(n, "apply", coeff, u=u, E=E, nu=NU, mixed=precision == "mixed")
    assert rel(y, yo) < tol
    # residual through the level fields
    H = hom.hierarchy()
    H.set_field(0, "u", u)
    H.set_field(0, "f", f)
    H.compute_residual(0)
    ro = orc.fem(n, "residual", coeff, u=u, f=f, E=E, nu=NU, mixed=precision == "mixed")
    assert rel(H.field(0, "r"), ro) < tol


@pytest.mark.parametrize("precision,tol", [("double", 1e-11), ("mixed", 2e-6)])
@pytest.mark.parametrize("n", [8, (10, 8, 12), 32])
def test_level0_gauss_seidel_sweep(ih, orc, precision, tol, n):
    nv = int(np.prod(n)) if not np.isscalar(n) else n ** 3
    rho = mt_uniform(nv, 3, 1e-3, 1.0)
    hom = make_hom(ih, n, precision)
    hom.set_density(rho)
    H = hom.hierarchy()
    coeff = H.coeff()
    u = mt_uniform(3 * nv, 11, -1, 1).reshape(nv, 3)
    f = mt_uniform(3 * nv, 12, -1, 1).reshape(nv, 3)
    H.set_field(0, "u", u)
    H.set_field(0, "f", f)
    H.relax(0, 1)
    uo = orc.fem(n, "gs", coeff, u=u, f=f, E=E, nu=NU, mixed=precision == "mixed")
    assert rel(H.field(0, "u"), uo) < tol


@pytest.mark.parametrize("precision", ["double", "mixed"])
def test_macro_force(ih, orc, precision):
    n, nv = 8, 512
    rho = mt_uniform(nv, 5, 1e-3, 1.0)
    hom = make_hom(ih, n, precision)
    hom.set_density(rho)
    coeff = hom.hierarchy().coeff()
    for load in range(6):
        f = hom.hierarchy().macro_force(load)
        fo = orc.fem(n, "macro", coeff, E=E, nu=NU, mixed=precision == "mixed", load=load)
        assert rel(f, fo) < 1e-13


# ---------------------------------------------------------------- Galerkin / coarse levels
@pytest.mark.parametrize("precision,tol", [("double", 1e-12), ("mixed", 1e-6)])
def test_galerkin_stencils(ih, orc, precision, tol):
    n = 16
    rho = mt_uniform(n ** 3, 223, 1e-3, 1.0)
    hom = make_hom(ih, n, precision)
    hom.set_density(rho)
    oh = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=precision == "mixed")
    oh.set_density(rho)
    assert hom.hierarchy().num_levels() == oh.num_levels() == 3
    for l in (1, 2):
        assert rel(hom.hierarchy().stencil(l), oh.stencil(l)) < tol


@pytest.mark.parametrize("precision,tol", [("double", 1e-11), ("mixed", 2e-6)])
@pytest.mark.parametrize("n", [16, 32, (32, 16, 24)])
def test_coarse_level_apply_gs_residual(ih, orc, precision, tol, n):
    """Stencil levels directly (src/multigrid.cpp:186-239, 392-424): on levels 1 and 2 the device
    apply (y = K_l x), one 8-colour GS sweep and the residual r = f - K_l u equal the oracle's on the
    same seeded u, f (the level operators themselves are pinned by test_galerkin_stencils)."""
    n3 = (n,) * 3 if np.isscalar(n) else n
    nv0 = int(np.prod(n3))
    rho = mt_uniform(nv0, 401, 1e-3, 1.0)
    hom = make_hom(ih, n3, precision)
    hom.set_density(rho)
    oh = orc.Homogenizer(n3, E=E, nu=NU, penal=3.0, mixed=precision == "mixed")
    oh.set_density(rho)
    H = hom.hierarchy()
    for l in (1, 2):
        nv = int(np.prod([x >> l for x in n3]))
        u = mt_uniform(3 * nv, 410 + l, -1, 1).reshape(nv, 3)
        f = mt_uniform(3 * nv, 420 + l, -1, 1).reshape(nv, 3)
        assert rel(H.apply(l, u), _oracle_apply(oh, l, u)) < tol
        for which, v in (("u", u), ("f", f)):
            H.set_field(l, which, v)
            oh.level_field(l, which, v)
        H.compute_residual(l)
        oh.compute_residual(l)
        assert rel(H.field(l, "r"), oh.level_field(l, "r")) < tol
        H.relax(l, 1)
        oh.relax(l, 1)
        assert rel(H.field(l, "u"), oh.level_field(l, "u")) < tol


def _oracle_apply(oh, l, x):
    """K_l x on the oracle: residual with f = 0 is -K_l x."""
    oh.level_field(l, "u", x)
    oh.level_field(l, "f", np.zeros_like(x))
    oh.compute_residual(l)
    return -oh.level_field(l, "r")


def test_coarse_operator_annihilates_constants(ih):
    hom = make_hom(ih, 16, "double")
    hom.set_density(mt_uniform(16 ** 3, 229, 1e-3, 1.0))
    H = hom.hierarchy()
    for l in range(H.num_levels()):
        nv = int(np.prod(H.level_dims(l)))
        c = np.tile([1.0, -2.0, 0.5], (nv, 1))
        y = H.apply(l, c)
        assert np.linalg.norm(y) < 1e-9 * np.linalg.norm(c) * max(1.0, H.op_scale())


@pytest.mark.parametrize("n", [8, (10, 8, 12), 32])
@pytest.mark.parametrize("f32", [False, True])
def test_transfer_restrict_prolong(ih, orc, n, f32):
    """Device restrict / prolong-add (f64 and the f32 inner-cycle kernels) against the oracle's
    restrict_residual_field / prolong_add_field (src/multigrid.cpp:19-79)."""
    nf = (n, n, n) if isinstance(n, int) else n
    nvf = int(np.prod(nf))
    fine = mt_uniform(3 * nvf, 101, -1, 1)
    coarse = mt_uniform(3 * nvf // 8, 103, -1, 1)
    base = mt_uniform(3 * nvf, 107, -1, 1)
    if f32:  # the f32 kernels see f32-rounded inputs; powers-of-two weights, f32 sums
        fine, coarse, base = (a.astype(np.float32).astype(np.float64) for a in (fine, coarse, base))
    tol = 1e-6 if f32 else 1e-15
    r = ih.transfer(nf, fine, "restrict", f32=f32)
    ro = orc.restrict(nf, fine)
    assert rel(r, ro) < tol
    p = ih.transfer(nf, coarse, "prolong", f32=f32, out=base)
    po = orc.prolong_add(nf, coarse, base)
    assert rel(p, po) < tol
    # adjointness R = P^T (tests/test_multigrid.cpp:59-72) on the device kernels
    if not f32:
        lhs = float(np.dot(ih.transfer(nf, fine, "restrict").ravel(), coarse))
        rhs = float(np.dot(fine, ih.transfer(nf, coarse, "prolong").ravel()))
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


# ---------------------------------------------------------------- V-cycle / solve
@pytest.mark.parametrize("precision,tol", [("double", 1e-8), ("mixed", 1e-4)])
def test_vcycle_trajectory_matches_oracle(ih, orc, precision, tol):
    n = 16
    rho = mt_uniform(n ** 3, 257, 0.1, 1.0)
    hom = make_hom(ih, n, precision)
    hom.set_density(rho)
    oh = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=precision == "mixed")
    oh.set_density(rho)
    f = hom.hierarchy().macro_force(0)
    f = f - f.mean(axis=0)
    H = hom.hierarchy()
    H.set_field(0, "f", f)
    H.set_field(0, "u", np.zeros_like(f))
    oh.level_field(0, "f", f)
    oh.level_field(0, "u", np.zeros_like(f))
    for _ in range(8):
        a, b = H.v_cycle(), oh.v_cycle()
        assert abs(a - b) <= tol * b + 1e-14
    assert rel(H.field(0, "u"), oh.level_field(0, "u")) < tol


@pytest.mark.parametrize("precision", ["double", "mixed"])
def test_solve_tight_matches_oracle(ih, orc, precision):
    n = 8
    rho = mt_uniform(512, 263, 0.1, 1.0)
    # f32 stencils bound the attainable mixed-precision residual (reference mixed mode stalls near 1e-7)
    tol = 1e-10 if precision == "double" else 1e-5
    hom = make_hom(ih, n, precision, tol=tol, max_cycles=100)
    hom.set_density(rho)
    oh = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=precision == "mixed", tol=tol, max_cycles=100)
    oh.set_density(rho)
    f = mt_uniform(3 * 512, 264, -1, 1).reshape(512, 3)
    u, st = hom.hierarchy().solve(f, np.zeros_like(f))
    uo, sto = oh.solve(f, np.zeros_like(f))
    assert st["converged"] and sto["converged"]
    assert abs(st["cycles"] - sto["cycles"]) <= 1
    assert rel(u, uo) < (1e-8 if precision == "double" else 1e-5)


# ---------------------------------------------------------------- homogenization known answers
def test_solid_tensor_known_values(ih):
    hom = make_hom(ih, 8, "double", tol=1e-10, max_cycles=200)
    hom.set_density(np.ones(512))
    st = hom.solve_cell_problems()
    assert st["converged"]
    c = hom.effective_tensor()  # tests/test_homogenization.cpp:30-33
    assert c[0, 0] == pytest.approx(1346153.846153846, rel=1e-9)
    assert c[0, 1] == pytest.approx(576923.0769230769, rel=1e-9)
    assert c[3, 3] == pytest.approx(384615.3846153846, rel=1e-9)
    for i in range(6):
        assert np.linalg.norm(hom.displacement(i)) < 1e-12


def test_laminate_harmonic_mean(ih):
    n = 8
    x = np.arange(512) % 8
    rho = np.where(x < 4, 0.4, 0.9)
    hom = make_hom(ih, n, "double", tol=1e-10, max_cycles=200)
    hom.set_density(rho)
    assert hom.solve_cell_problems()["converged"]
    lam, mu = E * NU / ((1 + NU) * (1 - 2 * NU)), E / (2 * (1 + NU))
    q1, q2 = 0.4 ** 3, 0.9 ** 3
    assert hom.effective_tensor()[0, 0] == pytest.approx((lam + 2 * mu) * 2 / (1 / q1 + 1 / q2), rel=1e-8)


@pytest.mark.parametrize("precision,tol", [("double", 1e-9), ("mixed", 1e-5)])
def test_tensor_and_sensitivity_vs_oracle(ih, orc, precision, tol):
    n = 8
    rho = mt_uniform(512, 1008, 1e-3, 1.0)
    stol = 1e-10 if precision == "double" else 1e-6  # f32 stencils bound the mixed-mode residual
    hom = make_hom(ih, n, precision, tol=stol, max_cycles=200)
    oh = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=precision == "mixed", tol=stol, max_cycles=200)
    hom.set_density(rho)
    oh.set_density(rho)
    s1, s2 = hom.solve_cell_problems(), oh.solve_cell_problems()
    assert s1["converged"] and s2["converged"]
    c, co = hom.effective_tensor(), oh.effective_tensor()
    assert np.abs(c - co).max() < tol * np.abs(co).max()
    seed = np.arange(36, dtype=float).reshape(6, 6) / 36.0
    g, go = hom.tensor_sensitivity(seed), oh.tensor_sensitivity(seed)
    assert rel(g, go) < tol * 10


def test_tensor_from_oracle_displacements_is_exact(ih, orc):
    """Same u -> same C^H to rounding: isolates the C^H kernel from the solver."""
    n = 8
    rho = mt_uniform(512, 77, 0.2, 1.0)
    oh = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=False, tol=1e-6)
    oh.set_density(rho)
    oh.solve_cell_problems()
    hom = make_hom(ih, n, "double")
    hom.set_density(rho)
    for i in range(6):
        hom.set_displacement(i, oh.displacement(i))
    c, co = hom.effective_tensor(), oh.effective_tensor()
    assert np.abs(c - co).max() < 1e-10 * np.abs(co).max()
    seed = np.eye(6)
    assert rel(hom.tensor_sensitivity(seed), oh.tensor_sensitivity(seed)) < 1e-10


# ---------------------------------------------------------------- density side
@pytest.mark.parametrize("kernel", ["linear", "spline4"])
@pytest.mark.parametrize("radius", [0.5, 1.0, 2.0, 2.5])
def test_radial_filter(ih, orc, kernel, radius):
    n = (8, 6, 10)
    f = mt_uniform(480, 31, 0, 1)
    assert rel(ih.radial_filter(n, f, radius, kernel), orc.radial_filter(n, f, radius, kernel)) < 1e-14


@pytest.mark.parametrize("n", [(8, 6, 12), (16, 16, 16), (12, 10, 8)])
@pytest.mark.parametrize("kernel", ["linear", "spline4"])
def test_radial_filter_four_plane_path(ih, orc, n, kernel):
    """nz % 4 == 0 grids take the four-z-planes-per-thread filter (FILTER_NZ, default on): it equals the
    one-plane kernel bit for bit and the oracle to 1e-14."""
    m = int(np.prod(n))
    f = mt_uniform(m, 37, 0, 1)
    a = ih.radial_filter(n, f, 2.0, kernel)
    ih.set_knob("FILTER_NZ", 0)
    try:
        b = ih.radial_filter(n, f, 2.0, kernel)
    finally:
        ih.set_knob("FILTER_NZ", 1)
    np.testing.assert_array_equal(a, b)
    assert rel(a, orc.radial_filter(n, f, 2.0, kernel)) < 1e-14


def _ulps(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b) / np.spacing(np.maximum(np.abs(b), 1e-300)))


@pytest.mark.parametrize("p", [1.0, 2.0, 3.0, 4.0, 2.5])
@pytest.mark.parametrize("radius", [None, 2.0])
def test_density_expr_eval_backward(ih, orc, p, radius):
    """DensityExpr eval / backward on the device (src/density.cpp:65-83): pre = filter(design) (or the
    design), out = pre^p; backward = filter(g p pre^(p-1)). Integer exponents use repeated
    multiplication (POW_INT) -- within 2 ulp of std::pow (numpy's pow is the same libm call); the
    fractional exponent goes through pow and the filter is the oracle's to 1e-14."""
    n = (8, 10, 12)
    m = int(np.prod(n))
    design = mt_uniform(m, 41, 1e-3, 1.0)
    g = mt_uniform(m, 43, -1.0, 1.0)
    de = ih.DensityExpr(radius, "spline4", p)
    out = de.eval(n, design)
    pre = orc.radial_filter(n, design, radius, "spline4") if radius else design
    assert rel(de._pre, pre) < 1e-14
    assert _ulps(out, np.asarray(de._pre) ** p) <= 2  # repeated products / device pow vs glibc pow
    back = de.backward(g)
    gp = g * p * pre ** (p - 1.0)
    expect = orc.radial_filter(n, gp, radius, "spline4") if radius else gp
    assert rel(back, expect) < 1e-14
    if p == int(p):  # POW_INT against std::pow, bitwise structure of the off switch
        ih.set_knob("POW_INT", 0)
        try:
            de0 = ih.DensityExpr(radius, "spline4", p)
            out0 = de0.eval(n, design)
        finally:
            ih.set_knob("POW_INT", 1)
        assert _ulps(out, out0) <= 2
        if radius is None:
            assert _ulps(out0, pre ** p) <= 1  # CUDA pow vs glibc pow


@pytest.mark.parametrize("sym", ["reflect3", "reflect6", "rotate3"])
@pytest.mark.parametrize("n", [8, 16, 24, 12, (7, 9, 11)])
def test_symmetrize(ih, orc, sym, n):
    n3 = (n,) * 3 if np.isscalar(n) else n
    if sym != "reflect3" and len(set(n3)) > 1:
        with pytest.raises(ValueError):
            ih.symmetrize(n3, np.zeros(int(np.prod(n3))), sym)
        return
    f = mt_uniform(int(np.prod(n3)), 41, 0, 1)
    assert rel(ih.symmetrize(n3, f, sym), orc.symmetrize(n3, f, sym)) < 1e-15


def test_oc_update_matches_oracle(ih, orc):
    rho = mt_uniform(4096, 13, 0.2, 0.4)
    g = mt_uniform(4096, 17, -3.0, -0.1)
    a, lam, ok = ih.oc_update(rho, g, ih.OCConfig(volume=0.3))
    b, lamo, oko = orc.oc_update(rho, g, volume=0.3)
    assert ok and oko
    assert lam == pytest.approx(lamo, rel=1e-12)
    assert np.abs(a - b).max() < 1e-14


def test_sensitivity_filter(ih, orc):
    n = 6
    g = mt_uniform(216, 29, -1, 1)
    r = mt_uniform(216, 31, 0.1, 1)
    assert rel(ih.sensitivity_filter(n, g, r, 2.0), orc.sensitivity_filter(n, g, r, 2.0)) < 1e-14


def test_init_trig(ih, orc):
    a, fa = ih.init_trig(32, 2, 0, 0.2)
    b, fb = orc.init_trig(32, 2, 0, 0.2)
    assert not fa and not fb
    assert np.abs(a - b).max() < 1e-9
    assert abs(a.mean() - 0.200091854) < 1e-8  # reference mean for this spec


# ---------------------------------------------------------------- whole iteration (BASELINE configs[0])
@pytest.mark.parametrize("mode", ["vcycle", "mixed_defect"])
def test_32cubed_bulk_5_iterations_matches_oracle(ih, orc, mode):
    cfg = ih.RunConfig(reso=32, vol=0.2, obj="bulk", max_iter=5, precision="mixed", solver_mode=mode)
    rep = ih.run_optimization(cfg)
    recs, rho_o, flags = orc.run(reso=32, vol=0.2, obj="bulk", max_iter=5, mixed=True)
    assert not rep.solver_failed and not flags["solver_failed"]
    assert len(rep.records) == len(recs) == 5
    for r, ro in zip(rep.records, recs):
        assert abs(r["objective"] - ro["objective"]) <= 1e-4 * abs(ro["objective"])
        assert np.abs(r["C"] - ro["C"]).max() <= 1e-4 * np.abs(ro["C"]).max()
    assert np.abs(rep.density - rho_o).max() <= 1e-3


@pytest.mark.parametrize("mode", ["pcg", "mixed_defect"])
def test_fast_modes_tight_tolerance_match_oracle(ih, orc, mode):
    """Solver-independent comparison (SURVEY 8d config 1 'also at tight tol'): with both
    sides converged tightly the per-iteration C^H must agree whatever the solver."""
    tol = 1e-6
    cfg = ih.RunConfig(reso=16, vol=0.3, obj="shear", max_iter=3, precision="mixed", solver_mode=mode, tol=tol,
                       max_cycles=200)
    rep = ih.run_optimization(cfg)
    recs, rho_o, _ = orc.run(reso=16, vol=0.3, obj="shear", max_iter=3, mixed=True, tol=tol, max_cycles=200)
    assert len(rep.records) == len(recs) == 3
    for r, ro in zip(rep.records, recs):
        assert np.abs(r["C"] - ro["C"]).max() <= 1e-5 * np.abs(ro["C"]).max()
    assert np.abs(rep.density - rho_o).max() <= 1e-4


def test_pcg_converges_in_fewer_cycles_than_vcycle(ih):
    n = 32
    rho, _ = ih.init_trig(n, 2, 0, 0.2)
    phys = ih.radial_filter(n, rho, 2.0, "spline4") ** 3
    cyc = {}
    for mode in ("vcycle", "pcg"):
        hom = make_hom(ih, n, "mixed", penal=1.0, tol=1e-6, max_cycles=200, mode=mode)
        hom.set_density(phys)
        st = hom.solve_cell_problems()
        assert st["converged"]
        cyc[mode] = st["total_cycles"]
    assert cyc["pcg"] <= cyc["vcycle"]


# ---------------------------------------------------------------- runner option space vs the oracle
@pytest.mark.parametrize("opts", [
    dict(obj="npr-log", sym="reflect6"),
    dict(obj="shear", sym="reflect3"),
    dict(obj="bulk", sym="rotate3"),
    dict(obj="shear", sym="none", kernel="linear"),
    dict(obj="bulk", sym="reflect6", filter_placement="sensitivity"),
    dict(obj="npr-relaxed", sym="reflect6", init="constant", vol=0.3),
    dict(obj="bulk", sym="reflect6", penal=1.0, filter_radius=1.5),
])
def test_runner_options_3_iterations_match_oracle(ih, orc, opts):
    """Whole optimisation iterations on the bench's solver path (mixed precision, mixed_defect) across the
    runner's option space (objectives, symmetry groups, filter kernel / radius / placement, init, SIMP
    power): per-iteration objective and C^H within 1e-4 of the oracle, final design within 1e-3."""
    o = {"vol": 0.2, **opts}
    cfg = ih.RunConfig(reso=32, max_iter=3, precision="mixed", solver_mode="mixed_defect", **o)
    rep = ih.run_optimization(cfg)
    recs, rho_o, flags = orc.run(reso=32, max_iter=3, mixed=True, **o)
    assert not rep.solver_failed and not flags["solver_failed"]
    assert len(rep.records) == len(recs)
    for r, ro in zip(rep.records, recs):
        assert abs(r["objective"] - ro["objective"]) <= 1e-4 * abs(ro["objective"])
        assert np.abs(r["C"] - ro["C"]).max() <= 1e-4 * np.abs(ro["C"]).max()
    assert np.abs(rep.density - rho_o).max() <= 1e-3


@pytest.mark.parametrize("obj", ["bulk", "npr-relaxed"])
def test_all_double_3_iterations_match_oracle(ih, orc, obj):
    """Homogenizer<double> (all-f64 coefficients, stencils and nodal data, the reference's double mode) with
    its V-cycle: whole iterations against the oracle's double mode."""
    cfg = ih.RunConfig(reso=32, vol=0.2, obj=obj, max_iter=3, precision="double", solver_mode="vcycle")
    rep = ih.run_optimization(cfg)
    recs, rho_o, flags = orc.run(reso=32, vol=0.2, obj=obj, max_iter=3, mixed=False)
    assert not rep.solver_failed and not flags["solver_failed"]
    assert len(rep.records) == len(recs) == 3
    for r, ro in zip(rep.records, recs):
        assert r["cycles"] == ro["cycles"]
        assert abs(r["objective"] - ro["objective"]) <= 1e-8 * abs(ro["objective"])
        assert np.abs(r["C"] - ro["C"]).max() <= 1e-8 * np.abs(ro["C"]).max()
    assert np.abs(rep.density - rho_o).max() <= 1e-8
