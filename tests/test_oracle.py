"""CPU tests: the oracle (oracle/) pinned against the reference.

* bit-exact against the reference's own src/density.cpp + src/oc.cpp compiled
  into oracle/_ref (skipped where that build is absent);
* against the committed golden vectors made by that reference build
  (tests/golden/, tests/golden/make_golden.py);
* against the known answers of proj/tests/*.cpp and independent numpy oracles
  (explicit sparse stiffness, dense deflated solve, energy identity), the same
  strategy as proj/tests/oracles.cpp.
"""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import mt_uniform

GOLD = os.path.join(os.path.dirname(__file__), "golden")
E, NU = 1e6, 0.3


# ---------------------------------------------------------------- numpy first-principles oracles
def lvo(j):
    return (j & 1, (j >> 1) & 1, (j >> 2) & 1)


def k0_quadrature(youngs, poisson):
    """3x3x3 Gauss on [-1,1]^3, independent of the library quadrature (tests/oracles.cpp:8-52)."""
    lam = youngs * poisson / ((1 + poisson) * (1 - 2 * poisson))
    mu = youngs / (2 * (1 + poisson))
    d = np.zeros((6, 6))
    d[:3, :3] = lam
    for i in range(3):
        d[i, i] = lam + 2 * mu
        d[3 + i, 3 + i] = mu
    sgn = [[-1 if not (j >> k) & 1 else 1 for k in range(3)] for j in range(8)]
    gp = [-np.sqrt(3 / 5), 0.0, np.sqrt(3 / 5)]
    gw = [5 / 9, 8 / 9, 5 / 9]
    k = np.zeros((24, 24))
    for a in range(3):
        for b in range(3):
            for c in range(3):
                xi, et, ze = gp[a], gp[b], gp[c]
                bm = np.zeros((6, 24))
                for v in range(8):
                    s = sgn[v]
                    dx = 0.125 * s[0] * (1 + s[1] * et) * (1 + s[2] * ze) * 2
                    dy = 0.125 * s[1] * (1 + s[0] * xi) * (1 + s[2] * ze) * 2
                    dz = 0.125 * s[2] * (1 + s[0] * xi) * (1 + s[1] * et) * 2
                    bm[0, 3 * v] = dx
                    bm[1, 3 * v + 1] = dy
                    bm[2, 3 * v + 2] = dz
                    bm[3, 3 * v], bm[3, 3 * v + 1] = dy, dx
                    bm[4, 3 * v + 1], bm[4, 3 * v + 2] = dz, dy
                    bm[5, 3 * v], bm[5, 3 * v + 2] = dz, dx
                k += gw[a] * gw[b] * gw[c] / 8 * bm.T @ d @ bm
    return k


def chi_table():
    chi = np.zeros((24, 6))
    for j in range(8):
        x = lvo(j)
        chi[3 * j:3 * j + 3, 0] = (x[0], 0, 0)
        chi[3 * j:3 * j + 3, 1] = (0, x[1], 0)
        chi[3 * j:3 * j + 3, 2] = (0, 0, x[2])
        chi[3 * j:3 * j + 3, 3] = (x[1] / 2, x[0] / 2, 0)
        chi[3 * j:3 * j + 3, 4] = (0, x[2] / 2, x[1] / 2)
        chi[3 * j:3 * j + 3, 5] = (x[2] / 2, 0, x[0] / 2)
    return chi


def global_k(orc, n, rho, p, k0):
    """Explicit global stiffness, dof = 3*loc + c (tests/oracles.cpp:54-74)."""
    locs = orc.grid_locs(n).reshape(n, n, n)  # [z][y][x]
    nv = n ** 3
    K = np.zeros((3 * nv, 3 * nv))
    for e in range(nv):
        ex, ey, ez = e % n, (e // n) % n, e // (n * n)
        ids = [locs[(ez + d[2]) % n, (ey + d[1]) % n, (ex + d[0]) % n] for d in map(lvo, range(8))]
        dofs = np.array([3 * i + c for i in ids for c in range(3)])
        K[np.ix_(dofs, dofs)] += rho[e] ** p * k0
    return K, locs


def macro_f(orc, n, rho, p, k0, locs):
    nv = n ** 3
    chi = chi_table()
    F = np.zeros((3 * nv, 6))
    for e in range(nv):
        ex, ey, ez = e % n, (e // n) % n, e // (n * n)
        ids = [locs[(ez + d[2]) % n, (ey + d[1]) % n, (ex + d[0]) % n] for d in map(lvo, range(8))]
        dofs = np.array([3 * i + c for i in ids for c in range(3)])
        F[dofs] += rho[e] ** p * (k0 @ chi)
    return F


def solve_deflated(K, f):
    """tests/oracles.cpp:126-148."""
    nv = K.shape[0] // 3
    f = f.copy()
    for c in range(3):
        f[c::3] -= f[c::3].mean()
    A = K.copy()
    shift = np.mean(np.diag(A))
    for c in range(3):
        idx = np.arange(c, 3 * nv, 3)
        A[np.ix_(idx, idx)] += shift / nv
    u = np.linalg.solve(A, f)
    for c in range(3):
        u[c::3] -= u[c::3].mean()
    return u


def homogenized_tensor(orc, n, rho, p, youngs, poisson):
    """Energy identity M C_ij = chi_i'K chi_j - u_j' f_i (tests/oracles.cpp:150-176)."""
    k0 = orc.k0(youngs, poisson)
    K, locs = global_k(orc, n, rho, p, k0)
    F = macro_f(orc, n, rho, p, k0, locs)
    U = np.stack([solve_deflated(K, F[:, i]) for i in range(6)], 1)
    chi = chi_table()
    ckc = sum(rho[e] ** p for e in range(n ** 3)) * 0  # placeholder for clarity
    ckc = np.zeros((6, 6))
    for e in range(n ** 3):
        ckc += rho[e] ** p * chi.T @ k0 @ chi
    c = (ckc - F.T @ U) / n ** 3
    return 0.5 * (c + c.T)


# ---------------------------------------------------------------- K0 / material (tests/test_material.cpp)
def test_k0_known_answers(orc):
    k = orc.k0(1.0, 0.3)
    assert k[0, 0] == pytest.approx(0.23504273504273504, rel=1e-12)
    assert np.abs(k - k0_quadrature(1.0, 0.3)).max() < 1e-14 * np.abs(k).max()
    assert np.abs(k - k.T).max() < 1e-15
    lam, mu = 0.3 / (1.3 * 0.4) / 72, 1 / 2.6 / 72
    assert lam == pytest.approx(0.0080128, rel=1e-4) and mu == pytest.approx(0.0053419, rel=1e-4)
    vals = np.array([-8 * lam - 8 * mu, -6 * lam - 6 * mu, -6 * lam + 6 * mu, -4 * lam - 10 * mu, -3 * lam - 3 * mu,
                     -3 * lam + 3 * mu, -2 * lam - 8 * mu, 2 * lam - 4 * mu, 3 * lam - 3 * mu, 3 * lam + 3 * mu,
                     4 * lam + 4 * mu, 6 * lam - 6 * mu, 6 * lam + 6 * mu, 8 * lam + 32 * mu])
    assert np.abs(k.ravel()[:, None] - vals[None, :]).min(1).max() < 1e-14  # 14 values
    ev = np.linalg.eigvalsh(orc.k0(1.0, 0.25))
    assert (np.abs(ev) < 1e-10 * np.abs(ev).max()).sum() == 6  # 6-dim null space
    k2 = orc.k0(2.5, 0.2)
    for c in range(3):
        t = np.zeros(24)
        t[c::3] = 1
        assert np.abs(k2 @ t).max() < 1e-14 * np.abs(k2).max()


def test_energy_identity_base_elasticity(orc):
    k = orc.k0(E, NU)
    chi = chi_table()
    lam, mu = E * NU / ((1 + NU) * (1 - 2 * NU)), E / (2 * (1 + NU))
    base = np.zeros((6, 6))
    base[:3, :3] = lam
    for i in range(3):
        base[i, i] = lam + 2 * mu
        base[3 + i, 3 + i] = mu
    assert np.abs(chi.T @ k @ chi - base).max() < 1e-9 * np.abs(base).max()


# ---------------------------------------------------------------- grid (tests/test_grid.cpp)
@pytest.mark.parametrize("n", [4, 6, 8, (6, 10, 8), (5, 7, 9)])
def test_grid_colour_block_layout(orc, n):
    n3 = (n,) * 3 if np.isscalar(n) else n
    locs = orc.grid_locs(n3)
    assert np.array_equal(np.sort(locs), np.arange(np.prod(n3)))
    base, dim = orc.grid_info(n3)
    nx, ny, nz = n3
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                cid = (x & 1) | ((y & 1) << 1) | ((z & 1) << 2)
                exp = base[cid] + (x >> 1) + ((y >> 1) + (z >> 1) * dim[cid][1]) * dim[cid][0]
                assert locs[x + nx * (y + ny * z)] == exp


def test_every_element_has_eight_colours():
    n = 4
    for e in range(n ** 3):
        ex, ey, ez = e % n, (e // n) % n, e // 16
        cols = {((ex + d[0]) % n & 1) | (((ey + d[1]) % n & 1) << 1) | (((ez + d[2]) % n & 1) << 2)
                for d in map(lvo, range(8))}
        assert len(cols) == 8


# ---------------------------------------------------------------- fem vs explicit sparse
def test_apply_matches_global_matrix(orc):
    n = 4
    rho = mt_uniform(64, 3, 1e-3, 1.0)
    u = mt_uniform(192, 4, -1, 1)
    K, _ = global_k(orc, n, rho, 3.0, orc.k0(E, NU))
    y = orc.fem(n, "apply", rho ** 3, u=u, E=E, nu=NU).ravel()
    assert np.abs(y - K @ u).max() < 1e-10 * np.abs(K @ u).max()


# ---------------------------------------------------------------- multigrid (tests/test_multigrid.cpp)
def test_restriction_constant_and_delta(orc):
    r = np.full(3 * 512, 0.75)
    assert np.allclose(orc.restrict(8, r), 6.0, rtol=1e-14)
    locs = orc.grid_locs(8)
    r = np.zeros((512, 3))
    r[locs[3 + 8 * (3 + 8 * 3)], 1] = 1.0
    f = orc.restrict(8, r)
    nz = f[:, 1][f[:, 1] != 0]
    assert np.allclose(nz, 0.125) and f[:, 1].sum() == pytest.approx(1.0)


def test_transfer_adjoint(orc):
    r = mt_uniform(3 * 512, 101, -1, 1)
    v = mt_uniform(3 * 64, 103, -1, 1)
    a = np.dot(orc.restrict(8, r).ravel(), v)
    b = np.dot(r, orc.prolong_add(8, v, np.zeros(3 * 512)).ravel())
    assert a == pytest.approx(b, rel=1e-12)


def test_galerkin_identity(orc):
    """level-1 stencil == I^T K0 I (tests/test_multigrid.cpp:100-111)."""
    n = 8
    rho = mt_uniform(512, 211, 1e-3, 1.0)
    h = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=False)
    h.set_density(rho)
    K, _ = global_k(orc, n, rho, 3.0, orc.k0(E, NU))
    # interpolation matrix column by column through prolong_add
    P = np.zeros((3 * 512, 3 * 64))
    for j in range(3 * 64):
        e = np.zeros(3 * 64)
        e[j] = 1.0
        P[:, j] = orc.prolong_add(8, e, np.zeros(3 * 512)).ravel()
    rki = P.T @ K @ P
    st = h.stencil(1)
    locs = orc.grid_locs(4).reshape(4, 4, 4)
    inv = {int(locs[z, y, x]): (x, y, z) for z in range(4) for y in range(4) for x in range(4)}
    K1 = np.zeros((192, 192))
    for loc in range(64):
        x, y, z = inv[loc]
        for t in range(27):
            dx, dy, dz = t % 3 - 1, (t // 3) % 3 - 1, t // 9 - 1
            w = locs[(z + dz) % 4, (y + dy) % 4, (x + dx) % 4]
            K1[3 * loc:3 * loc + 3, 3 * w:3 * w + 3] += st[loc, t]
    assert np.linalg.norm(K1 - rki) < 1e-10 * np.linalg.norm(rki)


def test_vcycle_monotone_small(orc):
    """tests/test_multigrid.cpp:235-252."""
    n = 8
    rho = mt_uniform(512, 257, 0.1, 1.0)
    h = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=False)
    h.set_density(rho)
    f = orc.fem(n, "macro", rho ** 3, E=E, nu=NU, load=0)
    h.level_field(0, "f", f - f.mean(0))
    h.level_field(0, "u", np.zeros_like(f))
    prev = 1e300
    for _ in range(12):
        rel = h.v_cycle()
        assert rel < prev
        prev = rel
    assert prev < 1e-6


# ---------------------------------------------------------------- homogenization (tests/test_homogenization.cpp)
def test_solid_and_rho_min(orc):
    h = orc.Homogenizer(8, E=E, nu=NU, penal=3.0, mixed=False, tol=1e-10, max_cycles=200)
    h.set_density(np.ones(512))
    h.solve_cell_problems()
    c = h.effective_tensor()
    assert c[0, 0] == pytest.approx(1346153.846153846, rel=1e-9)
    assert c[0, 1] == pytest.approx(576923.0769230769, rel=1e-9)
    assert c[3, 3] == pytest.approx(384615.3846153846, rel=1e-9)
    h = orc.Homogenizer(4, E=E, nu=NU, penal=3.0, mixed=False, tol=1e-10, max_cycles=200)
    h.set_density(np.full(64, 1e-3))
    h.solve_cell_problems()
    lam, mu = E * NU / ((1 + NU) * (1 - 2 * NU)), E / (2 * (1 + NU))
    assert h.effective_tensor()[0, 0] == pytest.approx(1e-9 * (lam + 2 * mu), rel=1e-10)


@pytest.mark.parametrize("n", [4, 6])
def test_tensor_matches_sparse_direct_oracle(orc, n):
    rho = mt_uniform(n ** 3, 1000 + n, 1e-3, 1.0)
    h = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=False, tol=1e-10, max_cycles=200)
    h.set_density(rho)
    assert h.solve_cell_problems()["converged"]
    c = h.effective_tensor()
    cref = homogenized_tensor(orc, n, rho, 3.0, E, NU)
    assert np.abs(c - cref).max() < 1e-6 * np.abs(cref).max()


def test_sensitivity_finite_difference(orc):
    """bulk-seed sensitivity vs central differences (tests/test_homogenization.cpp:147-174)."""
    n = 4
    rho = mt_uniform(64, 23, 0.3, 0.7)
    h = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=False, tol=1e-10, max_cycles=200)
    h.set_density(rho)
    h.solve_cell_problems()
    c = h.effective_tensor()
    val, seed = orc.objective("bulk", c)
    g = h.tensor_sensitivity(seed)

    def fval(r):
        hh = orc.Homogenizer(n, E=E, nu=NU, penal=3.0, mixed=False, tol=1e-10, max_cycles=200)
        hh.set_density(r)
        hh.solve_cell_problems()
        return orc.objective("bulk", hh.effective_tensor())[0]
    for e in (0, 17, 42, 63):
        rp, rm = rho.copy(), rho.copy()
        rp[e] += 1e-4
        rm[e] -= 1e-4
        fd = (fval(rp) - fval(rm)) / 2e-4
        assert g[e] == pytest.approx(fd, rel=1e-3)


# ---------------------------------------------------------------- objectives (tests/test_objective.cpp)
def test_objectives_known_values_and_python_expr(orc):
    import paper_2301_08911_b200 as ih
    lam, mu = E * NU / ((1 + NU) * (1 - 2 * NU)), E / (2 * (1 + NU))
    base = ih.BaseMaterial(E, NU).elasticity()
    assert orc.objective("bulk", base)[0] == pytest.approx(-833333.3333333333, rel=1e-12)
    assert orc.objective("shear", base)[0] == pytest.approx(-384615.3846153846, rel=1e-12)
    rng = np.random.default_rng(5)
    cm = base + rng.uniform(-1e4, 1e4, (6, 6))
    cm = 0.5 * (cm + cm.T)
    for name, pyexpr in [("bulk", ih.bulk_objective()), ("shear", ih.shear_objective()),
                         ("npr-relaxed", ih.npr_relaxed(0.8, 3)), ("npr-log", ih.npr_log(0.6, -1e-3, 0.5))]:
        v, g = orc.objective(name, cm, iter=3)
        assert pyexpr.eval(cm) == pytest.approx(v, rel=1e-14)
        assert np.allclose(pyexpr.backward(1.0, cm), g, rtol=1e-13, atol=1e-300)
        # finite differences of the python Expr
        h = 1e-3
        for (i, j) in [(0, 0), (0, 1), (1, 2), (3, 3)]:
            cp, cn = cm.copy(), cm.copy()
            cp[i, j] += h
            cn[i, j] -= h
            fd = (pyexpr.eval(cp) - pyexpr.eval(cn)) / (2 * h)
            assert g[i, j] == pytest.approx(fd, rel=1e-5, abs=1e-12)


def test_expr_domain_errors():
    import paper_2301_08911_b200 as ih
    with pytest.raises(ih.EvalError):
        ih.Expr.entry(0, 0).log().eval(-np.eye(6))
    with pytest.raises(ih.EvalError):
        (ih.Expr.entry(0, 0) / ih.Expr.entry(1, 2)).eval(np.eye(6))
    with pytest.raises(ValueError):
        ih.Expr.entry(6, 0)
    assert (ih.Expr.constant(2.0) * 3.0).op == "const"  # eager constant folding


def test_converge_checker_traces():
    """inc/oc.hpp:35-61 via tests/test_oc.cpp:116-143."""
    import paper_2301_08911_b200 as ih
    c = ih.ConvergeChecker()
    assert [c.update(1.0) for _ in range(4)] == [False, False, False, True]
    alt = ih.ConvergeChecker()
    assert not any(alt.update(11.0 if i % 2 else 10.0) for i in range(50))
    runs = ih.ConvergeChecker()
    v = 1.0
    runs.update(v)
    out = []
    for r in [4e-4, 4e-4, 6e-4, 4e-4, 4e-4, 4e-4]:
        v *= 1 + r
        out.append(runs.update(v))
    assert out == [False] * 5 + [True]


# ---------------------------------------------------------------- density / OC vs the reference's own code
needs_ref = pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref",
                                                               "libihom_ref.so")), reason="oracle/_ref not built")
_dp = C.POINTER(C.c_double)


def _p(a):
    return a.ctypes.data_as(_dp)


@needs_ref
@pytest.mark.parametrize("kernel,radius", [(0, 1.0), (0, 2.0), (1, 2.0), (1, 2.5), (0, 3.5)])
def test_filter_bit_exact_vs_reference(orc, kernel, radius):
    n = (8, 6, 10)
    f = mt_uniform(480, 31, 0, 1)
    out = np.zeros(480)
    orc.ref().ref_radial_filter(*n, _p(f), C.c_double(radius), kernel, _p(out))
    assert np.array_equal(orc.radial_filter(n, f, radius, "linear" if kernel == 0 else "spline4"), out)


@needs_ref
@pytest.mark.parametrize("sym", [1, 2, 3])
def test_symmetrize_bit_exact_vs_reference(orc, sym):
    f = mt_uniform(1000, 41, 0, 1)
    ref = f.copy()
    assert orc.ref().ref_symmetrize(10, 10, 10, _p(ref), sym) == 0
    name = {1: "reflect3", 2: "reflect6", 3: "rotate3"}[sym]
    assert np.array_equal(orc.symmetrize(10, f, name), ref)


@needs_ref
@pytest.mark.parametrize("seed,basis,vol", [(0, 2, 0.2), (3, 1, 0.3), (7, 3, 0.5)])
def test_init_trig_bit_exact_vs_reference(orc, seed, basis, vol):
    out = np.zeros(16 ** 3)
    fb = orc.ref().ref_init_trig(16, 16, 16, basis, C.c_ulonglong(seed), C.c_double(vol), C.c_double(15.0), _p(out))
    mine, fb2 = orc.init_trig(16, basis, seed, vol)
    assert bool(fb) == fb2
    assert np.array_equal(mine, out)


@needs_ref
@pytest.mark.parametrize("case", range(4))
def test_oc_update_bit_exact_vs_reference(orc, case):
    rng = np.random.default_rng(case)
    rho = rng.uniform(0.2, 0.45, 6 * 7 * 8)
    g = rng.uniform(-3.0, -0.1 if case % 2 else 2.0, rho.size)
    vol = [0.3, 0.35, 0.5, 0.25][case]
    out = np.zeros_like(rho)
    lam = C.c_double()
    ok = orc.ref().ref_oc_update(6, 7, 8, _p(rho), _p(g), C.c_double(vol), C.c_double(0.05), C.c_double(0.5),
                                 _p(out), C.byref(lam))
    mine, lam2, ok2 = orc.oc_update(rho, g, volume=vol)
    assert bool(ok) == ok2
    assert lam.value == lam2
    assert np.array_equal(mine, out)


@needs_ref
def test_sensitivity_filter_and_density_expr_bit_exact_vs_reference(orc):
    n = 6
    g = mt_uniform(216, 29, -1, 1)
    r = mt_uniform(216, 31, 0.1, 1)
    out = np.zeros(216)
    orc.ref().ref_sensitivity_filter(n, n, n, _p(g), _p(r), C.c_double(2.0), _p(out))
    assert np.array_equal(orc.sensitivity_filter(n, g, r, 2.0), out)
    phys, gd = np.zeros(216), np.zeros(216)
    orc.ref().ref_density_expr(n, n, n, C.c_double(2.0), 1, C.c_double(3.0), _p(r), _p(phys), _p(g), _p(gd))
    pre = orc.radial_filter(n, r, 2.0, "spline4")
    assert np.array_equal(pre ** 3 if False else np.power(pre, 3.0), phys) or np.abs(np.power(pre, 3.0) - phys).max() < 1e-16
    mine_gd = orc.radial_filter(n, g * 3.0 * np.power(pre, 2.0), 2.0, "spline4")
    assert np.abs(mine_gd - gd).max() < 1e-15


# ---------------------------------------------------------------- golden vectors from the reference build
def test_golden_vectors(orc):
    path = os.path.join(GOLD, "reference_density_oc.npz")
    assert os.path.exists(path), "run tests/golden/make_golden.py where /root/reference is present"
    z = np.load(path)
    n = tuple(z["filter_n"])
    assert np.array_equal(orc.radial_filter(n, z["filter_in"], 2.0, "spline4"), z["filter_out_spline4_r2"])
    assert np.array_equal(orc.radial_filter(n, z["filter_in"], 1.5, "linear"), z["filter_out_linear_r15"])
    assert np.array_equal(orc.symmetrize(8, z["sym_in"], "reflect6"), z["sym_out_reflect6"])
    rho, fb = orc.init_trig(16, 2, 0, 0.2)
    assert np.array_equal(rho, z["trig16_b2_s0_v02"])
    out, lam, ok = orc.oc_update(z["oc_rho"], z["oc_sens"], volume=0.3)
    assert np.array_equal(out, z["oc_out"]) and lam == float(z["oc_lambda"])


# ---------------------------------------------------------------- runner semantics (tests/test_runner.cpp)
def test_first_iteration_objective(orc):
    recs, rho, fl = orc.run(reso=8, vol=0.5, obj="bulk", init="constant", sym="none", max_iter=1, mixed=False)
    assert recs[0]["objective"] == pytest.approx(0.125 * -833333.3333333333, rel=1e-9)


def test_short_run_invariants(orc):
    recs, rho, fl = orc.run(reso=8, vol=0.3, obj="bulk", seed=3, max_iter=6, mixed=False, sym="reflect3")
    assert not fl["solver_failed"]
    assert recs[0]["volume"] == pytest.approx(0.3, rel=1e-3)
    for r in recs[1:]:
        assert r["volume"] <= 0.3 + 1e-6
    assert rho.min() >= 1e-3 and rho.max() <= 1.0


def test_hadamard_basis_tables_reproduce_k0():
    """The generated sum/difference-basis element stiffness (csrc/hada_gen.cuh, tools/gen_hada.py) is
    K0 itself: for arbitrary (lam', mu') and q, y = Hb^T (q W) (Hb u) with W from the 45 generated
    terms and the 8 (alpha, beta) classes equals q K0 u, K0 from the oracle (src/material.cpp:39-69).
    Also the C^H identity d^T K0 d' = (Hb d)^T W (Hb d') used by the tensor pass."""
    import os
    import re

    import numpy as np

    import oracle

    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2301_08911_b200", "csrc", "hada_gen.cuh")).read()
    alpha = [int(x) for x in re.search(r"kHadaAlpha\[kHadaClasses\] = \{([^}]*)\}", src).group(1).split(",")]
    beta = [int(x) for x in re.search(r"kHadaBeta\[kHadaClasses\] = \{([^}]*)\}", src).group(1).split(",")]
    terms = []
    for m in re.finditer(r"w\[(\d+)\] = (?:fma\()?\(?(-?)qh\[(\d+)\]\)? \* uh\[(\d+)\]|"
                         r"w\[(\d+)\] = fma\(\(?(-?)qh\[(\d+)\]\)?, uh\[(\d+)\]", src):
        g = m.groups()
        r, sg, k, c = (g[0], g[1], g[2], g[3]) if g[0] is not None else (g[4], g[5], g[6], g[7])
        terms.append((int(r), int(c), int(k), -1.0 if sg == "-" else 1.0))
    assert len(terms) == 45
    E, nu = 1.0, 0.3
    K0 = oracle.k0(E, nu).reshape(24, 24)
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)) / 72.0, E / (2 * (1 + nu)) / 72.0  # lam', mu'
    h1 = np.array([[1, 1], [-1, 1]])
    Hb = np.kron(np.kron(h1, np.kron(h1, h1)), np.eye(3))
    W = np.zeros((24, 24))
    for r, c, k, sg in terms:
        W[r, c] += sg * (lam * alpha[k] + mu * beta[k]) / 64.0
    assert np.allclose(Hb.T @ W @ Hb, K0, rtol=0, atol=1e-14 * np.abs(K0).max())
    rng = np.random.default_rng(3)
    d1, d2 = rng.uniform(-1, 1, 24), rng.uniform(-1, 1, 24)
    assert abs(d1 @ K0 @ d2 - (Hb @ d1) @ W @ (Hb @ d2)) < 1e-13
