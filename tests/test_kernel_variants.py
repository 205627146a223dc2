"""Kernel variants that stay in the library are bit-identical to their reference forms,
except the sum-factorised sweep (tolerance). The f32 level-0 kernels run inside the mixed_defect inner
cycle, so whole cell solves are compared.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(ih, n, knobs, fabric_p=0, precision="mixed", mode="mixed_defect"):
    # the bitwise comparisons below are between stencil-form variants: the sum-factorised element
    # sweep (HSWEEP*, a different association of the same sums) is compared at tolerance separately
    knobs = {"HSWEEP": 0, "HSWEEP32": 0, "STENCIL_F32": 0, "TRANSFER_F32": 0, **knobs}
    for k, v in knobs.items():
        ih.set_knob(k, v)
    rho, _ = ih.init_trig(n if np.isscalar(n) else n[0], 2, 0, 0.3) if np.isscalar(n) else (None, None)
    nv = n ** 3 if np.isscalar(n) else int(np.prod(n))
    if rho is None:
        rho = np.random.default_rng(4).uniform(0.05, 1.0, nv)
    phys = np.asarray(rho) ** 3
    try:
        if fabric_p:
            fab = ih.Fabric.local(fabric_p)

            def body(r):
                hom = ih.Homogenizer(n, penal=1.0, precision=precision, opts=ih.SolverOptions(tol=1e-4, mode=mode),
                                     fabric=fab, rank=r)
                m = n * n * hom.planes
                hom.set_density(np.ascontiguousarray(phys[hom.z0 * n * n: hom.z0 * n * n + m]))
                st = hom.solve_cell_problems()
                out = (st["total_cycles"], hom.effective_tensor(), [hom.displacement(i) for i in range(6)])
                hom.close()
                return out
            res = ih.run_slabs(fabric_p, body)
            fab.close()
            return res[0][0], res[0][1], [np.concatenate([r[2][i] for r in res]) for i in range(6)]
        hom = ih.Homogenizer(n, penal=1.0, precision=precision, opts=ih.SolverOptions(tol=1e-4, mode=mode))
        hom.set_density(phys)
        st = hom.solve_cell_problems()
        out = (st["total_cycles"], hom.effective_tensor(), [hom.displacement(i) for i in range(6)])
        hom.close()
        return out
    finally:
        ih.set_knob("L0_SWEEP", 1)
        ih.set_knob("L0_SWEEP2", 1)
        ih.set_knob("ZERO_START", 1)
        ih.set_knob("SUBMEANS_FLAT", 1)
        ih.set_knob("FUSED_UPDATE", 1)
        ih.set_knob("RHS_PAIRS", 1)
        ih.set_knob("RHS_GROUP", 0)
        ih.set_knob("HSWEEP", 1)
        ih.set_knob("HSWEEP32", 1)
        ih.set_knob("HBM_LIMIT_MB", 0)
        ih.set_knob("STENCIL_F32", 1)
        ih.set_knob("TRANSFER_F32", 1)
        ih.set_knob("PROJECT_NORM", 1)
        ih.set_knob("MACRO_SUMS", 1)
        ih.set_knob("U_HOST", 0)
        ih.set_knob("BOTTOM_CYCLE", 1)
        ih.set_knob("GS_PAIR", 0)
        ih.set_knob("STENCIL_STREAM", 1)


@pytest.mark.parametrize("precision", ["mixed", "double"])
def test_energy_cache_bit_identical_and_invalidated(ih, precision):
    n = 16
    rho = np.random.default_rng(11).uniform(0.05, 1.0, n ** 3) ** 3
    seed = np.arange(36.0).reshape(6, 6) / 36.0

    def run(cache):
        ih.set_knob("ENERGY_CACHE", cache)
        try:
            hom = ih.Homogenizer(n, penal=1.0, precision=precision, opts=ih.SolverOptions(tol=1e-6))
            hom.set_density(rho)
            hom.solve_cell_problems()
            C = hom.effective_tensor()
            s1 = hom.tensor_sensitivity(seed)
            # a displacement written through the API must drop the cached energies
            u0 = hom.displacement(0)
            hom.set_displacement(0, 0.5 * u0)
            s2 = hom.tensor_sensitivity(seed)
            hom.close()
            return C, s1, s2
        finally:
            ih.set_knob("ENERGY_CACHE", 1)
    C0, a0, b0 = run(0)
    C1, a1, b1 = run(1)
    np.testing.assert_array_equal(C0, C1)
    np.testing.assert_array_equal(a0, a1)
    np.testing.assert_array_equal(b0, b1)
    assert np.max(np.abs(b1 - a1)) > 0


@pytest.mark.parametrize("precision,mode", [("mixed", "mixed_defect"), ("mixed", "vcycle"), ("double", "vcycle"),
                                            ("mixed", "pcg")])
@pytest.mark.parametrize("n", [32, 64])
def test_sweep_level0_kernels_bit_identical(ih, n, precision, mode):
    """z-plane sweep (shared-memory plane ring; x-paired FFMA2 form for f32 on 64-wide grids) vs the
    direct-load level-0 apply/residual kernels."""
    base = _solve(ih, n, {"L0_SWEEP": 0}, precision=precision, mode=mode)
    for knobs in ({"L0_SWEEP": 1, "L0_SWEEP2": 0}, {"L0_SWEEP": 1, "L0_SWEEP2": 1}):
        sw = _solve(ih, n, knobs, precision=precision, mode=mode)
        assert sw[0] == base[0]
        np.testing.assert_array_equal(sw[1], base[1])
        for a, b in zip(sw[2], base[2]):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("mode", ["mixed_defect", "vcycle"])
def test_sweep_level0_kernels_bit_identical_on_slabs(ih, mode):
    base = _solve(ih, 64, {"L0_SWEEP": 0}, fabric_p=2, mode=mode)
    sw = _solve(ih, 64, {"L0_SWEEP": 1}, fabric_p=2, mode=mode)
    assert sw[0] == base[0]
    np.testing.assert_array_equal(sw[1], base[1])
    for a, b in zip(sw[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("precision,mode", [("mixed", "mixed_defect"), ("mixed", "vcycle"), ("double", "vcycle"),
                                            ("mixed", "pcg")])
@pytest.mark.parametrize("n", [32, 64, (16, 16, 10)])
def test_zero_start_sweeps_bit_identical(ih, n, precision, mode):
    """Zero-start pre-smoothing (colours > c of the first sweep are known zeros: not read, not cleared)."""
    base = _solve(ih, n, {"ZERO_START": 0}, precision=precision, mode=mode)
    zs = _solve(ih, n, {"ZERO_START": 1}, precision=precision, mode=mode)
    assert zs[0] == base[0]
    np.testing.assert_array_equal(zs[1], base[1])
    for a, b in zip(zs[2], base[2]):
        np.testing.assert_array_equal(a, b)


def test_zero_start_sweeps_bit_identical_on_slabs(ih):
    base = _solve(ih, 64, {"ZERO_START": 0}, fabric_p=4)
    zs = _solve(ih, 64, {"ZERO_START": 1}, fabric_p=4)
    assert zs[0] == base[0]
    np.testing.assert_array_equal(zs[1], base[1])
    for a, b in zip(zs[2], base[2]):
        np.testing.assert_array_equal(a, b)


BASE = {"L0_SWEEP": 0, "ZERO_START": 0}
VARIANTS = [
    {"ZERO_START": 1, "L0_SWEEP": 0},
    {"ZERO_START": 1, "L0_SWEEP": 1, "L0_SWEEP2": 1},  # the default configuration
]


@pytest.mark.parametrize("precision,mode", [("mixed", "mixed_defect"), ("mixed", "pcg"), ("mixed", "vcycle")])
@pytest.mark.parametrize("n", [32, 128, (128, 64, 64)])
def test_gs_sweep_bit_identical(ih, n, precision, mode):
    """Zero-start GS passes and z-plane residual sweeps (the defaults) == plain direct-load kernels."""
    base = _solve(ih, n, BASE, precision=precision, mode=mode)
    for knobs in VARIANTS:
        v = _solve(ih, n, {**BASE, **knobs}, precision=precision, mode=mode)
        assert v[0] == base[0], knobs
        np.testing.assert_array_equal(v[1], base[1])
        for a, b in zip(v[2], base[2]):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("P", [2, 4])
def test_gs_sweep_bit_identical_on_slabs(ih, P):
    base = _solve(ih, 128, BASE, fabric_p=P)
    v = _solve(ih, 128, {**BASE, **VARIANTS[-1]}, fabric_p=P)
    assert v[0] == base[0]
    np.testing.assert_array_equal(v[1], base[1])
    for a, b in zip(v[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("precision", ["mixed", "double"])
@pytest.mark.parametrize("n", [16, 32])
def test_unrolled_element_galerkin_bit_identical(ih, n, precision):
    """Level-1 Galerkin with the compile-time term list == the table-driven kernel."""
    rho = np.random.default_rng(21).uniform(0.05, 1.0, n ** 3)
    out = []
    for unrolled in (0, 1):
        ih.set_knob("GAL_UNROLLED", unrolled)
        try:
            hom = ih.Homogenizer(n, penal=3.0, precision=precision)
            hom.set_density(rho)
            out.append(hom.hierarchy().stencil(1))
            hom.close()
        finally:
            ih.set_knob("GAL_UNROLLED", 1)
    np.testing.assert_array_equal(out[0], out[1])



@pytest.mark.parametrize("precision,mode", [("mixed", "mixed_defect"), ("double", "vcycle")])
def test_flat_sub_means_bit_identical(ih, precision, mode):
    base = _solve(ih, 32, {"SUBMEANS_FLAT": 0}, precision=precision, mode=mode)
    v = _solve(ih, 32, {"SUBMEANS_FLAT": 1}, precision=precision, mode=mode)
    assert v[0] == base[0]
    np.testing.assert_array_equal(v[1], base[1])
    for a, b in zip(v[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,P", [(32, 0), (64, 0), (64, 2), (64, 4)])
def test_fused_update_bit_identical(ih, n, P):
    """u += e folded into the defect-residual sweep (ping-pong buffers) == separate axpy + residual."""
    base = _solve(ih, n, {"FUSED_UPDATE": 0}, fabric_p=P)
    v = _solve(ih, n, {"FUSED_UPDATE": 1}, fabric_p=P)
    assert v[0] == base[0]
    np.testing.assert_array_equal(v[1], base[1])
    for a, b in zip(v[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,P", [(16, 0), (32, 0), (64, 0), ((64, 32, 48), 0), (32, 2), (64, 4)])
def test_rhs_pairs_bit_identical(ih, n, P):
    """Cell problems solved in lockstep pairs (coarse stencils streamed once per pair) == one by one:
    same cycle counts, tensors and displacements bit for bit."""
    base = _solve(ih, n, {"RHS_PAIRS": 0}, fabric_p=P)
    for group in (2, 3, 6):  # lockstep pairs, triples, all six cell problems
        v = _solve(ih, n, {"RHS_PAIRS": 1, "RHS_GROUP": group}, fabric_p=P)
        assert v[0] == base[0], group
        np.testing.assert_array_equal(v[1], base[1])
        for a, b in zip(v[2], base[2]):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n", [32, 64])
def test_hadamard_sweep_matches_stencil_sweep(ih, n):
    """The sum-factorised element sweep (HSWEEP / HSWEEP32, hsweep_kernels.cuh) is the same operator as
    the vertex-stencil sweep with a different association of the f64/f32 sums: whole cell solves agree
    to rounding (same cycle counts, C^H and displacements to ~1e-9 / 1e-6 relative)."""
    base = _solve(ih, n, {"HSWEEP": 0, "HSWEEP32": 0})
    for knobs in ({"HSWEEP": 1, "HSWEEP32": 0}, {"HSWEEP": 1, "HSWEEP32": 1}):
        h = _solve(ih, n, knobs)
        assert h[0] == base[0]
        tol = 1e-9 if knobs["HSWEEP32"] == 0 else 2e-6
        assert np.abs(h[1] - base[1]).max() <= tol * np.abs(base[1]).max()
        for a, b in zip(h[2], base[2]):
            assert np.linalg.norm(a - b) <= tol * 10 * max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("P", [0, 2])
def test_memory_levers_bit_identical(ih, P):
    """With the free HBM capped (HBM_LIMIT_MB) the solver drops the lockstep grouping (group size 1) and
    the energy cache; both are pure optimisations, so cycle counts, C^H and displacements are bitwise
    those of the default run (here: groups of six and the cache)."""
    # U_HOST=-1: the host-staged layout (which the cap would also select) is tested in test_host_staged.py
    base = _solve(ih, 32, {"U_HOST": -1}, fabric_p=P)
    low = _solve(ih, 32, {"HBM_LIMIT_MB": 256, "U_HOST": -1}, fabric_p=P)
    assert low[0] == base[0]
    np.testing.assert_array_equal(low[1], base[1])
    for a, b in zip(low[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,P", [(32, 0), (64, 0), (64, 2)])
def test_stencil_f32_accumulation_matches(ih, n, P):
    """Stencil-level (coarse) GS and residual of the inner f32 cycle with f32 products/sums
    (STENCIL_F32) instead of f64: the coarse-grid correction changes at f32 rounding, the outer f64
    defect residual is untouched, so whole solves agree to the solver tolerance (same cycle counts,
    C^H to 1e-6)."""
    base = _solve(ih, n, {"STENCIL_F32": 0}, fabric_p=P)
    v = _solve(ih, n, {"STENCIL_F32": 1}, fabric_p=P)
    assert v[0] == base[0]
    assert np.abs(v[1] - base[1]).max() <= 1e-6 * np.abs(base[1]).max()


@pytest.mark.parametrize("n,P", [(32, 0), (64, 0), (64, 2)])
def test_transfer_f32_matches(ih, n, P):
    """Restriction / prolongation of the inner f32 cycle in f32 arithmetic (TRANSFER_F32; the weights are
    powers of two, so only the sums round in f32): same cycle counts, C^H to 1e-6."""
    base = _solve(ih, n, {"TRANSFER_F32": 0}, fabric_p=P)
    v = _solve(ih, n, {"TRANSFER_F32": 1}, fabric_p=P)
    assert v[0] == base[0]
    assert np.abs(v[1] - base[1]).max() <= 1e-6 * np.abs(base[1]).max()


@pytest.mark.parametrize("P", [0, 2])
def test_project_norm_bit_identical(ih, P):
    """Load projection and its norm in one pass (PROJECT_NORM) == remove_translations + norm, bitwise."""
    base = _solve(ih, 32, {"PROJECT_NORM": 0, "MACRO_SUMS": 0}, fabric_p=P)  # both legs sum f separately
    v = _solve(ih, 32, {"PROJECT_NORM": 1, "MACRO_SUMS": 0}, fabric_p=P)
    assert v[0] == base[0]
    np.testing.assert_array_equal(v[1], base[1])
    for a, b in zip(v[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,P", [(32, 0), (48, 0), (32, 2)])
def test_macro_sums_match(ih, n, P):
    """Macro force with the load's component sums folded into the same pass (MACRO_SUMS: per-block
    partials of the macro-force grid, then the deterministic component-sum reduction) == macro force +
    the separate component-sum pass up to the order of the sums: same cycles, fields to rounding."""
    base = _solve(ih, n, {"MACRO_SUMS": 0}, fabric_p=P)
    v = _solve(ih, n, {"MACRO_SUMS": 1}, fabric_p=P)
    v2 = _solve(ih, n, {"MACRO_SUMS": 1}, fabric_p=P)
    assert v[0] == base[0]
    assert np.abs(v[1] - base[1]).max() <= 1e-12 * np.abs(base[1]).max()
    for a, b in zip(v[2], base[2]):  # f32 inner corrections turn last-bit load changes into ~1e-10
        assert np.linalg.norm(a - b) <= 1e-8 * max(np.linalg.norm(b), 1e-30)
    np.testing.assert_array_equal(v[1], v2[1])  # reproducible run to run
    for a, b in zip(v[2], v2[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,P,group", [(16, 0, 6), (64, 0, 2), (64, 0, 3), (64, 0, 6), (128, 0, 6),
                                       ((64, 32, 48), 0, 6), (128, 4, 2)])
def test_bottom_cycle_bit_identical(ih, n, P, group):
    """The small levels and the coarsest solve of the grouped inner V-cycle in one cooperative launch
    (BOTTOM_CYCLE: the same per-vertex kernels, grid-wide barriers between the passes) == one launch per
    pass, bitwise."""
    knobs = {"RHS_PAIRS": 1, "RHS_GROUP": group}
    base = _solve(ih, n, {**knobs, "BOTTOM_CYCLE": 0}, fabric_p=P)
    v = _solve(ih, n, {**knobs, "BOTTOM_CYCLE": 1}, fabric_p=P)
    assert v[0] == base[0]
    np.testing.assert_array_equal(v[1], base[1])
    for a, b in zip(v[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,P", [(32, 0), (64, 0), ((64, 32, 48), 0), (16, 0), (64, 2), (128, 4)])
def test_gs_pair_bit_identical(ih, n, P):
    """Level-0 f32 GS colour passes c, c + 1 in one launch (GS_PAIR: blocks own whole rows, the fresh
    colour-c values of a row handed to colour c + 1 through shared memory) == two launches, bitwise;
    plain and zero-start passes, z-slab links."""
    base = _solve(ih, n, {"GS_PAIR": 0}, fabric_p=P)
    v = _solve(ih, n, {"GS_PAIR": 1}, fabric_p=P)
    assert v[0] == base[0]
    np.testing.assert_array_equal(v[1], base[1])
    for a, b in zip(v[2], base[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,P", [(64, 0), (128, 0), (128, 2)])
def test_stencil_stream_bit_identical(ih, n, P):
    """Stencil-level residual and plain GS passes with each warp's stencil block streamed through a
    cp.async ring (STENCIL_STREAM) == the direct-load f32 kernels, bitwise (same arithmetic and order)."""
    base = _solve(ih, n, {"STENCIL_F32": 1, "STENCIL_STREAM": 0}, fabric_p=P)
    v = _solve(ih, n, {"STENCIL_F32": 1, "STENCIL_STREAM": 1}, fabric_p=P)
    assert v[0] == base[0]
    np.testing.assert_array_equal(v[1], base[1])
    for a, b in zip(v[2], base[2]):
        np.testing.assert_array_equal(a, b)
