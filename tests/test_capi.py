"""CPU tests of the drop-in boundary: libihom_b200.so loads, exports every
entry point include/ihom_b200.h declares, and fails loudly (no CPU fallback)
when no CUDA device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ihom_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ihom_[a-z0-9_]+)\s*\(", text)) - {"ihom_observer"})


def test_header_declares_the_reference_surface():
    syms = declared_symbols()
    # Homogenizer / Hierarchy / density / OC / runner surface
    for s in ["ihom_create", "ihom_set_density", "ihom_solve_cell_problems", "ihom_effective_tensor",
              "ihom_tensor_sensitivity", "ihom_v_cycle", "ihom_solve", "ihom_relax", "ihom_compute_residual",
              "ihom_coarsest_solve", "ihom_radial_filter", "ihom_symmetrize", "ihom_oc_update",
              "ihom_sensitivity_filter", "ihom_run_optimization", "ihom_opt_step"]:
        assert s in syms


def test_library_exports_every_declared_symbol(ih):
    L = ih.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_version_string(ih):
    assert "sm_100a" in ih.version()


def test_library_is_built_for_sm100a(ih):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", ih.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_fails_loudly_without_gpu(ih):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises((RuntimeError, ValueError)):
        ih.Homogenizer(8)
    with pytest.raises(Exception):
        ih.radial_filter(8, np.zeros(512))


def test_host_validation_before_device(ih):
    with pytest.raises(ValueError):
        ih.BaseMaterial(1.0, 0.5)
    with pytest.raises(ValueError):
        ih.BaseMaterial(-1.0, 0.3)


def test_no_undefined_library_symbols():
    """Every ihomgpu template the library calls is instantiated in it (a missing explicit
    instantiation links fine as -shared and only fails at dlopen)."""
    import subprocess
    lib = os.path.join(ROOT, "paper_2301_08911_b200", "libihom_b200.so")
    if not os.path.exists(lib):
        pytest.skip("library not built")
    out = subprocess.run(["nm", "-D", "--undefined-only", lib], capture_output=True, text=True).stdout
    assert "ihomgpu" not in out, out


@pytest.mark.parametrize("obj", ["bulk", "shear", "npr-relaxed", "npr-log"])
def test_objectives_bit_exact_with_oracle(ih, orc, obj):
    """The product's closed-form objectives (csrc/objective.cpp) against the oracle's expression-DAG
    restatement of src/objective.cpp:238-260: values and single-sided gradients bit for bit (host code,
    no device needed)."""
    rng = np.random.default_rng(11)
    for it in range(6):
        Cm = rng.uniform(0.1, 1.0, (6, 6))
        Cm = Cm + Cm.T + 3.0 * np.eye(6)
        v, g = orc.objective(obj, Cm, iter=it)
        v2, g2 = ih.objective_native(obj, Cm, iter=it)
        assert v == v2
        assert np.array_equal(g, np.asarray(g2).reshape(6, 6))


def test_objective_domain_errors(ih, orc):
    """npr-log domain failures raise (the reference's EvalError, inc/objective.hpp:11-14) in both."""
    Cm = np.eye(6)
    Cm[0, 1] = Cm[1, 2] = Cm[2, 0] = -10.0  # 1 + eta*ring/normal < 0
    with pytest.raises(Exception):
        orc.objective("npr-log", Cm)
    with pytest.raises(Exception):
        ih.objective_native("npr-log", Cm)
    with pytest.raises(Exception):
        ih.objective_native("npr-log", np.zeros((6, 6)))


def _build_reference_caller(tmp_path):
    exe = tmp_path / "reference_caller"
    lib_dir = os.path.join(ROOT, "paper_2301_08911_b200")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "reference_caller.cpp"), "-L", lib_dir, "-lihom_b200",
           f"-Wl,-rpath,{lib_dir}", "-o", str(exe)]
    import subprocess
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_wrapper_compiles_with_reference_constructor(tmp_path):
    """include/ihom_b200.hpp compiles and links for a reference-style caller (Homogenizer(IVec3,
    BaseMaterial, penal, SolverOptions), inc/homogenization.hpp:29); without a GPU it fails loudly."""
    import subprocess
    exe = _build_reference_caller(tmp_path)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except ImportError:
        has_gpu = False
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode in ((0,) if has_gpu else (3,)), r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_wrapper_solid_tensor_on_gpu(tmp_path):
    import subprocess
    exe = _build_reference_caller(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
