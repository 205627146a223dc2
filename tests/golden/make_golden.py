"""Generates tests/golden/reference_density_oc.npz from the REFERENCE's own
src/density.cpp + src/oc.cpp (compiled unmodified into oracle/_ref by
oracle/Makefile). Run where /root/reference exists:  python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py::test_golden_vectors)
on machines without the reference tree (e.g. the GPU box).
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

dp = C.POINTER(C.c_double)


def p(a):
    return a.ctypes.data_as(dp)


def main():
    oracle.build()
    R = oracle.ref()
    rng = np.random.default_rng(20230121)
    out = {}
    n = (8, 6, 10)
    f = rng.uniform(0, 1, int(np.prod(n)))
    out["filter_n"] = np.array(n)
    out["filter_in"] = f
    for name, k, r in [("filter_out_spline4_r2", 1, 2.0), ("filter_out_linear_r15", 0, 1.5)]:
        o = np.zeros_like(f)
        R.ref_radial_filter(*n, p(f), C.c_double(r), k, p(o))
        out[name] = o
    s = rng.uniform(0, 1, 512)
    out["sym_in"] = s.copy()
    R.ref_symmetrize(8, 8, 8, p(s), 2)
    out["sym_out_reflect6"] = s
    t = np.zeros(16 ** 3)
    R.ref_init_trig(16, 16, 16, 2, C.c_ulonglong(0), C.c_double(0.2), C.c_double(15.0), p(t))
    out["trig16_b2_s0_v02"] = t
    rho = rng.uniform(0.25, 0.35, 512)
    g = rng.uniform(-3.0, -0.1, 512)
    o = np.zeros(512)
    lam = C.c_double()
    R.ref_oc_update(8, 8, 8, p(rho), p(g), C.c_double(0.3), C.c_double(0.05), C.c_double(0.5), p(o), C.byref(lam))
    out.update(oc_rho=rho, oc_sens=g, oc_out=o, oc_lambda=np.array(lam.value))
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_density_oc.npz"), **out)
    print("wrote reference_density_oc.npz")


if __name__ == "__main__":
    main()
