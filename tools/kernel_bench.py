"""Isolated per-kernel timing at a given resolution (CUDA events via the library profiler).

python tools/kernel_bench.py --reso 512 --ops l0_gs_f32,l0_residual_f64 --reps 3
Prints one JSON line per op: device ms per launch family, algorithmic GB/s, fraction of MEASURED_PEAKS hbm_gbs.
Also the ncu target: ncu -k regex:<kernel> python tools/kernel_bench.py --ops <op> --reps 1
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2301_08911_b200 as ih  # noqa: E402

ALL = "l0_gs_f32,l0_gs_f64,l0_residual_f64,l0_defect_f64,l0_residual_f32,l1_gs_f32,l1_residual_f32,vcycle_f32,set_density,tensor,sensitivity"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reso", type=int, default=256)
    ap.add_argument("--ops", default=ALL)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", default="mixed")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    n = a.reso
    rho, _ = ih.init_trig(n, 2, 0, 0.2)
    phys = ih.radial_filter(n, rho, 2.0, "spline4") ** 3
    hom = ih.Homogenizer(n, ih.BaseMaterial(1e6, 0.3), 1.0, ih.SolverOptions(), precision=a.precision)
    hom.set_density(phys)
    H = hom.hierarchy()
    for op in a.ops.split(","):
        H.bench_op(op, 1)  # warm-up
        ih.profile_enable(True)
        H.bench_op(op, a.reps)
        tot = ih.profile_totals()
        ih.profile_enable(False)
        fams = {k: {"ms_per_launch": round(v["ms"] / v["launches"], 4), "launches": v["launches"],
                    "GB/s": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["bytes"] else None,
                    "frac": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9 / peak, 3) if v["bytes"] else None}
                for k, v in tot.items()}
        print(json.dumps({"op": op, "reso": n, "reps": a.reps, "families": fams}), flush=True)


if __name__ == "__main__":
    main()
