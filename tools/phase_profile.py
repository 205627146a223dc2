"""Per-phase device time of an optimisation iteration vs the kernel families inside it (host gaps =
phase time - kernel time). python tools/phase_profile.py --reso 512 --steps 6 --warmup 5"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_08911_b200 as ih  # noqa: E402

PHASE_FAMILIES = {
    "phase:density_eval": ["filter", "pow"],
    "phase:set_density": ["coeff", "galerkin_l1", "galerkin_coarse"],
    "phase:solve": ["l0_gs_f32", "l0_residual_f64", "l0_residual_f32", "l1_gs_f32", "l1_residual_f32", "l2_gs_f32",
                    "l2_residual_f32", "coarse_gs_f32", "coarse_residual_f32", "prolong", "restrict", "vector",
                    "reduce", "coarsest", "macro_force"],
    "phase:tensor": ["tensor"],
    "phase:sens_filter_oc": ["sensitivity", "symmetrize", "oc_trial"],
}

ap = argparse.ArgumentParser()
ap.add_argument("--reso", type=int, default=512)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--warmup", type=int, default=5)
a = ap.parse_args()
cfg = ih.RunConfig(reso=a.reso, vol=0.2, obj="npr-relaxed", max_iter=10 ** 6, precision="mixed",
                   solver_mode="mixed_defect")
opt = ih.Optimizer(cfg)
for _ in range(a.warmup):
    opt.step()
ih.set_knob("PHASE_PROF", 1)
ih.profile_enable(True)
t = time.time()
for _ in range(a.steps):
    opt.step()
wall = (time.time() - t) / a.steps * 1e3
tot = ih.profile_totals()
ih.profile_enable(False)
out = {"wall_ms_per_iter": round(wall, 2)}
for ph, fams in PHASE_FAMILIES.items():
    pt = tot.get(ph, {}).get("ms", 0.0) / a.steps
    kt = sum(tot.get(f, {}).get("ms", 0.0) for f in fams) / a.steps
    out[ph] = {"phase_ms": round(pt, 2), "kernel_ms": round(kt, 2), "gap_ms": round(pt - kt, 2)}
out["all_phases_ms"] = round(sum(v["phase_ms"] for k, v in out.items() if k.startswith("phase")), 2)
print(json.dumps(out, indent=1))
