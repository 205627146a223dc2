"""Long-run survival check on the GPU: one optimisation of `--iters` iterations at `--reso`
through the public API, printing per-iteration objective / cycles / wall ms.
--project 0 restores the reference's unprojected coarsest operator (knob COARSE_PROJECT).
Usage: python tools/long_run.py --reso 128 --obj npr-relaxed --iters 30 [--project 0]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_08911_b200 as ih  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reso", type=int, default=128)
ap.add_argument("--obj", default="npr-relaxed")
ap.add_argument("--vol", type=float, default=0.2)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--project", type=int, default=1)
ap.add_argument("--mode", default="mixed_defect")
ap.add_argument("--precision", default="mixed")
a = ap.parse_args()
ih.set_knob("COARSE_PROJECT", a.project)
cfg = ih.RunConfig(reso=a.reso, vol=a.vol, obj=a.obj, max_iter=a.iters, precision=a.precision, solver_mode=a.mode)
t = time.time()
try:
    rep = ih.run_optimization(cfg)
    out = {"ok": True, "solver_failed": rep.solver_failed, "n": len(rep.records),
           "records": [{k: r[k] for k in ("iter", "objective", "cycles", "residual", "ms")} for r in rep.records]}
except Exception as e:  # report, do not hide
    out = {"ok": False, "error": str(e)}
out.update(reso=a.reso, obj=a.obj, project=a.project, mode=a.mode, wall_s=round(time.time() - t, 2))
print(json.dumps(out))
