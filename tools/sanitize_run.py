"""Small hot-path run for compute-sanitizer (memcheck / racecheck / synccheck): one optimisation iteration
at 32^3 in the bench's mode (mixed precision, mixed_defect, default kernel variants) and one in the
reference-precision V-cycle mode. python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_08911_b200 as ih  # noqa: E402

for mode in ("mixed_defect", "vcycle"):
    rep = ih.run_optimization(ih.RunConfig(reso=32, vol=0.2, obj="npr-relaxed", max_iter=2, precision="mixed",
                                           solver_mode=mode))
    print(mode, [round(r["objective"], 4) for r in rep.records], flush=True)
print("sanitize run OK")
