"""Small hot-path run for compute-sanitizer (memcheck / racecheck / synccheck): two optimisation iterations
at 32^3 in the bench's mode (mixed precision, mixed_defect, default kernel variants: lockstep group of six
with the cooperative bottom cycle, last-block reductions, fused macro-force sums), the same with the
host-staged displacements (U_HOST=2), and the reference-precision V-cycle mode.
python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_08911_b200 as ih  # noqa: E402

for mode, host in (("mixed_defect", 0), ("mixed_defect", 2), ("vcycle", 0)):
    ih.set_knob("U_HOST", host)
    rep = ih.run_optimization(ih.RunConfig(reso=32, vol=0.2, obj="npr-relaxed", max_iter=2, precision="mixed",
                                           solver_mode=mode))
    print(mode, "U_HOST", host, [round(r["objective"], 4) for r in rep.records], flush=True)
ih.set_knob("U_HOST", 0)
print("sanitize run OK")
