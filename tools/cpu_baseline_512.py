"""Full-size CPU reference-loop timing (the oracle port of src/runner.cpp on all host cores) at 512^3
npr-relaxed: validates the bench's 128^3-sample x64 extrapolation. python tools/cpu_baseline_512.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the reference loop's CPU restatement)

threads = os.cpu_count() or 1
oracle.set_threads(threads)
out = {"reso": 512, "obj": "npr-relaxed", "cores": threads}
for reso, iters in ((128, 4), (512, 2)):
    t = time.time()
    recs, _, _ = oracle.run(reso=reso, vol=0.2, obj="npr-relaxed", max_iter=iters, mixed=True)
    out[f"{reso}"] = {"wall_s": round(time.time() - t, 1), "iter_s": [round(r["ms"] / 1e3, 2) for r in recs],
                      "cycles": [r["cycles"] for r in recs]}
    print(json.dumps(out), flush=True)
