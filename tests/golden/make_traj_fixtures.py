"""Generates tests/golden/traj_*.npz: per-iteration oracle trajectories (objective, C^H, volume,
V-cycle counts, a strided sample of the final design) for the BASELINE configs the GPU tests pin at
scale. Oracle = oracle/ (CPU restatement of src/runner.cpp:47-136 with the coarsest-operator
projection). CPU cost on 8 cores: ~25 min in total.
    python tests/golden/make_traj_fixtures.py [name ...]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

# name -> (reso, obj, vol, iterations); stride of the final-design sample
CASES = {
    "npr64": (64, "npr-relaxed", 0.2, 30),      # configs[3] objective, >= 20 iterations at 64^3
    "npr128": (128, "npr-relaxed", 0.2, 24),    # configs[3] objective past the reference's iteration-14 failure
    "shear128": (128, "shear", 0.2, 4),         # configs[1]
    "bulk256": (256, "bulk", 0.3, 3),           # configs[2]
}
STRIDE = 997


def make(name):
    reso, obj, vol, iters = CASES[name]
    t = time.time()
    recs, rho, flags = oracle.run(reso=reso, vol=vol, obj=obj, max_iter=iters, mixed=True)
    out = os.path.join(ROOT, "tests", "golden", f"traj_{name}.npz")
    np.savez_compressed(out, reso=reso, obj=obj, vol=vol, iters=iters,
                        objective=np.array([r["objective"] for r in recs]),
                        C=np.array([r["C"] for r in recs]), volume=np.array([r["volume"] for r in recs]),
                        cycles=np.array([r["cycles"] for r in recs]), rho_sample=rho[::STRIDE], stride=STRIDE,
                        rho_mean=rho.mean(), flags=np.array([flags[k] for k in sorted(flags)]))
    print(f"{name}: {len(recs)} iterations, flags {flags}, {time.time() - t:.0f} s -> {out}", flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or list(CASES):
        make(n)
