"""Per-GPU footprint of 1024^3 on two GPUs with the memory lever (host-staged displacements, U_HOST=2).

One B200 holds a 1024 x 1024 x 512 periodic grid: the element / vertex count of one z-slab of 1024^3 on
two GPUs. It runs whole cell-problem iterations (set_density, the six solves, C^H, sensitivities) with
the six displacement fields in pinned host memory, next to the optimiser's seven f64 density-side fields
(allocated here as one torch block: rho, next, pre, phys, grad, tmp, gd). Prints one JSON line with the
device memory the process holds and the time per iteration. A proxy for the slab: the same per-GPU
arrays and kernels, a periodic z wrap instead of the neighbour-slab halo.

usage: python tools/host_staged_1024.py [nx ny nz] [iterations]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2301_08911_b200 as ih  # noqa: E402


def mem_available_gb():
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 1e6
    return 0.0


def main():
    n = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (1024, 1024, 512)
    iters = int(sys.argv[4]) if len(sys.argv) >= 5 else 3
    nv = n[0] * n[1] * n[2]
    host_need = nv * (144 + 72 + 16) / 1e9  # pinned f64 + f32 fields, the density staging below
    if mem_available_gb() < host_need + 32:
        print(json.dumps({"skipped": f"host RAM {mem_available_gb():.0f} GB < {host_need + 32:.0f} GB needed"}))
        return
    torch.cuda.init()
    free0, total = torch.cuda.mem_get_info()
    ih.set_knob("U_HOST", 2)
    t0 = time.time()
    hom = ih.Homogenizer(n, penal=1.0, precision="mixed",
                         opts=ih.SolverOptions(tol=1e-2, max_cycles=50, mode="mixed_defect"))
    t_build = time.time() - t0
    side = torch.empty((7, nv), dtype=torch.float64, device="cuda")
    rho, _ = ih.init_trig(n, 2, 0, 0.2)
    side[0].copy_(torch.from_numpy(rho))
    del rho
    torch.pow(side[0], 3, out=side[3])  # phys = rho^p (DensityExpr, p = 3)
    sens = side[4]
    seed = -np.eye(6)  # bulk-like seed
    rows, min_free = [], free0
    gen = torch.Generator(device="cuda").manual_seed(1)
    for it in range(iters):
        if it:  # a design update: a small non-uniform change of the density (warm starts stay close)
            side[5].uniform_(-0.01, 0.01, generator=gen)
            side[0].add_(side[5]).clamp_(1e-3, 1.0)
            torch.pow(side[0], 3, out=side[3])
        torch.cuda.synchronize()
        t = time.time()
        hom.set_density(side[3])
        st = hom.solve_cell_problems()
        C = hom.effective_tensor()
        hom.tensor_sensitivity(seed, out=sens)
        torch.cuda.synchronize()
        rows.append({"iter": it, "s": round(time.time() - t, 3), "cycles": st["total_cycles"],
                     "C00": C[0, 0], "C33": C[3, 3]})
        min_free = min(min_free, torch.cuda.mem_get_info()[0])
    out = {"grid": list(n), "vertices": nv, "host_staged": hom.host_staged, "build_s": round(t_build, 1),
           "hbm_total_gb": round(total / 1e9, 1), "hbm_used_gb": round((total - min_free) / 1e9, 2),
           "hbm_this_process_gb": round((free0 - min_free) / 1e9, 2),
           "density_side_gb": round(7 * 8 * nv / 1e9, 2), "iterations": rows,
           "s_per_iteration_after_first": round(float(np.mean([r["s"] for r in rows[1:]])), 3) if iters > 1 else None}
    hom.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
