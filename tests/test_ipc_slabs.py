"""z-slab decomposition across PROCESSES (IPC fabric).

Two processes each own one slab and map the other's buffers with CUDA IPC, as
the bench does with one process per GPU. Here both processes share cuda:0
(gpurun gives one GPU; cross-process IPC on one device uses the same handles
and device-side release/acquire barriers as NVLink peers). The per-slab
results must equal the single-domain run of the same grid.
"""
import os
import socket

import numpy as np
import pytest

from paper_2301_08911_b200 import distributed as dd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _seed():
    s = np.zeros((6, 6))
    s[:3, :3] = 1.0 / 9.0
    s[3, 3] = s[4, 4] = s[5, 5] = 0.25
    return s


def _worker(rank, world, port, n, phys, mode, q, host=0):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import paper_2301_08911_b200 as ih
        from paper_2301_08911_b200 import distributed as dd2
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ih.set_knob("U_HOST", host)  # 2: host-staged displacements, snapshot links over CUDA IPC
        fab = dd2.ipc_fabric(rank, world, device=0)
        hom = ih.Homogenizer(n, penal=1.0, precision="mixed", opts=ih.SolverOptions(tol=1e-2, mode=mode),
                             fabric=fab, rank=rank)
        assert hom.host_staged == host
        z0, t = dd2.slab_planes(n, world, rank)
        assert (hom.z0, hom.planes) == (z0, t)
        hom.set_density(np.ascontiguousarray(phys[z0 * n * n:(z0 + t) * n * n]))
        st = hom.solve_cell_problems()
        C = hom.effective_tensor()
        sens = hom.tensor_sensitivity(_seed())
        hom.close()
        fab.close()
        q.put((rank, st, C, sens, None))
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001 - reported to the parent
        q.put((rank, None, None, None, repr(e)))


@pytest.mark.gpu
@pytest.mark.parametrize("mode,host", [("vcycle", 0), ("mixed_defect", 0), ("mixed_defect", 2)])
def test_ipc_two_process_slabs_match_single_domain(ih, mode, host):
    import torch.multiprocessing as mp
    n = 32
    rho, _ = ih.init_trig(n, 2, 0, 0.3)
    phys = ih.radial_filter(n, rho, 2.0, "spline4") ** 3
    hom = ih.Homogenizer(n, penal=1.0, precision="mixed", opts=ih.SolverOptions(tol=1e-2, mode=mode))
    hom.set_density(phys)
    st1 = hom.solve_cell_problems()
    C1, s1 = hom.effective_tensor(), hom.tensor_sensitivity(_seed())
    hom.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, phys, mode, q, host)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for rank, st, C, sens, err in res:
        assert err is None, f"rank {rank}: {err}"
        assert st["total_cycles"] == st1["total_cycles"]
        np.testing.assert_array_equal(C, res[0][2])
        assert np.max(np.abs(C - C1)) <= 1e-9 * np.max(np.abs(C1))
    sens = np.concatenate([r[3] for r in res])
    assert np.max(np.abs(sens - s1)) <= 1e-6 * np.max(np.abs(s1))


def test_slab_planes():
    assert dd.slab_planes(512, 8, 3) == (192, 64)
    assert dd.slab_planes(32, 2, 1) == (16, 16)
    with pytest.raises(ValueError):
        dd.slab_planes(32, 3, 0)
    with pytest.raises(ValueError):
        dd.slab_planes(24, 4, 0)  # 6 planes per slab: not a multiple of 4


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_bench_under_torchrun_same_device(world):
    """The bench's multi-GPU path as the driver launches it (torch.distributed.run, one process per rank,
    z-slabs over CUDA IPC), with every rank on cuda:0 (--same-device): it must complete and print one
    JSON line from rank 0 with the whole-job metric. Small grid: 64^3 (16 planes per slab at 4 ranks)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", str(world), "--same-device", "--reso", "64", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline"]
    env = dict(os.environ, IHOM_FABRIC_TIMEOUT_S="120")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["value"] > 0 and d["steps"] == 2
    assert "e2e" in d and d["e2e"]["h2d_bytes_per_step"] == 8 * 64 ** 3
