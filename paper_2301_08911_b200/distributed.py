"""Multi-GPU plumbing for the hot path (one process per GPU).

Two schemes:

* z-slabs (the default of ``bench.py --gpus N``): rank r owns z planes [r t, (r+1) t) of every field;
  kernels read the neighbour slabs' boundary planes directly through CUDA-IPC-mapped peer memory
  (``ipc_fabric``), ordered by device-side barriers (z-neighbour-only around halo reads, bounded by a
  timeout) and reduced through per-rank mailboxes folded in rank order.
* load-case split (``--multi loads``): the six periodic cell problems are independent solves, so rank r
  solves the load cases ``load_owners(n)`` assigns it; the library broadcasts every solved displacement
  field from its owner over NCCL (NVLink) and every rank evaluates C^H, the sensitivities and the OC
  update identically (bitwise equal to one GPU; no memory saving, stops scaling at six ranks).

``torch.distributed`` carries only host metadata (IPC handles, the NCCL unique id); the data plane runs
inside libihom_b200.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

NUM_LOADS = 6


def load_owners(nranks: int) -> list:
    """Rank that solves load case i (i % nranks; ranks >= 6 get none)."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    return [i % nranks for i in range(NUM_LOADS)]


def combine_cell_stats(per_load) -> dict:
    """CellSolveStats from per-load (cycles, rel_residual, converged), in load order
    exactly as src/homogenization.cpp:29-38 accumulates them."""
    out = dict(total_cycles=0, worst_residual=0.0, worst_load=-1, converged=True)
    for i, (cyc, rel, conv) in enumerate(per_load):
        out["total_cycles"] += int(cyc)
        if rel >= out["worst_residual"]:
            out["worst_residual"] = float(rel)
            out["worst_load"] = i
        if not conv:
            out["converged"] = False
    return out


def nccl_unique_id() -> bytes:
    from . import _check, lib
    buf = (C.c_char * 128)()
    _check(lib().ihom_nccl_unique_id(buf))
    return bytes(buf)


def share_unique_id(rank: int) -> bytes:
    """Rank 0 creates the NCCL id; torch.distributed (any backend) broadcasts it."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t[:] = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().astype(np.uint8).tobytes())


# ---------------------------------------------------------------- z-slab fabric over processes
def slab_planes(n: int, nranks: int, rank: int):
    """(z0, planes) of z-slab ``rank`` of an n^3 grid (include/ihom_b200.h: t = n / nranks, a multiple
    of 4 so every smoothed level keeps an even slab thickness)."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / slab count")
    t = n // nranks
    if n % nranks or t % 4:
        raise ValueError(f"{n} planes do not split into {nranks} slabs of a multiple of 4 planes")
    return rank * t, t


def torch_allgather(group=None):
    """bytes -> [bytes of every rank] over torch.distributed (any backend): the host allgather an
    IPC fabric exchanges its CUDA IPC handles with (plumbing only; no data-path traffic)."""
    import torch.distributed as dist

    def ag(blob: bytes):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, blob, group=group)
        return out
    return ag


def ipc_fabric(rank: int, nranks: int, device: int = 0):
    """One z-slab per process: peer buffers are mapped with CUDA IPC (NVLink between GPUs)."""
    from . import Fabric
    return Fabric.ipc(rank, nranks, torch_allgather(), device=device)


# ---------------------------------------------------------------- memory plan (estimate)
# Bytes per level-0 vertex (= per element) of one z-slab in mixed precision, mixed_defect solver
# (DESIGN.md 2/6/7): six persistent f64 u^i (144), level-0 f64 u/f/r + ping-pong u (96), f32 inner e/f/r
# on every level (36 x 8/7 = 41), coefficients (4), level-1/2/... f32 stencils (243 x 4 B x (1/8 + 1/64 +
# ...) = 139), density side (the optimiser's 7 f64 fields + the homogenizer's copy, 64); optional: f64
# energy cache (168), each extra RHS of a lockstep group (89).
# Host-staged layout (U_HOST, the memory lever): the six u^i in pinned host memory, level-0 f64 u and f
# only, no ping-pong, no groups, no cache: 48 + 41 + 4 + 139 + 64 = 296 B on the device (measured: 512^3
# 39.8 GB, 1024 x 1024 x 512 = one slab of 1024^3 on 2 GPUs 159 GB; profiles/host_staged_r02.md), plus
# 216 B of pinned host memory per vertex.
_BASE_B = 144 + 96 + 41 + 4 + 139 + 64
_HOST_STAGED_B = 48 + 41 + 4 + 139 + 64
_CACHE_B = 168
_GROUP_B = 89


def memory_plan(reso: int, nranks: int, group: int = 1, energy_cache: bool = False,
                host_staged: bool = False) -> dict:
    """Estimated HBM per GPU (GB) of a reso^3 run on nranks z-slabs, and whether it fits a 180 GB B200
    (leaving 8 GB headroom). The library adapts the group size and the energy cache to the free HBM and
    switches to the host-staged layout when even the minimal device-resident one does not fit."""
    nv = reso ** 3 / nranks
    if host_staged:
        per_vertex = _HOST_STAGED_B
        group, energy_cache = 1, False
    else:
        per_vertex = _BASE_B + (_CACHE_B if energy_cache else 0) + _GROUP_B * (group - 1)
    gb = nv * per_vertex / 1e9
    out = {"reso": reso, "nranks": nranks, "group": group, "energy_cache": energy_cache,
           "gb_per_gpu": round(gb, 1), "fits_b200": gb <= 172.0}
    if host_staged:
        out["host_staged"] = True
        out["pinned_host_gb_per_gpu"] = round(nv * 216 / 1e9, 1)
    return out
