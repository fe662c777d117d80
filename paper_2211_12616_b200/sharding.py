"""Multi-GPU plumbing for one-process-per-GPU runs (torchrun + NCCL).

The path shards by particle: rank r owns the contiguous block
`calc_device_workload_range(N, world, r)` (partition.py:28-41) and never
exchanges particle data.  The only data collectives are

* the met replication — every rank needs the whole snapshot; rank 0 builds
  (or reads) it and broadcasts the packed u/v/w/T fields (the reference
  deep-copies both snapshots into every device image on each rotation,
  device_runtime.py:178-186; here only the new snapshot moves, once);
* the statistics gather — timings (max over ranks) and counters (sum).

Everything here is backend-agnostic torch.distributed so the same code runs
over NCCL on B200s and over gloo in the CPU tests.
"""

from __future__ import annotations

import numpy as np

from .partition import WorkRange, calc_device_workload_range

FIELDS = ("u", "v", "w", "T")


def shard_range(n_total: int, world: int, rank: int) -> WorkRange:
    return calc_device_workload_range(n_total, world, rank)


def broadcast_snapshot(met, shape, dist, device, src: int = 0):
    """Replicate one snapshot's four fields as a (4, nx, ny, nz) float32
    tensor on `device`.  `met` is the MeteoField on rank `src` (ignored
    elsewhere); `shape` is (nx, ny, nz) of the fields."""
    import torch
    buf = torch.empty((4,) + tuple(int(s) for s in shape), dtype=torch.float32, device=device)
    if dist.get_rank() == src:
        for f, name in enumerate(FIELDS):
            a = np.ascontiguousarray(getattr(met, name), dtype=np.float32)
            buf[f].copy_(torch.from_numpy(a))
    dist.broadcast(buf, src=src)
    return buf


def broadcast_grid(lons, lats, levs, dist, device, src: int = 0):
    """Replicate the (already closed) grid axes; returns float64 numpy arrays."""
    import torch
    sizes = torch.tensor([len(lons), len(lats), len(levs)] if dist.get_rank() == src
                         else [0, 0, 0], dtype=torch.int64, device=device)
    dist.broadcast(sizes, src=src)
    nx, ny, nz = (int(v) for v in sizes.tolist())
    ax = torch.zeros(nx + ny + nz, dtype=torch.float64, device=device)
    if dist.get_rank() == src:
        ax.copy_(torch.from_numpy(np.concatenate([lons, lats, levs]).astype(np.float64)))
    dist.broadcast(ax, src=src)
    a = ax.cpu().numpy()
    return a[:nx].copy(), a[nx:nx + ny].copy(), a[nx + ny:].copy()


def max_over_ranks(values, dist, device) -> list[float]:
    """Element-wise max of per-rank floats (device timings)."""
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def sum_over_ranks(values, dist, device) -> list[int]:
    """Element-wise sum of per-rank integer counters."""
    import torch
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(v) for v in t.tolist()]
