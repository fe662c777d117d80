"""CPU, world_size 2 over gloo: the N>1 host path of bench.py — shard
ranges, met grid + snapshot broadcast from rank 0, max/sum over ranks."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2211_12616_b200 import sharding, synthetic
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cpu")
    n_total = 1001
    work = sharding.shard_range(n_total, world, rank)
    m0 = synthetic.analytic_pair(dlon=30.0, dlat=30.0, nlev=5)[0] if rank == 0 else None
    grid = (m0.lons, m0.lats, m0.levs) if rank == 0 else (None, None, None)
    lons, lats, levs = sharding.broadcast_grid(*grid, dist, dev)
    buf = sharding.broadcast_snapshot(m0, (len(lons), len(lats), len(levs)), dist, dev)
    mx = sharding.max_over_ranks([rank + 1.5, -rank], dist, dev)
    sm = sharding.sum_over_ranks([work.size, 1], dist, dev)
    np.savez(Path(outdir) / f"rank{rank}.npz", start=work.start, end=work.end,
             lons=lons, lats=lats, levs=levs, fields=buf.numpy(), mx=mx, sm=sm)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_met_broadcast(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(world)]
    # contiguous, disjoint, covering, front-loaded remainder (partition.py:28-41)
    assert (int(r[0]["start"]), int(r[0]["end"]), int(r[1]["start"]), int(r[1]["end"])) == \
        (0, 501, 501, 1001)
    sys.path.insert(0, str(ROOT))
    from paper_2211_12616_b200 import synthetic
    m0 = synthetic.analytic_pair(dlon=30.0, dlat=30.0, nlev=5)[0]
    want = np.stack([np.asarray(getattr(m0, f), dtype=np.float32) for f in ("u", "v", "w", "T")])
    for k in range(world):
        np.testing.assert_array_equal(r[k]["lons"], m0.lons)
        np.testing.assert_array_equal(r[k]["levs"], m0.levs)
        np.testing.assert_array_equal(r[k]["fields"], want)
        np.testing.assert_array_equal(r[k]["mx"], [2.5, 0.0])
        np.testing.assert_array_equal(r[k]["sm"], [1001, 2])
