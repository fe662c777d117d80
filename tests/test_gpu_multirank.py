"""GPU: the N > 1 paths end to end on the one B200 a gpurun box has.

* two torch.distributed ranks (gloo, both on GPU 0) each run the Engine on
  their shard (calc_device_workload_range) with the met snapshots rank 0
  built broadcast to them (sharding.broadcast_snapshot -> lt_met_load from
  device memory), exactly as bench.py's torchrun path does; the gathered
  result equals the one-rank run bit for bit (particles are independent
  and draws are keyed by global id);
* bench.py itself under torchrun (2 gloo ranks) and as the one-process
  `--gpus 2` driver prints a valid contract line (strong scaling).
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _chain(rank, world, port, outdir):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2211_12616_b200 import _capi as capi
    from paper_2211_12616_b200 import engine, sharding, synthetic
    from paper_2211_12616_b200.model_state import Control
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    n = 20_000
    work = sharding.shard_range(n, world, rank)
    ctl = Control(t_stop=86400.0, dt_model=180.0, met_dt=10800.0, rng_mode="counter",
                  rng_seed_global=31, precision="fast")
    mets = synthetic.analytic_pair(dlon=5.0, dlat=5.0, nlev=24, t0=0.0, t1=10800.0) \
        if rank == 0 else None
    grid = (mets[0].lons, mets[0].lats, mets[0].levs) if rank == 0 else (None,) * 3
    cpu = torch.device("cpu")
    lons, lats, levs = sharding.broadcast_grid(*grid, dist, cpu)
    ens = synthetic.particles(n, seed=6)
    eng = engine.Engine(device=0, first_id=work.start)
    eng.upload(ens, start=work.start, end=work.end)
    eng.set_grid(lons, lats, levs)
    shape = (len(lons), len(lats), len(levs))
    for slot, t_met in ((0, 0.0), (1, 10800.0)):
        buf = sharding.broadcast_snapshot(mets[slot] if rank == 0 else None, shape, dist, cpu)
        dev = buf.to("cuda:0")
        torch.cuda.synchronize()
        p = dev.data_ptr()
        fb = dev[0].numel() * 4
        capi.check(eng.ctx.lib.lt_met_load(eng.ctx.h, slot, t_met, 4, p, p + fb, p + 2 * fb,
                                           p + 3 * fb, capi.MET_DEVICE_SRC))
        eng.ctx.sync()
    eng.ctx.use_met(0, 1)
    eng._met_slots, eng._staged = (0, 1), None
    for step in range(12):
        if step % 5 == 0:
            eng.sort()
        eng.step(ctl, step, engine.ADV_DIFF)
    out = eng.download()   # this shard, in particle order
    assert out.np == work.size
    np.savez(Path(outdir) / f"rank{rank}.npz", start=work.start, end=work.end,
             lon=out.lon, lat=out.lat, p=out.p, time=out.time)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_equal_one_rank_bitwise(tmp_path):
    import torch.multiprocessing as mp
    outs = {}
    for world in (1, 2):
        d = tmp_path / f"w{world}"
        d.mkdir()
        mp.spawn(_chain, args=(world, _free_port(), str(d)), nprocs=world, join=True)
        parts = [dict(np.load(d / f"rank{k}.npz")) for k in range(world)]
        outs[world] = {k: np.concatenate([q[k] for q in parts]) for k in ("lon", "lat", "p", "time")}
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_array_equal(outs[2][k], outs[1][k])


def _bench_line(cmd, env=None):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_torchrun_two_ranks():
    line = _bench_line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()), "bench.py", "--workload", "cfg2",
                        "--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "0",
                        "--alt-steps", "0"], env={"LT_DIST_BACKEND": "gloo"})
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["particles"] == 10_000_000
    assert line["config"]["particles_per_gpu"] == 5_000_000
    assert line["value"] > 0 and line["gpu_launches"] >= 3


def test_bench_one_process_two_gpus():
    line = _bench_line([sys.executable, "bench.py", "--gpus", "2", "--workload", "cfg2",
                        "--steps", "3", "--warmup", "3"])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["particles_per_gpu"] == 5_000_000
    assert line["met_broadcast"]["nccl_version"] >= 22700
    assert line["value"] > 0
