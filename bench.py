"""Benchmark: particle-steps/s of the fused advection + diffusion step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3|cfg2|cfg1]
                    [--impl b200|reference]

Workload (BASELINE.json configs[2], the metric's "at 1/2/4/8 B200" config):
1e8 particles on the synthetic ERA5-like 0.25 deg grid (1440(+1) x 721 x
137), advection + turbulent + mesoscale diffusion (+ timesteps, in-kernel
counter RNG, position), sharded over N GPUs with the reference partition
rule, met replicated to every rank by an NCCL broadcast.  A "step" is one
fused time step of every particle; the box sort runs every `--sort-every`
steps inside the timed region.

`value` is device-timed (CUDA events on the engine stream, max over ranks,
inputs resident in HBM); `e2e` times the same step through the host-buffer
C-ABI path (pinned host SoA in, step, SoA out every step).  `cpu_baseline`
and `--impl reference` time the CPU oracle (a numpy restatement of the
reference, oracle/) on the host's cores on a bounded particle sample of the
same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-steps/s (advect+diffusion) at 1/2/4/8 B200; % of HBM roofline"
WORKLOADS = {
    # name: (total particles, dlon, dlat, nlev, p_min, modules, description)
    "cfg3": (100_000_000, 0.25, 0.25, 137, 0.01, "adv_diff",
             "1e8 particles, ERA5-like 0.25deg 1440x721x137, advection+turb+meso diffusion"),
    "cfg2": (10_000_000, 1.0, 1.0, 60, 1.0, "adv_diff",
             "1e7 particles, ERA5-like 1deg 360x181x60, advection+turb+meso diffusion"),
    "cfg1": (100_000, 1.0, 1.0, 60, 1.0, "adv",
             "1e5 particles, solid-body rotation 1deg x 60, advection only"),
}
STATE_BYTES = {"adv": 64, "adv_diff": 112}  # fp64 lon/lat/p/time r+w (+ fp64 uvwp r+w)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def algorithmic_bytes(mod: str, n_local: int, nodes: int) -> float:
    """b = b_state + 32*nodes*(1 - exp(-8 N/nodes)) / N per
    particle-step (two fp32 float4 snapshots over the touched nodes)."""
    b_met = 32.0 * nodes * (1.0 - math.exp(-8.0 * n_local / nodes)) / n_local
    return STATE_BYTES[mod] + b_met


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def build_met(wl, rank, ws, torch, dist):
    """Rank 0 builds the snapshot pair on the host; with N > 1 ranks it is
    replicated by an NCCL broadcast (the only data collective of the path)."""
    from paper_2211_12616_b200 import synthetic
    n_tot, dlon, dlat, nlev, pmin, mod, _ = WORKLOADS[wl]
    if wl == "cfg1":
        return synthetic.solid_body_pair(dlon, dlat, nlev)
    if ws == 1 or rank == 0:
        return synthetic.analytic_pair(dlon, dlat, nlev, 0.0, 10800.0, pmin)
    lons, lats, levs = synthetic.grid(dlon, dlat, nlev, pmin)
    return None, (lons, lats, levs)


def load_met_everywhere(eng, mets, ws, rank, torch, dist):
    """N = 1: H2D of both snapshots.  N > 1: rank 0's snapshots reach every
    rank by NCCL broadcast (sharding.broadcast_snapshot) and are packed into
    the met slots straight from device memory."""
    m0, m1 = mets
    if ws == 1:
        eng.bind_met(m0, m1)
        return m0, m1
    from paper_2211_12616_b200 import _capi as capi
    from paper_2211_12616_b200 import sharding
    dev = torch.device("cuda", torch.cuda.current_device())
    if rank == 0:
        grid = (m0.lons, m0.lats, m0.levs)
    else:
        lons, lats, levs = m1
        grid = (np.append(lons, lons[0] + 360.0), lats, levs)
    eng.set_grid(*grid)
    shape = (len(grid[0]), len(grid[1]), len(grid[2]))
    for slot, t_met in ((0, 0.0), (1, 10800.0)):
        src = (m0, m1)[slot] if rank == 0 else None
        buf = sharding.broadcast_snapshot(src, shape, dist, dev)
        torch.cuda.synchronize()
        p = buf.data_ptr()
        fb = buf[0].numel() * 4
        capi.check(eng.ctx.lib.lt_met_load(eng.ctx.h, slot, t_met, 4, p, p + fb, p + 2 * fb,
                                           p + 3 * fb, capi.MET_DEVICE_SRC))
        eng.ctx.sync()
        del buf
    eng.ctx.use_met(0, 1)
    return None, None


def cpu_sample_rate(wl, mets, ctl, n_sample, steps, threads, target_s=0.0):
    """The CPU oracle on `threads` host threads over a particle sample
    (DevicePool-style static partition); returns (particle-steps/s, wall s,
    sample size).  With target_s > 0 the sample is sized from a probe so the
    timed steps take about target_s seconds."""
    if target_s > 0:
        probe, _, _ = cpu_sample_rate(wl, mets, ctl, n_sample, 1, threads)
        n_sample = int(min(max(probe * target_s / steps, 10_000), 20_000_000))
    from concurrent.futures import ThreadPoolExecutor

    from oracle import lagtrans_oracle as orc
    from paper_2211_12616_b200 import synthetic
    m0, m1 = mets
    s0 = orc.Snapshot(m0.t_met, m0.lons, m0.lats, m0.levs, m0.u, m0.v, m0.w, m0.T)
    s1 = orc.Snapshot(m1.t_met, m1.lons, m1.lats, m1.levs, m1.u, m1.v, m1.w, m1.T)
    ens = synthetic.particles(n_sample, seed=12616)
    st = {"time": ens.time.copy(), "lon": ens.lon.copy(), "lat": ens.lat.copy(),
          "p": ens.p.copy(), "uvwp": np.zeros((3, n_sample)), "iso_var": np.zeros(n_sample),
          "q": np.zeros((5, n_sample))}
    mods = ("advection", "position") if WORKLOADS[wl][5] == "adv" else \
        ("advection", "turb", "meso", "position")
    ranges = [orc.split_range(n_sample, threads, d) for d in range(threads)]
    with ThreadPoolExecutor(threads) as pool:
        def one(step):
            list(pool.map(lambda r: orc.full_step(ctl, s0, s1, st, r[0], r[1], step, modules=mods),
                          ranges))
        one(0)  # warm-up
        t0 = time.perf_counter()
        for k in range(steps):
            one(1 + k)
        wall = time.perf_counter() - t0
    return n_sample * steps / wall, wall, n_sample


def make_ctl(wl, precision="exact"):
    from paper_2211_12616_b200.model_state import Control
    return Control(np_max=10 ** 10, t_stop=10 * 86400.0, dt_model=180.0, met_dt=10800.0,
                   turb_dx=50.0, turb_dz=0.1, turb_meso=0.16, rng_mode="counter",
                   rng_seed_global=12616, precision=precision)


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, wl):
    """--impl reference: the CPU oracle port of the reference path."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    n_tot, *_, desc = WORKLOADS[wl]
    mets = build_met(wl, 0, 1, None, None)
    ctl = make_ctl(wl)
    threads = host_threads()
    n_sample = args.cpu_sample or (100_000 if wl == "cfg1" else 20_000 * threads)
    rates = []
    for _ in range(max(1, min(3, args.steps // 10))):
        r, wall, n_used = cpu_sample_rate(wl, mets, ctl, n_sample, 2, threads, target_s=10.0)
        rates.append(r)
    v = statistics.median(rates)
    n_sample = n_used
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "particle-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n_tot / v, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "description": desc, "particles": n_tot},
        "cpu_baseline": {"value": v, "unit": "particle-steps/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{n_sample} particles x 2 steps per repeat on the same met grid"},
        "e2e": {"value": v, "unit": "particle-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--sort-every", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--precision", default="exact", choices=("exact", "fast"))
    ap.add_argument("--met-store", default="f32", choices=("f32", "f64"))
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = args.workload
    if args.impl == "reference":
        run_reference(args, wl)
        return

    import torch
    import torch.distributed as dist

    from paper_2211_12616_b200 import engine, sharding, synthetic

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_tot, dlon, dlat, nlev, pmin, mod, desc = WORKLOADS[wl]
    mask = engine.ADV if mod == "adv" else engine.ADV_DIFF
    work = sharding.shard_range(n_tot, ws, rank)
    ctl = make_ctl(wl, args.precision)

    mets = build_met(wl, rank, ws, torch, dist)
    eng = engine.Engine(device=local, first_id=work.start, met_precision=args.met_store)
    ens = synthetic.particles(work.size, seed=12616 + rank)
    eng.upload(ens)
    m0, m1 = load_met_everywhere(eng, mets, ws, rank, torch, dist)
    nodes = (eng.ctx._grid_key and 1) and None
    nx = len(mets[0].lons) if mets[0] is not None else len(mets[1][0]) + 1
    lats_n = len(mets[0].lats) if mets[0] is not None else len(mets[1][1])
    nlev_n = len(mets[0].levs) if mets[0] is not None else len(mets[1][2])
    nodes = nx * lats_n * nlev_n

    stream = torch.cuda.ExternalStream(eng.ctx.stream_handle())
    sort_every = args.sort_every if mod != "adv" or work.size > 10 ** 6 else 0

    def barrier():
        eng.sync()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    step = 0
    n_sorts = 0
    for _ in range(args.warmup):
        if sort_every and step % sort_every == 0:
            eng.sort()
        eng.step(ctl, step, mask)
        step += 1
    barrier()

    # timed region: K steps, CUDA events on the engine stream around each launch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 2)]
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for k in range(args.steps):
            if sort_every and step % sort_every == 0:
                eng.sort()
                n_sorts += 1
            ev[2 + 2 * k].record(stream)
            eng.step(ctl, step, mask)
            ev[3 + 2 * k].record(stream)
            step += 1
        ev[1].record(stream)
        barrier()
    total_ms = ev[0].elapsed_time(ev[1])
    kern_ms = [ev[2 + 2 * k].elapsed_time(ev[3 + 2 * k]) for k in range(args.steps)]
    total_ms, kern_avg = sharding.max_over_ranks([total_ms, statistics.mean(kern_ms)], dist,
                                                 "cuda")
    value = n_tot * args.steps / (total_ms / 1e3)

    # e2e: the public host-buffer API (Engine.step_host -> lt_run_host): the
    # shard's SoA sits in pinned host memory; every step streams it through
    # the GPU (H2D, fused step, D2H overlapped in chunks) and lands back.
    e2e = None
    if args.e2e_steps > 0:
        from paper_2211_12616_b200 import model_state as ms
        from paper_2211_12616_b200.context import pinned_empty
        n = work.size
        hens = ms.ParticleEnsemble(n, pinned_empty(n), pinned_empty(n), np.zeros(1),
                                   pinned_empty(n), pinned_empty(n), np.zeros((5, 1)))
        hcache = ms.CacheState(uvwp=pinned_empty((3, n)), iso_var=np.zeros(1))
        for k in ("time", "p", "lon", "lat"):
            getattr(hens, k)[:] = getattr(ens, k)
        hcache.uvwp[:] = 0.0
        eng.step_host(ctl, hens, hcache, step, mask)   # warm-up (allocations, events)
        step += 1
        barrier()
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            eng.step_host(ctl, hens, hcache, step, mask)
            step += 1
        barrier()
        te = sharding.max_over_ranks([time.perf_counter() - t0], dist, "cuda")[0]
        rows_in = 4 + (3 if mod != "adv" else 0)
        rows_out = rows_in
        e2e = {"value": n_tot * args.e2e_steps / te, "unit": "particle-steps/s",
               "h2d_bytes_per_step": 8 * rows_in * n_tot, "d2h_bytes_per_step": 8 * rows_out * n_tot,
               "path": "Engine.step_host -> lt_run_host: pinned host SoA, chunked H2D / fused "
                       "step / D2H on three streams, every step"}

    # roofline of the dominant kernel (step_kernel), algorithmic bytes
    b = algorithmic_bytes(mod, work.size, nodes)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = b * work.size / (kern_avg / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / f"ncu_step_{wl}.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = host_threads()
        n_sample = args.cpu_sample or (100_000 if wl == "cfg1" else 20_000 * threads)
        mh = mets if wl == "cfg1" else (m0, m1)
        rate, wall, n_sample = cpu_sample_rate(wl, mh, make_ctl(wl), n_sample, 2, threads,
                                               target_s=15.0)
        cpu = {"value": rate, "unit": "particle-steps/s", "cores": threads, "kind": "port",
               "sample": f"oracle/ numpy port, {n_sample} particles x 2 timed steps on the "
                         f"same {wl} met grid ({wall:.1f} s)"}

    launches = args.steps + n_sorts * 13  # keys 1 + CUB 6 + row gathers 5 + ids 1
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl, "description": desc, "particles": n_tot,
                       "particles_per_gpu": work.size, "met_nodes": nodes,
                       "met_store": f"{args.met_store} node-pair records", "state": "fp64 SoA",
                       "precision": args.precision,
                       "rng": "counter (bit-identical to reference), in-kernel",
                       "sort_every": sort_every, "parallelism": f"particles sharded x{ws}",
                       "l2": "inputs larger than L2 (state %.1f GB/GPU)" % (
                           work.size * 144 / 1e9)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "step_kernel", "kernel_ms": kern_avg,
                         "algorithmic_bytes_per_particle_step": b,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": launches,
        }), flush=True)
    eng.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
