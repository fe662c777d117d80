"""Benchmark: particle-steps/s of the fused time step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3]
                    [--impl b200|reference] [--precision fast|exact]

Headline workload (BASELINE.json configs[2], the configuration the metric is
quoted on): **cfg3** — 1e8 particles on the synthetic ERA5-like 0.25 deg grid
(1440(+1) x 721 x 137), advection + turbulent + mesoscale diffusion
(+ timesteps, in-kernel Philox draws, position), sharded over N GPUs with the
reference partition rule (strong scaling: 1e8 in total; `--scaling weak`
keeps 1e8 per GPU), met replicated to every GPU by an NCCL broadcast.  N > 1
runs either as torchrun ranks (one GPU each) or, without torchrun, as ONE
process driving N GPUs (the paper's design; lt_met_broadcast).  A "step" is
one fused time step of every particle; the box sort runs every
`--sort-every` steps (15 for cfg3, the measured optimum — flat from 15 to
25; the default 30 timed steps hold exactly two sorts) inside the timed
region.

Other workloads (parity shapes, informational lines): cfg1 (SBR, 1e5,
advection), cfg2 (1e7, 1 deg), cfg4 (5e7 volcanic point release, advection
+ diffusion + sedimentation + decay, a new met snapshot streamed from pinned
host memory every simulated hour = every 20 steps, inside the timed region),
cfg5 (5e8 particles, the full module chain + decay, sort every 10 steps).

`value` is device-timed (CUDA events on the engine stream, max over ranks,
inputs resident in HBM); `roofline.achieved` counts SURVEY.md 8(d)'s
algorithmic bytes per particle-step.  `e2e` is the public host-buffer API
(Engine.step_host -> lt_run_host): the shard's SoA in pinned host memory
streams in, steps and streams out every step; the line carries the host
link's measured ceiling beside it.  `cpu_baseline` and `--impl
reference` time the CPU oracle (a numpy restatement of the reference,
oracle/) on the host's cores on a bounded particle sample of the same
workload.  `precision` "fast" (default) computes interpolation weights and
sums and the Box-Muller transform in fp32 with fp64 particle state; it stays
within the north star's 1e-5 run tolerance (tests/test_gpu_engine.py).
`--rng philox` (default) is the north star's counter-based generator keyed
by the full 32-bit particle id — the reference's splitmix64 counter key
packs only 24 bits of index, so at 1e8 particles it would hand particles i
and i + 2^24 identical draws; `counter` reproduces the reference's words
bit for bit.  The line also carries the same measurement with the
bit-faithful "exact" kernels (`alt_precision`), with the counter words
(`alt_rng`), with both — the like-for-like, fully reference-faithful
configuration (`alt_reference_faithful`) — and with the steps between two
sorts run as one multi-step launch each (`alt_multistep`, Engine.step_many;
identical results).  The headline is one launch per step, the unit its
roofline is stated for.  The reference arm builds its inputs without
importing the product package and reports `product_code_loaded`.
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
ADV = ("advection", "position")
ADV_DIFF = ("advection", "turb", "meso", "position")
PLUME = ("advection", "turb", "meso", "sedi", "decay", "position")
FULL = ("advection", "turb", "meso", "convection", "sedi", "decay", "isosurf", "position",
        "meteo")
WORKLOADS = {
    "cfg1": dict(n=100_000, grid=(1.0, 1.0, 60, 1.0), met="sbr", chain=ADV, init="uniform",
                 sort_every=0, desc="1e5 particles, solid-body rotation 1deg x 60, advection only"),
    "cfg2": dict(n=10_000_000, grid=(1.0, 1.0, 60, 1.0), met="era5", chain=ADV_DIFF,
                 init="uniform", sort_every=10,
                 desc="1e7 particles, ERA5-like 1deg 360x181x60, advection+turb+meso diffusion"),
    "cfg3": dict(n=100_000_000, grid=(0.25, 0.25, 137, 0.01), met="era5", chain=ADV_DIFF,
                 init="uniform", sort_every=15,
                 desc="1e8 particles, ERA5-like 0.25deg 1440x721x137, advection+turb+meso "
                      "diffusion"),
    "cfg4": dict(n=50_000_000, grid=(0.25, 0.25, 137, 0.01), met="stream", chain=PLUME,
                 init="point", sort_every=0, met_dt=3600.0,
                 ctl=dict(sedi_radius=5e-6, sedi_density=2000.0, decay_tau=3 * 86400.0,
                          decay_slot=5, nq=6),
                 desc="volcanic point release of 5e7 particles (-175.4E, -20.5N, 30 hPa), "
                      "advection+diffusion+sedimentation+decay, 0.25deg met streamed hourly "
                      "from pinned host memory"),
    "cfg5": dict(n=500_000_000, grid=(0.25, 0.25, 137, 0.01), met="era5", chain=FULL,
                 init="uniform", sort_every=10,
                 ctl=dict(conv_prob=0.05, sedi_radius=1e-6, isosurf_mode="theta",
                          decay_tau=3 * 86400.0, decay_slot=5, nq=6),
                 desc="5e8 particles, full module chain (+decay) with box sort every 10 "
                      "steps"),
}
# algorithmic state bytes per particle-step, SURVEY.md 8(d) ("fp64
# lon/lat/p/time + fp32 uvwp" column): lon/lat/p/time read + written (64 B),
# + the meso AR(1) state uvwp as fp32 read + written (24 B), + for the
# longer chains the decayed q slot read + written (16 B) and, for the full
# chain, iso_var read (8 B) and q0..4 written (40 B)
STATE_BYTES = {ADV: 64, ADV_DIFF: 88, PLUME: 104, FULL: 152}
# what this implementation's rows actually move per particle-step: uvwp is
# kept in fp64 (the reference's CacheState dtype; the exact kernels need it),
# i.e. +24 B over 8(d), plus the 4-byte particle-id row (RNG key) once sorted
MOVED_STATE_BYTES = {ADV: 64, ADV_DIFF: 116, PLUME: 132, FULL: 180}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def algorithmic_bytes(chain, n_local: int, nodes: int) -> float:
    """b = b_state + 32*nodes*(1 - exp(-8 N/nodes)) / N per
    particle-step (two fp32 snapshots' node-pair records over the touched
    cells, each read once per step)."""
    b_met = 32.0 * nodes * (1.0 - math.exp(-8.0 * n_local / nodes)) / n_local
    return STATE_BYTES[chain] + b_met


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
            # nvidia-smi takes a while to start: begin the timed region only
            # once it is sampling, so short regions are covered too
            t0 = time.time()
            while not self.rows and self.proc.poll() is None and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.rows.clear()
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
            # at least one sample taken during (or right at the end of) the region
            t0 = time.time()
            while not self.rows and self.proc.poll() is None and time.time() - t0 < 2.0:
                time.sleep(0.01)
            time.sleep(0.05)
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


def pure_modules():
    """(synthetic, model_state) loaded WITHOUT the package's __init__ (which
    loads liblagtrans_b200.so): the --impl reference arm builds the same
    inputs with no product code mapped into the process."""
    import importlib
    import types
    name = "_lt_inputs"
    if name not in sys.modules:
        pkg = types.ModuleType(name)
        pkg.__path__ = [str(ROOT / "paper_2211_12616_b200")]
        sys.modules[name] = pkg
    return importlib.import_module(name + ".synthetic"), importlib.import_module(name + ".model_state")


def make_ctl(wl, precision="fast", rng_mode="counter"):
    _, ms = pure_modules()
    Control = ms.Control
    cfg = WORKLOADS[wl]
    kw = dict(np_max=10 ** 10, t_stop=30 * 86400.0, dt_model=180.0,
              met_dt=cfg.get("met_dt", 10800.0), turb_dx=50.0, turb_dz=0.1, turb_meso=0.16,
              rng_mode=rng_mode, rng_seed_global=12616, precision=precision)
    kw.update(cfg.get("ctl", {}))
    return Control(**kw)


def make_particles(wl, n, seed):
    synthetic, _ = pure_modules()
    cfg = WORKLOADS[wl]
    nq = cfg.get("ctl", {}).get("nq", 5)
    if cfg["init"] == "point":
        ens = synthetic.point_release(n, nq=nq)
    else:
        ens = synthetic.particles(n, seed=seed, nq=nq)
    if nq > 5:
        ens.q[5] = 1.0   # the decayed tracer mass
    return ens


def build_met(wl, rank, ws):
    """Rank 0 (or the only rank) builds the first snapshot pair on the host;
    other ranks only need the grid (the fields arrive by broadcast)."""
    synthetic, _ = pure_modules()
    cfg = WORKLOADS[wl]
    dlon, dlat, nlev, pmin = cfg["grid"]
    if cfg["met"] == "sbr":
        return synthetic.solid_body_pair(dlon, dlat, nlev)
    t1 = cfg.get("met_dt", 10800.0)
    if ws == 1 or rank == 0:
        return synthetic.analytic_pair(dlon, dlat, nlev, 0.0, t1, pmin)
    return None, synthetic.grid(dlon, dlat, nlev, pmin)


def load_met_everywhere(eng, mets, wl, ws, rank, torch, dist):
    """N = 1: H2D of both snapshots.  N > 1: rank 0's snapshots reach every
    rank by NCCL broadcast (sharding.broadcast_snapshot) and are packed into
    the met slots straight from device memory."""
    m0, m1 = mets
    if ws == 1:
        eng.bind_met(m0, m1)
        return
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
    for slot, t_met in ((0, 0.0), (1, WORKLOADS[wl].get("met_dt", 10800.0))):
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
    eng._met_slots, eng._staged = (0, 1), None


def streamed_nodes(wl, ws, rank, torch, dist):
    """cfg4: two hourly snapshots as pinned (nx, ny, nz, 4) fp32 node arrays
    (without the +360 column); the stream alternates them at increasing
    t_met.  N > 1: rank 0 builds them and broadcasts."""
    from paper_2211_12616_b200 import synthetic
    from paper_2211_12616_b200.context import pinned_empty
    dlon, dlat, nlev, pmin = WORKLOADS[wl]["grid"]
    lons, lats, levs = synthetic.grid(dlon, dlat, nlev, pmin)
    shape = (len(lons), len(lats), len(levs), 4)
    out = []
    for phase in (20.0, 30.0):
        host = pinned_empty(shape, np.float32)
        if ws == 1 or rank == 0:
            f = synthetic.era5_like(lons, lats, levs, phase)
            for c, k in enumerate(("u", "v", "w", "T")):
                host[..., c] = f[k]
        if ws > 1:
            dev = torch.device("cuda", torch.cuda.current_device())
            buf = torch.from_numpy(host).to(dev) if rank == 0 else \
                torch.empty(shape, dtype=torch.float32, device=dev)
            dist.broadcast(buf, src=0)
            torch.from_numpy(host).copy_(buf.cpu())
            del buf
        out.append(host)
    return out


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
    m0, m1 = mets
    s0, s1 = orc.Snapshot.like(m0), orc.Snapshot.like(m1)
    ens = make_particles(wl, n_sample, 12616)
    st = {"time": ens.time.copy(), "lon": ens.lon.copy(), "lat": ens.lat.copy(),
          "p": ens.p.copy(), "uvwp": np.zeros((3, n_sample)), "iso_var": np.zeros(n_sample),
          "q": ens.q.copy()}
    chain = WORKLOADS[wl]["chain"]
    clim = orc.climatology_tables() if "meteo" in chain else None
    if "isosurf" in chain:
        st["iso_var"] = orc.isosurface_value(ctl, s0, s1, st["lon"], st["lat"], st["p"],
                                             st["time"], st["iso_var"])
    ranges = [orc.split_range(n_sample, threads, d) for d in range(threads)]
    with ThreadPoolExecutor(threads) as pool:
        def one(step):
            list(pool.map(lambda r: orc.full_step(ctl, s0, s1, st, r[0], r[1], step, clim=clim,
                                                  modules=chain), ranges))
        one(0)  # warm-up
        t0 = time.perf_counter()
        for k in range(steps):
            one(1 + k)
        wall = time.perf_counter() - t0
    return n_sample * steps / wall, wall, n_sample


def pcie_duplex_gbs(torch, gpu, gib=1):
    """Measured host-link ceiling: pinned H2D and D2H of `gib` GiB running
    at once on two streams (the e2e path's traffic pattern); GB/s per
    direction, best of 3."""
    n = (gib << 30) // 8
    h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.float64, device=f"cuda:{gpu}")
    d2 = torch.empty(n, dtype=torch.float64, device=f"cuda:{gpu}")
    s1, s2 = torch.cuda.Stream(gpu), torch.cuda.Stream(gpu)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(gpu)
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(gpu)
        best = min(best, time.perf_counter() - t0)
    del h1, h2, d1, d2
    return n * 8 / best / 1e9


def e2e_driver_run(wl, steps=30, met_dt=3600.0):
    """The reference's whole run loop through the drop-in's public driver
    (driver.run_simulation, driver_cli.py:84-209 without file I/O) at the
    workload's shape: particles from host memory, hourly met snapshots
    (three, the third prefetched and rotated in while stepping), outputs
    copied back every simulated hour.  Wall clock of the call; an
    informational line beside `e2e` (which moves every particle through
    PCIe every step)."""
    import dataclasses

    from paper_2211_12616_b200 import driver, engine, synthetic
    cfg = WORKLOADS[wl]
    dlon, dlat, nlev, pmin = cfg["grid"]
    lons, lats, levs = synthetic.grid(dlon, dlat, nlev, pmin)
    mets = [synthetic.snapshot(k * met_dt, lons, lats, levs,
                               synthetic.era5_like(lons, lats, levs, 10.0 * k, periodic=True))
            for k in range(3)]
    from paper_2211_12616_b200 import model_state as ms
    from paper_2211_12616_b200.context import pinned_empty
    ctl = dataclasses.replace(make_ctl(wl, "fast", "philox"), t_stop=steps * 180.0,
                              met_dt=met_dt, output_dt=met_dt)
    src = make_particles(wl, cfg["n"], 12616)
    n = src.np
    # the host ensemble and cache in pinned memory, as a production caller would
    rows = {k: pinned_empty(n) for k in ("time", "p", "zeta", "lon", "lat")}
    for k, a in rows.items():
        a[:] = getattr(src, k)
    q = pinned_empty(src.q.shape)
    q[:] = src.q
    ens = ms.ParticleEnsemble(n, rows["time"], rows["p"], rows["zeta"], rows["lon"], rows["lat"], q)
    cache = ms.CacheState(uvwp=pinned_empty((3, n)), iso_var=pinned_empty(n))
    cache.uvwp[:] = 0.0
    cache.iso_var[:] = 0.0
    outputs = []

    class Sink:   # the driver's timer rows (timers.py names), summed
        def __init__(self):
            self.s = {}

        def record(self, name, group, scope, ns):
            self.s[name] = self.s.get(name, 0) + ns
    sink = Sink()
    t0 = time.perf_counter()
    status, _ = driver.run_simulation(ctl, ens, mets, num_devices=1, fused=True,
                                      modules=engine.modules_mask(cfg["chain"]), cache=cache,
                                      timers=sink, on_output=lambda c, e, ca, t: outputs.append(t))
    wall = time.perf_counter() - t0
    if status != 0:
        return {"error": "run_simulation failed"}
    return {"value": cfg["n"] * steps / wall, "unit": "particle-steps/s", "wall_s": wall,
            "steps": steps, "outputs": len(outputs),
            "timers_s": {k: round(v / 1e9, 4) for k, v in sorted(sink.s.items())},
            "path": "driver.run_simulation (fused, multi-step launches, box sort every 15): "
                    "1e8 particles uploaded from pinned host memory, 3 hourly snapshots (the "
                    "third streamed on the copy stream while stepping), every particle's "
                    "state copied back at each hourly output; wall clock including setup "
                    "(met content fingerprints, device allocation)"}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, wl):
    """--impl reference: the CPU oracle port of the reference path on all
    host threads, rank 0 only."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = WORKLOADS[wl]
    n_job = cfg["n"] * (ws if args.scaling == "weak" else 1)
    mets = build_met(wl, 0, 1)
    ctl = make_ctl(wl, "exact")
    threads = host_threads()
    n_sample = args.cpu_sample or (100_000 if wl == "cfg1" else 20_000 * threads)
    rates = []
    for _ in range(max(1, min(3, args.steps // 10))):
        r, wall, n_used = cpu_sample_rate(wl, mets, ctl, n_sample, 2, threads, target_s=10.0)
        rates.append(r)
    v = statistics.median(rates)
    try:   # the arm must not have mapped any product library (checked, reported)
        maps = Path("/proc/self/maps").read_text()
        product_loaded = "liblagtrans_b200" in maps
    except OSError:
        product_loaded = None
    print(json.dumps({
        "impl": "reference", "product_code_loaded": product_loaded, "metric": METRIC, "value": v, "unit": "particle-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n_job / v, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "description": cfg["desc"], "particles": n_job,
                   "modules": list(cfg["chain"]), "precision": "exact (numpy fp64, the "
                   "reference's operation sequence)", "rng": "counter (reference splitmix64 "
                   "words)", "parallelism": f"{threads} host threads, DevicePool-style static "
                   "partition (device_runtime.py:136-161)"},
        "cpu_baseline": {"value": v, "unit": "particle-steps/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{n_used} particles x 2 steps per repeat on the same "
                                   f"{wl} met grid, {len(rates)} repeats (median); "
                                   "ms_per_step is the sample rate scaled to the "
                                   "workload's particle count"},
        "e2e": {"value": v, "unit": "particle-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def run_one_process(args, wl):
    """--gpus N without torchrun: ONE process drives N GPUs (the paper's
    design, arXiv 2211.12616 / device_runtime.DevicePool): one Engine and one
    host thread per GPU, particles sharded by calc_device_workload_range,
    met uploaded once to GPU 0 and replicated by lt_met_broadcast (one NCCL
    broadcast group over NVLink/NVSwitch).  Timing: CUDA events on every
    engine's stream after a common barrier, max over GPUs.  (More devices
    than GPUs present share them round-robin: the functional path on a
    single-GPU box, where the broadcast degenerates to device-local copies.)"""
    import torch
    from concurrent.futures import ThreadPoolExecutor

    from paper_2211_12616_b200 import engine
    from paper_2211_12616_b200.context import met_broadcast, nccl_info
    from paper_2211_12616_b200.partition import partition_all
    cfg = WORKLOADS[wl]
    G = args.gpus
    ngpu = torch.cuda.device_count()
    devs = [d % ngpu for d in range(G)]
    n_tot = cfg["n"] * (G if args.scaling == "weak" else 1)
    ranges = partition_all(n_tot, G)
    mask = engine.modules_mask(cfg["chain"])
    ctl = make_ctl(wl, args.precision, args.rng)
    m0, m1 = build_met(wl, 0, 1)
    pool = ThreadPoolExecutor(G)
    engs = [None] * G

    def setup(d):
        torch.cuda.set_device(devs[d])
        w = ranges[d]
        e = engine.Engine(device=devs[d], first_id=w.start, nq=ctl.nq)
        e.upload(make_particles(wl, w.size, 12616 + d))
        e.set_grid(m0.lons, m0.lats, m0.levs)
        engs[d] = e
    list(pool.map(setup, range(G)))
    # met: one host upload (GPU 0), one broadcast per snapshot to the others
    t0 = time.perf_counter()
    engs[0].ctx.load_met(0, m0, key="m0")
    engs[0].ctx.load_met(1, m1, key="m1")
    if G > 1:
        for slot in (0, 1):
            met_broadcast([e.ctx for e in engs], 0, [slot] * G)
    for e in engs:
        e.ctx.use_met(0, 1)
        e._met_slots, e._staged = (0, 1), None
        e.sync()
    t_met = time.perf_counter() - t0
    sort_every = args.sort_every if args.sort_every >= 0 else cfg["sort_every"]
    state = {"step": 0}

    def steps(d, k, ev=None):
        torch.cuda.set_device(devs[d])
        e = engs[d]
        st = state["step"]
        sh = torch.cuda.ExternalStream(e.ctx.stream_handle())
        if ev:
            ev[0].record(sh)
        for i in range(k):
            if sort_every and (st + i) % sort_every == 0:
                e.sort(mask)
            e.step(ctl, st + i, mask, device_id=d,
                   sort_next=bool(sort_every) and (st + i + 1) % sort_every == 0)
        if ev:
            ev[1].record(sh)
        e.sync()

    def run(k, timed=False):
        evs = None
        if timed:
            evs = []
            for d in range(G):
                with torch.cuda.device(devs[d]):
                    evs.append([torch.cuda.Event(enable_timing=True) for _ in range(2)])
        list(pool.map(lambda d: steps(d, k, evs[d] if evs else None), range(G)))
        state["step"] += k
        return max(ev[0].elapsed_time(ev[1]) for ev in evs) if evs else None

    run(args.warmup)
    with ClockSampler(devs[0]) as clk:
        total_ms = run(args.steps, timed=True)
    value = n_tot * args.steps / (total_ms / 1e3)
    dlon, dlat, nlev, pmin = cfg["grid"]
    nodes = (int(round(360.0 / dlon)) + 1) * (int(round(180.0 / dlat)) + 1) * nlev
    b = algorithmic_bytes(cfg["chain"], ranges[0].size, nodes)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    per_gpu_ms = total_ms / args.steps
    achieved = b * ranges[0].size / (per_gpu_ms / 1e3) / 1e9
    from paper_2211_12616_b200 import _capi as capi
    selftest = "ok"
    try:   # NCCL over the distinct GPUs of this run, checked byte for byte
        capi.check(capi.load().lt_nccl_selftest(len(set(devs)), 1 << 20))
    except Exception as exc:  # reported, not fatal: the timed run did not need it
        selftest = f"failed: {exc}"
    info = nccl_info()
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": G,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_gpu_ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64 state / f32 interpolation" if args.precision == "fast" else "f64",
        "data": "synthetic",
        "config": {"workload": wl, "description": cfg["desc"], "particles": n_tot,
                   "particles_per_gpu": ranges[0].size, "modules": list(cfg["chain"]),
                   "precision": args.precision, "rng": args.rng, "sort_every": sort_every,
                   "parallelism": f"one process drives {G} GPUs (threads), particles sharded "
                                  f"(calc_device_workload_range), met replicated by "
                                  "lt_met_broadcast (NCCL), no data-path collective",
                   "devices": devs, "l2": "inputs larger than L2"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "kernel": "step_kernel (per GPU, "
                     "ms/step incl. sorts)", "algorithmic_bytes_per_particle_step": b},
        "met_broadcast": {"nccl_version": info["version"], "nccl_ranks": info["ranks"],
                          "nccl_selftest": selftest,
                          "gpus_distinct": len(set(devs)),
                          "setup_s_upload_plus_broadcast": t_met},
        "clocks": clk.summary(),
        "gpu_launches": args.steps * G + G * sum(1 for i in range(args.steps)
                                                 if sort_every and (args.warmup + i) % sort_every == 0) * 7,
    }), flush=True)
    for e in engs:
        e.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--sort-every", type=int, default=-1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=0,
                    help="particles per host-path chunk (0: the library default)")
    ap.add_argument("--alt-steps", type=int, default=-1,
                    help="timed steps with the other precision's kernels (default: --steps)")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--precision", default="fast", choices=("exact", "fast"))
    ap.add_argument("--met-store", default="f32", choices=("f32", "f64"))
    ap.add_argument("--rng", default="philox", choices=("counter", "faithful", "philox"))
    ap.add_argument("--scaling", default="strong", choices=("weak", "strong"),
                    help="strong (default, BASELINE cfg3: 1e8 sharded over 1/2/4/8 GPUs): "
                         "the workload's total is sharded over the GPUs; weak: each GPU "
                         "advances the workload's particle count")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = args.workload
    if args.impl == "reference":
        run_reference(args, wl)
        return
    if args.gpus > 1 and dist_env()[0] == 1:
        run_one_process(args, wl)
        return

    import torch
    import torch.distributed as dist

    from paper_2211_12616_b200 import engine, sharding

    cfg = WORKLOADS[wl]
    ws, rank, local = dist_env()
    # one rank per GPU; LT_DIST_BACKEND=gloo with more ranks than GPUs maps
    # ranks round-robin onto the GPUs present (tests the N > 1 path on one GPU)
    gpu = local % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    if ws > 1:
        backend = os.environ.get("LT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    # weak scaling (default): every rank advances the workload's particle
    # count, global ids offset per rank (independent particles, no data-path
    # collective); strong: the workload's total is sharded over the ranks
    n_tot = cfg["n"] * ws if args.scaling == "weak" else cfg["n"]
    mask = engine.modules_mask(cfg["chain"])
    work = sharding.shard_range(n_tot, ws, rank)
    ctl = make_ctl(wl, args.precision, args.rng)

    mets = build_met(wl, rank, ws)
    eng = engine.Engine(device=gpu, first_id=work.start, met_precision=args.met_store,
                        nq=ctl.nq)
    ens = make_particles(wl, work.size, 12616 + rank)
    eng.upload(ens)
    load_met_everywhere(eng, mets, wl, ws, rank, torch, dist)
    if "meteo" in cfg["chain"]:
        from paper_2211_12616_b200.model_state import read_clim
        eng.load_clim(read_clim(ctl))
    eng.init_isosurf(ctl)
    dlon, dlat, nlev, pmin = cfg["grid"]
    nodes = (int(round(360.0 / dlon)) + 1) * (int(round(180.0 / dlat)) + 1) * nlev

    # met streaming (cfg4): the next snapshot is staged on the copy stream
    # right after every rotation; rotation follows driver_cli.py:139-149
    stream = None
    if cfg["met"] == "stream":
        stream = {"nodes": streamed_nodes(wl, ws, rank, torch, dist), "k": 0,
                  "t1": cfg["met_dt"], "rotations": 0}

        def stage_next():
            s = stream
            eng.prefetch(nodes=s["nodes"][s["k"] % 2].ctypes.data,
                         t_met=s["t1"] + cfg["met_dt"], close_lon=True)
            s["k"] += 1
        stage_next()
    t_model = [0.0]

    stream_h = torch.cuda.ExternalStream(eng.ctx.stream_handle())
    sort_every = args.sort_every if args.sort_every >= 0 else cfg["sort_every"]

    def barrier():
        eng.sync()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    step = 0
    n_sorts = 0

    def one_step(c, record=None):
        nonlocal step, n_sorts
        t_next = t_model[0] + ctl.dt_model
        if stream is not None and stream["t1"] < t_next:   # rotate + stage the next hour
            eng.rotate()
            stream["t1"] += cfg["met_dt"]
            stream["rotations"] += 1
            stage_next()
        if sort_every and step % sort_every == 0:
            eng.sort(mask)
            n_sorts += 1
        if record:
            record[0].record(stream_h)
        # a sort opens the next step: this launch writes the sort keys
        eng.step(c, step, mask, sort_next=bool(sort_every) and (step + 1) % sort_every == 0)
        if record:
            record[1].record(stream_h)
        step += 1
        t_model[0] = t_next

    for _ in range(args.warmup):
        one_step(ctl)
    barrier()

    fused_sorts = [0]   # sorts of the headline timed region that used step-written keys

    def timed(c, k_steps):
        sorts0 = n_sorts
        info0 = eng.ctx.sort_info()[1]
        rot0 = stream["rotations"] if stream else 0
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * k_steps + 2)]
        with ClockSampler(gpu) as clk:
            ev[0].record(stream_h)
            for k in range(k_steps):
                one_step(c, (ev[2 + 2 * k], ev[3 + 2 * k]))
            ev[1].record(stream_h)
            barrier()
        total = ev[0].elapsed_time(ev[1])
        per = [ev[2 + 2 * k].elapsed_time(ev[3 + 2 * k]) for k in range(k_steps)]
        kern = statistics.mean(per)
        if os.environ.get("LT_BENCH_PER_STEP"):
            print("per-step kernel ms:", " ".join(f"{t:.3f}" for t in per), file=sys.stderr)
        fused_sorts[0] = eng.ctx.sort_info()[1] - info0
        total, kern = sharding.max_over_ranks([total, kern], dist, "cuda")
        return total, kern, clk.summary(), n_sorts - sorts0, \
            (stream["rotations"] - rot0 if stream else 0)

    total_ms, kern_avg, clocks, sorts_timed, rots = timed(ctl, args.steps)
    fused_timed = fused_sorts[0]
    value = n_tot * args.steps / (total_ms / 1e3)
    b = algorithmic_bytes(cfg["chain"], work.size, nodes)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = b * work.size / (kern_avg / 1e3) / 1e9

    # the same steps with the other kernels, same state, same protocol:
    # the other precision, and the reference's bit-identical counter words
    def alt_run(precision, rng, k):
        t2, k2, clk2, _, _ = timed(make_ctl(wl, precision, rng), k)
        return {"precision": precision, "rng": rng, "value": n_tot * k / (t2 / 1e3),
                "ms_per_step": t2 / k, "kernel_ms": k2,
                "roofline_frac": b * work.size / (k2 / 1e3) / 1e9 / peak, "steps": k,
                "clocks": clk2}

    other = alt_rng = alt_ref = None
    k_other = args.steps if args.alt_steps < 0 else args.alt_steps
    if k_other > 0:
        other = alt_run("exact" if args.precision == "fast" else "fast", args.rng, k_other)
        if args.rng != "counter":
            alt_rng = alt_run(args.precision, "counter", k_other)
        if (args.precision, args.rng) != ("exact", "counter") and \
                (other["precision"], other["rng"]) != ("exact", "counter"):
            # the fully reference-faithful configuration: numpy-exact fp64
            # kernels fed the reference's own counter words (like for like
            # with the --impl reference arm)
            alt_ref = alt_run("exact", "counter", k_other)

    # the same steps with the sort cadence, but every run of steps between
    # two sorts is one multi-step launch (Engine.step_many: each particle
    # advanced in registers; identical results) — informational beside the
    # one-launch-per-step headline
    multi = None
    if k_other > 0 and stream is None and args.rng in ("counter", "philox") and \
            not any(m in cfg["chain"] for m in ("meteo", "decay")):
        nonlocal_step = [step]

        def run_multi(k_steps):
            ev0, ev1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            st = nonlocal_step[0]
            with ClockSampler(gpu) as clk:
                ev0.record(stream_h)
                done = 0
                while done < k_steps:
                    if sort_every and st % sort_every == 0:
                        eng.sort(mask)
                    run = k_steps - done
                    if sort_every:
                        run = min(run, sort_every - st % sort_every)
                    eng.step_many(ctl, st, run, mask,
                                  sort_next=bool(sort_every) and (st + run) % sort_every == 0)
                    st += run
                    done += run
                ev1.record(stream_h)
                barrier()
            nonlocal_step[0] = st
            t = sharding.max_over_ranks([ev0.elapsed_time(ev1)], dist, "cuda")[0]
            return t, clk.summary()

        run_multi(min(k_other, 15))            # warm-up of the multi-step kernels
        t_m, clk_m = run_multi(k_other)
        step = nonlocal_step[0]
        multi = {"value": n_tot * k_other / (t_m / 1e3), "ms_per_step": t_m / k_other,
                 "steps": k_other, "sort_every": sort_every, "clocks": clk_m,
                 "launches": "one per run of steps between sorts (the first step after a "
                             "sort applies its permutation alone)"}

    # e2e: the public host-buffer API (Engine.step_host -> lt_run_host): the
    # shard's SoA sits in pinned host memory; every step streams it through
    # the GPU (H2D, fused step, D2H overlapped in chunks) and lands back.
    e2e = None
    if args.e2e_steps > 0 and stream is None:
        from paper_2211_12616_b200 import _capi as capi
        from paper_2211_12616_b200 import model_state as ms
        from paper_2211_12616_b200.context import pinned_empty
        n = work.size
        want_q = any(m in cfg["chain"] for m in ("meteo", "decay"))
        want_iso = "isosurf" in cfg["chain"]
        hens = ms.ParticleEnsemble(n, pinned_empty(n), pinned_empty(n), np.zeros(1),
                                   pinned_empty(n), pinned_empty(n),
                                   pinned_empty((ctl.nq, n)) if want_q else np.zeros((5, 1)))
        hcache = ms.CacheState(uvwp=pinned_empty((3, n)),
                               iso_var=pinned_empty(n) if want_iso else np.zeros(1))
        for k in ("time", "p", "lon", "lat"):
            getattr(hens, k)[:] = getattr(ens, k)
        if want_q:
            hens.q[:] = ens.q
        hcache.uvwp[:] = 0.0
        if want_iso:
            eng.ctx.d2h_ordered(capi.F_ISO_VAR, 0, 0, n, eng.first_id, out=hcache.iso_var)
        eng.step_host(ctl, hens, hcache, step, mask, chunk=args.e2e_chunk)   # warm-up
        step += 1
        barrier()
        # K steps in one call: every step still moves every particle host ->
        # device -> host; chunks of step s+1 start as chunks of step s land
        t0 = time.perf_counter()
        eng.step_host(ctl, hens, hcache, step, mask, chunk=args.e2e_chunk, steps=args.e2e_steps)
        step += args.e2e_steps
        barrier()
        te = sharding.max_over_ranks([time.perf_counter() - t0], dist, "cuda")[0]
        chain = cfg["chain"]
        rows_in = 4 + (3 if "meso" in chain else 0) + (1 if want_iso else 0) + \
            (1 if "decay" in chain else 0)
        rows_out = 4 + (3 if "meso" in chain else 0) + \
            (5 if "meteo" in chain else (1 if "decay" in chain else 0))
        bw = pcie_duplex_gbs(torch, gpu)
        h2d_b, d2h_b = 8 * rows_in * n_tot, 8 * rows_out * n_tot
        ceiling = n_tot / (max(h2d_b, d2h_b) / ws / (bw * 1e9))
        e2e = {"value": n_tot * args.e2e_steps / te, "unit": "particle-steps/s",
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
               "steps": args.e2e_steps,
               "bound": "host link (PCIe): every step moves the state rows in and out",
               "pcie_duplex_gbs_per_direction": bw, "pcie_ceiling": ceiling,
               "frac_of_pcie_ceiling": n_tot * args.e2e_steps / te / ceiling,
               "path": "Engine.step_host(steps=K) -> lt_run_host_steps: pinned host SoA, every "
                       "step chunked H2D / fused step / D2H on three streams, pipelined across "
                       "steps (wall clock, max over ranks)"}

    traffic = None
    issue = None
    prof = ROOT / "profiles" / f"ncu_step_{wl}.json"
    if prof.exists():
        pj = json.loads(prof.read_text()).get(args.precision, {})
        if pj.get("dram_bytes_per_particle_step") is not None:
            traffic = pj["dram_bytes_per_particle_step"] * work.size
        if pj.get("issue_active_pct") is not None:
            # the bound that binds: instruction issue / latency, from the same capture
            issue = {"issue_active": pj["issue_active_pct"] / 100.0,
                     "thread_instructions_per_particle_step":
                         pj.get("thread_instructions_per_particle"),
                     "source": f"profiles/ncu_step_{wl}.json (ncu --set full)"}

    e2e_drv = None
    if ws == 1 and args.e2e_steps > 0 and stream is None and wl == "cfg3":
        eng.close()   # the driver builds its own device image
        # and its own pinned host ensemble: release the e2e leg's first
        # (a process holding both measured cudaFree-bound region deletes
        # of 0.03-1.5 s inside the driver's wall clock)
        import gc
        hens = hcache = None
        gc.collect()
        e2e_drv = e2e_driver_run(wl)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = host_threads()
        n_sample = args.cpu_sample or (100_000 if wl == "cfg1" else 20_000 * threads)
        rate, wall, n_sample = cpu_sample_rate(wl, mets, make_ctl(wl, "exact"), n_sample, 2,
                                               threads, target_s=15.0)
        cpu = {"value": rate, "unit": "particle-steps/s", "cores": threads, "kind": "port",
               "sample": f"oracle/ numpy port, {n_sample} particles x 2 timed steps on the "
                         f"same {wl} met grid ({wall:.1f} s)"}

    # launches of our kernels in the headline timed region: one fused step
    # per step; per sort: CUB's histogram, scan and three onesweep passes (5),
    # plus the key and compression kernels (2) unless the step before wrote
    # the keys (lt_sort_info), plus — unless every cold row is in particle
    # order and the next step applies the permutation — row gathers (8 hot
    # rows, plus the q rows when meteo/decay keep them in slot order, 4 per
    # launch) + ids 1; per streamed snapshot: one packing kernel, and the
    # spread table of the new met1 when the chain has meso
    q_hot = any(m in cfg["chain"] for m in ("meteo", "decay"))
    deferred = not q_hot and "isosurf" not in cfg["chain"]
    per_sort = 5 + (0 if deferred else 2 + (-(-ctl.nq // 4) if q_hot else 0) + 1)
    launches = args.steps + sorts_timed * per_sort + 2 * (sorts_timed - fused_timed) + \
        rots * (2 if "meso" in cfg["chain"] else 1)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64 state / f32 interpolation" if args.precision == "fast" else "f64",
            "data": "synthetic",
            "config": {"workload": wl, "description": cfg["desc"], "particles": n_tot,
                       "particles_per_gpu": work.size, "met_nodes": nodes,
                       "modules": list(cfg["chain"]),
                       "met_store": f"{args.met_store} node-pair records", "state": "fp64 SoA",
                       "precision": args.precision,
                       "rng": f"{args.rng} (reference splitmix64 words), in-kernel"
                              if args.rng != "philox" else
                              "philox4x32-10 keyed by (seed, step, 32-bit particle id), "
                              "in-kernel (the north star's counter-based generator)",
                       "sort_every": sort_every, "sorts_timed": sorts_timed,
                       "sorts_with_step_keys": fused_timed, "met_rotations_timed": rots,
                       "per_snapshot_precompute": "node-pair record packing and the per-cell "
                                                  "mesoscale spread table (2.1 ms at 0.25 deg), "
                                                  "once per met snapshot: inside the timed region "
                                                  "only when snapshots rotate in it "
                                                  "(met_rotations_timed)",
                       "parallelism": f"particles sharded x{ws} ({args.scaling} scaling), met "
                                      "replicated (NCCL broadcast), no data-path collective",
                       "l2": "inputs larger than L2 (state %.1f GB/GPU, met %.1f GB)" % (
                           work.size * 120 / 1e9, 2 * nodes * 16 / 1e9)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "step_kernel", "kernel_ms": kern_avg,
                         "algorithmic_bytes_per_particle_step": b,
                         "algorithmic_bytes_source": "SURVEY.md 8(d): b_state (fp64 "
                         "lon/lat/p/time + fp32 uvwp column) + b_met = 32*nodes*(1-exp(-8N/"
                         "nodes))/N",
                         "moved_bytes_per_particle_step": MOVED_STATE_BYTES[cfg["chain"]] +
                         b - STATE_BYTES[cfg["chain"]],
                         "issue": issue,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks
                         else "fallback"},
            "alt_precision": other, "alt_rng": alt_rng, "alt_reference_faithful": alt_ref,
            "alt_multistep": multi,
            "cpu_baseline": cpu, "e2e": e2e, "e2e_driver": e2e_drv, "clocks": clocks,
            "gpu_launches": launches,
        }), flush=True)
    if e2e_drv is None:
        eng.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
