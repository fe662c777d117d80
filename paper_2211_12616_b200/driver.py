"""The time loop around the hot path on device-resident GPU images —
`lagtrans.driver_cli.run_simulation`'s step loop (driver_cli.py:84-209)
without its file I/O and CLI (out of scope: SURVEY.md §2.1).

Two stepping modes over a `device_runtime.DevicePool`:

* ``fused=False`` — the reference's per-device closure verbatim
  (driver_cli.py:151-183): module_timesteps, generate_random_nums and the
  eight physics modules called through the drop-in module API on each
  device's HBM image, one kernel launch per module.  Each module is timed
  with CUDA events into the caller's timer sink under the reference names,
  groups and scopes (the c10 contract, test_acceptance.py:284-305).
* ``fused=True`` (production) — one launch of the fused step kernel per
  device per step with in-kernel draws (identical numbers in counter mode),
  an optional periodic box sort, and met snapshots prefetched into the
  third met slot on each device's copy stream while steps run.

Met snapshots come from memory (a list of `MeteoField`, already closed with
`met_periodic`), replacing the text reader `ingest.read_met`; rotation
follows driver_cli.py:139-149.  Output cadence (driver_cli.py:188-195)
copies every device's owned range back into the host ensemble and calls
`on_output(ctl, ens, cache, t)`.
"""

from __future__ import annotations

import math
import time

import numpy as np

from . import _capi as capi
from . import engine as eng
from . import physics
from .device_runtime import REGION_FIELDS, DevicePool, DeviceTaskError, ModelImage
from .model_state import cache_allocate, validate_control
from .partition import partition_all
from .rng import batch_allocate, generate_random_nums, module_rng_init

_OUT_EPS = 1e-9  # driver_cli.py:35
PIPELINE = ("module_advection", "module_diffusion_turb", "module_diffusion_meso",
            "module_convection", "module_sedi", "module_isosurf", "module_position",
            "module_meteo")  # driver_cli.py:31-33


def device_scope(d: int) -> str:
    return f"device{d}"


class _NullTimers:
    def record(self, name, group, scope, elapsed_ns):
        pass


def n_steps_for(ctl) -> int:
    """driver_cli.py:131-132."""
    return max(0, math.ceil((ctl.t_stop - ctl.t_start) / ctl.dt_model - _OUT_EPS))


def bracketing(mets, t_start):
    """driver_cli.py:67-81 over in-memory snapshots: (met0, met1, rest)."""
    if not mets:
        raise ValueError("no met snapshots")
    met0 = mets[0]
    rest = list(mets[1:])
    met1 = rest.pop(0) if rest else met0
    while met1.t_met < t_start and rest:
        met0, met1 = met1, rest.pop(0)
    if met0.t_met > t_start:
        raise ValueError(f"first met snapshot ({met0.t_met} s) is after t_start ({t_start} s)")
    return met0, met1, rest


DEFAULT_SORT_EVERY = 15   # measured optimum at cfg3


def run_simulation(ctl, ens, mets, num_devices: int = 1, *, fused: bool = True,
                   modules: int | None = None, sort_every: int | None = None, clim=None,
                   timers=None, on_output=None, parallel: bool = True,
                   device_map=None, module_timers: bool = False, cache=None):
    """Advance `ens` (host ParticleEnsemble, updated in place at every
    output time) from ctl.t_start to ctl.t_stop.  Returns (status, cache):
    status 0 on success, 1 when a device task failed (driver_cli.py:196-199).

    module_timers (fused mode): every step is one instrumented fused launch
    that charges SM cycles to the module that spends them, and the launch's
    CUDA-event time is split by those shares into the reference's PHYSICS
    rows (module_timesteps, generate_random_nums, module_advection, ...;
    driver_cli.py:151-183, test_acceptance.py:284-305).  Off by default:
    the production steps run the specialised, uninstrumented kernels.
    """
    if sort_every is None:      # box-sort the fused path by default (results never change)
        sort_every = DEFAULT_SORT_EVERY if fused else 0
    violations = validate_control(ctl)
    if violations:
        raise ValueError("invalid control: " + "; ".join(violations))
    timers = timers or _NullTimers()
    if clim is None:
        from .model_state import read_clim
        clim = read_clim(ctl)
    if modules is None:
        modules = eng.FULL
    met0, met1, rest = bracketing(list(mets), ctl.t_start)
    if cache is None:   # (a caller may pass its own, e.g. in pinned host memory)
        cache = cache_allocate(ens.np)
    host = ModelImage(ctl=ctl, ens=ens, cache=cache, clim=clim, met0=met0, met1=met1,
                      dt=np.zeros(ens.np), batch=batch_allocate(ens.np) if not fused else None)
    rng = module_rng_init(ctl, num_devices)
    ranges = partition_all(ens.np, num_devices)
    pool = DevicePool(num_devices, debug=True, device_map=device_map)
    regions = []
    status = 0

    def timed(name, group, scope, fn):
        t0 = time.perf_counter_ns()
        fn()
        timers.record(name, group, scope, time.perf_counter_ns() - t0)

    try:
        for d in range(num_devices):
            timed("ACC_INIT", "INIT", device_scope(d),
                  lambda d=d: pool.dispatch(d, lambda: None).result())
        fields = tuple(f for f in REGION_FIELDS if not (fused and f == "batch"))
        for d in range(num_devices):
            timed("CREATE_DATA_REGION", "MEMORY", device_scope(d),
                  lambda d=d: regions.append(pool.region_create(d, host, ranges[d],
                                                                with_batch=not fused)))
            timed("UPDATE_DEVICE", "MEMORY", device_scope(d),
                  lambda d=d: pool.region_update_device(regions[d], host, fields))

        def init(d):
            img = regions[d].image
            physics.module_isosurf_init(img.ctl, img.ens, met0, met1, img.cache, ranges[d])
        pool.for_each_device_parallel(init, parallel=parallel)

        # fused mode: device 0 stages the next snapshot from the host into its
        # free slot (copy stream); ONE met broadcast (NCCL over NVLink, every
        # device's copy stream) replicates it into the other devices' free
        # slots while they keep stepping — the paper's met replication
        def prefetch_all():
            if not rest:
                return
            eng0 = regions[0].image.engine
            pool.dispatch(0, lambda: eng0.prefetch(met=rest[0])).result()
            if num_devices > 1:
                timed("MET_BROADCAST", "MEMORY", device_scope(0),
                      lambda: eng.Engine.broadcast_staged(
                          eng0, [regions[d].image.engine for d in range(1, num_devices)]))
        if fused:
            prefetch_all()

        t = ctl.t_start
        next_out = ctl.t_start + ctl.output_dt
        n_steps = n_steps_for(ctl)
        step = 0
        while step < n_steps:
            t_next = min(t + ctl.dt_model, ctl.t_stop)
            while met1.t_met < t_next:      # driver_cli.py:139-149
                if not rest:
                    raise ValueError(f"t_stop {ctl.t_stop} s exceeds the last met snapshot "
                                     f"time {met1.t_met} s")
                met0, met1 = met1, rest.pop(0)
                host.met0, host.met1 = met0, met1
                for d in range(num_devices):
                    img = regions[d].image
                    if fused:
                        def rot(img=img):
                            img.engine.rotate()
                            img.met0, img.met1 = met0, met1
                        timed("UPDATE_DEVICE", "MEMORY", device_scope(d),
                              lambda d=d, rot=rot: pool.dispatch(d, rot).result())
                    else:
                        timed("UPDATE_DEVICE", "MEMORY", device_scope(d),
                              lambda d=d: pool.region_update_device(regions[d], host,
                                                                    ("met0", "met1")))
                if fused:
                    prefetch_all()

            # fused mode runs the steps up to the next event (met rotation,
            # box sort, output) as one multi-step launch (Engine.step_many:
            # identical results, each particle advanced in registers)
            run, t_end = 1, t_next
            if fused and not module_timers:
                while step + run < n_steps:
                    t_more = min(t_end + ctl.dt_model, ctl.t_stop)
                    if (met1.t_met < t_more or (sort_every and (step + run) % sort_every == 0)
                            or t_end >= next_out - _OUT_EPS or t_end >= ctl.t_stop):
                        break
                    run, t_end = run + 1, t_more
            if fused:
                def device_step(d, step=step, run=run):
                    img = regions[d].image
                    if sort_every and step % sort_every == 0:
                        img.engine.sort(modules)
                    ctx = img.engine.ctx
                    ctx.timing(True)
                    # a sort opens the next launch: this one writes its keys
                    sort_next = bool(sort_every) and (step + run) % sort_every == 0 and \
                        step + run < n_steps
                    if run > 1:
                        img.engine.step_many(img.ctl, step, run, modules, device_id=d,
                                             sort_next=sort_next)
                    else:
                        img.engine.step(img.ctl, step, modules, device_id=d,
                                        num_devices=num_devices, module_clocks=module_timers,
                                        sort_next=sort_next)
                    ms = ctx.last_elapsed_ms()
                    ctx.timing(False)
                    timers.record("module_fused_step", "PHYSICS", device_scope(d),
                                  int(ms * 1e6))
                    if module_timers:
                        _record_module_split(ctx, modules, ms, timers, device_scope(d))
            else:
                def device_step(d, step=step, t_next=t_next):
                    _module_step(regions[d].image, ranges[d], d, step, t_next, rng,
                                 met0, met1, timers)
            pool.for_each_device_parallel(device_step, parallel=parallel)
            t = t_end
            step += run

            if t >= next_out - _OUT_EPS or t >= ctl.t_stop:   # driver_cli.py:188-195
                for d in range(num_devices):
                    timed("UPDATE_HOST", "MEMORY", device_scope(d),
                          lambda d=d: pool.region_update_host(regions[d], host, ranges[d]))
                if on_output is not None:
                    on_output(ctl, ens, cache, t)
                while next_out <= t + _OUT_EPS:
                    next_out += ctl.output_dt
    except DeviceTaskError as exc:
        import sys
        for d, err in sorted(exc.failures.items()):
            print(f"device {d} failed: {err!r}", file=sys.stderr)
        status = 1
    finally:
        for region in regions:
            pool.device_wait(region.device_id)
            if region.state != "deleted":
                timed("DELETE_DATA_REGION", "MEMORY", device_scope(region.device_id),
                      lambda r=region: pool.region_delete(r))
        pool.shutdown()
    return status, cache


_SPLIT_BITS = {"module_timesteps": capi.MOD_TIMESTEPS, "module_advection": capi.MOD_ADVECTION,
               "module_diffusion_turb": capi.MOD_TURB, "module_diffusion_meso": capi.MOD_MESO,
               "module_convection": capi.MOD_CONVECTION, "module_sedi": capi.MOD_SEDI,
               "module_decay": capi.MOD_DECAY, "module_isosurf": capi.MOD_ISOSURF,
               "module_position": capi.MOD_POSITION, "module_meteo": capi.MOD_METEO}


def _record_module_split(ctx, modules, ms, timers, scope):
    """One instrumented fused launch of `ms` milliseconds: each enabled
    module's row gets its share of the launch's SM cycles (random draws as
    generate_random_nums, as the reference times them); modules that are
    enabled but did no work (e.g. isosurf off in the control) get 0 ns."""
    cyc = ctx.module_cycles(reset=True).astype(np.float64)
    total = cyc.sum()
    for name, c in zip(capi.MODULE_CLOCK_NAMES, cyc):
        bit = _SPLIT_BITS.get(name)
        if name == "generate_random_nums":
            on = bool(modules & (capi.MOD_TURB | capi.MOD_MESO | capi.MOD_CONVECTION))
        elif name == "module_isosurf_init":
            on = False
        else:
            on = bool(modules & bit)
        if on:
            timers.record(name, "PHYSICS", scope, int(ms * 1e6 * (c / total if total else 0.0)))


def _module_step(img, work, d, step, t_next, rng, met0, met1, timers):
    """driver_cli.py:151-183 on one device image, each module CUDA-event timed."""
    ctx = img.engine.ctx
    scope = device_scope(d)

    def timed(name, fn):
        ctx.timing(True)
        fn()
        ms = ctx.last_elapsed_ms()
        ctx.timing(False)
        timers.record(name, "PHYSICS", scope, int(ms * 1e6))

    c, e = img.ctl, img.ens
    timed("module_timesteps", lambda: physics.module_timesteps(c, e, t_next, work, img.dt))
    timed("generate_random_nums", lambda: generate_random_nums(rng, step, work, d, img.batch))
    timed("module_advection", lambda: physics.module_advection(c, e, met0, met1, img.dt, work))
    timed("module_diffusion_turb",
          lambda: physics.module_diffusion_turb(c, e, met0, met1, img.dt, img.batch, work))
    timed("module_diffusion_meso",
          lambda: physics.module_diffusion_meso(c, e, met0, met1, img.dt, img.batch, img.cache,
                                                work))
    timed("module_convection", lambda: physics.module_convection(c, e, img.dt, img.batch, work))
    timed("module_sedi", lambda: physics.module_sedi(c, e, met0, met1, img.dt, work))
    if getattr(c, "decay_tau", 0.0) > 0:
        timed("module_decay", lambda: physics.module_decay(c, e, img.dt, work))
    timed("module_isosurf", lambda: physics.module_isosurf(c, e, met0, met1, img.cache, work))
    timed("module_position", lambda: physics.module_position(c, e, work))
    timed("module_meteo", lambda: physics.module_meteo(c, e, met0, met1, img.clim, work))
