"""The drop-in module API: `lagtrans.physics` signatures on B200 kernels.

Every `module_*` here has the reference signature
(/root/reference/pkg/src/lagtrans/physics.py:69-301) and the same in-place,
range-restricted semantics.  Two call paths:

* host objects (numpy ensembles, as the reference's own tests use): the
  work-range slice is copied to the default GPU context, the module runs as
  one launch of the fused step kernel with a single module bit, and the
  changed fields are copied back;
* device-resident images (`device_runtime.DeviceEnsemble`, what
  `device_runtime.DevicePool.region_create` builds): the kernel runs in
  place in HBM and nothing crosses PCIe.

There is no CPU fallback: without the CUDA library these functions raise.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _capi as capi
from .context import DeviceContext

RE = 6_371_000.0
G0 = 9.80665
R_AIR = 287.058
ETA_AIR = 1.8205e-5
KAPPA = 0.2857
DEG_PER_M = 180.0 / (np.pi * RE)

_local = threading.local()
_contexts: dict[int, DeviceContext] = {}
_lock = threading.Lock()


def default_context(device: int | None = None) -> DeviceContext:
    """The per-device scratch context used by host-array calls."""
    dev = getattr(_local, "device", 0) if device is None else device
    with _lock:
        ctx = _contexts.get(dev)
        if ctx is None or ctx.closed:
            ctx = DeviceContext(dev)
            _contexts[dev] = ctx
        return ctx


def set_device(device: int) -> None:
    """Select the GPU used by host-array calls from this thread."""
    _local.device = device


def _is_device(ens) -> bool:
    return getattr(ens, "is_device_resident", False)


# fields each module reads / writes beyond (time, lon, lat, p)
_NEEDS = {
    capi.MOD_TIMESTEPS: ((), ("dt",)),
    capi.MOD_ADVECTION: (("dt",), ("time", "lon", "lat", "p")),
    capi.MOD_TURB: (("dt", "turb"), ("lon", "lat", "p")),
    capi.MOD_MESO: (("dt", "meso", "uvwp"), ("lon", "lat", "p", "uvwp")),
    capi.MOD_CONVECTION: (("dt", "conv"), ("p",)),
    capi.MOD_SEDI: (("dt",), ("p",)),
    capi.MOD_DECAY: (("dt", "qdecay"), ("qdecay",)),
    capi.MOD_ISOSURF: (("iso",), ("p",)),
    capi.MOD_ISOSURF_INIT: ((), ("iso",)),
    capi.MOD_POSITION: ((), ("lon", "lat", "p")),
    capi.MOD_METEO: ((), ("q5",)),
}
_STATE = {"time": capi.F_TIME, "lon": capi.F_LON, "lat": capi.F_LAT, "p": capi.F_P}


def _run_host(module, ctl, ens, met0, met1, dt, rnd, cache, clim, work):
    """Copy the work slice in, launch one module, copy the results out."""
    n = work.size
    if n == 0:
        return
    s = work.slice
    reads, writes = _NEEDS[module]
    ctx = default_context()
    nq = ens.q.shape[0] if ens.q.ndim == 2 else 5
    ctx.ensure_capacity(n, nq=max(nq, 5), with_batch=bool(set(reads) & {"turb", "meso", "conv"}))
    for name, fid in _STATE.items():
        ctx.h2d(fid, 0, 0, getattr(ens, name)[s])
    flags = 0
    if "dt" in reads:
        ctx.h2d(capi.F_DT, 0, 0, dt[s])
        flags |= capi.RUN_DT_ARRAY
    if module == capi.MOD_TIMESTEPS:
        flags |= capi.RUN_WRITE_DT
    if "turb" in reads:
        ctx.h2d(capi.F_RND_TURB, 0, 0, rnd.diff_turb[3 * work.start:3 * work.end])
    if "meso" in reads:
        ctx.h2d(capi.F_RND_MESO, 0, 0, rnd.diff_meso[3 * work.start:3 * work.end])
    if "conv" in reads:
        ctx.h2d(capi.F_RND_CONV, 0, 0, rnd.convection[s])
    if "uvwp" in reads:
        for c in range(3):
            ctx.h2d(capi.F_UVWP, c, 0, cache.uvwp[c, s])
    if "iso" in reads:
        ctx.h2d(capi.F_ISO_VAR, 0, 0, cache.iso_var[s])
    slot = int(getattr(ctl, "decay_slot", -1))
    if "qdecay" in reads and 0 <= slot < nq:
        ctx.h2d(capi.F_Q, slot, 0, ens.q[slot, s])
    if module & (capi.MOD_ADVECTION | capi.MOD_TURB | capi.MOD_MESO | capi.MOD_SEDI |
                 capi.MOD_ISOSURF | capi.MOD_ISOSURF_INIT | capi.MOD_METEO):
        ctx.bind_pair(met0, met1)
    if module & capi.MOD_METEO:
        ctx.load_clim(clim)
    if module & capi.MOD_ISOSURF:
        ctx.iso_counter(reset=True)
    ctx.run(ctl, module, 0, n, flags=flags)
    for name in writes:
        if name in _STATE:
            getattr(ens, name)[s] = ctx.d2h(_STATE[name], 0, 0, n)
        elif name == "dt":
            dt[s] = ctx.d2h(capi.F_DT, 0, 0, n)
        elif name == "uvwp":
            for c in range(3):
                cache.uvwp[c, s] = ctx.d2h(capi.F_UVWP, c, 0, n)
        elif name == "iso":
            cache.iso_var[s] = ctx.d2h(capi.F_ISO_VAR, 0, 0, n)
        elif name == "q5":
            for k in range(5):
                ens.q[k, s] = ctx.d2h(capi.F_Q, k, 0, n)
        elif name == "qdecay" and 0 <= slot < nq:
            ens.q[slot, s] = ctx.d2h(capi.F_Q, slot, 0, n)
    if module & capi.MOD_ISOSURF and ctl.isosurf_mode == "theta":
        cache.iso_nonconverged += ctx.iso_counter(reset=True)


def _run(module, ctl, ens, met0=None, met1=None, dt=None, rnd=None, cache=None, clim=None,
         work=None):
    if _is_device(ens):
        ens.image.run_module(module, ctl, work, met0=met0, met1=met1, clim=clim, cache=cache)
    else:
        _run_host(module, ctl, ens, met0, met1, dt, rnd, cache, clim, work)


# ------------------------------------------------------------------ module API

def interpolate_met(met0, met1, t, lon, lat, p, fields=("u", "v", "w", "T")):
    """physics.py:69-79 on the GPU: trilinear in space per snapshot, linear
    in time; returns a tuple of arrays in `fields` order."""
    ctx = default_context()
    ctx.bind_pair(met0, met1)
    lon = np.atleast_1d(np.asarray(lon, dtype=np.float64))
    out = ctx.interpolate(t, lon, lat, p)
    idx = {"u": 0, "v": 1, "w": 2, "T": 3}
    return tuple(out[idx[f]] for f in fields)


def module_timesteps(ctl, ens, t_next, work, dt) -> None:
    """physics.py:82-88 (t_next unused, as in the reference)."""
    _run(capi.MOD_TIMESTEPS, ctl, ens, dt=dt, work=work)


def module_advection(ctl, ens, met0, met1, dt, work) -> None:
    """physics.py:91-116, explicit midpoint."""
    _run(capi.MOD_ADVECTION, ctl, ens, met0, met1, dt=dt, work=work)


def module_diffusion_turb(ctl, ens, met0, met1, dt, rnd, work) -> None:
    """physics.py:119-147."""
    _run(capi.MOD_TURB, ctl, ens, met0, met1, dt=dt, rnd=rnd, work=work)


def module_diffusion_meso(ctl, ens, met0, met1, dt, rnd, cache, work) -> None:
    """physics.py:150-188."""
    _run(capi.MOD_MESO, ctl, ens, met0, met1, dt=dt, rnd=rnd, cache=cache, work=work)


def module_convection(ctl, ens, dt, rnd, work) -> None:
    """physics.py:191-203."""
    _run(capi.MOD_CONVECTION, ctl, ens, dt=dt, rnd=rnd, work=work)


def module_sedi(ctl, ens, met0, met1, dt, work) -> None:
    """physics.py:206-222."""
    _run(capi.MOD_SEDI, ctl, ens, met0, met1, dt=dt, work=work)


def module_decay(ctl, ens, dt, work) -> None:
    """New module (no reference counterpart): q[decay_slot] *= exp(-dt/decay_tau)
    for particles with dt > 0; a no-op when decay_tau <= 0."""
    _run(capi.MOD_DECAY, ctl, ens, dt=dt, work=work)


def module_isosurf_init(ctl, ens, met0, met1, cache, work) -> None:
    """physics.py:225-235."""
    if ctl.isosurf_mode == "off":
        return
    _run(capi.MOD_ISOSURF_INIT, ctl, ens, met0, met1, cache=cache, work=work)


def module_isosurf(ctl, ens, met0, met1, cache, work) -> None:
    """physics.py:238-264."""
    if ctl.isosurf_mode == "off":
        return
    _run(capi.MOD_ISOSURF, ctl, ens, met0, met1, cache=cache, work=work)


def module_position(ctl, ens, work) -> None:
    """physics.py:267-287."""
    _run(capi.MOD_POSITION, ctl, ens, work=work)


def module_meteo(ctl, ens, met0, met1, clim, work) -> None:
    """physics.py:290-301."""
    _run(capi.MOD_METEO, ctl, ens, met0, met1, clim=clim, work=work)
