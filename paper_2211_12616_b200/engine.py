"""Engine: device-resident fused time stepping for one GPU's particle shard.

The production path behind the drop-in.  Where the reference driver calls
eight module functions per device per step on a deep-copied image
(driver_cli.py:151-183), the engine keeps the shard's SoA state in HBM and
runs the whole chain as ONE kernel launch per step with the random draws
generated in-kernel (same numbers as `generate_random_nums`, no batch in
memory).  It also owns the two extensions the north star asks for:

* met streaming: the next snapshot is staged from (pinned) host memory on a
  side stream into the free met slot while steps run, then the slots rotate
  (replaces driver_cli.py:139-149 + device_runtime.py:178-186 deep copies);
* box sort: particles are periodically stably sorted by met0 cell so the
  gathers of neighbouring threads hit the same L1/L2 lines; ids travel with
  the particles, the RNG is keyed by id, and downloads undo the permutation,
  so sorting never changes a result.
"""

from __future__ import annotations

import numpy as np

from . import _capi as capi
from .context import DeviceContext, met_fingerprint
from .model_state import ParticleEnsemble
from .rng import advance_faithful, rng_seed_for

ADV = capi.MOD_TIMESTEPS | capi.MOD_ADVECTION | capi.MOD_POSITION
ADV_DIFF = capi.MOD_TIMESTEPS | capi.MOD_ADVECTION | capi.MOD_TURB | capi.MOD_MESO | \
    capi.MOD_POSITION
FULL = (capi.MOD_TIMESTEPS | capi.MOD_ADVECTION | capi.MOD_TURB | capi.MOD_MESO |
        capi.MOD_CONVECTION | capi.MOD_SEDI | capi.MOD_DECAY | capi.MOD_ISOSURF |
        capi.MOD_POSITION | capi.MOD_METEO)
MODULE_BITS = {
    "advection": capi.MOD_ADVECTION, "turb": capi.MOD_TURB, "meso": capi.MOD_MESO,
    "convection": capi.MOD_CONVECTION, "sedi": capi.MOD_SEDI, "decay": capi.MOD_DECAY,
    "isosurf": capi.MOD_ISOSURF, "position": capi.MOD_POSITION, "meteo": capi.MOD_METEO,
}


def modules_mask(names) -> int:
    m = capi.MOD_TIMESTEPS
    for n in names:
        m |= MODULE_BITS[n]
    return m


class Engine:
    """One shard of the particle set on one GPU: local slot t holds global
    particle first_id + t (until a sort permutes slots; ids travel along)."""

    def __init__(self, device: int = 0, capacity: int = 0, nq: int = 5,
                 met_precision: str = "f32", first_id: int = 0):
        self.ctx = DeviceContext(device, met_precision=met_precision)
        self.device = device
        self.n = 0
        self.nq = nq
        self.first_id = int(first_id)
        self.faithful_state = None
        self.sorted = False
        self._met_slots = (0, 1)   # (met0 slot, met1 slot)
        self._staged = None         # slot holding the prefetched next snapshot
        if capacity:
            self.ctx.alloc(capacity, nq)

    # -- particles ---------------------------------------------------------
    def upload(self, ens, cache=None, start: int = 0, end: int | None = None) -> None:
        """Copy ensemble slice [start, end) into the device shard."""
        end = ens.np if end is None else end
        n = end - start
        nq = ens.q.shape[0]
        if n > self.ctx.capacity or nq > self.ctx.nq:
            self.ctx.alloc(n, max(nq, self.nq))
        self.n, self.nq = n, max(nq, self.nq)
        s = slice(start, end)
        for fid, arr in ((capi.F_TIME, ens.time), (capi.F_P, ens.p), (capi.F_ZETA, ens.zeta),
                         (capi.F_LON, ens.lon), (capi.F_LAT, ens.lat)):
            self.ctx.h2d(fid, 0, 0, arr[s])
        for k in range(nq):
            self.ctx.h2d(capi.F_Q, k, 0, ens.q[k, s])
        if cache is not None:
            for c in range(3):
                self.ctx.h2d(capi.F_UVWP, c, 0, cache.uvwp[c, s])
            self.ctx.h2d(capi.F_ISO_VAR, 0, 0, cache.iso_var[s])
        else:
            for c in range(3):
                self.ctx.fill(capi.F_UVWP, c, 0, n, 0.0)
            self.ctx.fill(capi.F_ISO_VAR, 0, 0, n, 0.0)
        self.ctx.ids_reset(0, n, self.first_id)   # global id of local slot t
        self.sorted = False

    def download(self, ens=None, cache=None, start: int = 0) -> ParticleEnsemble:
        """Copy the shard back in original particle order (undoing sorts),
        into ens[start:start+n] (range-restricted copy-back,
        device_runtime.py:188-219)."""
        n = self.n
        if ens is None:
            ens = ParticleEnsemble(n, np.empty(n), np.empty(n), np.empty(n), np.empty(n),
                                   np.empty(n), np.empty((self.nq, n)))
            start = 0
        s = slice(start, start + n)
        get = lambda fid, row=0: self.ctx.d2h_ordered(fid, row, 0, n, self.first_id)
        ens.time[s], ens.p[s], ens.zeta[s] = get(capi.F_TIME), get(capi.F_P), get(capi.F_ZETA)
        ens.lon[s], ens.lat[s] = get(capi.F_LON), get(capi.F_LAT)
        for k in range(min(self.nq, ens.q.shape[0])):
            ens.q[k, s] = get(capi.F_Q, k)
        if cache is not None:
            for c in range(3):
                cache.uvwp[c, s] = get(capi.F_UVWP, c)
            cache.iso_var[s] = get(capi.F_ISO_VAR)
        return ens

    # -- met ---------------------------------------------------------------
    def bind_met(self, met0, met1) -> None:
        """Load the first snapshot pair into slots 0 and 1."""
        self.ctx.set_grid(met0.lons, met0.lats, met0.levs)
        self.ctx.load_met(0, met0, key=met_fingerprint(met0))
        self.ctx.load_met(1, met1, key=met_fingerprint(met1))
        self._met_slots = (0, 1)
        self._staged = None
        self.ctx.use_met(0, 1)

    def bind_pair(self, met0, met1, donor=None) -> None:
        """Select (met0, met1), uploading only snapshots the slots lack
        (or replicating them from a donor context, see DeviceContext)."""
        self._met_slots = self.ctx.bind_pair(met0, met1, donor)
        self._staged = None

    def set_grid(self, lons, lats, levs) -> None:
        self.ctx.set_grid(lons, lats, levs)

    def load_slot(self, slot, met=None, nodes=None, t_met=None, close_lon=False) -> None:
        if met is not None:
            self.ctx.load_met(slot, met, key=met_fingerprint(met), close_lon=close_lon)
        else:
            self.ctx.load_met_nodes(slot, t_met, nodes, close_lon=close_lon)

    def prefetch(self, met=None, nodes=None, t_met=None, close_lon=False) -> None:
        """Stage the next snapshot into the free slot on the copy stream; the
        compute stream keeps stepping on the current pair meanwhile."""
        free = min({0, 1, 2} - set(self._met_slots))
        self.load_slot(free, met=met, nodes=nodes, t_met=t_met, close_lon=close_lon)
        self._staged = free

    def prefetch_from(self, other: "Engine") -> None:
        """Stage the snapshot `other` has staged by a GPU-to-GPU copy
        (NVLink peer copy) instead of another host upload."""
        if other._staged is None:
            raise RuntimeError("prefetch_from() an engine without a staged snapshot")
        free = min({0, 1, 2} - set(self._met_slots))
        self.ctx.copy_slot_from(other.ctx, other._staged, free)
        self._staged = free

    @staticmethod
    def broadcast_staged(root: "Engine", others) -> None:
        """Stage `root`'s prefetched snapshot on every engine in `others` by
        ONE met broadcast (lt_met_broadcast: an NCCL broadcast group over
        NVLink/NVSwitch, each GPU's copy stream; the paper's met replication)
        instead of one host upload per GPU."""
        if root._staged is None:
            raise RuntimeError("broadcast_staged() from an engine without a staged snapshot")
        others = [e for e in others if e is not root]
        if not others:
            return
        frees = [min({0, 1, 2} - set(e._met_slots)) for e in others]
        from .context import met_broadcast
        met_broadcast([root.ctx] + [e.ctx for e in others], 0, [root._staged] + frees)
        for e, f in zip(others, frees):
            e._staged = f

    def rotate(self) -> None:
        """met0 <- met1, met1 <- staged (driver_cli.py:139-145)."""
        if self._staged is None:
            raise RuntimeError("rotate() without a prefetched snapshot")
        self._met_slots = (self._met_slots[1], self._staged)
        self._staged = None
        self.ctx.use_met(*self._met_slots)

    def load_clim(self, clim) -> None:
        self.ctx.load_clim(clim)

    # -- stepping ----------------------------------------------------------
    def init_isosurf(self, ctl) -> None:
        if ctl.isosurf_mode != "off":
            self.ctx.run(ctl, capi.MOD_ISOSURF_INIT, 0, self.n)

    def step(self, ctl, step: int, modules: int = ADV_DIFF, device_id: int = 0,
             num_devices: int = 1, module_clocks: bool = False, sort_next: bool = False) -> None:
        """One fused time step of every particle in the shard.  With
        module_clocks the launch also charges its SM cycles per module
        (ctx.module_cycles; the generic, instrumented kernel runs).  With
        sort_next (a box sort follows) the launch also writes the particles'
        sort keys, which the sort then uses instead of computing its own."""
        fstate = 0
        if ctl.rng_mode == "faithful":   # the reference fills a batch every step
            if self.faithful_state is None:
                self.faithful_state = rng_seed_for(ctl.mpi_rank, device_id)
            fstate = self.faithful_state
            self.faithful_state = advance_faithful(fstate, self.n)
        flags = capi.RUN_RNG_INKERNEL | (capi.RUN_MODULE_CLOCKS if module_clocks else 0) | \
            (capi.RUN_SORT_KEYS if sort_next else 0)
        self.ctx.run(ctl, modules, 0, self.n, step=step, faithful_state=fstate,
                     faithful_base=self.first_id, flags=flags)
        self._last_modules = modules

    def step_many(self, ctl, step: int, nsteps: int, modules: int = ADV_DIFF,
                  device_id: int = 0, sort_next: bool = False) -> None:
        """`nsteps` fused steps of every particle (lt_run_steps: the
        production chain in one launch, state in registers across the steps;
        identical results).  The bound met pair must cover all of them — call
        between rotations.  Faithful draws step one launch at a time here
        (their per-step stream state lives on the host)."""
        if nsteps <= 1 or ctl.rng_mode == "faithful":
            for k in range(nsteps):
                self.step(ctl, step + k, modules, device_id=device_id,
                          sort_next=sort_next and k == nsteps - 1)
            return
        self.ctx.run_steps(ctl, modules, 0, self.n, step, nsteps,
                           flags=capi.RUN_RNG_INKERNEL | (capi.RUN_SORT_KEYS if sort_next else 0))
        self._last_modules = modules

    def step_host(self, ctl, ens, cache, step: int, modules: int = ADV_DIFF,
                  device_id: int = 0, chunk: int = 0, steps: int = 1) -> None:
        """`steps` fused steps (step, step+1, ...) of a HOST ensemble (numpy
        SoA, ideally in pinned memory — see context.pinned_empty), updated
        in place: every step streams every particle through this GPU's store
        in chunks with H2D, kernel and D2H overlapped, and across steps
        (lt_run_host_steps).  Particle i has global id first_id + i."""
        n = int(ens.np)
        if self.ctx.capacity == 0:
            self.ctx.alloc(min(max(n, 1), 1 << 24), max(self.nq, ens.q.shape[0]))
        fstate = 0
        if ctl.rng_mode == "faithful":
            if self.faithful_state is None:
                self.faithful_state = rng_seed_for(ctl.mpi_rank, device_id)
            fstate = self.faithful_state
            for _ in range(steps):
                self.faithful_state = advance_faithful(self.faithful_state, n)
        want = lambda bits: bool(modules & bits)
        self.ctx.run_host(ctl, modules, n, step, self.first_id, ens.time, ens.p, ens.lon, ens.lat,
                          uvwp=cache.uvwp if want(capi.MOD_MESO) else None,
                          iso_var=cache.iso_var if want(capi.MOD_ISOSURF |
                                                        capi.MOD_ISOSURF_INIT) else None,
                          q=ens.q if want(capi.MOD_METEO | capi.MOD_DECAY) else None,
                          faithful_state=fstate, chunk=chunk, steps=steps)
        self.sorted = False

    def sort(self, modules: int | None = None) -> None:
        """Stable box sort of the shard.  Rows the stepping modules do not
        touch (zeta, dt; q unless meteo/decay run; iso_var unless isosurf
        runs) stay in particle order, so the sort moves only the rows the step
        kernel streams — and with all of those cold, the next production-chain
        step applies the permutation itself while it streams them
        (lt_sort_by_box defers it, lt_run fuses it).  `modules` is the chain
        the next steps run (default: the last step's); a row those modules
        touch kept in particle order would be read and written scattered."""
        last = modules if modules is not None else getattr(self, "_last_modules", 0)
        home = capi.HOME_ZETA | capi.HOME_DT
        if not (last & (capi.MOD_METEO | capi.MOD_DECAY)):
            home |= capi.HOME_Q      # (a later meteo/decay step still works, via the ids)
        if not (last & (capi.MOD_ISOSURF | capi.MOD_ISOSURF_INIT)):
            home |= capi.HOME_ISO
        self.ctx.set_home_rows(home)
        self.ctx.sort_by_box(0, self.n)
        self.sorted = True

    def sync(self) -> None:
        self.ctx.sync()

    def close(self) -> None:
        self.ctx.close()
