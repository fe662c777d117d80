"""DevicePool over real GPUs — the dispatch and data-region API of
`lagtrans.device_runtime` (/root/reference/pkg/src/lagtrans/device_runtime.py)
with device-resident images.

Reference model (device_runtime.py:1-7,88-244): a "device" is a worker
thread holding a deep-copied image of the whole model state; results come
back only through range-restricted copy-back.  Here a device is a CUDA
device driven by one host worker thread (the paper's one-process-drives-
all-GPUs design), and its image is an `lt_ctx`:

* region_create      -> lt_ctx_create + lt_particles_alloc of the OWNED range
                        only (the reference copies all N particles to every
                        device; a shard never reads another shard's slots)
* region_update_device("ens"/"cache"/"dt"/"batch")
                     -> H2D of the owned slice; ("met0","met1") -> the met
                        store binds the pair, uploading only snapshots it
                        does not already hold; ("clim") -> lt_clim_load
* region_update_host -> D2H of the owned slice, in original particle order
                        (undoing any box sort), into host[start:end)
* region_delete      -> lt_ctx_destroy (refused while tasks are in flight)

The module API (`physics.module_*`) recognises the image's ensemble as
device resident and launches in place; nothing crosses PCIe per step.
Lifecycle errors, the debug copy-back overlap check and per-device
failure aggregation keep the reference's types and messages.

Devices beyond the GPUs present map onto them round-robin (`device_map`),
so an N-device pool runs on fewer GPUs with N independent contexts — the
multi-device invariance tests use this on a single B200.
"""

from __future__ import annotations

from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _capi as capi
from . import physics
from ._capi import LifecycleError
from .engine import Engine
from .model_state import deep_copy
from .partition import WorkRange

MAX_DEVICES = 64

REGION_FIELDS = ("ctl", "ens", "cache", "clim", "met0", "met1", "dt", "batch")

__all__ = ["MAX_DEVICES", "REGION_FIELDS", "LifecycleError", "DeviceTaskError",
           "available_devices", "enumerate_devices", "ModelImage", "DeviceRegion",
           "DevicePool", "DeviceImage"]


class DeviceTaskError(RuntimeError):
    """One or more device tasks failed; maps device id to its exception
    (device_runtime.py:30-36)."""

    def __init__(self, failures: dict[int, BaseException]):
        self.failures = failures
        details = "; ".join(f"device {d}: {e!r}" for d, e in sorted(failures.items()))
        super().__init__(f"device task failure(s): {details}")


def available_devices() -> int:
    """CUDA devices visible to this process (device_runtime.py:39-44 counts
    host cores, the simulated devices of the reference)."""
    return capi.device_count()


def enumerate_devices(requested: int, available: int | None = None) -> int:
    """Resolve a device-count request; negative means all available
    (device_runtime.py:47-55)."""
    if requested == 0:
        raise ValueError("device count 0 is invalid (negative means all available)")
    if available is None:
        available = available_devices()
    if requested < 0:
        return min(max(available, 1), MAX_DEVICES)
    return min(requested, MAX_DEVICES)


@dataclass
class ModelImage:
    """The host model state bundle (device_runtime.py:58-69)."""

    ctl: object
    ens: object
    cache: object
    clim: object
    met0: object
    met1: object
    dt: np.ndarray
    batch: object


# ---------------------------------------------------------------- device image

class DeviceRow:
    """One per-particle field of a device image, indexed like the reference
    image's numpy array over the GLOBAL particle range (the reference's
    image is a deep copy of the whole model, device_runtime.py:165-186).
    The owned range lives in HBM — every access copies that part in or out,
    in particle order — and the particles outside it are the image's
    host-side copy (`outside`: the rows before and after the owned range
    only, so a one-device image holds none), which, as in the reference, is
    never computed on or copied back.  For tests and inspection; the module
    API and the driver never go through it."""

    def __init__(self, image: "DeviceImage", fid: int, row: int, host_row=None,
                 n_total: int = 0):
        self.image, self.fid, self.row = image, fid, row
        self.n_total = int(n_total if host_row is None else np.asarray(host_row).size)
        self.before = np.zeros(image.base)
        self.after = np.zeros(max(self.n_total - image.base - image.n, 0))
        if host_row is not None:
            self.refresh(host_row)

    def refresh(self, host_row) -> None:
        img = self.image
        h = np.asarray(host_row, dtype=np.float64)
        self.before[:] = h[:img.base]
        self.after[:] = h[img.base + img.n:]

    def _full(self) -> np.ndarray:
        img = self.image
        a = np.empty(self.n_total)
        a[:img.base] = self.before
        a[img.base + img.n:] = self.after
        if img.n:
            img.engine.ctx.d2h_ordered(self.fid, self.row, 0, img.n, img.base,
                                       out=a[img.base:img.base + img.n])
        return a

    def __array__(self, dtype=None, copy=None):
        a = self._full()
        return a if dtype is None else a.astype(dtype)

    def __getitem__(self, key):
        return self._full()[key]

    def __setitem__(self, key, value) -> None:
        img = self.image
        a = self._full()
        a[key] = value
        self.refresh(a)
        if img.n:
            img.engine.ctx.h2d_ordered(self.fid, self.row, 0, a[img.base:img.base + img.n], img.base)

    def __len__(self) -> int:
        return self.n_total

    @property
    def shape(self):
        return (self.n_total,)

    @property
    def dtype(self):
        return np.dtype(np.float64)


class DeviceRows:
    """A (rows, np) field of a device image (q, uvwp) as a stack of DeviceRow."""

    def __init__(self, rows: list[DeviceRow]):
        self.rows = rows

    def _full(self) -> np.ndarray:
        return np.stack([r._full() for r in self.rows])

    def __array__(self, dtype=None, copy=None):
        a = self._full()
        return a if dtype is None else a.astype(dtype)

    def __getitem__(self, key):
        if isinstance(key, (int, np.integer)):
            return self.rows[key]
        return self._full()[key]

    def __setitem__(self, key, value) -> None:
        a = self._full()
        a[key] = value
        for r, v in zip(self.rows, a):
            r[:] = v

    @property
    def shape(self):
        return (len(self.rows),) + self.rows[0].shape


class DeviceEnsemble:
    """Stand-in for `ParticleEnsemble` inside a device image: the SoA lives
    in HBM; `np` is the global particle count, as in the reference image.
    time, p, zeta, lon, lat and q read and write like the reference image's
    arrays (DeviceRow)."""

    is_device_resident = True

    def __init__(self, image: "DeviceImage", n_total: int, nq: int, host_ens=None):
        self.image = image
        self.np = n_total
        self.nq = nq
        self._rows = {}
        for name, fid in (("time", capi.F_TIME), ("p", capi.F_P), ("zeta", capi.F_ZETA),
                          ("lon", capi.F_LON), ("lat", capi.F_LAT)):
            h = getattr(host_ens, name) if host_ens is not None else None
            self._rows[name] = DeviceRow(image, fid, 0, h, n_total)
        self._q = DeviceRows([DeviceRow(image, capi.F_Q, k,
                                        host_ens.q[k] if host_ens is not None else None, n_total)
                              for k in range(nq)])

    def __getattr__(self, name):
        rows = self.__dict__.get("_rows", {})
        if name in rows:
            return rows[name]
        if name == "q":
            return self.__dict__["_q"]
        raise AttributeError(name)

    def refresh_shadow(self, host_ens) -> None:
        """The image's copy of particles outside the owned range (upload)."""
        for name, row in self._rows.items():
            row.refresh(getattr(host_ens, name))
        for k, row in enumerate(self._q.rows):
            row.refresh(host_ens.q[k])


class DeviceCache:
    """`CacheState` inside a device image (uvwp, iso_var in HBM).  The
    theta-isosurface counter stays on the device, as in the reference image
    (never copied back)."""

    is_device_resident = True

    def __init__(self, image: "DeviceImage", host_cache=None, n_total: int = 0):
        self.image = image
        hc = host_cache
        self.uvwp = DeviceRows([DeviceRow(image, capi.F_UVWP, c,
                                          hc.uvwp[c] if hc is not None else None, n_total)
                                for c in range(3)])
        self.iso_var = DeviceRow(image, capi.F_ISO_VAR, 0, hc.iso_var if hc is not None else None,
                                 n_total)

    def refresh_shadow(self, host_cache) -> None:
        for c, row in enumerate(self.uvwp.rows):
            row.refresh(host_cache.uvwp[c])
        self.iso_var.refresh(host_cache.iso_var)

    @property
    def iso_nonconverged(self) -> int:
        return self.image.engine.ctx.iso_counter()


class DeviceArray:
    """Marker for a per-particle device array (the image's `dt`)."""

    is_device_resident = True

    def __init__(self, image: "DeviceImage", name: str):
        self.image = image
        self.name = name


class DeviceImage:
    """One device's data region: an Engine (lt_ctx) holding the owned range
    [base, base + n) of the global ensemble."""

    def __init__(self, gpu: int, host: ModelImage, work: WorkRange, with_batch: bool = True,
                 donor=None):
        n_total = int(host.ens.np)
        nq = int(host.ens.q.shape[0])
        self.gpu = gpu
        self.base = work.start
        self.n = work.size
        self.engine = Engine(device=gpu, nq=max(nq, 5), first_id=work.start)
        self.engine.ctx.alloc(max(self.n, 1), max(nq, 5), with_batch=with_batch)
        self.engine.n = self.n
        self.engine.ctx.ids_reset(0, self.n, self.base)
        self.ctl = deep_copy(host.ctl)
        self.ens = DeviceEnsemble(self, n_total, nq, host.ens)
        self.cache = DeviceCache(self, host.cache, n_total)
        self.dt = DeviceArray(self, "dt")
        self.batch = DeviceArray(self, "batch")
        self.clim = host.clim
        self.met0 = None
        self.met1 = None
        self.donor = donor   # key -> (context, slot) of another device holding it

    # -- module execution (physics._run dispatches here) -------------------
    def local(self, work: WorkRange) -> tuple[int, int]:
        lo, hi = work.start - self.base, work.end - self.base
        if not (0 <= lo <= hi <= self.n):
            raise IndexError(f"range [{work.start}, {work.end}) outside the device's range "
                             f"[{self.base}, {self.base + self.n})")
        return lo, hi

    def bind(self, met0, met1) -> None:
        if met0 is not self.met0 or met1 is not self.met1:
            self.engine.bind_pair(met0, met1, self.donor)
            self.met0, self.met1 = met0, met1

    def run_module(self, module: int, ctl, work: WorkRange, met0=None, met1=None, clim=None,
                   cache=None) -> None:
        lo, hi = self.local(work)
        ctx = self.engine.ctx
        flags = 0
        if module & (capi.MOD_ADVECTION | capi.MOD_TURB | capi.MOD_MESO | capi.MOD_CONVECTION |
                     capi.MOD_SEDI | capi.MOD_DECAY):
            flags |= capi.RUN_DT_ARRAY
        if module == capi.MOD_TIMESTEPS:
            flags |= capi.RUN_WRITE_DT
        if module & (capi.MOD_ADVECTION | capi.MOD_TURB | capi.MOD_MESO | capi.MOD_SEDI |
                     capi.MOD_ISOSURF | capi.MOD_ISOSURF_INIT | capi.MOD_METEO):
            self.bind(met0, met1)
        if module & capi.MOD_METEO:
            ctx.load_clim(clim)
        if module & (capi.MOD_TURB | capi.MOD_MESO | capi.MOD_CONVECTION) and not ctx.with_batch:
            raise LifecycleError("module needs the random batch, but the region was created "
                                 "without one (use the fused step)")
        ctx.run(ctl, module, lo, hi, flags=flags)

    def rng_fill(self, mode: str, seed: int, step: int, work: WorkRange) -> None:
        lo, hi = self.local(work)
        self.engine.ctx.rng_fill(capi.RNG_MODES[mode], seed, step, lo, hi)

    # -- transfers ----------------------------------------------------------
    def upload(self, host: ModelImage, name: str) -> None:
        eng, ctx = self.engine, self.engine.ctx
        s = slice(self.base, self.base + self.n)
        if name == "ctl":
            self.ctl = deep_copy(host.ctl)
        elif name == "ens":
            ens = host.ens
            for fid, arr in ((capi.F_TIME, ens.time), (capi.F_P, ens.p), (capi.F_ZETA, ens.zeta),
                             (capi.F_LON, ens.lon), (capi.F_LAT, ens.lat)):
                ctx.h2d_ordered(fid, 0, 0, arr[s], self.base)
            for k in range(ens.q.shape[0]):
                ctx.h2d_ordered(capi.F_Q, k, 0, ens.q[k, s], self.base)
            self.ens.np = int(ens.np)
            self.ens.refresh_shadow(ens)
        elif name == "cache":
            for c in range(3):
                ctx.h2d_ordered(capi.F_UVWP, c, 0, host.cache.uvwp[c, s], self.base)
            ctx.h2d_ordered(capi.F_ISO_VAR, 0, 0, host.cache.iso_var[s], self.base)
            self.cache.refresh_shadow(host.cache)
        elif name == "dt":
            ctx.h2d_ordered(capi.F_DT, 0, 0, np.asarray(host.dt)[s], self.base)
        elif name == "batch":
            if ctx.with_batch and self.n:
                b = host.batch
                ctx.h2d(capi.F_RND_CONV, 0, 0, b.convection[s])
                ctx.h2d(capi.F_RND_TURB, 0, 0, b.diff_turb[3 * self.base:3 * (self.base + self.n)])
                ctx.h2d(capi.F_RND_MESO, 0, 0, b.diff_meso[3 * self.base:3 * (self.base + self.n)])
        elif name in ("met0", "met1"):
            self.bind(host.met0, host.met1)
        elif name == "clim":
            self.clim = host.clim
            if host.clim is not None:
                ctx.load_clim(host.clim)
        else:
            raise ValueError(f"unknown region field {name!r}")

    def download(self, host: ModelImage, work: WorkRange) -> None:
        """Owned slices of ens and cache back to the host, in particle order
        (device_runtime.py:212-219)."""
        lo, hi = self.local(work)
        if hi == lo:
            return
        ctx = self.engine.ctx
        s = slice(work.start, work.end)
        n = hi - lo
        if lo != 0 or hi != self.n:
            raise LifecycleError("copy-back must cover the device's whole range")
        def get(dst, fid, row=0):
            # straight into the caller's row when it is a contiguous float64
            # slice (pinned host memory then moves at full PCIe rate)
            v = dst[s]
            if v.flags.c_contiguous and v.dtype == np.float64:
                ctx.d2h_ordered(fid, row, 0, n, self.base, out=v)
            else:
                dst[s] = ctx.d2h_ordered(fid, row, 0, n, self.base)
        ens = host.ens
        for name, fid in (("time", capi.F_TIME), ("p", capi.F_P), ("zeta", capi.F_ZETA),
                          ("lon", capi.F_LON), ("lat", capi.F_LAT)):
            get(getattr(ens, name), fid)
        for k in range(min(ens.q.shape[0], ctx.nq)):
            get(ens.q[k], capi.F_Q, k)
        for c in range(3):
            get(host.cache.uvwp[c], capi.F_UVWP, c)
        get(host.cache.iso_var, capi.F_ISO_VAR)

    def close(self) -> None:
        self.engine.close()


@dataclass
class DeviceRegion:
    """One device's image with an explicit lifecycle
    (device_runtime.py:72-85): empty -> created -> populated -> deleted."""

    device_id: int
    state: str = "empty"
    image: DeviceImage | None = None
    work_range: WorkRange | None = None

    def _check_live(self, op: str) -> None:
        if self.state == "deleted":
            raise LifecycleError(f"{op} on deleted region of device {self.device_id}")
        if self.state == "empty":
            raise LifecycleError(f"{op} before create on device {self.device_id}")


class DevicePool:
    """A fixed set of GPU devices, each driven by one host worker thread;
    tasks on one device run in submission order, devices run concurrently
    (device_runtime.py:88-161).  ctypes drops the GIL around every library
    call, so per-device threads overlap their launches and copies."""

    def __init__(self, num_devices: int, debug: bool = False,
                 device_map: list[int] | None = None):
        if num_devices < 1:
            raise ValueError(f"num_devices must be >= 1, got {num_devices}")
        gpus = capi.device_count()
        if gpus < 1:
            raise RuntimeError("DevicePool needs at least one CUDA device")
        self.num_devices = num_devices
        self.debug = debug
        self.device_map = list(device_map) if device_map else [d % gpus for d in range(num_devices)]
        if len(self.device_map) != num_devices:
            raise ValueError("device_map must name one GPU per device")
        self._executors = [
            ThreadPoolExecutor(max_workers=1, thread_name_prefix=f"device{d}",
                               initializer=physics.set_device, initargs=(self.device_map[d],))
            for d in range(num_devices)]
        self._pending: list[list[Future]] = [[] for _ in range(num_devices)]
        self._regions: dict[int, DeviceRegion] = {}

    # -- dispatch ------------------------------------------------------------
    def _check_device_id(self, device_id: int) -> None:
        if not 0 <= device_id < self.num_devices:
            raise ValueError(f"device_id {device_id} out of range [0, {self.num_devices})")

    def dispatch(self, device_id: int, fn) -> Future:
        self._check_device_id(device_id)
        fut = self._executors[device_id].submit(fn)
        pending = self._pending[device_id]
        pending.append(fut)
        if len(pending) > 64:
            self._pending[device_id] = [f for f in pending if not f.done()]
        return fut

    def busy(self, device_id: int) -> bool:
        return any(not f.done() for f in self._pending[device_id])

    def device_wait(self, device_id: int) -> None:
        """Block until every task dispatched to the device has completed and
        its GPU work has drained (device_runtime.py:118-127)."""
        self._check_device_id(device_id)
        for fut in self._pending[device_id]:
            try:
                fut.result()
            except BaseException:
                pass
        self._pending[device_id] = []
        region = self._regions.get(device_id)
        if region is not None and region.image is not None:
            region.image.engine.sync()

    def for_each_device_parallel(self, task, parallel: bool = True) -> None:
        """Run task(device_id) once per device; failures are gathered per
        device and raised together (device_runtime.py:136-161).  Each task
        ends with a device sync, so asynchronous CUDA errors surface here."""

        def run(d):
            task(d)
            region = self._regions.get(d)
            if region is not None and region.image is not None:
                region.image.engine.sync()

        failures: dict[int, BaseException] = {}
        if parallel:
            futures = [self.dispatch(d, lambda d=d: run(d)) for d in range(self.num_devices)]
            for d, fut in enumerate(futures):
                try:
                    fut.result()
                except BaseException as exc:
                    failures[d] = exc
            for d in range(self.num_devices):
                self._pending[d] = []
        else:
            for d in range(self.num_devices):
                physics.set_device(self.device_map[d])
                try:
                    run(d)
                except BaseException as exc:
                    failures[d] = exc
        if failures:
            raise DeviceTaskError(failures)

    # -- data-region lifecycle -----------------------------------------------
    def region_create(self, device_id: int, host: ModelImage,
                      work_range: WorkRange | None = None, with_batch: bool = True) -> DeviceRegion:
        """Allocate the device image of `work_range` (the whole ensemble when
        None); content is defined by the first update_device."""
        self._check_device_id(device_id)
        live = self._regions.get(device_id)
        if live is not None and live.state in ("created", "populated"):
            raise LifecycleError(f"device {device_id} already has a live region")
        work = work_range or WorkRange(device_id, 0, int(host.ens.np))
        gpu = self.device_map[device_id]
        image = self._executors[device_id].submit(
            lambda: DeviceImage(gpu, host, work, with_batch, donor=self._met_donor)).result()
        region = DeviceRegion(device_id=device_id, state="created", image=image,
                              work_range=work_range)
        self._regions[device_id] = region
        return region

    def region_update_device(self, region: DeviceRegion, host: ModelImage, fields) -> None:
        region._check_live("update_device")
        for name in fields:
            if name not in REGION_FIELDS:
                raise ValueError(f"unknown region field {name!r}")
        img = region.image
        self._executors[region.device_id].submit(
            lambda: [img.upload(host, name) for name in fields]).result()
        region.state = "populated"

    def region_update_host(self, region: DeviceRegion, host: ModelImage, work: WorkRange) -> None:
        """Copy the owned ensemble/cache slices back; host bytes outside
        [work.start, work.end) are untouched (device_runtime.py:188-219)."""
        region._check_live("update_host")
        if region.state != "populated":
            raise LifecycleError(f"update_host on unpopulated region of device {region.device_id}")
        if self.debug:
            if region.work_range is not None and (work.start, work.end) != \
                    (region.work_range.start, region.work_range.end):
                raise LifecycleError(
                    f"device {region.device_id} copy-back range [{work.start}, {work.end}) is "
                    f"not its own range [{region.work_range.start}, {region.work_range.end})")
            for other in self._regions.values():
                if other is region or other.work_range is None or other.state == "deleted":
                    continue
                if work.overlaps(other.work_range):
                    raise LifecycleError(f"copy-back range of device {region.device_id} "
                                         f"overlaps device {other.device_id}'s range")
        img = region.image
        host.ens.np = img.ens.np
        self._executors[region.device_id].submit(lambda: img.download(host, work)).result()

    def region_delete(self, region: DeviceRegion) -> None:
        if region.state == "deleted":
            raise LifecycleError(f"double delete on device {region.device_id}")
        region._check_live("delete")
        if self.busy(region.device_id):
            raise LifecycleError(f"delete with in-flight task on device {region.device_id}")
        img = region.image
        self._executors[region.device_id].submit(img.close).result()
        region.image = None
        region.state = "deleted"

    def _met_donor(self, key):
        """A live image already holding snapshot `key`: new images replicate
        it GPU to GPU (peer copy over NVLink) instead of re-uploading it
        from the host — the met broadcast of the paper's design."""
        for region in self._regions.values():
            img = region.image
            if img is None:
                continue
            slot = img.engine.ctx.find_slot(key)
            if slot is not None:
                return img.engine.ctx, slot
        return None

    def region(self, device_id: int) -> DeviceRegion:
        return self._regions[device_id]

    def shutdown(self) -> None:
        for ex in self._executors:
            ex.shutdown(wait=True)
        for region in self._regions.values():
            if region.image is not None:
                region.image.close()
                region.image = None
                region.state = "deleted"

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.shutdown()
        return False
