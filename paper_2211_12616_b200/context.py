"""DeviceContext — one GPU's data region, a thin owner of an `lt_ctx`.

Equivalent of one DevicePool worker's ModelImage in the reference
(device_runtime.py:58-69,165-230), but resident in HBM: SoA particle
fields, up to three met snapshot slots, climatology tables and the CUDA
streams, all owned by liblagtrans_b200.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import zlib

import numpy as np

from . import _capi as capi


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


_HASH_CHUNK = 1 << 26   # 64 MiB per checksum task


def _chunk_sums(m) -> tuple:
    return zlib.crc32(m), zlib.adler32(m), m.nbytes


def _digest(a: np.ndarray, pool) -> bytes:
    """Content digest of EVERY byte of `a` (C order): CRC-32 and Adler-32 of
    each 64 MiB chunk (zlib releases the GIL, so the chunks run on a thread
    pool at memory speed), combined in order by blake2b — any change to any
    element changes the digest except with probability ~2^-64 per chunk."""
    buf = memoryview(np.ascontiguousarray(a)).cast("B")
    parts = [buf[o:o + _HASH_CHUNK] for o in range(0, max(buf.nbytes, 1), _HASH_CHUNK)]
    sums = list(pool.map(_chunk_sums, parts)) if len(parts) > 1 else [_chunk_sums(buf)]
    return hashlib.blake2b(repr(sums).encode(), digest_size=16).digest()


def met_fingerprint(met) -> tuple:
    """Content identity of a MeteoField: its time and a digest of every byte
    of its axes and fields (with shapes and dtypes).  A snapshot rewritten in
    place — even one element, even with the same t_met — gets a new key, so
    the met-slot cache (bind_pair) never reuses stale fields.  ~0.1–0.3 s
    for a 0.25 deg snapshot on a multi-core host."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    h = hashlib.blake2b(digest_size=16)
    with ThreadPoolExecutor(min(32, os.cpu_count() or 1)) as pool:
        for name in ("lons", "lats", "levs", "u", "v", "w", "T"):
            a = np.asarray(getattr(met, name))
            h.update(f"{name}{a.shape}{a.dtype.str}".encode())
            h.update(_digest(a, pool))
    return (float(met.t_met), h.hexdigest())


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (cudaHostAlloc), freed when
    the array is garbage collected; host-path copies from it run at full
    PCIe rate and overlap the kernels."""
    import weakref
    lib = capi.load()
    count = int(np.prod(shape))
    nbytes = max(count * np.dtype(dtype).itemsize, 8)
    p = C.c_void_p()
    capi.check(lib.lt_host_alloc(nbytes, C.byref(p)))
    buf = (C.c_char * nbytes).from_address(p.value)
    arr = np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
    weakref.finalize(buf, lib.lt_host_free, C.c_void_p(p.value))
    return arr


def met_broadcast(ctxs, root: int, slots) -> None:
    """lt_met_broadcast: slot slots[root] of ctxs[root] into slot slots[i] of
    every other context — one NCCL broadcast group over the distinct GPUs
    (device-to-device copies for contexts sharing a GPU).  Asynchronous on
    the contexts' copy streams; use_met orders compute after it."""
    lib = capi.load()
    n = len(ctxs)
    handles = (C.c_void_p * n)(*[c.h for c in ctxs])
    sl = (C.c_int32 * n)(*[int(s) for s in slots])
    capi.check(lib.lt_met_broadcast(handles, n, int(root), sl))
    key = ctxs[root]._slot_keys[slots[root]]
    for c, s in zip(ctxs, slots):
        c._slot_keys[s] = key


def nccl_info() -> dict:
    """Version of the libnccl the broadcast loads, and the NCCL ranks created."""
    lib = capi.load()
    v, r = C.c_int32(0), C.c_int32(0)
    rc = lib.lt_nccl_version(C.byref(v))
    lib.lt_nccl_ranks(C.byref(r))
    return {"version": int(v.value) if rc == capi.LT_OK else None, "ranks": int(r.value)}


class DeviceContext:
    """Owns one lt_ctx on `device`; all methods raise the reference's
    exception types on failure (ValueError, IndexError, LifecycleError)."""

    def __init__(self, device: int = 0, met_precision: str = "f32"):
        self.lib = capi.load()
        self.device = device
        h = C.c_void_p()
        capi.check(self.lib.lt_ctx_create(device, C.byref(h)))
        self.h = h
        self.capacity = 0
        self.nq = 0
        self.with_batch = False
        self.met_precision = met_precision
        self._grid_key = None
        self._slot_keys = [None, None, None]
        self._clim_key = None
        self.closed = False

    # -- lifecycle -------------------------------------------------------
    def close(self) -> None:
        if not self.closed:
            self.closed = True
            capi.check(self.lib.lt_ctx_destroy(self.h))

    def __del__(self):  # best effort
        try:
            if not self.closed:
                self.lib.lt_ctx_destroy(self.h)
                self.closed = True
        except Exception:
            pass

    def sync(self) -> None:
        capi.check(self.lib.lt_sync(self.h))

    def stream_handle(self) -> int:
        s = C.c_void_p()
        capi.check(self.lib.lt_stream(self.h, C.byref(s)))
        return s.value or 0

    # -- particles -------------------------------------------------------
    def alloc(self, capacity: int, nq: int = 5, with_batch: bool = False) -> None:
        capi.check(self.lib.lt_particles_alloc(self.h, int(capacity), int(nq), int(with_batch)))
        self.capacity, self.nq, self.with_batch = int(capacity), int(nq), bool(with_batch)

    def ensure_capacity(self, n: int, nq: int = 5, with_batch: bool = False) -> None:
        if n > self.capacity or nq > self.nq or (with_batch and not self.with_batch) \
                or self.capacity == 0:
            self.alloc(max(n, 1), max(nq, 5), with_batch or self.with_batch)

    def h2d(self, field: int, row: int, offset: int, arr) -> None:
        a = _f64(arr)
        capi.check(self.lib.lt_field_h2d(self.h, field, row, offset, a.size, capi.ptr(a)))

    def d2h(self, field: int, row: int, offset: int, count: int, out=None) -> np.ndarray:
        out = np.empty(count) if out is None else out
        capi.check(self.lib.lt_field_d2h(self.h, field, row, offset, count, capi.ptr(out)))
        return out

    def h2d_ordered(self, field, row, offset, arr, first_id) -> None:
        a = _f64(arr)
        capi.check(self.lib.lt_field_h2d_ordered(self.h, field, row, offset, a.size, first_id,
                                                 capi.ptr(a)))

    def d2h_ordered(self, field, row, offset, count, first_id, out=None) -> np.ndarray:
        out = np.empty(count) if out is None else out
        capi.check(self.lib.lt_field_d2h_ordered(self.h, field, row, offset, count, first_id,
                                                 capi.ptr(out)))
        return out

    def fill(self, field, row, offset, count, value) -> None:
        capi.check(self.lib.lt_field_fill(self.h, field, row, offset, count, float(value)))

    def ids(self, offset: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint32)
        capi.check(self.lib.lt_field_d2h(self.h, capi.F_ID, 0, offset, count, capi.ptr(out)))
        return out

    def ids_reset(self, offset: int, count: int, first_id: int) -> None:
        capi.check(self.lib.lt_ids_reset(self.h, offset, count, first_id))

    def devptr(self, field: int, row: int = 0) -> int:
        p = C.c_void_p()
        capi.check(self.lib.lt_field_devptr(self.h, field, row, C.byref(p)))
        return p.value or 0

    # -- met ---------------------------------------------------------------
    def set_grid(self, lons, lats, levs, precision: str | None = None) -> None:
        prec = precision or self.met_precision
        lons, lats, levs = _f64(lons), _f64(lats), _f64(levs)
        key = (lons.tobytes(), lats.tobytes(), levs.tobytes(), prec)
        if key == self._grid_key:
            return
        capi.check(self.lib.lt_met_grid(self.h, lons.size, lats.size, levs.size,
                                        capi.ptr(lons), capi.ptr(lats), capi.ptr(levs),
                                        capi.MET_F64 if prec == "f64" else capi.MET_F32))
        self._grid_key = key
        self._slot_keys = [None, None, None]

    def load_met(self, slot: int, met, key=None, close_lon: bool = False) -> None:
        """Upload a MeteoField-like snapshot into `slot` (copy stream)."""
        arrs = []
        src_bytes = 8
        for name in ("u", "v", "w", "T"):
            a = np.asarray(getattr(met, name))
            if a.dtype == np.float32:
                src_bytes = 4
            arrs.append(a)
        dt = np.float32 if src_bytes == 4 else np.float64
        arrs = [np.ascontiguousarray(a, dtype=dt) for a in arrs]
        self._met_arrays = arrs  # keep alive until the copy is staged
        capi.check(self.lib.lt_met_load(self.h, slot, float(met.t_met), src_bytes,
                                        *[capi.ptr(a) for a in arrs],
                                        capi.MET_CLOSE_LON if close_lon else 0))
        self._slot_keys[slot] = key

    def load_met_nodes(self, slot: int, t_met: float, nodes: np.ndarray | int,
                       close_lon: bool = False, key=None) -> None:
        """Upload (nx, ny, nz, 4) float32 nodes (numpy array or pinned pointer)."""
        p = nodes if isinstance(nodes, int) else capi.ptr(nodes)
        capi.check(self.lib.lt_met_load_nodes(self.h, slot, float(t_met), C.c_void_p(p),
                                              capi.MET_CLOSE_LON if close_lon else 0))
        self._slot_keys[slot] = key

    def copy_slot_from(self, src: "DeviceContext", src_slot: int, slot: int, key=None) -> None:
        """Replicate src's packed snapshot into `slot` (peer copy / D2D)."""
        capi.check(self.lib.lt_met_copy_slot(self.h, slot, src.h, src_slot))
        self._slot_keys[slot] = key if key is not None else src._slot_keys[src_slot]

    def use_met(self, slot0: int, slot1: int) -> None:
        capi.check(self.lib.lt_met_use(self.h, slot0, slot1))

    def slot_key(self, slot: int):
        return self._slot_keys[slot]

    def bind_pair(self, met0, met1, donor=None) -> tuple[int, int]:
        """Make (met0, met1) the active snapshot pair, uploading only what
        changed (module-API path; grids must be identical).  `donor(key)`
        may name another context already holding a snapshot — (ctx, slot) —
        which is then replicated GPU to GPU instead of uploaded again.
        Returns the (met0, met1) slot numbers."""
        for name in ("lons", "lats", "levs"):
            if not np.array_equal(np.asarray(getattr(met0, name)), np.asarray(getattr(met1, name))):
                raise ValueError("met0 and met1 must share one grid on the B200 met store")
        self.set_grid(met0.lons, met0.lats, met0.levs)
        k0 = met_fingerprint(met0)
        k1 = k0 if met1 is met0 else met_fingerprint(met1)
        slots = {}
        for key in (k0, k1):
            if key in slots:
                continue
            for s in range(3):
                if self._slot_keys[s] == key and s not in slots.values():
                    slots[key] = s
                    break
        for key, met in ((k0, met0), (k1, met1)):
            if key in slots:
                continue
            free = next(s for s in range(3) if s not in slots.values())
            src = donor(key) if donor is not None else None
            if src is not None and src[0] is not self and src[0]._grid_key == self._grid_key:
                self.copy_slot_from(src[0], src[1], free, key)
            else:
                self.load_met(free, met, key)
            slots[key] = free
        self.use_met(slots[k0], slots[k1])
        return slots[k0], slots[k1]

    def find_slot(self, key):
        """Slot holding the snapshot with fingerprint `key`, or None."""
        for s in range(3):
            if self._slot_keys[s] == key:
                return s
        return None

    def load_clim(self, clim) -> None:
        lat, pg = _f64(clim.lat_grid), _f64(clim.p_grid)
        hno3, pt = _f64(clim.hno3_tab), _f64(clim.p_trop_tab)
        key = hashlib.blake2b(b"".join(a.tobytes() for a in (lat, pg, hno3, pt))).hexdigest()
        if key == self._clim_key:
            return
        capi.check(self.lib.lt_clim_load(self.h, lat.size, pg.size, capi.ptr(lat), capi.ptr(pg),
                                         capi.ptr(hno3), capi.ptr(pt)))
        self._clim_key = key

    # -- compute -----------------------------------------------------------
    def run(self, ctl, modules: int, start: int, end: int, step: int = 0,
            faithful_state: int = 0, faithful_base: int = 0, flags: int = 0) -> None:
        c = ctl if isinstance(ctl, capi.LtControl) else capi.control_struct(ctl)
        capi.check(self.lib.lt_run(self.h, C.byref(c), modules, start, end, step,
                                   faithful_state & 0xFFFFFFFFFFFFFFFF, faithful_base, flags))

    def run_steps(self, ctl, modules: int, start: int, end: int, step: int, nsteps: int,
                  flags: int = 0) -> None:
        """lt_run_steps: `nsteps` consecutive steps in one launch."""
        c = ctl if isinstance(ctl, capi.LtControl) else capi.control_struct(ctl)
        capi.check(self.lib.lt_run_steps(self.h, C.byref(c), modules, start, end, step,
                                          int(nsteps), flags))

    def run_host(self, ctl, modules: int, n: int, step: int, first_id: int, time, p, lon, lat,
                 uvwp=None, iso_var=None, q=None, faithful_state: int = 0,
                 chunk: int = 0, steps: int = 1) -> None:
        """lt_run_host_steps on C-contiguous float64 host arrays (updated in
        place): `steps` consecutive steps, each a full host round trip."""
        c = ctl if isinstance(ctl, capi.LtControl) else capi.control_struct(ctl)
        arrs = [time, p, lon, lat]
        for a in arrs + [x for x in (uvwp, iso_var, q) if x is not None]:
            if a.dtype != np.float64 or not a.flags.c_contiguous or not a.flags.writeable:
                raise ValueError("host rows must be writeable C-contiguous float64 arrays")
        rows2 = [x for x in (uvwp, q) if x is not None]
        stride = rows2[0].shape[1] if rows2 else n
        if any(x.shape[1] != stride for x in rows2):
            raise ValueError("uvwp and q must share one row stride")
        io = capi.LtHostSoa(*[capi.ptr(a) for a in arrs],
                            capi.ptr(uvwp) if uvwp is not None else None,
                            capi.ptr(iso_var) if iso_var is not None else None,
                            capi.ptr(q) if q is not None else None, stride,
                            q.shape[0] if q is not None else 0)
        capi.check(self.lib.lt_run_host_steps(self.h, C.byref(c), modules, n, step, int(steps),
                                              first_id, faithful_state & 0xFFFFFFFFFFFFFFFF,
                                              C.byref(io), chunk))

    def rng_fill(self, mode: int, seed: int, step: int, start: int, end: int) -> None:
        capi.check(self.lib.lt_rng_fill(self.h, mode, seed & 0xFFFFFFFFFFFFFFFF, step, start, end))

    def iso_counter(self, reset: bool = False) -> int:
        v = C.c_int64()
        capi.check(self.lib.lt_iso_counter(self.h, C.byref(v), int(reset)))
        return int(v.value)

    def set_home_rows(self, mask: int) -> None:
        """Keep the HOME_* row groups in particle order (not moved by sorts)."""
        capi.check(self.lib.lt_set_home_rows(self.h, mask))

    def sort_by_box(self, start: int, end: int) -> None:
        capi.check(self.lib.lt_sort_by_box(self.h, start, end))

    def sort_info(self) -> tuple[int, int]:
        """(sorts, sorts that used the keys of the step launched just before)."""
        a, b = C.c_int64(0), C.c_int64(0)
        capi.check(self.lib.lt_sort_info(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def interpolate(self, t, lon, lat, p) -> np.ndarray:
        lon = _f64(lon)
        n = lon.size
        t = _f64(np.broadcast_to(np.asarray(t, dtype=np.float64), (n,)))
        lat, p = _f64(lat), _f64(p)
        out = np.empty((4, n))
        capi.check(self.lib.lt_interpolate(self.h, n, capi.ptr(t), capi.ptr(lon), capi.ptr(lat),
                                           capi.ptr(p), capi.ptr(out)))
        return out

    def locate_cells(self, lon, lat, p, precision: str = "exact") -> np.ndarray:
        """(3, n) int32 cell indices (i, j, k) of the exact or fast kernels'
        lookup at host points (lt_locate_cells; the box-index audit)."""
        lon, lat, p = _f64(lon), _f64(lat), _f64(p)
        out = np.empty((3, lon.size), dtype=np.int32)
        capi.check(self.lib.lt_locate_cells(self.h, capi.PRECISIONS[precision], lon.size,
                                            capi.ptr(lon), capi.ptr(lat), capi.ptr(p),
                                            capi.ptr(out)))
        return out

    def timing(self, on: bool) -> None:
        capi.check(self.lib.lt_timing(self.h, int(on)))

    def module_cycles(self, reset: bool = True) -> np.ndarray:
        """SM cycles per module of the RUN_MODULE_CLOCKS launches so far
        (slots in capi.MODULE_CLOCK_NAMES order)."""
        out = np.zeros(len(capi.MODULE_CLOCK_NAMES), dtype=np.uint64)
        capi.check(self.lib.lt_module_cycles(self.h, capi.ptr(out), int(reset)))
        return out

    def last_elapsed_ms(self) -> float:
        v = C.c_float()
        capi.check(self.lib.lt_last_elapsed_ms(self.h, C.byref(v)))
        return float(v.value)
