"""Output-side statistics on the GPU — `lagtrans.output.write_grid` and
`write_ens` (/root/reference/pkg/src/lagtrans/output.py:28-64) computed
where the particles live.

* `grid_counts` — output.py:33-38: particles per lon/lat bin, upper edges
  in the last bin; exact int64 counts (block-privatised shared-memory
  histogram, lt_grid_counts).
* `group_stats` — output.py:52-63: groups from int64(q[slot]), ascending;
  count and mean/std (ddof 0) of lon, lat and p (radix sort by group then
  particle id, segmented two-pass reductions, lt_group_stats).  Means and
  stds agree with numpy to rounding (numpy sums pairwise, the device sums
  in a fixed tree); counts and group ids are exact.

`write_grid` / `write_ens` keep the reference's CSV format byte for byte
(`repr` floats).  `pool_*` combine the shards of a `DevicePool`: counts
add, group moments merge with Chan's parallel formula.  The file writers
themselves are host I/O and otherwise out of scope.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import _capi as capi
from .partition import WorkRange


def _fmt(x: float) -> str:
    return repr(float(x))


def _ctx_range(ens, work):
    """(context, local start, local end) for a host or device ensemble."""
    if getattr(ens, "is_device_resident", False):
        img = ens.image
        w = work or WorkRange(0, img.base, img.base + img.n)
        lo, hi = img.local(w)
        return img.engine.ctx, lo, hi
    from .physics import default_context
    w = work or WorkRange(0, 0, int(ens.np))
    ctx = default_context()
    n = w.size
    nq = ens.q.shape[0]
    ctx.ensure_capacity(n, nq=max(nq, 5))
    s = w.slice
    for fid, arr in ((capi.F_LON, ens.lon), (capi.F_LAT, ens.lat), (capi.F_P, ens.p)):
        ctx.h2d(fid, 0, 0, arr[s])
    for k in range(nq):
        ctx.h2d(capi.F_Q, k, 0, ens.q[k, s])
    ctx.ids_reset(0, n, w.start)
    return ctx, 0, n


def grid_counts(ctl, ens, work: WorkRange | None = None) -> np.ndarray:
    """(grid_nx, grid_ny) int64 particle counts (output.py:33-38)."""
    nx, ny = int(ctl.grid_nx), int(ctl.grid_ny)
    out = np.zeros((nx, ny), dtype=np.int64)
    if nx * ny == 0:
        return out
    ctx, lo, hi = _ctx_range(ens, work)
    capi.check(ctx.lib.lt_grid_counts(ctx.h, nx, ny, lo, hi, capi.ptr(out)))
    return out


def group_stats(ctl, ens, work: WorkRange | None = None, max_groups: int = 1024):
    """(gids, counts, means[3, G], stds[3, G]) over (lon, lat, p) per group
    (output.py:52-63); ValueError as the reference for a bad slot or a
    negative group id."""
    slot = int(ctl.ens_group_slot)
    nq = ens.nq if getattr(ens, "is_device_resident", False) else ens.q.shape[0]
    if not 0 <= slot < nq:
        raise ValueError(f"ens_group_slot {slot} is not a valid quantity slot")
    ctx, lo, hi = _ctx_range(ens, work)
    while True:
        G = max(int(max_groups), 1)
        ng = C.c_int64(0)
        gid = np.zeros(G, dtype=np.int64)
        cnt = np.zeros(G, dtype=np.int64)
        mean = np.zeros((3, G))
        std = np.zeros((3, G))
        rc = ctx.lib.lt_group_stats(ctx.h, slot, lo, hi, G, C.byref(ng), capi.ptr(gid),
                                    capi.ptr(cnt), capi.ptr(mean), capi.ptr(std))
        if rc == capi.LT_ERR_RANGE and ng.value > G:
            max_groups = ng.value
            continue
        capi.check(rc)
        g = ng.value
        return gid[:g], cnt[:g], mean[:, :g].copy(), std[:, :g].copy()


def merge_group_stats(parts):
    """Chan et al. pairwise merge of per-shard (gids, counts, means, stds)."""
    acc: dict[int, list] = {}
    for gids, cnts, means, stds in parts:
        for k, g in enumerate(gids):
            n_b, m_b, v_b = int(cnts[k]), means[:, k], stds[:, k] ** 2
            if int(g) not in acc:
                acc[int(g)] = [n_b, m_b.copy(), v_b * n_b]
                continue
            n_a, m_a, m2_a = acc[int(g)]
            n = n_a + n_b
            d = m_b - m_a
            acc[int(g)] = [n, m_a + d * (n_b / n), m2_a + v_b * n_b + d * d * (n_a * n_b / n)]
    gids = np.array(sorted(acc), dtype=np.int64)
    cnts = np.array([acc[g][0] for g in gids], dtype=np.int64)
    means = np.array([acc[g][1] for g in gids]).T.reshape(3, -1)
    stds = np.sqrt(np.array([acc[g][2] / acc[g][0] for g in gids]).T.reshape(3, -1))
    return gids, cnts, means, stds


def pool_grid_counts(ctl, pool) -> np.ndarray:
    """Sum of every live region's counts (C6: per-GPU partials, one sum)."""
    total = np.zeros((int(ctl.grid_nx), int(ctl.grid_ny)), dtype=np.int64)
    for d in range(pool.num_devices):
        img = pool.region(d).image
        total += pool._executors[d].submit(lambda img=img: grid_counts(ctl, img.ens)).result()
    return total


def pool_group_stats(ctl, pool):
    parts = [pool._executors[d].submit(
        lambda img=pool.region(d).image: group_stats(ctl, img.ens)).result()
        for d in range(pool.num_devices)]
    return merge_group_stats(parts)


def format_double(x: float) -> str:
    """repr(float(x)) computed by the library (lt_format_double)."""
    lib = capi.load()
    buf = C.create_string_buffer(40)
    n = C.c_int32(0)
    capi.check(lib.lt_format_double(float(x), buf, 40, C.byref(n)))
    return buf.value.decode()


def write_atm(ens, path, threads: int = 0) -> None:
    """output.py:17-25, byte for byte, formatted by native threads
    (lt_write_atm) instead of a per-particle Python loop."""
    lib = capi.load()
    n = int(ens.np)
    rows = [np.ascontiguousarray(getattr(ens, k)[:n], dtype=np.float64)
            for k in ("time", "p", "zeta", "lon", "lat")]
    q = np.ascontiguousarray(ens.q[:, :n], dtype=np.float64)
    nq = q.shape[0]
    rc = lib.lt_write_atm(str(path).encode(), n, nq, *[capi.ptr(r) for r in rows],
                          capi.ptr(q) if nq else None, n, int(threads))
    if rc != capi.LT_OK:
        raise OSError(f"lt_write_atm failed for {path}")


def write_grid(ctl, ens, path) -> None:
    """output.py:28-44 with the counts from the GPU."""
    nx, ny = int(ctl.grid_nx), int(ctl.grid_ny)
    counts = grid_counts(ctl, ens)
    wx, wy = 360.0 / nx, 180.0 / ny
    lines = ["lon_center,lat_center,count"]
    for i in range(nx):
        for j in range(ny):
            lines.append(f"{_fmt(-180.0 + (i + 0.5) * wx)},{_fmt(-90.0 + (j + 0.5) * wy)},"
                         f"{counts[i, j]}")
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")


def write_ens(ctl, ens, path) -> None:
    """output.py:47-64 with the statistics from the GPU."""
    gids, cnts, means, stds = group_stats(ctl, ens)
    lines = ["group,count,lon_mean,lon_std,lat_mean,lat_std,p_mean,p_std"]
    for k, g in enumerate(gids):
        stats = [means[0, k], stds[0, k], means[1, k], stds[1, k], means[2, k], stds[2, k]]
        lines.append(f"{g},{int(cnts[k])}," + ",".join(_fmt(v) for v in stats))
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")
