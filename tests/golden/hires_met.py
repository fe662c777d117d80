"""Met recipe of the 0.25 deg x 137-level golden fixture (hires.npz) and of
the global 1 deg x 60-level one (deg1.npz, with lon_scale = 180 and the
+360 column of met_periodic appended as a copy of column 0).

The fixture is the headline grid's shape — 0.25 deg spacing and all 137
levels of geomspace(1013.25, 0.01, 137) — on a 40 x 40 deg window
(161 x 161 columns at the south-west corner of the globe: the -180 edge,
the pole).  The fields are too large to commit (2 x 14 MB of float32), so
the fixture stores the axes and the particle in/out vectors, and both the
generator (make_golden.py, which runs the reference) and the GPU tests
rebuild the fields here from the stored axes.

Only + - * / appear below, so the float64 values — and their float32
roundings, which is what the reference and the GPU met store both see —
are the same on every IEEE machine (no libm, whose last bits differ
between CPUs).  `fields_digest` pins that: make_golden stores the digest of
the fields the reference ran on and the tests check they rebuilt the same
bytes.  Shapes are ERA5-like in magnitude: u up to ~35 m/s,
v ~5 m/s, w ~1e-3 hPa/s, T 200-290 K.
"""

from __future__ import annotations

import hashlib

import numpy as np

WINDOW = dict(lon0=-180.0, lat0=-90.0, n_lon=161, n_lat=161, step=0.25)


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def axes():
    """(lons, lats, levs) as the generator builds them (levels surface
    first); the tests use the copies stored in hires.npz instead."""
    lons = f32(np.arange(-180.0, 180.0, 0.25))[:WINDOW["n_lon"]]
    lats = f32(np.linspace(-90.0, 90.0, 721))[:WINDOW["n_lat"]]
    levs = f32(np.geomspace(1013.25, 0.01, 137))
    return lons, lats, levs


def fields(lons, lats, levs, phase=0.0, lon_scale=20.0):
    """u, v, w, T as float32-valued float64 (nx, ny, nz) arrays.  lon_scale
    180 keeps the longitude polynomial O(1) on a global grid (deg1.npz)."""
    X = ((np.asarray(lons, dtype=np.float64) + phase) / lon_scale)[:, None, None]
    Y = (np.asarray(lats, dtype=np.float64) / 90.0)[None, :, None]
    Z = (np.asarray(levs, dtype=np.float64) / 1000.0)[None, None, :]
    c = 1.0 - Y * Y                           # cos-like in latitude
    s = X * (1.0 - X * X / 6.0)               # sin-like in longitude
    shape = (X.shape[0], Y.shape[1], Z.shape[2])
    u = 20.0 * c + 10.0 * s * (c * c) + 5.0 * Z
    v = 5.0 * (X * X - 0.5) * c + 0.0 * Z
    w = 1e-3 * Y * (1.0 - 0.5 * X * X) + 0.0 * Z
    T = 200.0 + 80.0 * Z + 10.0 * c + 0.0 * X
    return {k: f32(np.broadcast_to(a, shape)) for k, a in (("u", u), ("v", v), ("w", w),
                                                           ("T", T))}


def fields_digest(f) -> str:
    h = hashlib.sha256()
    for k in ("u", "v", "w", "T"):
        h.update(np.ascontiguousarray(f[k], dtype=np.float32).tobytes())
    return h.hexdigest()
