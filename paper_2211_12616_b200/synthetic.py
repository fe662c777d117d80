"""Synthetic met snapshots and particle clouds for the benchmark configs.

Recipes follow SURVEY.md Appendix B (there is no network for reanalysis
data).  Every value is rounded through float32, so the float32 met store on
the GPU and the float64 CPU oracle see exactly the same numbers.
"""

from __future__ import annotations

import numpy as np

from .model_state import ClimData, MeteoField, ParticleEnsemble, met_periodic, read_clim  # noqa: F401


def f32(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def grid(dlon: float, dlat: float, nlev: int, p_min: float = 1.0):
    """lon -180..180-dlon, lat -90..90, levels geomspace(1013.25, p_min, nlev)."""
    lons = f32(np.arange(-180.0, 180.0, dlon))
    lats = f32(np.linspace(-90.0, 90.0, int(round(180.0 / dlat)) + 1))
    levs = f32(np.geomspace(1013.25, p_min, nlev))
    return lons, lats, levs


def era5_like(lons, lats, levs, phase_deg: float = 0.0, periodic: bool = False,
              chunk: int = 16, threads: int | None = None):
    """'ERA5-like' multi-scale fields (App. B) as float32 (nx, ny, nz) arrays:
    u = 20cos(lat) + 10sin(3lon)cos^2(lat) + 5lev/1000, v = 5sin(2lon)cos(lat),
    w = 1e-3 sin(lat)cos(4lon) hPa/s, T = 200 + 0.08lev + 10cos(lat).

    With periodic=True the arrays get one more longitude column, a copy of
    column 0 (what met_periodic, ingest.py:195-207, appends)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    nx, ny, nz = len(lons), len(lats), len(levs)
    shape = (nx + (1 if periodic else 0), ny, nz)
    out = {k: np.empty(shape, dtype=np.float32) for k in ("u", "v", "w", "T")}
    ra = np.deg2rad(lats)[None, :, None]
    ca, sa = np.cos(ra), np.sin(ra)
    le = np.asarray(levs, dtype=np.float64)[None, None, :]

    def fill(i0):
        rl = np.deg2rad(np.asarray(lons[i0:i0 + chunk]) + phase_deg)[:, None, None]
        sl = slice(i0, min(i0 + chunk, nx))
        out["u"][sl] = 20 * ca + 10 * np.sin(3 * rl) * ca ** 2 + 5 * le / 1000
        out["v"][sl] = 5 * np.sin(2 * rl) * ca
        out["w"][sl] = 1e-3 * sa * np.cos(4 * rl)
        out["T"][sl] = 200 + 0.08 * le + 10 * ca

    with ThreadPoolExecutor(threads or min(32, os.cpu_count() or 1)) as pool:
        list(pool.map(fill, range(0, nx, chunk)))
    if periodic:
        for a in out.values():
            a[nx] = a[0]
    return out


def snapshot(t_met, lons, lats, levs, fields, periodic=True) -> MeteoField:
    """MeteoField from float32 fields; periodic closes the longitude circle
    (fields already carrying the extra column are used as they are)."""
    if periodic and fields["u"].shape[0] == len(lons) + 1:
        return MeteoField(float(t_met), np.append(lons, lons[0] + 360.0), lats, levs,
                          fields["u"], fields["v"], fields["w"], fields["T"])
    met = MeteoField(float(t_met), lons, lats, levs, fields["u"], fields["v"], fields["w"],
                     fields["T"])
    return met_periodic(met) if periodic else met


def analytic_pair(dlon=1.0, dlat=1.0, nlev=60, t0=0.0, t1=10800.0, p_min=1.0,
                  periodic=True):
    """Two ERA5-like snapshots, the second phase-shifted by 10 deg in lon."""
    lons, lats, levs = grid(dlon, dlat, nlev, p_min)
    m0 = snapshot(t0, lons, lats, levs, era5_like(lons, lats, levs, 0.0, periodic), periodic)
    m1 = snapshot(t1, lons, lats, levs, era5_like(lons, lats, levs, 10.0, periodic), periodic)
    return m0, m1


def solid_body_pair(dlon=1.0, dlat=1.0, nlev=60, t_end=86400.0):
    """cfg1: u = Omega*Re*cos(lat), v = w = 0, T = 250, two identical snapshots
    at t = 0 and t_end (so the kernel exercises the two-slot blend)."""
    lons, lats, levs = grid(dlon, dlat, nlev)
    omega = 2.0 * np.pi / 86400.0
    ulat = f32(omega * 6371000.0 * np.cos(np.deg2rad(lats))).astype(np.float32)
    shape = (lons.size, lats.size, levs.size)
    u = np.ascontiguousarray(np.broadcast_to(ulat[None, :, None], shape))
    z = np.zeros(shape, dtype=np.float32)
    T = np.full(shape, 250.0, dtype=np.float32)
    f = {"u": u, "v": z, "w": z, "T": T}
    return snapshot(0.0, lons, lats, levs, f), snapshot(t_end, lons, lats, levs, f)


def particles(n: int, seed: int = 12616, lat_span: float = 80.0, p_lo: float = 300.0,
              p_hi: float = 900.0, nq: int = 5) -> ParticleEnsemble:
    """Uniform cloud (test_acceptance.py:62-64 ranges), fp32-rounded, time 0."""
    rs = np.random.default_rng(seed)
    lon = f32(rs.uniform(-180.0, 180.0, n))
    lat = f32(rs.uniform(-lat_span, lat_span, n))
    p = f32(rs.uniform(p_lo, p_hi, n))
    return ParticleEnsemble(n, np.zeros(n), p, np.zeros(n), lon, lat, np.zeros((nq, n)))


def point_release(n: int, lon=-175.4, lat=-20.5, p=30.0, nq: int = 6) -> ParticleEnsemble:
    """cfg4 volcanic point release: every particle at one point."""
    full = lambda v: np.full(n, float(np.float32(v)))
    return ParticleEnsemble(n, np.zeros(n), full(p), np.zeros(n), full(lon), full(lat),
                            np.zeros((nq, n)))
