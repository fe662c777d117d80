"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference particle time step (`lagtrans`,
`/root/reference/pkg/src/lagtrans/physics.py` and `rng.py`).  Only
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` may import this module, and only as the
checker or the timed CPU baseline.  The CUDA path in
`paper_2211_12616_b200` never calls it.

Parity status: PINNED.  `tests/test_oracle_golden.py` checks every
function here against (a) the reference's own known-answer tests
(splitmix64 vectors, `test_physics.py` analytic cases) and (b) golden
input/output vectors produced by running the reference itself in the
build container (`tests/golden/make_golden.py`, fixtures in
`tests/golden/*.npz`).  Decay (`decay_factor`) and the box sort
(`box_keys`) have no reference counterpart: decay is specified in
DESIGN.md ("parity unpinned" for that row); the sort is pinned by
construction (stable argsort of keys computed from the pinned locate).

Style: functions take plain float64 arrays (one particle per element)
and return new arrays; nothing here mutates its inputs.  Every function
cites the reference lines it restates.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# physics.py:17-24 — physical constants, bit-identical literals
EARTH_RADIUS = 6_371_000.0
GRAVITY = 9.80665
GAS_CONST_AIR = 287.058
AIR_VISCOSITY = 1.8205e-5
KAPPA = 0.2857
DEG_PER_METRE = 180.0 / (np.pi * EARTH_RADIUS)
COS_LAT_FLOOR = np.cos(np.deg2rad(89.999))

# rng.py:24-31 — splitmix64 increment, stream ids
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
U64 = 0xFFFFFFFFFFFFFFFF
STREAM_CONV, STREAM_TURB, STREAM_MESO = 0, 1, 2
TWO_POW_M64 = 2.0 ** -64


# --------------------------------------------------------------------------
# grid geometry
# --------------------------------------------------------------------------

@dataclass
class Snapshot:
    """One met time level (restates model_state.py:126-137).

    `levs` is surface-first (strictly decreasing) exactly as the reference
    stores it; fields are (nx, ny, nz) float64, level index fastest."""
    t_met: float
    lons: np.ndarray
    lats: np.ndarray
    levs: np.ndarray
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    T: np.ndarray

    @classmethod
    def like(cls, met) -> "Snapshot":
        """Adopt any object exposing the reference MeteoField attributes."""
        a = lambda x: np.asarray(x, dtype=np.float64)
        return cls(float(met.t_met), a(met.lons), a(met.lats), a(met.levs),
                   a(met.u), a(met.v), a(met.w), a(met.T))


def close_longitudes(snap: Snapshot) -> Snapshot:
    """Append the +360 column when the longitudes span the globe.

    Restates ingest.py:195-207 (met_periodic): the test is
    |lon[-1] - lon[0] + (lon[1]-lon[0]) - 360| <= 1e-6 (math.isclose with
    abs_tol, rel_tol 1e-9)."""
    step = snap.lons[1] - snap.lons[0]
    if not math.isclose(snap.lons[-1] - snap.lons[0] + step, 360.0, abs_tol=1e-6):
        return snap
    extend = lambda f: np.concatenate([f, f[:1]], axis=0)
    return Snapshot(snap.t_met, np.append(snap.lons, snap.lons[0] + 360.0),
                    snap.lats, snap.levs, extend(snap.u), extend(snap.v),
                    extend(snap.w), extend(snap.T))


def bracket(axis_ascending: np.ndarray, x: np.ndarray):
    """Cell index and fraction on an ascending axis (physics.py:31-37).

    x is first clamped to [axis[0], axis[-1]]; the index is
    (#nodes strictly below x) - 1, clipped to [0, n-2] (numpy
    searchsorted side='left'); the fraction uses the clamped x."""
    n = axis_ascending.shape[0]
    xc = np.minimum(np.maximum(x, axis_ascending[0]), axis_ascending[-1])
    below = np.searchsorted(axis_ascending, xc, side="left")
    idx = np.minimum(np.maximum(below - 1, 0), n - 2)
    lo = axis_ascending[idx]
    hi = axis_ascending[idx + 1]
    return idx, (xc - lo) / (hi - lo)


def cell_of(snap: Snapshot, lon, lat, p):
    """(i, j, k, fx, fy, fz) of the enclosing cell (physics.py:42-47).

    The vertical axis is bracketed on the reversed (ascending) levels, then
    mapped back: k = nz - 2 - k_rev and fz = 1 - f_rev."""
    i, fx = bracket(snap.lons, lon)
    j, fy = bracket(snap.lats, lat)
    k_rev, f_rev = bracket(snap.levs[::-1], p)
    k = snap.levs.shape[0] - 2 - k_rev
    return i, j, k, fx, fy, 1.0 - f_rev


def corner_weights(fx, fy, fz):
    """Eight trilinear weights in reference order (physics.py:49-56).

    Order (di,dj,dk): 000,100,010,110,001,101,011,111; each product is
    evaluated left to right as numpy does."""
    gx, gy, gz = 1 - fx, 1 - fy, 1 - fz
    return (gx * gy * gz, fx * gy * gz, gx * fy * gz, fx * fy * gz,
            gx * gy * fz, fx * gy * fz, gx * fy * fz, fx * fy * fz)


_CORNERS = ((0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0),
            (0, 0, 1), (1, 0, 1), (0, 1, 1), (1, 1, 1))


def trilinear(snap: Snapshot, lon, lat, p, names):
    """Spatial interpolation of each named field (physics.py:40-66).

    The eight weighted corner terms are summed strictly left to right."""
    i, j, k, fx, fy, fz = cell_of(snap, lon, lat, p)
    wts = corner_weights(fx, fy, fz)
    out = []
    for name in names:
        field = getattr(snap, name)
        acc = None
        for wgt, (di, dj, dk) in zip(wts, _CORNERS):
            term = wgt * field[i + di, j + dj, k + dk]
            acc = term if acc is None else acc + term
        out.append(acc)
    return out


def sample(m0: Snapshot, m1: Snapshot, t, lon, lat, p, names):
    """Space then time interpolation (physics.py:69-79).

    Equal snapshot times short-circuit to m0; otherwise
    wt = clip((t - t0)/(t1 - t0), 0, 1) and (1-wt)*a + wt*b."""
    first = trilinear(m0, lon, lat, p, names)
    if m1.t_met == m0.t_met:
        return first
    second = trilinear(m1, lon, lat, p, names)
    wt = (np.asarray(t, dtype=np.float64) - m0.t_met) / (m1.t_met - m0.t_met)
    wt = np.minimum(np.maximum(wt, 0.0), 1.0)
    return [(1.0 - wt) * a + wt * b for a, b in zip(first, second)]


def inv_metric_cos(lat):
    """max(cos(lat * pi/180), cos(89.999 deg)) (physics.py:27-28)."""
    return np.maximum(np.cos(np.deg2rad(lat)), COS_LAT_FLOOR)


# --------------------------------------------------------------------------
# process modules — each returns the updated arrays
# --------------------------------------------------------------------------

def timestep_lengths(ctl, time):
    """physics.py:82-88: clip(min(dt_model, t_stop - time), 0, dt_model)."""
    dt = np.minimum(ctl.dt_model, ctl.t_stop - time)
    return np.minimum(np.maximum(dt, 0.0), ctl.dt_model)


def advect(m0, m1, dt, lon, lat, p, time):
    """Explicit midpoint trajectory step (physics.py:91-116)."""
    moving = dt > 0.0
    u0, v0, w0 = sample(m0, m1, time, lon, lat, p, ("u", "v", "w"))
    h = 0.5 * dt
    lon_h = lon + u0 * h * DEG_PER_METRE / inv_metric_cos(lat)
    lat_h = lat + v0 * h * DEG_PER_METRE
    p_h = p + w0 * h
    u1, v1, w1 = sample(m0, m1, time + h, lon_h, lat_h, p_h, ("u", "v", "w"))
    new_lon = lon + u1 * dt * DEG_PER_METRE / inv_metric_cos(lat_h)
    new_lat = lat + v1 * dt * DEG_PER_METRE
    new_p = p + w1 * dt
    return (np.where(moving, new_lon, lon), np.where(moving, new_lat, lat),
            np.where(moving, new_p, p), np.where(moving, time + dt, time))


def turbulent_hop(ctl, m0, m1, dt, xi3, lon, lat, p, time):
    """Gaussian turbulent displacement (physics.py:119-147).

    xi3 is (n, 3).  The vertical part samples T at the post-hop lon/lat,
    the pre-hop p and the (already advanced) particle time, matching the
    reference's in-place view semantics (physics.py:133,139-143)."""
    if ctl.turb_dx == 0.0 and ctl.turb_dz == 0.0:
        return lon, lat, p
    moving = dt > 0.0
    if ctl.turb_dx > 0.0:
        s = np.sqrt(2.0 * ctl.turb_dx * dt)
        lon = np.where(moving, lon + s * xi3[:, 0] * DEG_PER_METRE / inv_metric_cos(lat), lon)
        lat = np.where(moving, lat + s * xi3[:, 1] * DEG_PER_METRE, lat)
    if ctl.turb_dz > 0.0:
        (temp,) = sample(m0, m1, time, lon, lat, p, ("T",))
        dz = np.sqrt(2.0 * ctl.turb_dz * dt) * xi3[:, 2]
        dens = 100.0 * p / (GAS_CONST_AIR * temp)
        p = np.where(moving, p + (-(dens * GRAVITY * dz) / 100.0), p)
    return lon, lat, p


def pairwise8(cols):
    """numpy's 8-term pairwise sum ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)),
    the order np.std(axis=1) uses on an (n, 8) array (physics.py:179)."""
    return ((cols[0] + cols[1]) + (cols[2] + cols[3])) + \
           ((cols[4] + cols[5]) + (cols[6] + cols[7]))


def corner_std(field, i, j, k):
    """Population std of the 8 cell corners (np.std, ddof=0)."""
    cols = [field[i + di, j + dj, k + dk] for di, dj, dk in _CORNERS_MESO]
    mean = pairwise8(cols) / 8
    dev = [(c - mean) * (c - mean) for c in cols]
    return np.sqrt(pairwise8(dev) / 8)


# physics.py:173-175 — corner order used by the mesoscale module
_CORNERS_MESO = tuple(zip((0, 1, 0, 1, 0, 1, 0, 1),
                          (0, 0, 1, 1, 0, 0, 1, 1),
                          (0, 0, 0, 0, 1, 1, 1, 1)))


def mesoscale_hop(ctl, m0, dt, xi3, uvwp, lon, lat, p):
    """AR(1) subgrid wind perturbation (physics.py:150-188).

    uvwp is (3, n).  sigma_c = turb_meso * std over the 8 met0 corners;
    r = clip(1 - 2 dt / met_dt, 0, 1); amp = sqrt(1 - r^2)."""
    if ctl.turb_meso == 0.0:
        return lon, lat, p, uvwp
    moving = dt > 0.0
    i, j, k, _, _, _ = cell_of(m0, lon, lat, p)
    r = np.minimum(np.maximum(1.0 - 2.0 * dt / ctl.met_dt, 0.0), 1.0)
    amp = np.sqrt(1.0 - r * r)
    new = np.empty_like(uvwp)
    for c, name in enumerate(("u", "v", "w")):
        sigma = ctl.turb_meso * corner_std(getattr(m0, name), i, j, k)
        new[c] = np.where(moving, r * uvwp[c] + amp * sigma * xi3[:, c], uvwp[c])
    lon = np.where(moving, lon + new[0] * dt * DEG_PER_METRE / inv_metric_cos(lat), lon)
    lat_new = np.where(moving, lat + new[1] * dt * DEG_PER_METRE, lat)
    p = np.where(moving, p + new[2] * dt, p)
    return lon, lat_new, p, new


def convective_mix(ctl, dt, r, p):
    """Random vertical redistribution (physics.py:191-203)."""
    if ctl.conv_prob == 0.0:
        return p
    hit = (dt > 0.0) & (p > ctl.conv_p_top) & (r < ctl.conv_prob)
    target = ctl.conv_p_top + (r / ctl.conv_prob) * (ctl.p_surf - ctl.conv_p_top)
    return np.where(hit, target, p)


def settle(ctl, m0, m1, dt, lon, lat, p, time):
    """Stokes settling as a pressure increase (physics.py:206-222)."""
    if ctl.sedi_radius == 0.0:
        return p
    (temp,) = sample(m0, m1, time, lon, lat, p, ("T",))
    dens = 100.0 * p / (GAS_CONST_AIR * temp)
    vs = 2.0 * ctl.sedi_radius ** 2 * (ctl.sedi_density - dens) * GRAVITY / (9.0 * AIR_VISCOSITY)
    return np.where(dt > 0.0, p + (dens * GRAVITY * vs * dt) / 100.0, p)


def isosurface_value(ctl, m0, m1, lon, lat, p, time, iso_var):
    """module_isosurf_init (physics.py:225-235)."""
    if ctl.isosurf_mode == "pressure":
        return p.copy()
    if ctl.isosurf_mode == "theta":
        (temp,) = sample(m0, m1, time, lon, lat, p, ("T",))
        return temp * (1000.0 / p) ** KAPPA
    return iso_var


def isosurface_pull(ctl, m0, m1, lon, lat, p, time, iso_var):
    """module_isosurf (physics.py:238-264). Returns (p, n_nonconverged)."""
    if ctl.isosurf_mode == "pressure":
        return iso_var.copy(), 0
    if ctl.isosurf_mode != "theta":
        return p, 0
    cur = p.copy()
    todo = np.ones(cur.shape[0], dtype=bool)
    for _ in range(10):
        if not todo.any():
            break
        (temp,) = sample(m0, m1, time, lon, lat, cur, ("T",))
        nxt = 1000.0 * (temp / iso_var) ** (1.0 / KAPPA)
        step = np.where(todo, nxt - cur, 0.0)
        cur = np.where(todo, nxt, cur)
        todo &= np.abs(step) >= 0.1
    return cur, int(np.count_nonzero(todo))


def numpy_mod(a, b):
    """np.mod on floats: fmod, then add b when the remainder's sign
    differs from b's (ingest.py:87-88, physics.py:284)."""
    return np.mod(a, b)


def fold_position(ctl, lon, lat, p):
    """Pole reflection, longitude wrap, pressure clamp (physics.py:267-287)."""
    lon = lon.copy()
    lat = lat.copy()
    while True:
        over = np.abs(lat) > 90.0
        if not over.any():
            break
        lat[over] = np.sign(lat[over]) * (180.0 - np.abs(lat[over]))
        lon[over] = lon[over] + 180.0
    wrap = (lon < -180.0) | (lon >= 180.0)
    lon[wrap] = numpy_mod(lon[wrap] + 180.0, 360.0) - 180.0
    return lon, lat, np.minimum(np.maximum(p, ctl.p_top), ctl.p_surf)


def climatology_tables():
    """Analytic climatology (ingest.py:210-224): lat grid 5 deg, p grid
    10 hPa; p_trop = 300 - 200 cos^2(lat); hno3 gaussian in p."""
    lat_grid = np.arange(-90.0, 90.0 + 1e-9, 5.0)
    p_grid = np.arange(10.0, 1000.0 + 1e-9, 10.0)
    rad = np.deg2rad(lat_grid)
    p_trop = 300.0 - 200.0 * np.cos(rad) ** 2
    hno3 = (1e-8 * np.exp(-(((p_grid[None, :] - 50.0) / 40.0) ** 2))
            * (0.5 + 0.5 * np.cos(rad))[:, None])
    return lat_grid, p_grid, hno3, p_trop


def hno3_lookup(lat_grid, p_grid, tab, lat, p):
    """Bilinear clamped table lookup (model_state.py:169-181)."""
    i, fi = bracket(lat_grid, lat)
    j, fj = bracket(p_grid, p)
    return ((1 - fi) * (1 - fj) * tab[i, j] + fi * (1 - fj) * tab[i + 1, j]
            + (1 - fi) * fj * tab[i, j + 1] + fi * fj * tab[i + 1, j + 1])


def sample_along(m0, m1, clim, lon, lat, p, time):
    """module_meteo (physics.py:290-301): q0..q4 = T, u, v, hno3, strat."""
    lat_grid, p_grid, hno3, p_trop = clim
    temp, u, v = sample(m0, m1, time, lon, lat, p, ("T", "u", "v"))
    strat = np.where(p < np.interp(lat, lat_grid, p_trop), 1.0, 0.0)
    return temp, u, v, hno3_lookup(lat_grid, p_grid, hno3, lat, p), strat


def decay_factor(ctl, dt, q):
    """Exponential decay (new north-star module):
    q * exp(-dt / tau) where dt > 0, tau = ctl.decay_tau > 0."""
    tau = getattr(ctl, "decay_tau", 0.0)
    if tau <= 0.0:
        return q
    return np.where(dt > 0.0, q * np.exp(-dt / tau), q)


def part1by1(x):
    """Spread the low 16 bits of x to the even bit positions."""
    x = np.asarray(x, dtype=np.uint64) & np.uint64(0xFFFF)
    for shift, mask in ((8, 0x00FF00FF), (4, 0x0F0F0F0F), (2, 0x33333333), (1, 0x55555555)):
        x = (x | (x << np.uint64(shift))) & np.uint64(mask)
    return x


BOX_LEVELS = 2   # level cells per sort box (lt_kernels.cuh LT_BOX_ZDIV)


def box_keys(snap: Snapshot, lon, lat, p):
    """Sort key of the met cell (i, j, k) of each particle (new north-star
    component; the cell is pinned through the reference locate): the lon/lat
    column in Z (Morton) order, bits of i above those of j, times the number
    of level boxes, plus the level box k // BOX_LEVELS — when that fits 32
    bits, else the linear record index ((i*ny)+j)*(nz-1)+k.  Mirrors
    lt_sort_by_box."""
    i, j, k, _, _, _ = cell_of(snap, lon, lat, p)
    nx, ny, nz = snap.lons.shape[0], snap.lats.shape[0], snap.levs.shape[0]
    nb = (nz - 2) // BOX_LEVELS + 1
    top = int((part1by1(nx - 1) << np.uint64(1)) | part1by1(ny - 1)) * nb + (nb - 1)
    if nx <= 65536 and ny <= 65536 and top < 2 ** 32:
        col = (part1by1(i) << np.uint64(1)) | part1by1(j)
        return (col * np.uint64(nb) + (k // BOX_LEVELS).astype(np.uint64)).astype(np.int64)
    return ((i.astype(np.int64) * ny + j) * (nz - 1) + k).astype(np.int64)


# --------------------------------------------------------------------------
# random numbers (rng.py)
# --------------------------------------------------------------------------

def seed_for(rank, device):
    """rng.py:54-56."""
    return rank + 83 * device


def splitmix64_step(state: int):
    """Scalar splitmix64 (rng.py:71-77): returns (output, new_state)."""
    state = (state + GOLDEN_GAMMA) & U64
    z = ((state ^ (state >> 30)) * 0xBF58476D1CE4E5B9) & U64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & U64
    return z ^ (z >> 31), state


def finalize64(x: np.ndarray) -> np.ndarray:
    """Vector splitmix64 output mix (rng.py:80-89) on uint64 arrays."""
    with np.errstate(over="ignore"):
        z = np.array(x, dtype=np.uint64, copy=True)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit_interval(words: np.ndarray) -> np.ndarray:
    """uint64 -> float64 (round to nearest) times 2^-64 (rng.py:92-94)."""
    return words.astype(np.float64) * TWO_POW_M64


def gauss_pair(ua, ub):
    """Box-Muller with the u<=0 nudge (rng.py:97-102): (r cos, r sin)."""
    ua = np.where(ua <= 0.0, TWO_POW_M64, ua)
    rad = np.sqrt(-2.0 * np.log(ua))
    ang = 2.0 * np.pi * ub
    return rad * np.cos(ang), rad * np.sin(ang)


def faithful_words(state: int, n: int) -> np.ndarray:
    """The 7n sequential splitmix64 outputs of one fill (rng.py:115-119)."""
    with np.errstate(over="ignore"):
        k = np.arange(1, 7 * n + 1, dtype=np.uint64)
        return finalize64(np.uint64(state) + k * np.uint64(GOLDEN_GAMMA))


def faithful_batch(state: int, n: int):
    """Faithful-mode fill (rng.py:105-126).

    Returns (conv[n], turb[n,3], meso[n,3], new_state)."""
    u = unit_interval(faithful_words(state, n)).reshape(n, 7)
    a0, a1 = gauss_pair(u[:, 1], u[:, 2])
    b0, b1 = gauss_pair(u[:, 3], u[:, 4])
    c0, c1 = gauss_pair(u[:, 5], u[:, 6])
    return (u[:, 0], np.stack([a0, a1, b0], axis=1),
            np.stack([b1, c0, c1], axis=1), (state + 7 * n * GOLDEN_GAMMA) & U64)


def counter_words(seed, step, idx, stream, comp):
    """Keyed splitmix64 words (rng.py:129-147): key = seed ^ (step[0:32] |
    idx[0:24]<<32 | (stream*4+comp)[0:8]<<56), word = mix(key + gamma).
    Note the reference keeps only 24 bits of the particle index."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = (np.uint64(step & 0xFFFFFFFF)
               | ((idx & np.uint64(0xFFFFFF)) << np.uint64(32))
               | (np.uint64((stream * 4 + comp) & 0xFF) << np.uint64(56)))
        key = np.uint64(seed & U64) ^ key
        return finalize64(key + np.uint64(GOLDEN_GAMMA))


def counter_uniform(seed, step, idx, stream, comp):
    return unit_interval(counter_words(seed, step, idx, stream, comp))


def counter_gauss(seed, step, idx, stream, comp):
    """rng.py:150-153: cos branch only; shares u_{c+1} with comp+1."""
    ua = counter_uniform(seed, step, idx, stream, comp)
    ub = counter_uniform(seed, step, idx, stream, comp + 1)
    ua = np.where(ua <= 0.0, TWO_POW_M64, ua)
    return np.sqrt(-2.0 * np.log(ua)) * np.cos(2.0 * np.pi * ub)


def counter_batch(seed, step, start, end):
    """Counter-mode fill of particles [start, end) (rng.py:172-177)."""
    idx = np.arange(start, end, dtype=np.uint64)
    conv = counter_uniform(seed, step, idx, STREAM_CONV, 0)
    turb = np.stack([counter_gauss(seed, step, idx, STREAM_TURB, c) for c in range(3)], 1)
    meso = np.stack([counter_gauss(seed, step, idx, STREAM_MESO, c) for c in range(3)], 1)
    return conv, turb, meso


def split_range(n, parts, part):
    """Contiguous block partition, remainder to the front (partition.py:28-41)."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if not 0 <= part < parts:
        raise ValueError("part out of range")
    base, extra = divmod(n, parts)
    lo = part * base + min(part, extra)
    return lo, lo + base + (1 if part < extra else 0)


# --------------------------------------------------------------------------
# whole step (driver_cli.py:151-183 order) — used by the CPU baseline
# --------------------------------------------------------------------------

def full_step(ctl, m0, m1, st, lo, hi, step, rng_state=None, clim=None,
              modules=("advection", "turb", "meso", "convection", "sedi",
                       "isosurf", "position", "meteo")):
    # decay (new module, not in the reference) runs after sedi when listed
    """Advance particles [lo, hi) of the state dict `st` by one step.

    st holds arrays time, lon, lat, p, uvwp(3,n), iso_var, q(nq,n).
    Random numbers: counter mode unless rng_state (faithful device state)
    is given; returns the new faithful state (or None)."""
    s = slice(lo, hi)
    time, lon, lat, p = st["time"][s], st["lon"][s], st["lat"][s], st["p"][s]
    dt = timestep_lengths(ctl, time)
    n = hi - lo
    new_state = None
    need_rng = any(m in modules for m in ("turb", "meso", "convection"))
    if need_rng:
        if rng_state is None:
            conv, turb, meso = counter_batch(ctl.rng_seed_global, step, lo, hi)
        else:
            conv, turb, meso, new_state = faithful_batch(rng_state, n)
    if "advection" in modules:
        lon, lat, p, time = advect(m0, m1, dt, lon, lat, p, time)
    if "turb" in modules:
        lon, lat, p = turbulent_hop(ctl, m0, m1, dt, turb, lon, lat, p, time)
    if "meso" in modules:
        lon, lat, p, uvwp = mesoscale_hop(ctl, m0, dt, meso, st["uvwp"][:, s], lon, lat, p)
        st["uvwp"][:, s] = uvwp
    if "convection" in modules:
        p = convective_mix(ctl, dt, conv, p)
    if "sedi" in modules:
        p = settle(ctl, m0, m1, dt, lon, lat, p, time)
    slot = getattr(ctl, "decay_slot", -1)
    if "decay" in modules and 0 <= slot < st["q"].shape[0]:
        st["q"][slot, s] = decay_factor(ctl, dt, st["q"][slot, s])
    if "isosurf" in modules:
        p, _ = isosurface_pull(ctl, m0, m1, lon, lat, p, time, st["iso_var"][s])
    if "position" in modules:
        lon, lat, p = fold_position(ctl, lon, lat, p)
    if "meteo" in modules and clim is not None:
        q = sample_along(m0, m1, clim, lon, lat, p, time)
        for slot in range(5):
            st["q"][slot, s] = q[slot]
    st["time"][s], st["lon"][s], st["lat"][s], st["p"][s] = time, lon, lat, p
    return new_state


# --------------------------------------------------------------------------
# output-side statistics (output.py:28-64)
# --------------------------------------------------------------------------

def bin_counts(lon, lat, nx, ny):
    """Particles per lon/lat bin over [-180,180) x [-90,90], upper edges in
    the last bin (output.py:33-38: clip(floor((x+off)/w)) then add.at)."""
    wx, wy = 360.0 / nx, 180.0 / ny
    ix = np.clip(np.floor((np.asarray(lon) + 180.0) / wx).astype(np.int64), 0, nx - 1)
    iy = np.clip(np.floor((np.asarray(lat) + 90.0) / wy).astype(np.int64), 0, ny - 1)
    return np.bincount(ix * ny + iy, minlength=nx * ny).astype(np.int64).reshape(nx, ny)


def grouped_moments(qslot, lon, lat, p):
    """Ascending group ids int64(qslot) (>= 0, else ValueError) with count,
    mean and population std of lon, lat, p per group (output.py:52-63)."""
    gids = np.asarray(qslot).astype(np.int64)
    if np.any(gids < 0):
        raise ValueError("group ids must be non-negative")
    groups = np.unique(gids)
    counts = np.array([np.count_nonzero(gids == g) for g in groups], dtype=np.int64)
    means = np.array([[np.mean(a[gids == g]) for g in groups] for a in (lon, lat, p)])
    stds = np.array([[np.std(a[gids == g]) for g in groups] for a in (lon, lat, p)])
    return groups, counts, means.reshape(3, -1), stds.reshape(3, -1)
