"""Generate golden vectors by running the REFERENCE `lagtrans` package.

Run in the build container only (it imports /root/reference, which does
not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs `tests/golden/*.npz`.  All synthetic inputs (met values, particle
positions, random draws fed to modules) are rounded through float32 so a
float32 met store on the GPU sees exactly the values the reference saw.
"""

from __future__ import annotations

import copy
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))

from lagtrans import ingest, physics, rng as lrng  # noqa: E402
from lagtrans.model_state import (Control, MeteoField, cache_allocate,  # noqa: E402
                                  ensemble_allocate)
from lagtrans.partition import WorkRange, partition_all  # noqa: E402


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def grid(dlon, dlat, levs):
    lons = f32(np.arange(-180.0, 180.0, dlon))
    lats = f32(np.linspace(-90.0, 90.0, int(round(180.0 / dlat)) + 1))
    return lons, lats, f32(levs)


def analytic_met(t_met, lons, lats, levs, phase=0.0, periodic=True):
    """Smooth multi-scale fields (SURVEY App. B 'ERA5-like'), fp32-rounded."""
    LO, LA, LE = np.meshgrid(lons, lats, levs, indexing="ij")
    rl, ra = np.deg2rad(LO + phase), np.deg2rad(LA)
    u = 20 * np.cos(ra) + 10 * np.sin(3 * rl) * np.cos(ra) ** 2 + 5 * LE / 1000
    v = 5 * np.sin(2 * rl) * np.cos(ra)
    w = 1e-3 * np.sin(ra) * np.cos(4 * rl)
    T = 200 + 0.08 * LE + 10 * np.cos(ra)
    met = MeteoField(t_met=float(t_met), lons=lons, lats=lats, levs=levs,
                     u=f32(u), v=f32(v), w=f32(w), T=f32(T))
    met.validate()
    return ingest.met_periodic(met) if periodic else met


def particles(ctl, n, seed, lat_span=85.0):
    rs = np.random.default_rng(seed)
    ens = ensemble_allocate(ctl, n)
    ens.lon[:] = f32(rs.uniform(-180.0, 180.0, n))
    ens.lat[:] = f32(rs.uniform(-lat_span, lat_span, n))
    ens.p[:] = f32(rs.uniform(ctl.p_top + 1, ctl.p_surf - 1, n))
    return ens


def met_arrays(prefix, met):
    return {f"{prefix}_t": np.float64(met.t_met), f"{prefix}_lons": met.lons,
            f"{prefix}_lats": met.lats, f"{prefix}_levs": met.levs,
            f"{prefix}_u": met.u.astype(np.float32), f"{prefix}_v": met.v.astype(np.float32),
            f"{prefix}_w": met.w.astype(np.float32), f"{prefix}_T": met.T.astype(np.float32)}


def ens_arrays(prefix, ens):
    return {f"{prefix}_{k}": getattr(ens, k).copy()
            for k in ("time", "p", "zeta", "lon", "lat", "q")}


def gen_interp():
    """Locate + interpolate_met on awkward points: exact nodes, hull edges,
    out-of-hull, decreasing levels, time blend and equal-time snapshots."""
    lons, lats, levs = grid(10.0, 5.0, np.geomspace(1013.25, 1.0, 20))
    m0 = analytic_met(0.0, lons, lats, levs)
    m1 = analytic_met(10800.0, lons, lats, levs, phase=10.0)
    rs = np.random.default_rng(7)
    n = 4000
    lon = f32(rs.uniform(-200.0, 200.0, n))
    lat = f32(rs.uniform(-95.0, 95.0, n))
    p = f32(rs.uniform(0.5, 1100.0, n))
    t = f32(rs.uniform(-100.0, 11000.0, n))
    # exact grid nodes and hull corners exercise searchsorted side='left'
    lon[:400] = rs.choice(m0.lons, 400)
    lat[400:800] = rs.choice(m0.lats, 400)
    p[800:1200] = rs.choice(m0.levs, 400)
    lon[1200:1210] = m0.lons[0]; lon[1210:1220] = m0.lons[-1]
    lat[1220:1230] = -90.0; lat[1230:1240] = 90.0
    p[1240:1250] = m0.levs[0]; p[1250:1260] = m0.levs[-1]
    i, fx = physics._locate(m0.lons, lon)
    j, fy = physics._locate(m0.lats, lat)
    krev, fz = physics._locate(m0.levs[::-1], p)
    out = physics.interpolate_met(m0, m1, t, lon, lat, p)
    same = physics.interpolate_met(m0, m0, t, lon, lat, p)
    np.savez_compressed(OUT / "interp.npz", lon=lon, lat=lat, p=p, t=t,
                        i=i, j=j, krev=krev, fx=fx, fy=fy, fz=fz,
                        uvwT=np.stack(out), uvwT_same=np.stack(same),
                        **met_arrays("m0", m0), **met_arrays("m1", m1))


def modules_control():
    return Control(np_max=10**6, t_stop=9000.0, met_dt=10800.0, turb_dx=50.0,
                   turb_dz=0.1, turb_meso=0.16, conv_prob=0.3, conv_p_top=300.0,
                   sedi_radius=5e-6, sedi_density=2000.0, isosurf_mode="theta",
                   rng_mode="counter", rng_seed_global=12616)


def gen_modules():
    """Single-call in/out pairs for every module from identical inputs."""
    lons, lats, levs = grid(10.0, 5.0, np.geomspace(1013.25, 1.0, 20))
    m0 = analytic_met(0.0, lons, lats, levs)
    m1 = analytic_met(10800.0, lons, lats, levs, phase=10.0)
    ctl = modules_control()
    ens = particles(ctl, 3000, 11)
    np.savez_compressed(OUT / "modules.npz", **module_pairs(ctl, m0, m1, ens))


def module_pairs(ctl, m0, m1, ens, seed=12, lon_span=(-900.0, 900.0)):
    """Every module called once, in pipeline order, on the reference; the
    ensemble before and after each call (plus the batch it drew)."""
    n = ens.np
    rs = np.random.default_rng(seed)
    ens.time[:] = f32(rs.uniform(0.0, 9000.0, n))
    ens.time[:50] = 9000.0           # finished particles
    ens.time[50:100] = 8950.0        # partial final step
    ens.q[:] = f32(rs.uniform(0, 1, ens.q.shape))
    cache = cache_allocate(n)
    cache.uvwp[:] = f32(rs.standard_normal((3, n)) * 0.5)
    dt = np.zeros(n)
    work = WorkRange(0, 0, n)
    batch = lrng.batch_allocate(n)
    rstate = lrng.module_rng_init(ctl, 1)
    lrng.generate_random_nums(rstate, 5, work, 0, batch)
    clim = ingest.read_clim(ctl)
    rec = {"n": n}
    rec.update(met_arrays("m0", m0)); rec.update(met_arrays("m1", m1))
    rec.update(ens_arrays("in", ens))
    rec["in_uvwp"] = cache.uvwp.copy()
    rec["rnd_conv"] = batch.convection.copy()
    rec["rnd_turb"] = batch.diff_turb.copy()
    rec["rnd_meso"] = batch.diff_meso.copy()

    def snap(tag):
        rec.update(ens_arrays(tag, ens))
        rec[f"{tag}_uvwp"] = cache.uvwp.copy()
        rec[f"{tag}_iso"] = cache.iso_var.copy()
        rec[f"{tag}_dt"] = dt.copy()

    physics.module_timesteps(ctl, ens, 0.0, work, dt); snap("timesteps")
    physics.module_isosurf_init(ctl, ens, m0, m1, cache, work); snap("isoinit")
    physics.module_advection(ctl, ens, m0, m1, dt, work); snap("advection")
    physics.module_diffusion_turb(ctl, ens, m0, m1, dt, batch, work); snap("turb")
    physics.module_diffusion_meso(ctl, ens, m0, m1, dt, batch, cache, work); snap("meso")
    physics.module_convection(ctl, ens, dt, batch, work); snap("convection")
    physics.module_sedi(ctl, ens, m0, m1, dt, work); snap("sedi")
    # perturb p so the theta iteration has work to do
    ens.p[:] = f32(ens.p * (1.0 + 0.05 * rs.standard_normal(n)))
    ens.p[:] = np.clip(ens.p, 20.0, 1000.0); snap("preiso")
    cache.iso_nonconverged = 0
    physics.module_isosurf(ctl, ens, m0, m1, cache, work); snap("isosurf")
    rec["iso_nonconverged"] = cache.iso_nonconverged
    ens.lat[:200] = f32(rs.uniform(-300.0, 300.0, 200))   # pole reflections
    ens.lon[:400] = f32(rs.uniform(*lon_span, 400))        # wraps
    ens.lon[400:410] = [180.0, -180.0, 540.0, -540.0, 179.99998, -180.00002,
                        360.0, 0.0, -0.0, 720.0]
    ens.p[400:420] = f32(rs.uniform(0.0, 1200.0, 20)); snap("preposition")
    physics.module_position(ctl, ens, work); snap("position")
    physics.module_meteo(ctl, ens, m0, m1, clim, work); snap("meteo")
    ctl_p = copy.copy(ctl); ctl_p.isosurf_mode = "pressure"
    physics.module_isosurf_init(ctl_p, ens, m0, m1, cache, work)
    ens.p[:] = ens.p + 3.0
    physics.module_isosurf(ctl_p, ens, m0, m1, cache, work); snap("isopressure")
    return rec


STAGES = ("in", "timesteps", "isoinit", "advection", "turb", "meso", "convection", "sedi",
          "preiso", "isosurf", "preposition", "position", "meteo", "isopressure")
FIELDS = ("time", "p", "zeta", "lon", "lat", "q", "uvwp", "iso", "dt")


def dedupe_stages(rec, prefix=""):
    """Drop a stage's array when it equals the previous stage's (most modules
    change one or two fields); tests/conftest.py:golden_module_set restores
    them.  Keeps the fixtures small."""
    out = dict(rec)
    for f in FIELDS:
        prev = None
        for tag in STAGES:
            k = f"{prefix}{tag}_{f}"
            if k not in out:
                continue
            if prev is not None and np.array_equal(out[k], prev, equal_nan=True):
                cur = out.pop(k)
            else:
                cur = out[k]
            prev = cur
    return out


def gen_hires():
    """The headline grid's shape (0.25 deg, all 137 levels down to 0.01 hPa)
    on a 40 x 40 deg window (hires_met.py): every module once from
    identical inputs (module_pairs), and a 20-step advection + turbulent +
    mesoscale diffusion + position chain with the reference's counter draws
    (the production chain), 1e4 particles each."""
    sys.path.insert(0, str(OUT))
    import hires_met as hm
    lons, lats, levs = hm.axes()
    f0, f1 = hm.fields(lons, lats, levs, 0.0), hm.fields(lons, lats, levs, 5.0)
    m0 = MeteoField(t_met=0.0, lons=lons, lats=lats, levs=levs, **f0)
    m1 = MeteoField(t_met=10800.0, lons=lons, lats=lats, levs=levs, **f1)
    m0.validate(); m1.validate()
    n = 10000

    def cloud(ctl, seed):
        rs = np.random.default_rng(seed)
        ens = ensemble_allocate(ctl, n)
        ens.lon[:] = f32(rs.uniform(-180.5, -139.5, n))   # a few outside the window
        ens.lat[:] = f32(rs.uniform(-90.0, -50.5, n))
        p = rs.uniform(300.0, 900.0, n)                     # cfg3's particles
        k = n // 10
        p[:3 * k] = np.exp(rs.uniform(np.log(0.01), np.log(1013.25), 3 * k))  # every level
        p[3 * k:4 * k] = rs.choice(levs, k)                 # exact level nodes
        p[4 * k:5 * k] = rs.uniform(0.001, 1100.0, k)       # incl. beyond the hull
        ens.p[:] = f32(p)
        return ens

    ctl = modules_control()
    rec = module_pairs(ctl, m0, m1, cloud(ctl, 31), seed=32, lon_span=(-400.0, 400.0))
    rec = {f"mod_{k}": v for k, v in rec.items() if not k.startswith(("m0_", "m1_"))}
    cctl = Control(np_max=10**6, t_stop=86400.0, dt_model=180.0, met_dt=10800.0,
                   turb_dx=50.0, turb_dz=0.1, turb_meso=0.16, rng_mode="counter",
                   rng_seed_global=2211)
    ens = cloud(cctl, 33)
    init = ens_arrays("chain_init", ens)
    cache = run_chain(cctl, ens, m0, m1, None, 20, ("advection", "turb", "meso", "position"))
    np.savez_compressed(OUT / "hires.npz", lons=lons, lats=lats, levs=levs,
                        digest0=np.array(hm.fields_digest(f0)),
                        digest1=np.array(hm.fields_digest(f1)),
                        **dedupe_stages(rec, "mod_"), **init, **ens_arrays("chain_final", ens),
                        chain_final_uvwp=cache.uvwp)


def gen_deg1():
    """cfg1/cfg2's grid in full — 1 deg x 60 levels (geomspace(1013.25, 1,
    60)), global, closed by met_periodic — every module once from identical
    inputs (module_pairs), 1e4 particles."""
    sys.path.insert(0, str(OUT))
    import hires_met as hm
    lons = f32(np.arange(-180.0, 180.0, 1.0))
    lats = f32(np.linspace(-90.0, 90.0, 181))
    levs = f32(np.geomspace(1013.25, 1.0, 60))
    f0 = hm.fields(lons, lats, levs, 0.0, lon_scale=180.0)
    f1 = hm.fields(lons, lats, levs, 7.0, lon_scale=180.0)
    m0 = ingest.met_periodic(MeteoField(t_met=0.0, lons=lons, lats=lats, levs=levs, **f0))
    m1 = ingest.met_periodic(MeteoField(t_met=10800.0, lons=lons, lats=lats, levs=levs, **f1))
    ctl = modules_control()
    ens = particles(ctl, 10000, 41, lat_span=90.0)
    rs = np.random.default_rng(42)
    ens.lon[:500] = f32(rs.choice(lons, 500))            # on nodes, incl. the seam
    ens.lon[500:520] = [180.0, -180.0, 179.5, 179.99998, -179.99998] * 4
    ens.p[:1000] = f32(np.exp(rs.uniform(np.log(0.5), np.log(1100.0), 1000)))
    rec = module_pairs(ctl, m0, m1, ens, seed=43)
    rec = {f"mod_{k}": v for k, v in rec.items() if not k.startswith(("m0_", "m1_"))}
    np.savez_compressed(OUT / "deg1.npz", lons=lons, lats=lats, levs=levs,
                        digest0=np.array(hm.fields_digest(f0)),
                        digest1=np.array(hm.fields_digest(f1)), **dedupe_stages(rec, "mod_"))


def gen_rng():
    seq, s = [], 0
    for _ in range(8):
        v, s = lrng.splitmix64_next(s)
        seq.append(v)
    n = 1000
    rec = {"splitmix_seq": np.array(seq, dtype=np.uint64)}
    ctl = Control(rng_mode="counter", rng_seed_global=99, np_max=10**6)
    st = lrng.module_rng_init(ctl, 3)
    b = lrng.batch_allocate(n)
    for w in partition_all(n, 3):
        lrng.generate_random_nums(st, 7, w, w.device_id, b)
    rec.update(counter_conv=b.convection, counter_turb=b.diff_turb,
               counter_meso=b.diff_meso)
    # particles 2^24 apart alias in the reference key (rng.py:137)
    big = lrng.batch_allocate(2**24 + 8)
    lrng.generate_random_nums(st, 7, WorkRange(0, 2**24 - 4, 2**24 + 4), 0, big)
    rec["alias_conv"] = big.convection[2**24 - 4: 2**24 + 4].copy()
    ctlf = Control(rng_mode="faithful", mpi_rank=3, np_max=10**6)
    stf = lrng.module_rng_init(ctlf, 2)
    bf = lrng.batch_allocate(n)
    w0, w1 = partition_all(n, 2)
    lrng.generate_random_nums(stf, 0, w1, 1, bf)
    lrng.generate_random_nums(stf, 1, w1, 1, bf)   # second call: advanced state
    rec.update(faithful_state_in=np.uint64(lrng.rng_seed_for(3, 1)),
               faithful_state_out=np.uint64(stf.device_states[1]),
               faithful_conv=bf.convection, faithful_turb=bf.diff_turb,
               faithful_meso=bf.diff_meso, faithful_start=w1.start,
               faithful_end=w1.end)
    np.savez_compressed(OUT / "rng.npz", **rec)


def run_chain(ctl, ens, m0, m1, clim, n_steps, modules, nd=1):
    """The driver's per-device pipeline (driver_cli.py:151-183), no files."""
    cache = cache_allocate(ens.np)
    dt = np.zeros(ens.np)
    batch = lrng.batch_allocate(ens.np)
    st = lrng.module_rng_init(ctl, nd)
    ranges = partition_all(ens.np, nd)
    for w in ranges:
        physics.module_isosurf_init(ctl, ens, m0, m1, cache, w)
    t = ctl.t_start
    for step in range(n_steps):
        t_next = min(t + ctl.dt_model, ctl.t_stop)
        for w in ranges:
            physics.module_timesteps(ctl, ens, t_next, w, dt)
            lrng.generate_random_nums(st, step, w, w.device_id, batch)
            if "advection" in modules:
                physics.module_advection(ctl, ens, m0, m1, dt, w)
            if "turb" in modules:
                physics.module_diffusion_turb(ctl, ens, m0, m1, dt, batch, w)
            if "meso" in modules:
                physics.module_diffusion_meso(ctl, ens, m0, m1, dt, batch, cache, w)
            if "convection" in modules:
                physics.module_convection(ctl, ens, dt, batch, w)
            if "sedi" in modules:
                physics.module_sedi(ctl, ens, m0, m1, dt, w)
            if "isosurf" in modules:
                physics.module_isosurf(ctl, ens, m0, m1, cache, w)
            if "position" in modules:
                physics.module_position(ctl, ens, w)
            if "meteo" in modules:
                physics.module_meteo(ctl, ens, m0, m1, clim, w)
        t = t_next
    return cache


def gen_chain():
    """50-step all-physics run, counter RNG (acceptance c1 shape)."""
    lons, lats, levs = grid(10.0, 5.0, np.geomspace(1013.25, 1.0, 20))
    m0 = analytic_met(0.0, lons, lats, levs)
    m1 = analytic_met(10800.0, lons, lats, levs, phase=10.0)
    ctl = Control(np_max=10**6, t_stop=9000.0, dt_model=180.0, met_dt=10800.0,
                  turb_dx=50.0, turb_dz=0.1, turb_meso=0.16, conv_prob=0.05,
                  sedi_radius=1e-6, isosurf_mode="theta", rng_mode="counter",
                  rng_seed_global=4242)
    ens = particles(ctl, 2048, 21, lat_span=80.0)
    init = ens_arrays("init", ens)
    clim = ingest.read_clim(ctl)
    mods = ("advection", "turb", "meso", "convection", "sedi", "isosurf",
            "position", "meteo")
    cache = run_chain(ctl, ens, m0, m1, clim, 50, mods, nd=2)
    np.savez_compressed(OUT / "chain.npz", **init, **ens_arrays("final", ens),
                        final_uvwp=cache.uvwp, final_iso=cache.iso_var,
                        **met_arrays("m0", m0), **met_arrays("m1", m1))


def gen_sbr():
    """cfg1 in full: 1e5 particles, solid-body rotation on 1 deg x 60 levels,
    480 steps of advection + position (about 5 min on one core); only the
    1-D u(lat) profile is stored, and only the rows that change."""
    omega = 2.0 * np.pi / 86400.0
    lons, lats, levs = grid(1.0, 1.0, np.geomspace(1013.25, 1.0, 60))
    ulat = f32(omega * 6371000.0 * np.cos(np.deg2rad(lats)))
    shape = (lons.size, lats.size, levs.size)
    u = np.broadcast_to(ulat[None, :, None], shape).copy()
    zero = np.zeros(shape)
    mk = lambda t: ingest.met_periodic(MeteoField(t, lons, lats, levs, u, zero,
                                                  zero, np.full(shape, 250.0)))
    m0, m1 = mk(0.0), mk(86400.0)
    ctl = Control(np_max=10**6, t_stop=86400.0, dt_model=180.0)
    rs = np.random.default_rng(12616)
    n = 100_000
    ens = ensemble_allocate(ctl, n)
    ens.lon[:] = f32(rs.uniform(-180, 180, n))
    ens.lat[:] = f32(rs.uniform(-80, 80, n))
    ens.p[:] = f32(rs.uniform(300, 900, n))
    keep = ("time", "p", "lon", "lat")
    init = {f"init_{k}": getattr(ens, k).copy() for k in keep}
    run_chain(ctl, ens, m0, m1, None, 480, ("advection", "position"), nd=1)
    np.savez_compressed(OUT / "sbr.npz", **init,
                        **{f"final_{k}": getattr(ens, k).copy() for k in keep},
                        lons=lons, lats=lats, levs=levs, ulat=ulat)


def gen_output():
    """write_grid / write_ens of the reference on a seeded ensemble with
    bin-edge particles and 5 groups (one a single point)."""
    import tempfile
    from lagtrans import output
    ctl = Control(grid_nx=36, grid_ny=18, ens_group_slot=5, nq=6)
    ens = particles(ctl, 4000, 33, lat_span=90.0)
    ens.lon[:6] = [-180.0, 180.0 - 1e-9, 0.0, 10.0, -170.0, 179.99999]
    ens.lat[:6] = [-90.0, 90.0, 0.0, 10.0, 89.99999, -85.0]
    rs = np.random.default_rng(34)
    ens.q[5, :] = rs.integers(0, 4, ens.np) + 0.25
    ens.q[5, 10:20] = 7.9     # group 7: ten particles at one point
    ens.lon[10:20], ens.lat[10:20], ens.p[10:20] = 5.0, 6.0, 700.0
    with tempfile.TemporaryDirectory() as d:
        output.write_grid(ctl, ens, Path(d) / "grid.csv")
        output.write_ens(ctl, ens, Path(d) / "ens.csv")
        output.write_atm(ens, Path(d) / "atm.csv")
        atm_csv = (Path(d) / "atm.csv").read_text()
        grid_csv = (Path(d) / "grid.csv").read_text()
        ens_csv = (Path(d) / "ens.csv").read_text()
    np.savez_compressed(OUT / "output.npz", **ens_arrays("ens", ens), grid_nx=36, grid_ny=18,
                        slot=5, grid_csv=np.array(grid_csv), ens_csv=np.array(ens_csv),
                        atm_csv=np.array(atm_csv))


if __name__ == "__main__":
    which = sys.argv[1:] or ["interp", "modules", "rng", "chain", "sbr", "output", "hires", "deg1"]
    for name in which:
        globals()[f"gen_{name}"]()
        print("wrote", name)
