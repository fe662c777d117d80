"""Pin the CPU oracle: reference known-answer tests and golden vectors.

The golden vectors were produced by the reference itself
(tests/golden/make_golden.py).  Integer, index and IEEE-only results must
match bit for bit; results through libm transcendentals (cos, log, pow,
exp) are held to 1e-13 relative in case the CPU's SIMD libm differs from
the one that generated the fixtures."""

import numpy as np
import pytest

from conftest import (chain_ctl, control, golden_module_set, hires_chain_ctl, load_golden,
                      snapshot_from)
from oracle import lagtrans_oracle as orc

TRANS = dict(rtol=1e-13, atol=1e-300)


def exact(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


# ---------------------------------------------------------------- rng KATs

def test_splitmix64_reference_vector(golden_rng):
    # test_rng.py:31-51 and the published splitmix64 sequence
    state, seq = 0, []
    for _ in range(8):
        v, state = orc.splitmix64_step(state)
        seq.append(v)
    assert seq[:3] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    exact(np.array(seq, dtype=np.uint64), golden_rng["splitmix_seq"])


def test_seed_formula():
    assert [orc.seed_for(0, d) for d in range(4)] == [0, 83, 166, 249]
    assert orc.seed_for(2, 3) == 251


def test_counter_batch_matches_reference(golden_rng):
    conv, turb, meso = orc.counter_batch(99, 7, 0, 1000)
    exact(conv, golden_rng["counter_conv"])
    np.testing.assert_allclose(turb.ravel(), golden_rng["counter_turb"], **TRANS)
    np.testing.assert_allclose(meso.ravel(), golden_rng["counter_meso"], **TRANS)


def test_counter_index_alias_is_reproduced(golden_rng):
    # rng.py:137 keeps 24 bits of the particle index
    conv, _, _ = orc.counter_batch(99, 7, 2**24 - 4, 2**24 + 4)
    exact(conv, golden_rng["alias_conv"])
    assert conv[4] == orc.counter_batch(99, 7, 0, 1)[0][0]


def test_faithful_batch_matches_reference(golden_rng):
    g = golden_rng
    lo, hi = int(g["faithful_start"]), int(g["faithful_end"])
    st = int(g["faithful_state_in"])
    _, _, _, st = orc.faithful_batch(st, hi - lo)          # first call
    conv, turb, meso, st = orc.faithful_batch(st, hi - lo)  # second call
    assert st == int(g["faithful_state_out"])
    exact(conv, g["faithful_conv"][lo:hi])
    np.testing.assert_allclose(turb.ravel(), g["faithful_turb"][3 * lo:3 * hi], **TRANS)
    np.testing.assert_allclose(meso.ravel(), g["faithful_meso"][3 * lo:3 * hi], **TRANS)


# ------------------------------------------------------- interpolation

def test_locate_bit_exact(golden_interp):
    g = golden_interp
    m0 = snapshot_from(g, "m0")
    i, fx = orc.bracket(m0.lons, g["lon"])
    j, fy = orc.bracket(m0.lats, g["lat"])
    k, fz = orc.bracket(m0.levs[::-1], g["p"])
    exact(i, g["i"]); exact(j, g["j"]); exact(k, g["krev"])
    exact(fx, g["fx"]); exact(fy, g["fy"]); exact(fz, g["fz"])


def test_interpolate_bit_exact(golden_interp):
    g = golden_interp
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    out = orc.sample(m0, m1, g["t"], g["lon"], g["lat"], g["p"], ("u", "v", "w", "T"))
    exact(np.stack(out), g["uvwT"])
    same = orc.sample(m0, m0, g["t"], g["lon"], g["lat"], g["p"], ("u", "v", "w", "T"))
    exact(np.stack(same), g["uvwT_same"])


def test_interpolation_known_answers():
    # test_physics.py:13-50 restated on the oracle
    lons = np.arange(-180.0, 180.0, 30.0)
    lats = np.arange(-90.0, 90.0 + 1e-9, 10.0)
    levs = np.array([1000.0, 700.0, 500.0, 300.0, 100.0, 50.0, 10.0])
    LO, LA, LE = np.meshgrid(lons, lats, levs, indexing="ij")
    const = lambda v: np.full(LO.shape, v)
    s = orc.Snapshot(0.0, lons, lats, levs, const(10.0), const(0.0), const(0.0), LE)
    (u,) = orc.sample(s, s, 0.0, np.array([13.7]), np.array([-42.1]), np.array([333.0]), ("u",))
    assert u[0] == pytest.approx(10.0)
    (T,) = orc.sample(s, s, 0.0, np.array([0.0]), np.array([0.0]), np.array([600.0]), ("T",))
    assert T[0] == pytest.approx(600.0)
    s1 = orc.Snapshot(100.0, lons, lats, levs, const(0.0), const(0.0), const(0.0), const(300.0))
    s0 = orc.Snapshot(0.0, lons, lats, levs, const(0.0), const(0.0), const(0.0), const(200.0))
    (T,) = orc.sample(s0, s1, 25.0, np.array([0.0]), np.array([0.0]), np.array([500.0]), ("T",))
    assert T[0] == pytest.approx(225.0)


# ------------------------------------------------------- module stages

def _state(g, tag):
    return {k: g[f"{tag}_{k}"].copy() for k in ("time", "p", "lon", "lat", "q", "uvwp", "iso", "dt")
            if f"{tag}_{k}" in g}


@pytest.fixture(scope="module", params=["modules", "hires", "deg1"])
def mods(request):
    """Every stage on the 10 x 5 deg x 20 fixture and on the headline
    0.25 deg x 137-level window (levels down to 0.01 hPa)."""
    return golden_module_set(request.param)


def test_stage_timesteps(mods):
    g, ctl, m0, m1 = mods
    exact(orc.timestep_lengths(ctl, g["isoinit_time"]), g["timesteps_dt"])


def test_stage_isosurf_init(mods):
    g, ctl, m0, m1 = mods
    iso = orc.isosurface_value(ctl, m0, m1, g["timesteps_lon"], g["timesteps_lat"],
                               g["timesteps_p"], g["timesteps_time"], g["timesteps_iso"])
    np.testing.assert_allclose(iso, g["isoinit_iso"], **TRANS)


def test_stage_advection(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "isoinit")
    lon, lat, p, t = orc.advect(m0, m1, s["dt"], s["lon"], s["lat"], s["p"], s["time"])
    np.testing.assert_allclose(lon, g["advection_lon"], **TRANS)
    np.testing.assert_allclose(lat, g["advection_lat"], **TRANS)
    np.testing.assert_allclose(p, g["advection_p"], **TRANS)
    exact(t, g["advection_time"])


def test_stage_turb(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "advection")
    xi = g["rnd_turb"].reshape(-1, 3)
    lon, lat, p = orc.turbulent_hop(ctl, m0, m1, s["dt"], xi, s["lon"], s["lat"], s["p"], s["time"])
    np.testing.assert_allclose(lon, g["turb_lon"], **TRANS)
    np.testing.assert_allclose(lat, g["turb_lat"], **TRANS)
    np.testing.assert_allclose(p, g["turb_p"], **TRANS)


def test_stage_meso(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "turb")
    xi = g["rnd_meso"].reshape(-1, 3)
    lon, lat, p, uvwp = orc.mesoscale_hop(ctl, m0, s["dt"], xi, s["uvwp"], s["lon"], s["lat"], s["p"])
    exact(uvwp, g["meso_uvwp"])   # pairwise std + IEEE ops: bit exact
    np.testing.assert_allclose(lon, g["meso_lon"], **TRANS)
    exact(lat, g["meso_lat"]); exact(p, g["meso_p"])


def test_stage_convection(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "meso")
    exact(orc.convective_mix(ctl, s["dt"], g["rnd_conv"], s["p"]), g["convection_p"])


def test_stage_sedi(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "convection")
    p = orc.settle(ctl, m0, m1, s["dt"], s["lon"], s["lat"], s["p"], s["time"])
    np.testing.assert_allclose(p, g["sedi_p"], **TRANS)


def test_stage_isosurf_theta(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "preiso")
    p, bad = orc.isosurface_pull(ctl, m0, m1, s["lon"], s["lat"], s["p"], s["time"], s["iso"])
    np.testing.assert_allclose(p, g["isosurf_p"], **TRANS)
    assert bad == int(g["iso_nonconverged"])


def test_stage_position(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "preposition")
    lon, lat, p = orc.fold_position(ctl, s["lon"], s["lat"], s["p"])
    exact(lon, g["position_lon"]); exact(lat, g["position_lat"]); exact(p, g["position_p"])


def test_stage_meteo(mods):
    g, ctl, m0, m1 = mods
    s = _state(g, "position")
    q = orc.sample_along(m0, m1, orc.climatology_tables(), s["lon"], s["lat"], s["p"], s["time"])
    for slot in range(5):
        np.testing.assert_allclose(q[slot], g["meteo_q"][slot], **TRANS)


def test_stage_isosurf_pressure(mods):
    g, ctl, m0, m1 = mods
    c = control(isosurf_mode="pressure")
    iso = orc.isosurface_value(c, m0, m1, g["meteo_lon"], g["meteo_lat"], g["meteo_p"],
                               g["meteo_time"], g["meteo_iso"])
    p, _ = orc.isosurface_pull(c, m0, m1, g["meteo_lon"], g["meteo_lat"], g["meteo_p"] + 3.0,
                               g["meteo_time"], iso)
    exact(p, g["isopressure_p"])


# ------------------------------------------------------- whole runs

def _run_chain(ctl, g, m0, m1, steps, modules, parts):
    st = {k: g[f"init_{k}"].astype(np.float64).copy() for k in ("time", "p", "lon", "lat", "q")}
    n = st["p"].shape[0]
    st["uvwp"] = np.zeros((3, n))
    st["iso_var"] = np.zeros(n)
    ranges = [orc.split_range(n, parts, d) for d in range(parts)]
    for lo, hi in ranges:
        sl = slice(lo, hi)
        st["iso_var"][sl] = orc.isosurface_value(ctl, m0, m1, st["lon"][sl], st["lat"][sl],
                                                 st["p"][sl], st["time"][sl], st["iso_var"][sl])
    clim = orc.climatology_tables()
    for step in range(steps):
        for lo, hi in ranges:
            orc.full_step(ctl, m0, m1, st, lo, hi, step, clim=clim, modules=modules)
    return st


def test_chain_50_steps_all_physics(golden_chain):
    g = golden_chain
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    st = _run_chain(chain_ctl(), g, m0, m1, 50,
                    ("advection", "turb", "meso", "convection", "sedi", "isosurf",
                     "position", "meteo"), parts=3)
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(st[k], g[f"final_{k}"], rtol=1e-11, atol=1e-9)
    exact(st["time"], g["final_time"])


def test_hires_chain_20_steps(golden_hires):
    """The production chain (advection + turbulent + mesoscale diffusion +
    position, counter draws) for 20 steps on the 0.25 deg x 137 window."""
    g, (m0, m1) = golden_hires
    st = _run_chain(hires_chain_ctl(), {k[6:]: v for k, v in g.items() if k.startswith("chain_")},
                    m0, m1, 20, ("advection", "turb", "meso", "position"), parts=2)
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(st[k], g[f"chain_final_{k}"], rtol=1e-11, atol=1e-9)
    exact(st["time"], g["chain_final_time"])
    np.testing.assert_allclose(st["uvwp"], g["chain_final_uvwp"], rtol=1e-11, atol=1e-12)


def test_sbr_cfg1_shape(golden_sbr):
    """The first 5000 of the fixture's 1e5 cfg1 particles (particles are
    independent, so a subsample of the reference's full run pins the oracle
    within seconds)."""
    g = {k: (v[:5000] if k.startswith(("init_", "final_")) else v) for k, v in golden_sbr.items()}
    lons, lats, levs = g["lons"], g["lats"], g["levs"]
    shape = (lons.size, lats.size, levs.size)
    u = np.broadcast_to(g["ulat"][None, :, None], shape).copy()
    z = np.zeros(shape)
    mk = lambda t: orc.close_longitudes(orc.Snapshot(t, lons, lats, levs, u, z, z, np.full(shape, 250.0)))
    m0, m1 = mk(0.0), mk(86400.0)
    ctl = control(t_stop=86400.0, dt_model=180.0)
    g["init_q"] = np.zeros((5, 5000))
    st = _run_chain(ctl, g, m0, m1, 480, ("advection", "position"), parts=1)
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_allclose(st[k], g[f"final_{k}"], rtol=1e-12, atol=1e-9)


def test_partition_rule():
    assert [orc.split_range(100, 4, d) for d in range(4)] == [(0, 25), (25, 50), (50, 75), (75, 100)]
    assert [orc.split_range(10, 3, d) for d in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert orc.split_range(3, 4, 3) == (3, 3)
    with pytest.raises(ValueError):
        orc.split_range(10, 2, 2)


# ------------------------------------------------------------ output statistics

def _csv_rows(text):
    return [line.split(",") for line in str(text).splitlines()[1:]]


def test_bin_counts_match_reference_write_grid():
    g = load_golden("output")
    counts = orc.bin_counts(g["ens_lon"], g["ens_lat"], int(g["grid_nx"]), int(g["grid_ny"]))
    ref = np.array([int(r[2]) for r in _csv_rows(g["grid_csv"])]).reshape(counts.shape)
    np.testing.assert_array_equal(counts, ref)
    assert counts.sum() == g["ens_lon"].size


def test_grouped_moments_match_reference_write_ens():
    g = load_golden("output")
    gids, cnts, means, stds = orc.grouped_moments(g["ens_q"][int(g["slot"])], g["ens_lon"],
                                                  g["ens_lat"], g["ens_p"])
    rows = _csv_rows(g["ens_csv"])
    assert [int(r[0]) for r in rows] == list(gids)
    assert [int(r[1]) for r in rows] == list(cnts)
    ref = np.array([[float(x) for x in r[2:]] for r in rows])   # lon_mean, lon_std, lat_mean ...
    np.testing.assert_array_equal(ref[:, 0::2].T, means)
    np.testing.assert_array_equal(ref[:, 1::2].T, stds)
    with pytest.raises(ValueError):
        orc.grouped_moments(np.array([1.0, -1.0]), *np.zeros((3, 2)))
