"""GPU parity: the drop-in module API (liblagtrans_b200 kernels) against the
golden vectors made by the reference and against the oracle.

Tolerance contract: cell indices, uint64 RNG words,
uniforms and every result built only from + - * / sqrt are bit-exact
(the library is compiled with -fmad=false and keeps numpy's operation
order); results that pass through cos/log/pow/exp (libdevice vs numpy's
SIMD libm, ~1 ulp apart) are held to 1e-12 relative per call."""

import numpy as np
import pytest

from conftest import chain_ctl, control, golden_module_set, snapshot_from
from oracle import lagtrans_oracle as orc

pytestmark = pytest.mark.gpu

ULP = dict(rtol=1e-12, atol=1e-12)


@pytest.fixture(scope="module")
def b200():
    import paper_2211_12616_b200.physics as phys
    import paper_2211_12616_b200.rng as rng
    from paper_2211_12616_b200 import model_state as ms
    return phys, rng, ms


def exact(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


def host_ensemble(ms, g, tag, nq=5):
    ens = ms.ParticleEnsemble(np=g[f"{tag}_p"].size, time=g[f"{tag}_time"].copy(),
                              p=g[f"{tag}_p"].copy(), zeta=g[f"{tag}_zeta"].copy(),
                              lon=g[f"{tag}_lon"].copy(), lat=g[f"{tag}_lat"].copy(),
                              q=g[f"{tag}_q"].copy())
    return ens


def cache_from(ms, g, tag):
    return ms.CacheState(uvwp=g[f"{tag}_uvwp"].copy(), iso_var=g[f"{tag}_iso"].copy())


# ------------------------------------------------------------ interpolation

def test_interpolate_met_bit_exact(b200, golden_interp):
    phys, _, _ = b200
    g = golden_interp
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    out = phys.interpolate_met(m0, m1, g["t"], g["lon"], g["lat"], g["p"])
    exact(np.stack(out), g["uvwT"])
    same = phys.interpolate_met(m0, m0, g["t"], g["lon"], g["lat"], g["p"])
    exact(np.stack(same), g["uvwT_same"])


def test_interpolate_met_f64_store(b200, golden_interp):
    """f64 met store on non-fp32 values (reference conftest.make_met style)."""
    phys, _, _ = b200
    from paper_2211_12616_b200.physics import default_context
    g = golden_interp
    m0 = snapshot_from(g, "m0")
    m0.u = m0.u + 1e-9 * np.arange(m0.u.size).reshape(m0.u.shape)  # not fp32-representable
    ctx = default_context()
    old = ctx.met_precision
    try:
        ctx.met_precision = "f64"
        ctx._grid_key = None
        (u,) = phys.interpolate_met(m0, m0, 0.0, g["lon"], g["lat"], g["p"], fields=("u",))
    finally:
        ctx.met_precision = old
        ctx._grid_key = None
    (ref,) = orc.sample(m0, m0, 0.0, g["lon"], g["lat"], g["p"], ("u",))
    exact(u, ref)


# ------------------------------------------------------------ module stages

@pytest.fixture(scope="module", params=["modules", "hires", "deg1"])
def mods(request):
    """Every module on the 10 x 5 deg x 20 fixture and on the headline
    0.25 deg x 137-level window (hires.npz, levels down to 0.01 hPa)."""
    return golden_module_set(request.param)


def _batch(rng, g):
    b = rng.batch_allocate(int(g["n"]))
    b.convection[:] = g["rnd_conv"]
    b.diff_turb[:] = g["rnd_turb"]
    b.diff_meso[:] = g["rnd_meso"]
    return b


def _work(g):
    from paper_2211_12616_b200.partition import WorkRange
    return WorkRange(0, 0, int(g["n"]))


def test_module_timesteps(b200, mods):
    phys, _, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "isoinit")
    dt = np.zeros(ens.np)
    phys.module_timesteps(ctl, ens, 0.0, _work(g), dt)
    exact(dt, g["timesteps_dt"])


def test_module_isosurf_init(b200, mods):
    phys, _, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "timesteps")
    cache = cache_from(ms, g, "timesteps")
    phys.module_isosurf_init(ctl, ens, m0, m1, cache, _work(g))
    np.testing.assert_allclose(cache.iso_var, g["isoinit_iso"], **ULP)


def test_module_advection(b200, mods):
    phys, _, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "isoinit")
    phys.module_advection(ctl, ens, m0, m1, g["isoinit_dt"].copy(), _work(g))
    # the longitude hop divides by cos(lat): within ~0.1 deg of a pole numpy's
    # cos(fl(lat * pi/180)) carries the argument's rounding, ulp(pi/2) /
    # cos(lat) relative (~1e-12 at 89.99 deg), which the hop passes on; the
    # kernels' cos(pi * lat/180) is within 1 ulp of the exact cosine there
    polar = np.abs(g["isoinit_lat"]) > 89.9
    np.testing.assert_allclose(ens.lon[~polar], g["advection_lon"][~polar], **ULP)
    np.testing.assert_allclose(ens.lon[polar], g["advection_lon"][polar], rtol=1e-9, atol=1e-9)
    for k in ("lat", "p"):
        np.testing.assert_allclose(getattr(ens, k), g[f"advection_{k}"], **ULP)
    exact(ens.time, g["advection_time"])
    # lat/p only see cos through the midpoint longitude: almost all bit-exact
    assert np.mean(ens.lat == g["advection_lat"]) > 0.9


def test_module_turb(b200, mods):
    phys, rng, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "advection")
    phys.module_diffusion_turb(ctl, ens, m0, m1, g["advection_dt"].copy(), _batch(rng, g), _work(g))
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(getattr(ens, k), g[f"turb_{k}"], **ULP)
    exact(ens.lat, g["turb_lat"])


def test_module_meso(b200, mods):
    phys, rng, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "turb")
    cache = cache_from(ms, g, "turb")
    phys.module_diffusion_meso(ctl, ens, m0, m1, g["turb_dt"].copy(), _batch(rng, g), cache, _work(g))
    exact(cache.uvwp, g["meso_uvwp"])
    exact(ens.lat, g["meso_lat"])
    exact(ens.p, g["meso_p"])
    np.testing.assert_allclose(ens.lon, g["meso_lon"], **ULP)


def test_module_convection(b200, mods):
    phys, rng, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "meso")
    phys.module_convection(ctl, ens, g["meso_dt"].copy(), _batch(rng, g), _work(g))
    exact(ens.p, g["convection_p"])


def test_module_sedi(b200, mods):
    phys, _, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "convection")
    phys.module_sedi(ctl, ens, m0, m1, g["convection_dt"].copy(), _work(g))
    exact(ens.p, g["sedi_p"])


def test_module_isosurf_theta(b200, mods):
    phys, _, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "preiso")
    cache = cache_from(ms, g, "preiso")
    cache.iso_nonconverged = 0
    phys.module_isosurf(ctl, ens, m0, m1, cache, _work(g))
    np.testing.assert_allclose(ens.p, g["isosurf_p"], rtol=1e-10, atol=1e-10)
    assert cache.iso_nonconverged == int(g["iso_nonconverged"])


def test_module_position(b200, mods):
    phys, _, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "preposition")
    phys.module_position(ctl, ens, _work(g))
    exact(ens.lon, g["position_lon"])
    exact(ens.lat, g["position_lat"])
    exact(ens.p, g["position_p"])


def test_module_meteo(b200, mods):
    phys, _, ms = b200
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "position")
    phys.module_meteo(ctl, ens, m0, m1, ms.read_clim(ctl), _work(g))
    np.testing.assert_allclose(ens.q[:5], g["meteo_q"][:5], **ULP)
    exact(ens.q[4], g["meteo_q"][4])


def test_module_isosurf_pressure(b200, mods):
    phys, _, ms = b200
    g, _, m0, m1 = mods
    ctl = control(isosurf_mode="pressure")
    ens = host_ensemble(ms, g, "meteo")
    cache = cache_from(ms, g, "meteo")
    phys.module_isosurf_init(ctl, ens, m0, m1, cache, _work(g))
    ens.p[:] = ens.p + 3.0
    phys.module_isosurf(ctl, ens, m0, m1, cache, _work(g))
    exact(ens.p, g["isopressure_p"])


def test_range_purity_and_subrange(b200, mods):
    """physics.py:1-7: a module on [a, b) leaves every byte outside unchanged
    and equals the whole-range result inside."""
    phys, rng, ms = b200
    from paper_2211_12616_b200.partition import WorkRange
    g, ctl, m0, m1 = mods
    ens = host_ensemble(ms, g, "isoinit")
    before = ens.lon.copy(), ens.lat.copy(), ens.p.copy(), ens.time.copy()
    dt = g["isoinit_dt"].copy()
    phys.module_advection(ctl, ens, m0, m1, dt, WorkRange(0, 700, 1900))
    out = np.r_[0:700, 1900:ens.np]
    for a, b in zip((ens.lon, ens.lat, ens.p, ens.time), before):
        exact(a[out], b[out])
    whole = host_ensemble(ms, g, "isoinit")
    phys.module_advection(ctl, whole, m0, m1, dt, _work(g))
    exact(ens.lon[700:1900], whole.lon[700:1900])
    exact(ens.p[700:1900], whole.p[700:1900])


# ------------------------------------------------------------ random numbers

def test_counter_batch(b200, golden_rng):
    _, rng, ms = b200
    from paper_2211_12616_b200.partition import partition_all
    g = golden_rng
    ctl = ms.Control(rng_mode="counter", rng_seed_global=99)
    st = rng.module_rng_init(ctl, 3)
    b = rng.batch_allocate(1000)
    for w in partition_all(1000, 3):
        rng.generate_random_nums(st, 7, w, w.device_id, b)
    exact(b.convection, g["counter_conv"])
    np.testing.assert_allclose(b.diff_turb, g["counter_turb"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(b.diff_meso, g["counter_meso"], rtol=1e-13, atol=1e-13)


def test_faithful_batch(b200, golden_rng):
    _, rng, ms = b200
    from paper_2211_12616_b200.partition import partition_all
    g = golden_rng
    ctl = ms.Control(rng_mode="faithful", mpi_rank=3)
    st = rng.module_rng_init(ctl, 2)
    b = rng.batch_allocate(1000)
    w0, w1 = partition_all(1000, 2)
    rng.generate_random_nums(st, 0, w1, 1, b)
    rng.generate_random_nums(st, 1, w1, 1, b)
    assert st.device_states[1] == int(g["faithful_state_out"])
    lo, hi = int(g["faithful_start"]), int(g["faithful_end"])
    exact(b.convection[lo:hi], g["faithful_conv"][lo:hi])
    np.testing.assert_allclose(b.diff_turb, g["faithful_turb"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(b.diff_meso, g["faithful_meso"], rtol=1e-13, atol=1e-13)


def test_philox_moments(b200):
    """Fast mode matches distributionally (test_rng.py:157-165 bounds)."""
    _, rng, ms = b200
    from paper_2211_12616_b200.partition import WorkRange
    n = 10 ** 6
    st = rng.RngState("philox", 5)
    b = rng.batch_allocate(n)
    rng.generate_random_nums(st, 0, WorkRange(0, 0, n), 0, b)
    assert abs(b.convection.mean() - 0.5) < 0.002
    assert b.convection.min() >= 0.0 and b.convection.max() < 1.0
    for arr in (b.diff_turb, b.diff_meso):
        assert abs(arr.mean()) < 0.004
        assert abs(arr.var() - 1.0) < 0.01


# ------------------------------------------------------------ whole chains

def _module_chain(phys, rng, ms, ctl, g, m0, m1, steps, parts):
    from paper_2211_12616_b200.partition import partition_all
    ens = host_ensemble(ms, g, "init")
    n = ens.np
    cache = ms.cache_allocate(n)
    dt = np.zeros(n)
    batch = rng.batch_allocate(n)
    clim = ms.read_clim(ctl)
    st = rng.module_rng_init(ctl, parts)
    ranges = partition_all(n, parts)
    for w in ranges:
        phys.module_isosurf_init(ctl, ens, m0, m1, cache, w)
    for step in range(steps):
        for w in ranges:
            phys.module_timesteps(ctl, ens, 0.0, w, dt)
            rng.generate_random_nums(st, step, w, w.device_id, batch)
            phys.module_advection(ctl, ens, m0, m1, dt, w)
            phys.module_diffusion_turb(ctl, ens, m0, m1, dt, batch, w)
            phys.module_diffusion_meso(ctl, ens, m0, m1, dt, batch, cache, w)
            phys.module_convection(ctl, ens, dt, batch, w)
            phys.module_sedi(ctl, ens, m0, m1, dt, w)
            phys.module_isosurf(ctl, ens, m0, m1, cache, w)
            phys.module_position(ctl, ens, w)
            phys.module_meteo(ctl, ens, m0, m1, clim, w)
    return ens, cache


def test_chain_50_steps_module_api(b200, golden_chain):
    phys, rng, ms = b200
    g = golden_chain
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    ens, cache = _module_chain(phys, rng, ms, chain_ctl(), g, m0, m1, 50, parts=2)
    exact(ens.time, g["final_time"])
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(getattr(ens, k), g[f"final_{k}"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(ens.q, g["final_q"], rtol=1e-9, atol=1e-9)


def test_interpolate_irregular_axes_bit_exact(b200):
    """Irregular lon/lat axes (random, jittered; not fp32-representable lat
    nodes) with particles on the nodes: cell indices and values bit-exact."""
    phys, _, ms = b200
    rs = np.random.default_rng(17)
    lons = np.sort(rs.uniform(-180, 180, 40)).astype(np.float32).astype(np.float64)
    lats = np.linspace(-90, 90, 31)
    lats[1:-1] += rs.uniform(-1.5, 1.5, 29)
    levs = np.geomspace(1000.0, 5.0, 12).astype(np.float32).astype(np.float64)
    shape = (lons.size, lats.size, levs.size)
    f = lambda: rs.uniform(-20, 20, shape).astype(np.float32).astype(np.float64)
    m0 = ms.MeteoField(0.0, lons, lats, levs, f(), f(), f(), rs.uniform(200, 300, shape).astype(
        np.float32).astype(np.float64))
    m1 = ms.MeteoField(3600.0, lons, lats, levs, f(), f(), f(),
                       (m0.T + 1.0).astype(np.float32).astype(np.float64))
    n = 20000
    lon = rs.uniform(-200, 200, n)
    lat = rs.uniform(-95, 95, n)
    p = rs.uniform(1, 1100, n)
    lon[:40] = lons          # on nodes: searchsorted-left edge cases
    lat[:31] = lats
    p[:12] = levs
    t = rs.uniform(-100, 4000, n)
    got = np.stack(phys.interpolate_met(m0, m1, t, lon, lat, p))
    ref = np.stack(orc.sample(orc.Snapshot.like(m0), orc.Snapshot.like(m1), t, lon, lat, p,
                              ("u", "v", "w", "T")))
    exact(got, ref)


def test_rng_fill_unaffected_by_earlier_id_layouts(b200):
    """The scratch context may carry an id row from an earlier call
    (statistics, sorts); the host-path fill still keys draws by global index."""
    phys, rng, ms = b200
    from paper_2211_12616_b200 import output
    from paper_2211_12616_b200.partition import WorkRange
    ens = ms.ParticleEnsemble(50, np.zeros(50), np.full(50, 500.0), np.zeros(50),
                              np.zeros(50), np.zeros(50), np.zeros((6, 50)))
    output.group_stats(ms.Control(ens_group_slot=5, nq=6), ens, work=WorkRange(0, 10, 40))
    r = rng.module_rng_init(ms.Control(rng_mode="counter", rng_seed_global=77), 1)
    b = rng.batch_allocate(1000)
    rng.generate_random_nums(r, 3, WorkRange(0, 100, 900), 0, b)
    conv, turb, meso = orc.counter_batch(77, 3, 100, 900)
    exact(b.convection[100:900], conv)
    np.testing.assert_allclose(b.diff_turb.reshape(-1, 3)[100:900], turb, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(b.diff_meso.reshape(-1, 3)[100:900], meso, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------ generator KATs

# Random123 kat_vectors, philox4x32 10: (ctr[4], key[2]) -> out[4]
PHILOX_KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff), (0xffffffff, 0xffffffff),
     (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


def test_philox_device_known_answers(b200):
    """The in-kernel Philox4x32-10 block function, run on the device through
    lt_philox4x32_10, reproduces Random123's known-answer vectors."""
    import ctypes as C
    from paper_2211_12616_b200 import _capi as capi
    from paper_2211_12616_b200.physics import default_context
    ctx = default_context()
    ctr = np.array([v[0] for v in PHILOX_KAT], dtype=np.uint32)
    key = np.array([v[1] for v in PHILOX_KAT], dtype=np.uint32)
    out = np.zeros((len(PHILOX_KAT), 4), dtype=np.uint32)
    capi.check(ctx.lib.lt_philox4x32_10(ctx.h, len(PHILOX_KAT), capi.ptr(ctr), capi.ptr(key),
                                        capi.ptr(out)))
    exact(out, np.array([v[2] for v in PHILOX_KAT], dtype=np.uint32))


def test_philox_draws_follow_the_kat_words(b200):
    """Seed 0, step 0, particle 0 is Philox block (0, 0, 0, 0) under key
    (0, 0) — KAT vector 1 — so the batch's convection uniform is the 53-bit
    uniform of its first two words and the first turbulent normal the
    Box-Muller transform of words 3 and 4 (lt_device.cuh philox_draws)."""
    _, rng, _ = b200
    from paper_2211_12616_b200.partition import WorkRange
    w = PHILOX_KAT[0][2]
    b = rng.batch_allocate(4)
    rng.generate_random_nums(rng.RngState("philox", 0), 0, WorkRange(0, 0, 4), 0, b)
    conv = ((w[0] >> 5) * 67108864.0 + (w[1] >> 6)) / 9007199254740992.0
    assert b.convection[0] == conv
    u1 = (w[2] + 0.5) * 2.3283064365386963e-10
    u2 = (w[3] + 0.5) * 2.3283064365386963e-10
    z0 = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    np.testing.assert_allclose(b.diff_turb[0], z0, rtol=1e-13, atol=1e-15)


# ------------------------------------------------------------ met packing

@pytest.mark.parametrize("path", ["fields", "nodes"])
def test_close_lon_packing_on_device(b200, path):
    """LT_MET_CLOSE_LON (met_periodic, ingest.py:195-207, done by the
    packing kernel instead of on the host): a global snapshot WITHOUT its
    +360 column, loaded with the flag into a closed grid, interpolates bit
    for bit like the host-closed snapshot — for lt_met_load (separate
    fields) and lt_met_load_nodes (interleaved float32 nodes, the streaming
    path of cfg4)."""
    _, _, ms = b200
    from paper_2211_12616_b200 import synthetic as syn
    from paper_2211_12616_b200.context import DeviceContext
    lons, lats, levs = syn.grid(5.0, 5.0, 24)
    f = syn.era5_like(lons, lats, levs, 13.0)                    # nx columns, open
    closed = syn.snapshot(600.0, lons, lats, levs, f, periodic=True)
    assert closed.lons.size == lons.size + 1
    ref, got = DeviceContext(0), DeviceContext(0)
    for c in (ref, got):
        c.set_grid(closed.lons, closed.lats, closed.levs)
    ref.load_met(0, closed)
    if path == "fields":
        open_met = ms.MeteoField(600.0, lons, lats, levs, f["u"], f["v"], f["w"], f["T"])
        got.load_met(0, open_met, close_lon=True)
    else:
        nodes = np.stack([f["u"], f["v"], f["w"], f["T"]], axis=-1).astype(np.float32)
        got.load_met_nodes(0, 600.0, np.ascontiguousarray(nodes), close_lon=True)
    ref.use_met(0, 0)
    got.use_met(0, 0)
    rs = np.random.default_rng(3)
    n = 20000
    lon = rs.uniform(-181.0, 181.0, n)
    lon[:200] = rs.uniform(175.0, 180.0, 200)                   # inside the closing column
    lat, p = rs.uniform(-90, 90, n), rs.uniform(0.5, 1100, n)
    exact(got.interpolate(600.0, lon, lat, p), ref.interpolate(600.0, lon, lat, p))
    ref.close()
    got.close()


def test_exact_transcendentals_against_numpy(b200):
    """The exact kernels' own fp64 log and sin/cos(pi y) (lt_device.cuh
    lt_log / lt_sincospi2) behind the Box-Muller draws: 1e6 particles of
    counter-mode draws (6e6 normals through log, sqrt and cos) and 2e5 of
    faithful draws against the oracle's numpy evaluation, within the
    contract's 1e-13 relative for values through transcendentals — and
    1e-14 absolute where cos(2 pi u) crosses zero: numpy rounds the argument
    2 pi u first, the kernels reduce u exactly (cos_lat's note), so near a
    zero of the cosine the two differ by ~1e-15 absolute."""
    _, rng, ms = b200
    from paper_2211_12616_b200.partition import WorkRange
    n = 1_000_000
    st = rng.module_rng_init(ms.Control(rng_mode="counter", rng_seed_global=2211), 1)
    b = rng.batch_allocate(n)
    rng.generate_random_nums(st, 17, WorkRange(0, 0, n), 0, b)
    conv, turb, meso = orc.counter_batch(2211, 17, 0, n)
    exact(b.convection, conv)
    np.testing.assert_allclose(b.diff_turb, turb.ravel(), rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(b.diff_meso, meso.ravel(), rtol=1e-13, atol=1e-14)
    m = 200_000
    stf = rng.module_rng_init(ms.Control(rng_mode="faithful", mpi_rank=5), 1)
    s0 = stf.device_states[0]
    bf = rng.batch_allocate(m)
    rng.generate_random_nums(stf, 0, WorkRange(0, 0, m), 0, bf)
    fconv, fturb, fmeso, _ = orc.faithful_batch(s0, m)
    exact(bf.convection, fconv)
    np.testing.assert_allclose(bf.diff_turb, fturb.ravel(), rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(bf.diff_meso, fmeso.ravel(), rtol=1e-13, atol=1e-14)
