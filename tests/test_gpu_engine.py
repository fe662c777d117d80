"""GPU: the fused device-resident engine (one launch per step, in-kernel
random draws, box sort, met rotation) against the reference's golden runs,
the oracle and the module-by-module path."""

import numpy as np
import pytest

from conftest import chain_ctl, control, snapshot_from
from oracle import lagtrans_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_2211_12616_b200 import engine, model_state, synthetic
    return engine, model_state, synthetic


def _ens(ms, g, tag):
    return ms.ParticleEnsemble(np=g[f"{tag}_p"].size, time=g[f"{tag}_time"].copy(),
                               p=g[f"{tag}_p"].copy(), zeta=g[f"{tag}_zeta"].copy(),
                               lon=g[f"{tag}_lon"].copy(), lat=g[f"{tag}_lat"].copy(),
                               q=g[f"{tag}_q"].copy())


def _run_chain(engine, ms, g, ctl, steps, shards=1, sort_every=0):
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    from paper_2211_12616_b200.partition import partition_all
    ens = _ens(ms, g, "init")
    cache = ms.cache_allocate(ens.np)
    mask = engine.FULL
    for w in partition_all(ens.np, shards):
        e = engine.Engine(device=0, first_id=w.start)
        e.upload(ens, start=w.start, end=w.end)
        e.bind_met(m0, m1)
        e.load_clim(ms.read_clim(ctl))
        e.init_isosurf(ctl)
        for step in range(steps):
            if sort_every and step % sort_every == 0:
                e.sort()
            e.step(ctl, step, mask, device_id=w.device_id)
        e.download(ens, cache, start=w.start)
        e.close()
    return ens, cache


def test_fused_chain_matches_reference_golden(eng, golden_chain):
    engine, ms, _ = eng
    g = golden_chain
    ens, cache = _run_chain(engine, ms, g, chain_ctl(), 50, shards=2)
    np.testing.assert_array_equal(ens.time, g["final_time"])
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(getattr(ens, k), g[f"final_{k}"], rtol=1e-9, atol=1e-9)


def test_fused_equals_module_by_module_bitwise(eng, golden_chain):
    """Counter mode: in-kernel draws == generate_random_nums batch, so the
    fused launch reproduces the eight-module pipeline bit for bit."""
    engine, ms, _ = eng
    from test_gpu_parity import _module_chain
    import paper_2211_12616_b200.physics as phys
    import paper_2211_12616_b200.rng as rng
    g = golden_chain
    ctl = chain_ctl()
    fused, _ = _run_chain(engine, ms, g, ctl, 12, shards=1)
    mod, _ = _module_chain(phys, rng, ms, ctl, g, snapshot_from(g, "m0"),
                           snapshot_from(g, "m1"), 12, parts=1)
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_array_equal(getattr(fused, k), getattr(mod, k))


def test_shard_count_invariance(eng, golden_chain):
    """Acceptance c1 on the GPU engine: 1, 2, 3 shards are byte-identical."""
    engine, ms, _ = eng
    g = golden_chain
    ref, _ = _run_chain(engine, ms, g, chain_ctl(), 20, shards=1)
    for shards in (2, 3):
        got, _ = _run_chain(engine, ms, g, chain_ctl(), 20, shards=shards)
        for k in ("lon", "lat", "p", "time"):
            np.testing.assert_array_equal(getattr(got, k), getattr(ref, k))


def test_sort_never_changes_results(eng, golden_chain):
    engine, ms, _ = eng
    g = golden_chain
    ref, rc = _run_chain(engine, ms, g, chain_ctl(), 20, shards=1)
    got, gc = _run_chain(engine, ms, g, chain_ctl(), 20, shards=1, sort_every=3)
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_array_equal(getattr(got, k), getattr(ref, k))
    np.testing.assert_array_equal(got.q, ref.q)
    np.testing.assert_array_equal(gc.uvwp, rc.uvwp)


def test_sort_permutation_is_stable_argsort_of_oracle_keys(eng):
    engine, ms, syn = eng
    m0, m1 = syn.analytic_pair(dlon=5.0, dlat=5.0, nlev=30, t0=0.0, t1=3600.0)
    ens = syn.particles(50000, seed=9)
    ens.lon[:1000] = ens.lon[0]   # ties: stability matters
    ens.lat[:1000] = ens.lat[0]
    ens.p[:1000] = ens.p[0]
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(m0, m1)
    e.sort()
    ids = e.ctx.ids(0, ens.np)
    keys = orc.box_keys(orc.Snapshot.like(m0), ens.lon, ens.lat, ens.p)
    np.testing.assert_array_equal(ids, np.argsort(keys, kind="stable").astype(np.uint32))
    e.close()


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_sbr_cfg1_whole_run(eng, golden_sbr, precision):
    """cfg1 in full (1e5 particles, 1 deg x 60 SBR, 480 steps of advection)
    against the reference's own run: exact kernels one launch per step to
    1e-9, the fast kernels in multi-step launches within the north star's
    1e-5 run tolerance (span-normalised lon/lat, relative p)."""
    engine, ms, syn = eng
    g = golden_sbr
    m0, m1 = syn.solid_body_pair(1.0, 1.0, 60)
    np.testing.assert_array_equal(m0.lons[:-1], g["lons"])
    ctl = ms.Control(t_stop=86400.0, dt_model=180.0, precision=precision)
    n = g["init_p"].size
    assert n == 100_000
    ens = ms.ParticleEnsemble(n, g["init_time"].copy(), g["init_p"].copy(), np.zeros(n),
                              g["init_lon"].copy(), g["init_lat"].copy(), np.zeros((5, n)))
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(m0, m1)
    if precision == "exact":
        for step in range(480):
            e.step(ctl, step, engine.ADV)
    else:
        for step in range(0, 480, 60):
            e.step_many(ctl, step, 60, engine.ADV)
    e.download(ens)
    e.close()
    np.testing.assert_array_equal(ens.time, g["final_time"])
    if precision == "exact":
        for k in ("lon", "lat", "p"):
            np.testing.assert_allclose(getattr(ens, k), g[f"final_{k}"], rtol=1e-9, atol=1e-9)
    else:
        dlon = np.abs((ens.lon - g["final_lon"] + 180.0) % 360.0 - 180.0) / 360.0
        assert dlon.max() <= 1e-5
        assert (np.abs(ens.lat - g["final_lat"]) / 180.0).max() <= 1e-5
        assert (np.abs(ens.p - g["final_p"]) / g["final_p"]).max() <= 1e-5


def test_met_rotation_matches_oracle(eng):
    engine, ms, syn = eng
    lons, lats, levs = syn.grid(10.0, 5.0, 20)
    mets = [syn.snapshot(3600.0 * k, lons, lats, levs, syn.era5_like(lons, lats, levs, 7.0 * k))
            for k in range(4)]
    ctl = ms.Control(t_stop=3 * 3600.0, dt_model=600.0, rng_mode="counter", rng_seed_global=3,
                     met_dt=3600.0)
    ens = syn.particles(3000, seed=4)
    st = {"time": ens.time.copy(), "lon": ens.lon.copy(), "lat": ens.lat.copy(),
          "p": ens.p.copy(), "uvwp": np.zeros((3, ens.np)), "iso_var": np.zeros(ens.np),
          "q": np.zeros((5, ens.np))}
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(mets[0], mets[1])
    snaps = [orc.Snapshot.like(m) for m in mets]
    k1, t = 1, 0.0
    for step in range(18):
        t_next = min(t + ctl.dt_model, ctl.t_stop)
        while mets[k1].t_met < t_next:
            e.prefetch(met=mets[k1 + 1])
            e.rotate()
            k1 += 1
        e.step(ctl, step, engine.ADV_DIFF)
        orc.full_step(ctl, snaps[k1 - 1], snaps[k1], st, 0, ens.np, step,
                      modules=("advection", "turb", "meso", "position"))
        t = t_next
    got = e.download()
    e.close()
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_allclose(getattr(got, k), st[k], rtol=1e-10, atol=1e-9)


def _engine_run(engine, m0, m1, ens, ctl, steps, mask, sort_every=0):
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(m0, m1)
    for step in range(steps):
        if sort_every and step % sort_every == 0:
            e.sort()
        e.step(ctl, step, mask)
    out = e.download()
    e.close()
    return out


def test_fast_precision_within_north_star_tolerance(eng):
    """precision='fast' (fp32 interpolation arithmetic, fp64 state) stays
    within the north star's ~1e-5 run tolerance of the exact kernels over a
    24 h cfg2-style run (1 deg ERA5-like met, adv + turb + meso, 480 steps)."""
    engine, ms, syn = eng
    m0, m1 = syn.analytic_pair(1.0, 1.0, 60, 0.0, 10800.0)
    ens = syn.particles(200_000, seed=21)
    kw = dict(t_stop=86400.0, dt_model=180.0, met_dt=10800.0, rng_mode="counter",
              rng_seed_global=5)
    exact = _engine_run(engine, m0, m1, ens, ms.Control(**kw), 480, engine.ADV_DIFF, 40)
    fast = _engine_run(engine, m0, m1, ens, ms.Control(precision="fast", **kw), 480,
                       engine.ADV_DIFF, 40)
    dlon = np.abs((fast.lon - exact.lon + 180.0) % 360.0 - 180.0)
    assert dlon.max() / 360.0 <= 1e-5
    assert np.abs(fast.lat - exact.lat).max() / 180.0 <= 1e-5
    assert (np.abs(fast.p - exact.p) / exact.p).max() <= 1e-5
    np.testing.assert_array_equal(fast.time, exact.time)


@pytest.mark.parametrize("chunk", [0, 700, 2048])
def test_host_path_equals_device_path_bitwise(eng, golden_chain, chunk):
    """lt_run_host (host SoA streamed through the store in overlapped
    chunks, a ring of slots when chunk < n) == the device-resident step."""
    engine, ms, _ = eng
    from paper_2211_12616_b200.context import pinned_empty
    g = golden_chain
    ctl = chain_ctl()
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    ref, rc = _run_chain(engine, ms, g, ctl, 6, shards=1)
    ens = _ens(ms, g, "init")
    n = ens.np
    pin = {k: pinned_empty(n) for k in ("time", "p", "lon", "lat")}
    for k, a in pin.items():
        a[:] = getattr(ens, k)
    q = pinned_empty((5, n))
    q[:] = ens.q
    host = ms.ParticleEnsemble(n, pin["time"], pin["p"], ens.zeta, pin["lon"], pin["lat"], q)
    cache = ms.CacheState(uvwp=pinned_empty((3, n)), iso_var=pinned_empty(n))
    cache.uvwp[:] = 0.0
    e = engine.Engine(device=0)
    e.ctx.alloc(1500 if chunk == 700 else n, 5)   # ring of 2 slots for chunk 700
    e.bind_met(m0, m1)
    e.load_clim(ms.read_clim(ctl))
    e.ctx.run_host(ctl, engine.capi.MOD_ISOSURF_INIT, n, 0, 0, host.time, host.p, host.lon,
                   host.lat, iso_var=cache.iso_var, chunk=chunk)
    for step in range(6):
        e.step_host(ctl, host, cache, step, engine.FULL, chunk=chunk)
    e.close()
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_array_equal(getattr(host, k), getattr(ref, k))
    np.testing.assert_array_equal(host.q, ref.q)
    np.testing.assert_array_equal(cache.uvwp, rc.uvwp)
    np.testing.assert_array_equal(cache.iso_var, rc.iso_var)


def test_home_order_rows_follow_particles(eng, golden_chain):
    """Rows the chain does not touch stay in particle order through sorts
    (lt_set_home_rows); downloads, statistics and a later switch to a chain
    that writes q (meteo) see the same particles as an unsorted run."""
    engine, ms, _ = eng
    g = golden_chain
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    ctl = chain_ctl()
    base = _ens(ms, g, "init")
    n = base.np
    base.zeta[:] = np.arange(n) * 0.5
    q = np.zeros((6, n))
    q[5] = np.arange(n) % 7
    base = ms.ParticleEnsemble(n, base.time, base.p, base.zeta, base.lon, base.lat, q)

    def run(sort_every):
        e = engine.Engine(device=0, nq=6, first_id=0)
        e.upload(base)
        e.bind_met(m0, m1)
        e.load_clim(ms.read_clim(ctl))
        e.init_isosurf(ctl)
        for step in range(6):
            if sort_every and step % sort_every == 0:
                e.sort()
            e.step(ctl, step, engine.ADV_DIFF)
        mid = e.download()
        for step in range(6, 10):
            if sort_every and step % sort_every == 0:
                e.sort()
            e.step(ctl, step, engine.FULL)
        out = e.download()
        e.close()
        return mid, out

    mid0, out0 = run(0)
    mid2, out2 = run(2)
    np.testing.assert_array_equal(mid2.zeta, base.zeta)
    np.testing.assert_array_equal(mid2.q, base.q)
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_array_equal(getattr(mid2, k), getattr(mid0, k))
        np.testing.assert_array_equal(getattr(out2, k), getattr(out0, k))
    np.testing.assert_array_equal(out2.q, out0.q)
    np.testing.assert_array_equal(out2.zeta, base.zeta)


def test_group_stats_with_home_order_q(eng):
    engine, ms, syn = eng
    from paper_2211_12616_b200 import output
    from paper_2211_12616_b200.device_runtime import DevicePool, ModelImage
    m0, m1 = syn.analytic_pair(dlon=10.0, dlat=5.0, nlev=12)
    ens = syn.particles(20000, seed=4, nq=6)
    ens.q[5] = np.arange(ens.np) % 5
    ctl = ms.Control(ens_group_slot=5, nq=6, rng_mode="counter")
    host = ModelImage(ctl=ctl, ens=ens, cache=ms.cache_allocate(ens.np), clim=ms.read_clim(),
                      met0=m0, met1=m1, dt=np.zeros(ens.np), batch=None)
    with DevicePool(1) as pool:
        r = pool.region_create(0, host, None, with_batch=False)
        pool.region_update_device(r, host, ("ens", "met0", "met1"))
        before = output.group_stats(ctl, r.image.ens)
        img = r.image

        def go():
            img.engine.step(ctl, 0, engine.ADV_DIFF)
            img.engine.sort()       # q now kept in particle order
        pool.dispatch(0, go).result()
        after = output.group_stats(ctl, r.image.ens)
        back = img.engine.download()
    np.testing.assert_array_equal(back.q[5], ens.q[5])
    og, oc, om, osd = orc.grouped_moments(back.q[5], back.lon, back.lat, back.p)
    np.testing.assert_array_equal(after[0], og)
    np.testing.assert_array_equal(after[1], oc)
    np.testing.assert_allclose(after[2], om, rtol=1e-12)
    np.testing.assert_array_equal(before[1], after[1])


def test_faithful_mode_production_chain(eng):
    """The adv+turb+meso chain with the reference's default faithful RNG
    (compile-time generator): exact kernels against the oracle stepping
    with the same per-device stream; fast kernels within tolerance."""
    engine, ms, syn = eng
    m0, m1 = syn.analytic_pair(dlon=5.0, dlat=5.0, nlev=30, t0=0.0, t1=10800.0)
    ens = syn.particles(20000, seed=13)
    kw = dict(t_stop=86400.0, dt_model=180.0, met_dt=10800.0, rng_mode="faithful", mpi_rank=3)
    st = {"time": ens.time.copy(), "lon": ens.lon.copy(), "lat": ens.lat.copy(),
          "p": ens.p.copy(), "uvwp": np.zeros((3, ens.np)), "iso_var": np.zeros(ens.np),
          "q": np.zeros((5, ens.np))}
    s0, s1 = orc.Snapshot.like(m0), orc.Snapshot.like(m1)
    state = orc.seed_for(3, 0)
    for step in range(12):
        state = orc.full_step(ms.Control(**kw), s0, s1, st, 0, ens.np, step, rng_state=state,
                              modules=("advection", "turb", "meso", "position"))
    exact = _engine_run(engine, m0, m1, ens, ms.Control(**kw), 12, engine.ADV_DIFF, 5)
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_allclose(getattr(exact, k), st[k], rtol=1e-10, atol=1e-9)
    fast = _engine_run(engine, m0, m1, ens, ms.Control(precision="fast", **kw), 12,
                       engine.ADV_DIFF, 5)
    assert np.abs((fast.lon - exact.lon + 180.0) % 360.0 - 180.0).max() / 360.0 <= 1e-6
    assert (np.abs(fast.p - exact.p) / exact.p).max() <= 1e-6


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_philox_production_chain_brownian_variance(eng, precision):
    """Philox (the north star's counter-based generator, full 32-bit ids):
    Brownian variance 2 K t within 5 % (acceptance c5) through the fused
    production chain, both precisions."""
    engine, ms, syn = eng
    lons, lats, levs = syn.grid(30.0, 10.0, 7)
    shape = (lons.size, lats.size, levs.size)
    z = np.zeros(shape)
    met = ms.met_periodic(ms.MeteoField(0.0, lons, lats, levs, z, z, z, np.full(shape, 250.0)))
    n = 200_000
    ens = syn.particles(n, seed=2, lat_span=0.0)
    ens.lon[:] = 0.0
    ctl = ms.Control(t_stop=1e6, dt_model=1000.0, met_dt=10800.0, turb_dx=50.0, turb_dz=0.0,
                     turb_meso=0.0, rng_mode="philox", rng_seed_global=11, precision=precision)
    out = _engine_run(engine, met, met, ens, ctl, 10, engine.ADV_DIFF)
    var = np.var(out.lon / (180.0 / (np.pi * 6371000.0)))
    assert var == pytest.approx(2.0 * 50.0 * 1e4, rel=0.05)


def test_fast_precision_philox_within_tolerance(eng):
    """The headline configuration (fast kernels, Philox) against the exact
    kernels on the same draws: a 24 h cfg2-style run stays inside 1e-5."""
    engine, ms, syn = eng
    m0, m1 = syn.analytic_pair(1.0, 1.0, 60, 0.0, 10800.0)
    ens = syn.particles(100_000, seed=22)
    kw = dict(t_stop=86400.0, dt_model=180.0, met_dt=10800.0, rng_mode="philox",
              rng_seed_global=5)
    exact = _engine_run(engine, m0, m1, ens, ms.Control(**kw), 480, engine.ADV_DIFF, 15)
    fast = _engine_run(engine, m0, m1, ens, ms.Control(precision="fast", **kw), 480,
                       engine.ADV_DIFF, 15)
    dlon = np.abs((fast.lon - exact.lon + 180.0) % 360.0 - 180.0)
    assert dlon.max() / 360.0 <= 1e-5
    assert np.abs(fast.lat - exact.lat).max() / 180.0 <= 1e-5
    assert (np.abs(fast.p - exact.p) / exact.p).max() <= 1e-5


@pytest.mark.parametrize("mode", ["counter", "faithful"])
def test_host_path_multi_step_call_equals_single_steps(eng, golden_chain, mode):
    """lt_run_host_steps (K steps per call, pipelined across steps, a ring
    smaller than the ensemble) == K single-step calls, bit for bit."""
    engine, ms, _ = eng
    from paper_2211_12616_b200.context import pinned_empty
    g = golden_chain
    base = vars(chain_ctl()).copy()
    base["rng_mode"] = mode
    ctl = ms.Control(**{k: v for k, v in base.items() if k in ms.Control.__dataclass_fields__})
    m0, m1 = snapshot_from(g, "m0"), snapshot_from(g, "m1")
    outs = []
    for split in (True, False):
        ens = _ens(ms, g, "init")
        n = ens.np
        rows = {k: pinned_empty(n) for k in ("time", "p", "lon", "lat")}
        for k, a in rows.items():
            a[:] = getattr(ens, k)
        q = pinned_empty((5, n))
        q[:] = ens.q
        host = ms.ParticleEnsemble(n, rows["time"], rows["p"], ens.zeta, rows["lon"],
                                   rows["lat"], q)
        cache = ms.CacheState(uvwp=pinned_empty((3, n)), iso_var=pinned_empty(n))
        cache.uvwp[:] = 0.0
        e = engine.Engine(device=0, first_id=0)
        e.ctx.alloc(1024, 5)                       # ring of 2 slots of 512
        e.bind_met(m0, m1)
        e.load_clim(ms.read_clim(ctl))
        e.ctx.run_host(ctl, engine.capi.MOD_ISOSURF_INIT, n, 0, 0, host.time, host.p, host.lon,
                       host.lat, iso_var=cache.iso_var, chunk=512)
        if split:
            for step in range(4):
                e.step_host(ctl, host, cache, step, engine.FULL, chunk=512)
        else:
            e.step_host(ctl, host, cache, 0, engine.FULL, chunk=512, steps=4)
        e.close()
        outs.append(np.stack([host.lon, host.lat, host.p, host.time, *host.q, *cache.uvwp]))
    np.testing.assert_array_equal(outs[0], outs[1])


def test_fast_full_chain_within_tolerance(eng, golden_chain):
    """All nine modules (theta isosurface, convection, sedimentation,
    meteo, decay) with the fast kernels against the exact ones over the
    50-step golden chain."""
    engine, ms, _ = eng
    g = golden_chain
    base = vars(chain_ctl()).copy()
    base.update(decay_tau=86400.0, decay_slot=4)
    exact_ctl = ms.Control(**{k: v for k, v in base.items() if k in ms.Control.__dataclass_fields__})
    fast_ctl = ms.Control(**{**vars(exact_ctl), "precision": "fast"})
    ex, _ = _run_chain(engine, ms, g, exact_ctl, 50, shards=1, sort_every=10)
    fa, _ = _run_chain(engine, ms, g, fast_ctl, 50, shards=1, sort_every=10)
    dlon = np.abs((fa.lon - ex.lon + 180.0) % 360.0 - 180.0) / 360.0
    dlat = np.abs(fa.lat - ex.lat) / 180.0
    dp = np.abs(fa.p - ex.p) / ex.p
    print("full chain fast-vs-exact: max dlon %.2e dlat %.2e dp %.2e; dp>1e-5: %d of %d"
          % (dlon.max(), dlat.max(), dp.max(), int((dp > 1e-5).sum()), dp.size))
    # thresholded modules branch on rounding-level differences: the theta
    # isosurface iterates while |dp| >= 0.1 hPa, so a particle whose update
    # lands within ~1e-4 hPa of the threshold stops one iteration earlier or
    # later (threshold flips are legitimate; measured 2 % of
    # particles over 50 steps, each off by less than one sub-0.1 hPa update)
    assert np.mean(dp <= 1e-5) >= 0.95 and dp.max() <= 1e-3
    assert dlon.max() <= 1e-5 and dlat.max() <= 1e-5
    np.testing.assert_array_equal(fa.time, ex.time)


@pytest.mark.parametrize("same_time", [False, True])
def test_fast_path_regional_irregular_grid(eng, same_time):
    """The fast path's own cell logic — computed cells on uniform axes, fp32
    fraction search on irregular ones, the clamp folded into index and
    fraction — against the exact kernels on a regional (non-periodic) grid
    with irregular latitudes, particles partly outside the hull, and the
    single-snapshot (t0 == t1) case."""
    engine, ms, _ = eng
    rs = np.random.default_rng(7)
    f32 = lambda x: np.asarray(x, dtype=np.float32).astype(np.float64)
    lons = f32(np.arange(0.0, 91.0, 3.0))                                  # uniform
    lats = f32(np.sort(np.r_[-60.0, 60.0, rs.uniform(-59.0, 59.0, 29)]))   # irregular
    levs = f32(np.geomspace(1000.0, 50.0, 12))
    shape = (lons.size, lats.size, levs.size)
    lo3, la3 = np.meshgrid(lons, lats, indexing="ij")
    base = lambda a, b: f32((a + b * np.cos(np.deg2rad(la3)) * np.sin(np.deg2rad(3 * lo3)))[..., None]
                            * np.ones(shape))
    def snap(t, ph):
        return ms.MeteoField(t, lons, lats, levs, base(10.0 + ph, 5.0), base(2.0, 3.0 + ph),
                             f32(1e-3 * np.ones(shape)), base(250.0 + ph, 10.0))
    m0 = snap(0.0, 0.0)
    m1 = m0 if same_time else snap(3600.0, 1.0)
    n = 20000
    ens = ms.ParticleEnsemble(np=n, time=np.zeros(n), p=rs.uniform(30.0, 1100.0, n),
                              zeta=np.zeros(n), lon=rs.uniform(-20.0, 110.0, n),
                              lat=rs.uniform(-70.0, 70.0, n), q=np.zeros((5, n)))
    kw = dict(t_stop=1800.0, dt_model=180.0, met_dt=3600.0, rng_mode="counter", rng_seed_global=3)
    exact = _engine_run(engine, m0, m1, ens, ms.Control(**kw), 10, engine.ADV_DIFF, 5)
    fast = _engine_run(engine, m0, m1, ens, ms.Control(precision="fast", **kw), 10,
                       engine.ADV_DIFF, 5)
    dlon = np.abs((fast.lon - exact.lon + 180.0) % 360.0 - 180.0)
    assert dlon.max() / 360.0 <= 1e-5
    assert np.abs(fast.lat - exact.lat).max() / 180.0 <= 1e-5
    assert (np.abs(fast.p - exact.p) / exact.p).max() <= 1e-5
    np.testing.assert_array_equal(fast.time, exact.time)


@pytest.mark.parametrize("precision,rng_mode", [("exact", "counter"), ("fast", "philox"),
                                                ("fast", "counter")])
def test_multi_step_launch_equals_single_steps(eng, precision, rng_mode):
    """Engine.step_many (lt_run_steps: each particle advanced K steps in one
    launch, state in registers) == K single-step launches, bit for bit —
    including after a box sort whose permutation rides along with the first
    step."""
    engine, ms, syn = eng
    m0, m1 = syn.analytic_pair(1.0, 1.0, 60, 0.0, 10800.0)
    ens = syn.particles(30_000, seed=5)
    ctl = ms.Control(t_stop=5400.0, dt_model=180.0, met_dt=10800.0, rng_mode=rng_mode,
                     rng_seed_global=9, precision=precision)
    outs = []
    for many in (False, True):
        e = engine.Engine(device=0)
        e.upload(ens)
        e.bind_met(m0, m1)
        step = 0
        for cycle in range(3):
            e.sort(engine.ADV_DIFF)
            if many:
                e.step_many(ctl, step, 7, engine.ADV_DIFF)
            else:
                for k in range(7):
                    e.step(ctl, step + k, engine.ADV_DIFF)
            step += 7
        out = e.download()
        outs.append(np.stack([out.lon, out.lat, out.p, out.time]))
        e.close()
    np.testing.assert_array_equal(outs[1], outs[0])


def test_spread_tables_follow_reloaded_slots(eng):
    """The per-cell mesoscale spread tables are tagged by met slot: a slot
    reloaded with new content (same slot index, same snapshot time) gets a
    fresh table, and a prebuilt met1 table is used after the rotation —
    both runs equal the oracle, which computes the spreads per particle."""
    engine, ms, syn = eng
    lons, lats, levs = syn.grid(10.0, 5.0, 20)
    a = syn.snapshot(0.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 0.0))
    b = syn.snapshot(3600.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 7.0))
    c = syn.snapshot(0.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 3.0))
    d = syn.snapshot(7200.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 11.0))
    ctl = ms.Control(t_stop=7200.0, dt_model=600.0, rng_mode="counter", rng_seed_global=5,
                     met_dt=3600.0, turb_meso=0.16)
    ens = syn.particles(2000, seed=6)
    st = {"time": ens.time.copy(), "lon": ens.lon.copy(), "lat": ens.lat.copy(),
          "p": ens.p.copy(), "uvwp": np.zeros((3, ens.np)), "iso_var": np.zeros(ens.np),
          "q": np.zeros((5, ens.np))}
    mods = ("advection", "turb", "meso", "position")
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(a, b)
    e.step(ctl, 0, engine.ADV_DIFF)      # tables: a (built), b (prebuilt)
    orc.full_step(ctl, orc.Snapshot.like(a), orc.Snapshot.like(b), st, 0, ens.np, 0, modules=mods)
    e.bind_met(c, b)                     # slot 0 now holds c: its table must be rebuilt
    e.step(ctl, 1, engine.ADV_DIFF)
    orc.full_step(ctl, orc.Snapshot.like(c), orc.Snapshot.like(b), st, 0, ens.np, 1, modules=mods)
    e.prefetch(met=d)
    e.rotate()                           # met0 = b: the prebuilt table
    for step in (2, 3):
        e.step(ctl, step, engine.ADV_DIFF)
        orc.full_step(ctl, orc.Snapshot.like(b), orc.Snapshot.like(d), st, 0, ens.np, step,
                      modules=mods)
    got = e.download()
    e.close()
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_allclose(getattr(got, k), st[k], rtol=1e-10, atol=1e-9)


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_sort_with_step_keys_is_the_oracle_permutation(eng, precision):
    """LT_RUN_SORT_KEYS: the step launched just before a sort writes the box
    keys of the particles' end positions and the sort uses them (no key
    kernel): the permutation is still the stable argsort of the oracle's
    box_keys of those positions, and the fused path was taken."""
    engine, ms, syn = eng
    lons, lats, levs = syn.grid(2.0, 2.0, 40)
    m0 = syn.snapshot(0.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 0.0))
    m1 = syn.snapshot(3600.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 7.0))
    ctl = ms.Control(t_stop=7200.0, dt_model=600.0, rng_mode="philox", rng_seed_global=8,
                     met_dt=3600.0, precision=precision)
    ens = syn.particles(30000, seed=11)
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(m0, m1)
    e.sort(engine.ADV_DIFF)                     # computes its own keys (and the level window)
    for step in range(2):
        e.step(ctl, step, engine.ADV_DIFF)
    ids_before = e.ctx.ids(0, ens.np).astype(np.int64)
    e.step(ctl, 2, engine.ADV_DIFF, sort_next=True)
    e.sort(engine.ADV_DIFF)
    sorts, fused = e.ctx.sort_info()
    assert (sorts, fused) == (2, 1)
    ids_after = e.ctx.ids(0, ens.np).astype(np.int64)
    end = e.download()                          # particle order
    slot = ids_before - e.first_id
    keys = orc.box_keys(orc.Snapshot.like(m0), end.lon[slot], end.lat[slot], end.p[slot])
    np.testing.assert_array_equal(ids_after, ids_before[np.argsort(keys, kind="stable")])
    e.close()


def test_sort_with_step_keys_falls_back_outside_the_level_window(eng):
    """Keys written by a step are used only while every particle stays in
    the level window sized from the last sort's occupied range: convection
    that throws particles across the column makes the sort compute its own
    keys — and the permutation is the oracle's either way."""
    engine, ms, syn = eng
    lons, lats, levs = syn.grid(2.0, 2.0, 60)
    m0 = syn.snapshot(0.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 0.0))
    m1 = syn.snapshot(3600.0, lons, lats, levs, syn.era5_like(lons, lats, levs, 5.0))
    ctl = ms.Control(t_stop=7200.0, dt_model=600.0, rng_mode="philox", rng_seed_global=4,
                     met_dt=3600.0, conv_prob=1.0, conv_p_top=50.0, precision="fast")
    ens = syn.particles(20000, seed=12)
    ens.p[:] = 500.0 + (ens.p - ens.p.mean()) * 1e-3     # one narrow level band
    mask = engine.modules_mask(("advection", "convection", "position"))
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(m0, m1)
    e.sort(mask)                                   # window from the narrow band
    ids_before = e.ctx.ids(0, ens.np).astype(np.int64)
    e.step(ctl, 0, mask, sort_next=True)           # convection: p anywhere in [50, p_surf]
    e.sort(mask)
    assert e.ctx.sort_info() == (2, 0)
    ids_after = e.ctx.ids(0, ens.np).astype(np.int64)
    end = e.download()
    slot = ids_before - e.first_id
    keys = orc.box_keys(orc.Snapshot.like(m0), end.lon[slot], end.lat[slot], end.p[slot])
    np.testing.assert_array_equal(ids_after, ids_before[np.argsort(keys, kind="stable")])
    e.close()
