"""GPU parity at the headline shape: the 0.25 deg x 137-level grid (levels
geomspace(1013.25, 0.01, 137)), where the benchmark's fast
kernels take their geographic-grid lookups (computed lon/lat cells,
log-guessed levels).

* hires.npz (made by running the reference on a 40 x 40 deg window of that
  grid, make_golden.gen_hires): the 20-step production chain (advection +
  turbulent + mesoscale diffusion + position, counter draws) through the
  fused engine (exact kernels, sharded, box-sorted), through the module API,
  and through the fast kernels.  Per-module pairs on the same window run in
  test_gpu_parity.py (`mods` is parametrised over both fixtures).
* the full 1441 x 721 x 137 grid, 1e6 particles x 480 steps (24 h): the fast
  kernels against the exact kernels within the north star's 1e-5 run
  tolerance (span-normalised lon/lat, relative p).

Reference code on this path: physics.py:31-66 (_locate, _interp_snapshot),
physics.py:91-188 (advection, turb, meso), ingest.py:195-207 (met_periodic).
"""

import numpy as np
import pytest

from conftest import hires_chain_ctl

pytestmark = pytest.mark.gpu

TOL = 1e-5   # north star: positions within ~1e-5 of the CPU oracle over the run


@pytest.fixture(scope="module")
def eng():
    from paper_2211_12616_b200 import engine, model_state, synthetic
    return engine, model_state, synthetic


def _ens(ms, g, tag):
    return ms.ParticleEnsemble(np=g[f"{tag}_p"].size, time=g[f"{tag}_time"].copy(),
                               p=g[f"{tag}_p"].copy(), zeta=g[f"{tag}_zeta"].copy(),
                               lon=g[f"{tag}_lon"].copy(), lat=g[f"{tag}_lat"].copy(),
                               q=g[f"{tag}_q"].copy())


def _engine_chain(engine, ms, g, met, ctl, steps, shards=1, sort_every=0):
    from paper_2211_12616_b200.partition import partition_all
    ens = _ens(ms, g, "chain_init")
    cache = ms.cache_allocate(ens.np)
    for w in partition_all(ens.np, shards):
        e = engine.Engine(device=0, first_id=w.start)
        e.upload(ens, start=w.start, end=w.end)
        e.bind_met(*met)
        for step in range(steps):
            if sort_every and step % sort_every == 0:
                e.sort()
            e.step(ctl, step, engine.ADV_DIFF, device_id=w.device_id)
        e.download(ens, cache, start=w.start)
        e.close()
    return ens, cache


def _run_error(a_lon, a_lat, a_p, b_lon, b_lat, b_p):
    dlon = np.abs((a_lon - b_lon + 180.0) % 360.0 - 180.0) / 360.0
    dlat = np.abs(a_lat - b_lat) / 180.0
    dp = np.abs(a_p - b_p) / b_p
    return dlon.max(), dlat.max(), dp.max()


def test_hires_chain_exact_engine_matches_reference(eng, golden_hires):
    engine, ms, _ = eng
    g, met = golden_hires
    ens, cache = _engine_chain(engine, ms, g, met, hires_chain_ctl(), 20, shards=2, sort_every=7)
    np.testing.assert_array_equal(ens.time, g["chain_final_time"])
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(getattr(ens, k), g[f"chain_final_{k}"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(cache.uvwp, g["chain_final_uvwp"], rtol=1e-9, atol=1e-12)


def test_hires_chain_module_api_matches_reference(eng, golden_hires):
    """The eight-call pipeline of driver_cli.device_step through the drop-in
    module API (host arrays), as the reference's driver would call it."""
    engine, ms, _ = eng
    import paper_2211_12616_b200.physics as phys
    import paper_2211_12616_b200.rng as rng
    from paper_2211_12616_b200.partition import partition_all
    g, (m0, m1) = golden_hires
    ctl = hires_chain_ctl()
    ens = _ens(ms, g, "chain_init")
    n = ens.np
    cache = ms.cache_allocate(n)
    dt = np.zeros(n)
    batch = rng.batch_allocate(n)
    st = rng.module_rng_init(ctl, 3)
    ranges = partition_all(n, 3)
    for step in range(20):
        t_next = min(ctl.t_start + (step + 1) * ctl.dt_model, ctl.t_stop)
        for w in ranges:
            phys.module_timesteps(ctl, ens, t_next, w, dt)
            rng.generate_random_nums(st, step, w, w.device_id, batch)
            phys.module_advection(ctl, ens, m0, m1, dt, w)
            phys.module_diffusion_turb(ctl, ens, m0, m1, dt, batch, w)
            phys.module_diffusion_meso(ctl, ens, m0, m1, dt, batch, cache, w)
            phys.module_position(ctl, ens, w)
    np.testing.assert_array_equal(ens.time, g["chain_final_time"])
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(getattr(ens, k), g[f"chain_final_{k}"], rtol=1e-9, atol=1e-9)


def test_hires_chain_fast_kernels_within_tolerance(eng, golden_hires):
    """The benchmark's kernels (fp32 interpolation arithmetic, fp64 state)
    against the reference's own final state, same counter draws."""
    engine, ms, _ = eng
    g, met = golden_hires
    ctl = hires_chain_ctl()
    ctl.precision = "fast"
    ens, _ = _engine_chain(engine, ms, g, met, ctl, 20, shards=1, sort_every=5)
    np.testing.assert_array_equal(ens.time, g["chain_final_time"])
    err = _run_error(ens.lon, ens.lat, ens.p, g["chain_final_lon"], g["chain_final_lat"],
                     g["chain_final_p"])
    assert max(err) <= TOL, f"fast vs reference (lon, lat, p): {err}"


def test_full_grid_fast_vs_exact_24h(eng):
    """cfg3's grid in full (1441 x 721 x 137 fp32 records, 4.5 GB per
    snapshot), 1e6 particles, 480 steps with box sorts: fast vs exact within
    the run tolerance (tools/fast_error.py prints the distribution)."""
    engine, ms, syn = eng
    m0, m1 = syn.analytic_pair(0.25, 0.25, 137, 0.0, 10800.0, p_min=0.01)
    ens = syn.particles(1_000_000, seed=21)
    rs = np.random.default_rng(22)   # a third of them spread over every level to 0.02 hPa
    ens.p[::3] = np.exp(rs.uniform(np.log(0.02), np.log(1000.0), ens.p[::3].size)).astype(
        np.float32)
    kw = dict(t_stop=86400.0, dt_model=180.0, met_dt=10800.0, rng_mode="philox",
              rng_seed_global=5)
    out = {}
    for prec in ("exact", "fast"):
        e = engine.Engine(device=0)
        e.upload(ens)
        e.bind_met(m0, m1)
        ctl = ms.Control(precision=prec, **kw)
        for step in range(480):
            if step % 40 == 0:
                e.sort()
            e.step(ctl, step, engine.ADV_DIFF)
        out[prec] = e.download()
        e.close()
    ex, fa = out["exact"], out["fast"]
    np.testing.assert_array_equal(fa.time, ex.time)
    err = _run_error(fa.lon, fa.lat, fa.p, ex.lon, ex.lat, ex.p)
    assert max(err) <= TOL, f"fast vs exact over 24 h (lon, lat, p): {err}"
