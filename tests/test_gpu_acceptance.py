"""GPU: the reference's acceptance criteria and driver/runtime tests
(test_acceptance.py, test_driver.py, test_device_runtime.py) restated
against the B200 drop-in.  Criterion 9 (4-device speedup on host cores)
needs four GPUs and is covered by bench.py's multi-GPU path instead."""

import threading

import numpy as np
import pytest

from conftest import snapshot_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    from paper_2211_12616_b200 import device_runtime, driver, model_state, physics, rng
    from paper_2211_12616_b200 import synthetic
    from paper_2211_12616_b200.partition import WorkRange, partition_all
    return dict(dr=device_runtime, driver=driver, ms=model_state, phys=physics, rng=rng,
                syn=synthetic, WorkRange=WorkRange, partition_all=partition_all)


def _still_met(ms, syn, t, u=None):
    lons, lats, levs = syn.grid(30.0, 10.0, 7)
    shape = (lons.size, lats.size, levs.size)
    z = np.zeros(shape)
    uu = z if u is None else u(lons[:, None, None] + z, lats[None, :, None] + z)
    return ms.met_periodic(ms.MeteoField(t, lons, lats, levs, uu, z, z, np.full(shape, 250.0)))


def test_c2_deterministic_physics_invariance(m, golden_chain):
    """No stochastic module on: 1..4 devices byte-identical in both RNG
    modes, fused and module-by-module (test_acceptance.py:105-118)."""
    ms, driver = m["ms"], m["driver"]
    g = golden_chain
    mets = [snapshot_from(g, "m0"), snapshot_from(g, "m1")]
    outs = []
    for mode in ("faithful", "counter"):
        ctl = ms.Control(t_stop=9000.0, dt_model=180.0, met_dt=10800.0, turb_dx=0.0, turb_dz=0.0,
                         turb_meso=0.0, conv_prob=0.0, sedi_radius=1e-6, rng_mode=mode,
                         output_dt=9000.0)
        for fused, nd in ((True, 1), (True, 3), (False, 2), (False, 4)):
            ens = ms.ParticleEnsemble(np=g["init_p"].size, time=g["init_time"].copy(),
                                      p=g["init_p"].copy(), zeta=g["init_zeta"].copy(),
                                      lon=g["init_lon"].copy(), lat=g["init_lat"].copy(),
                                      q=g["init_q"].copy())
            status, _ = driver.run_simulation(ctl, ens, mets, num_devices=nd, fused=fused)
            assert status == 0
            outs.append(np.stack([ens.lon, ens.lat, ens.p, ens.time, *ens.q]))
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


def test_c5_turbulent_diffusion_variance(m):
    """Brownian oracle: var(x) = 2 K t within 5 % (test_acceptance.py:150-165)."""
    ms, phys, rng, syn = m["ms"], m["phys"], m["rng"], m["syn"]
    ctl = ms.Control(np_max=200000, turb_dx=50.0, turb_dz=0.0, rng_mode="counter")
    met = _still_met(ms, syn, 0.0)
    n = 100000
    ens = ms.ensemble_allocate(ctl, n)
    ens.p[:] = 500.0
    dt = np.full(n, 1000.0)
    work = m["WorkRange"](0, 0, n)
    r = rng.module_rng_init(ctl, 1)
    batch = rng.batch_allocate(n)
    for step in range(10):
        rng.generate_random_nums(r, step, work, 0, batch)
        phys.module_diffusion_turb(ctl, ens, met, met, dt, batch, work)
    var = np.var(ens.lon / phys.DEG_PER_M)
    assert var == pytest.approx(2.0 * 50.0 * 1e4, rel=0.05)


def test_c6_closed_orbit(m):
    """Solid-body rotation for two periods returns to the start
    (test_acceptance.py:168-183)."""
    ms, phys, syn = m["ms"], m["phys"], m["syn"]
    omega = 2.0 * np.pi / 86400.0
    period = 2.0 * np.pi / omega
    ctl = ms.Control(t_stop=2.0 * period)
    lons = np.arange(-180.0, 180.0, 30.0)
    lats = np.arange(-90.0, 90.0 + 1e-9, 5.0)
    levs = np.geomspace(1000.0, 100.0, 7)
    shape = (lons.size, lats.size, levs.size)
    u = np.broadcast_to(omega * 6371000.0 * np.cos(np.deg2rad(lats))[None, :, None], shape).copy()
    z = np.zeros(shape)
    met = ms.met_periodic(ms.MeteoField(0.0, lons, lats, levs, u, z, z, np.full(shape, 250.0)))
    ens = ms.ensemble_allocate(ctl, 1)
    ens.p[:] = 500.0
    dt = np.full(1, period / 1000.0)
    work = m["WorkRange"](0, 0, 1)
    for _ in range(1000):
        phys.module_advection(ctl, ens, met, met, dt, work)
        phys.module_position(ctl, ens, work)
    assert abs(ens.lon[0]) < 1e-3
    assert abs(ens.lat[0]) < 1e-3


def _host(m, n):
    ms, syn, dr = m["ms"], m["syn"], m["dr"]
    ens = syn.particles(n, seed=17)
    m0 = _still_met(ms, syn, 0.0)
    m1 = _still_met(ms, syn, 3600.0)
    return dr.ModelImage(ctl=ms.Control(), ens=ens, cache=ms.cache_allocate(n),
                         clim=ms.read_clim(), met0=m0, met1=m1, dt=np.zeros(n),
                         batch=m["rng"].batch_allocate(n))


def test_c7_range_restricted_copy_back(m):
    """Copy-back writes only the device's own range (test_acceptance.py:205-219)."""
    dr, capi = m["dr"], __import__("paper_2211_12616_b200._capi", fromlist=["x"])
    host = _host(m, 100)
    ranges = m["partition_all"](100, 4)
    snapshot = {k: getattr(host.ens, k).copy() for k in ("time", "p", "zeta", "lon", "lat")}
    q = host.ens.q.copy()
    with dr.DevicePool(4, debug=True) as pool:
        region = pool.region_create(1, host, work_range=ranges[1])
        pool.region_update_device(region, host, dr.REGION_FIELDS)
        ctx = region.image.engine.ctx
        ctx.fill(capi.F_LON, 0, 0, 25, 999.0)
        for k in range(5):
            ctx.fill(capi.F_Q, k, 0, 25, -1.0)
        for c in range(3):
            ctx.fill(capi.F_UVWP, c, 0, 25, 2.0)
        pool.region_update_host(region, host, ranges[1])
    outside = np.r_[0:25, 50:100]
    for k, v in snapshot.items():
        if k != "lon":
            np.testing.assert_array_equal(getattr(host.ens, k), v)
    np.testing.assert_array_equal(host.ens.lon[outside], snapshot["lon"][outside])
    np.testing.assert_array_equal(host.ens.q[:, outside], q[:, outside])
    assert np.all(host.ens.lon[25:50] == 999.0)
    assert np.all(host.ens.q[:5, 25:50] == -1.0)
    assert np.all(host.cache.uvwp[:, 25:50] == 2.0) and np.all(host.cache.uvwp[:, outside] == 0.0)


def test_c8_lifecycle_errors(m):
    """Lifecycle violations raise without corrupting state
    (test_acceptance.py:222-246)."""
    dr = m["dr"]
    from paper_2211_12616_b200._capi import LifecycleError
    from paper_2211_12616_b200.partition import calc_device_workload_range
    host = _host(m, 10)
    with dr.DevicePool(1) as pool:
        work = calc_device_workload_range(10, 1, 0)
        region = pool.region_create(0, host, work_range=work)
        with pytest.raises(LifecycleError):
            pool.region_create(0, host)
        pool.region_update_device(region, host, dr.REGION_FIELDS)
        release = threading.Event()
        pool.dispatch(0, release.wait)
        with pytest.raises(LifecycleError):
            pool.region_delete(region)
        release.set()
        pool.device_wait(0)
        assert region.state == "populated"
        pool.region_delete(region)
        with pytest.raises(LifecycleError):
            pool.region_delete(region)
        with pytest.raises(LifecycleError):
            pool.region_update_device(region, host, ("ens",))
        with pytest.raises(LifecycleError):
            pool.region_update_host(region, host, work)
        assert region.state == "deleted"
        again = pool.region_create(0, host, work_range=work)      # recreate after delete
        assert again.state == "created"


def test_device_image_isolation_and_order(m):
    """Host edits after update_device do not reach the image until the next
    update (test_device_runtime.py:123-129); tasks on one device run in
    submission order, waits are per device (:239-262)."""
    dr, capi = m["dr"], __import__("paper_2211_12616_b200._capi", fromlist=["x"])
    host = _host(m, 50)
    with dr.DevicePool(2) as pool:
        region = pool.region_create(0, host)
        pool.region_update_device(region, host, ("ens",))
        lon0 = host.ens.lon.copy()
        host.ens.lon[:] = 42.0
        got = region.image.engine.ctx.d2h(capi.F_LON, 0, 0, 50)
        np.testing.assert_array_equal(got, lon0)
        order = []
        futs = [pool.dispatch(1, lambda k=k: order.append(k)) for k in range(20)]
        pool.device_wait(1)
        assert all(f.done() for f in futs) and order == list(range(20))


def test_driver_edge_cases(m):
    """Degenerate duration, times capped at t_stop, met exhaustion,
    parallel == sequential (test_driver.py:67-135)."""
    ms, syn, driver = m["ms"], m["syn"], m["driver"]
    mets = [_still_met(ms, syn, 0.0, u=lambda lo, la: 10.0 + 0.0 * lo),
            _still_met(ms, syn, 3600.0, u=lambda lo, la: 12.0 + 0.0 * lo)]
    ens = syn.particles(500, seed=3)
    lon0 = ens.lon.copy()
    status, _ = driver.run_simulation(ms.Control(t_stop=0.0), ens, mets)
    assert status == 0 and np.array_equal(ens.lon, lon0)           # zero steps
    ctl = ms.Control(t_stop=1000.0, dt_model=180.0, output_dt=5000.0, rng_mode="counter")
    outs = []
    for par in (True, False):
        e = syn.particles(500, seed=3)
        status, _ = driver.run_simulation(ctl, e, mets, num_devices=3, parallel=par)
        assert status == 0
        assert np.all(e.time == 1000.0)                                # capped at t_stop
        outs.append(np.stack([e.lon, e.lat, e.p]))
    np.testing.assert_array_equal(outs[0], outs[1])
    with pytest.raises(ValueError):
        driver.run_simulation(ms.Control(t_stop=7200.0), syn.particles(10), mets)


def test_driver_multi_step_runs_equal_single_steps(m, golden_chain, monkeypatch):
    """run_simulation(fused) advances the steps between events (met rotation,
    sort, output) as multi-step launches; the result equals one launch per
    step bit for bit, with outputs and rotations inside the run."""
    ms, driver = m["ms"], m["driver"]
    from paper_2211_12616_b200 import engine as eng
    g = golden_chain
    mets = [snapshot_from(g, "m0"), snapshot_from(g, "m1")]
    ctl = ms.Control(t_stop=9000.0, dt_model=180.0, met_dt=10800.0, rng_mode="counter",
                     output_dt=1800.0)

    def run():
        ens = ms.ParticleEnsemble(np=g["init_p"].size, time=g["init_time"].copy(),
                                  p=g["init_p"].copy(), zeta=g["init_zeta"].copy(),
                                  lon=g["init_lon"].copy(), lat=g["init_lat"].copy(),
                                  q=g["init_q"].copy())
        outs = []
        status, _ = driver.run_simulation(ctl, ens, mets, num_devices=2, fused=True,
                                          modules=eng.ADV_DIFF, sort_every=7,
                                          on_output=lambda c, e, cache, t: outs.append(
                                              (t, e.lon.copy())))
        assert status == 0
        return np.stack([ens.lon, ens.lat, ens.p, ens.time]), outs

    multi, outs_m = run()

    def single(self, ctl, step, nsteps, modules=eng.ADV_DIFF, device_id=0, sort_next=False):
        for k in range(nsteps):
            self.step(ctl, step + k, modules, device_id=device_id,
                      sort_next=sort_next and k == nsteps - 1)
    monkeypatch.setattr(eng.Engine, "step_many", single)
    ref, outs_r = run()
    np.testing.assert_array_equal(multi, ref)
    assert [t for t, _ in outs_m] == [t for t, _ in outs_r] and len(outs_m) == 5
    for (_, a), (_, b) in zip(outs_m, outs_r):
        np.testing.assert_array_equal(a, b)
