"""GPU: the DevicePool mirror (device-resident images behind the module
API) and the driver loop, against the reference's golden run and against
each other.  Devices beyond the GPUs present share GPU 0 (device_map)."""

import numpy as np
import pytest

from conftest import chain_ctl, snapshot_from
from oracle import lagtrans_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rt():
    from paper_2211_12616_b200 import device_runtime, driver, engine, model_state, synthetic
    return device_runtime, driver, engine, model_state, synthetic


def _ens(ms, g, tag):
    return ms.ParticleEnsemble(np=g[f"{tag}_p"].size, time=g[f"{tag}_time"].copy(),
                               p=g[f"{tag}_p"].copy(), zeta=g[f"{tag}_zeta"].copy(),
                               lon=g[f"{tag}_lon"].copy(), lat=g[f"{tag}_lat"].copy(),
                               q=g[f"{tag}_q"].copy())


def _ctl(ms, **kw):
    base = vars(chain_ctl()).copy()
    base.update(kw)
    return ms.Control(**{k: v for k, v in base.items() if k in ms.Control.__dataclass_fields__})


@pytest.mark.parametrize("fused,ndev", [(False, 4), (True, 3), (True, 1)])
def test_driver_matches_reference_golden_chain(rt, golden_chain, fused, ndev):
    """driver_cli.run_simulation's loop over 1..4 device images reproduces
    the reference's 50-step all-physics run (acceptance c1 shape)."""
    _, driver, _, ms, _ = rt
    g = golden_chain
    ens = _ens(ms, g, "init")
    ctl = _ctl(ms, output_dt=1e9)
    status, cache = driver.run_simulation(ctl, ens, [snapshot_from(g, "m0"), snapshot_from(g, "m1")],
                                          num_devices=ndev, fused=fused)
    assert status == 0
    np.testing.assert_array_equal(ens.time, g["final_time"])
    for k in ("lon", "lat", "p"):
        np.testing.assert_allclose(getattr(ens, k), g[f"final_{k}"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(cache.uvwp, g["final_uvwp"], rtol=1e-9, atol=1e-12)


def test_device_count_invariance_bitwise(rt, golden_chain):
    """Counter mode: 1, 2 and 4 devices give byte-identical states
    (test_acceptance.py:93-102), fused and module-by-module alike."""
    _, driver, _, ms, _ = rt
    g = golden_chain
    mets = [snapshot_from(g, "m0"), snapshot_from(g, "m1")]
    ctl = _ctl(ms, output_dt=1e9, t_stop=1800.0)
    outs = []
    for fused, nd in ((True, 1), (True, 2), (True, 4), (False, 1), (False, 3)):
        ens = _ens(ms, g, "init")
        status, cache = driver.run_simulation(ctl, ens, mets, num_devices=nd, fused=fused,
                                              sort_every=3 if fused else 0)
        assert status == 0
        outs.append(np.stack([ens.lon, ens.lat, ens.p, ens.time, *ens.q, *cache.uvwp]))
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


def test_streamed_met_rotation_matches_oracle(rt):
    """Snapshots every hour, prefetched into the third met slot while the
    steps run (fused) vs the oracle stepping with driver_cli's rotation."""
    _, driver, engine, ms, syn = rt
    lons, lats, levs = syn.grid(10.0, 5.0, 16)
    mets = [syn.snapshot(3600.0 * k, lons, lats, levs,
                         syn.era5_like(lons, lats, levs, 7.0 * k, periodic=True))
            for k in range(4)]
    ctl = ms.Control(t_stop=3 * 3600.0, dt_model=600.0, met_dt=3600.0, turb_dx=50.0,
                     turb_dz=0.1, turb_meso=0.16, sedi_radius=5e-6, sedi_density=2000.0,
                     decay_tau=7200.0, decay_slot=5, nq=6, rng_mode="counter",
                     rng_seed_global=99, output_dt=3600.0)
    ens = syn.particles(3000, seed=5, nq=6)
    ens.q[5] = 1.0
    init = {k: getattr(ens, k).copy() for k in ("time", "lon", "lat", "p")}
    q5 = ens.q[5].copy()
    seen = []
    status, _ = driver.run_simulation(ctl, ens, mets, num_devices=2, fused=True,
                                      modules=engine.modules_mask(
                                          ("advection", "turb", "meso", "sedi", "decay",
                                           "position")),
                                      on_output=lambda c, e, ca, t: seen.append(t))
    assert status == 0
    assert seen == [3600.0, 7200.0, 10800.0]
    st = {"time": init["time"], "lon": init["lon"], "lat": init["lat"], "p": init["p"],
          "uvwp": np.zeros((3, ens.np)), "iso_var": np.zeros(ens.np), "q": np.zeros((5, ens.np))}
    snaps = [orc.Snapshot.like(m) for m in mets]
    t, k = 0.0, 0
    for step in range(driver.n_steps_for(ctl)):
        t_next = min(t + ctl.dt_model, ctl.t_stop)
        while snaps[k + 1].t_met < t_next:
            k += 1
        orc.full_step(ctl, snaps[k], snaps[k + 1], st, 0, ens.np, step,
                      modules=("advection", "turb", "meso", "sedi", "position"))
        t = t_next
    for key in ("lon", "lat", "p", "time"):
        np.testing.assert_allclose(getattr(ens, key), st[key], rtol=1e-9, atol=1e-9)
    # decay (new module): q *= exp(-dt / tau) per active step
    np.testing.assert_allclose(ens.q[5], q5 * np.exp(-3 * 3600.0 / 7200.0), rtol=1e-12)


def test_lifecycle_errors(rt):
    dr, _, _, ms, syn = rt
    from paper_2211_12616_b200._capi import LifecycleError
    from paper_2211_12616_b200.partition import partition_all
    ens = syn.particles(100)
    host = dr.ModelImage(ctl=ms.Control(), ens=ens, cache=ms.cache_allocate(100),
                         clim=ms.read_clim(), met0=None, met1=None, dt=np.zeros(100), batch=None)
    ranges = partition_all(100, 2)
    with dr.DevicePool(2, debug=True) as pool:
        with pytest.raises(ValueError):
            pool.dispatch(2, lambda: None)
        r0 = pool.region_create(0, host, ranges[0])
        with pytest.raises(LifecycleError):
            pool.region_create(0, host, ranges[0])
        with pytest.raises(LifecycleError):
            pool.region_update_host(r0, host, ranges[0])      # not populated
        with pytest.raises(ValueError):
            pool.region_update_device(r0, host, ("bogus",))
        pool.region_update_device(r0, host, ("ens", "cache"))
        with pytest.raises(LifecycleError):
            pool.region_update_host(r0, host, ranges[1])      # not its own range
        pool.region_update_host(r0, host, ranges[0])
        np.testing.assert_array_equal(host.ens.lon, ens.lon)
        pool.region_delete(r0)
        with pytest.raises(LifecycleError):
            pool.region_delete(r0)
        with pytest.raises(dr.DeviceTaskError) as ei:
            pool.for_each_device_parallel(lambda d: 1 / (d - 1))
        assert set(ei.value.failures) == {1}


def test_module_mode_timer_contract(rt, golden_chain):
    """Per-module, per-device PHYSICS records (test_acceptance.py:284-305),
    filled from CUDA events."""
    _, driver, _, ms, _ = rt
    g = golden_chain
    recs = []

    class Sink:
        def record(self, name, group, scope, ns):
            recs.append((group, name, scope, ns))

    ctl = _ctl(ms, output_dt=1e9, t_stop=360.0)
    status, _ = driver.run_simulation(ctl, _ens(ms, g, "init"),
                                      [snapshot_from(g, "m0"), snapshot_from(g, "m1")],
                                      num_devices=4, fused=False, timers=Sink())
    assert status == 0
    keys = {(gr, n, s) for gr, n, s, _ in recs}
    for d in range(4):
        for mod in driver.PIPELINE:
            assert ("PHYSICS", mod, f"device{d}") in keys
        assert ("INIT", "ACC_INIT", f"device{d}") in keys
        assert ("MEMORY", "DELETE_DATA_REGION", f"device{d}") in keys
    assert all(ns >= 0 for *_, ns in recs)


def test_fused_mode_timer_contract(rt, golden_chain):
    """The production (fused) path meets the same c10 contract: with
    module_timers each fused launch charges its SM cycles per module and its
    CUDA-event time is split into the reference's PHYSICS rows
    (module_advection ... module_meteo, generate_random_nums), per device;
    the per-module rows of a step add up to its module_fused_step row, and
    the instrumented kernel changes no result bit."""
    _, driver, _, ms, _ = rt
    g = golden_chain
    recs = []

    class Sink:
        def record(self, name, group, scope, ns):
            recs.append((group, name, scope, ns))

    ctl = _ctl(ms, output_dt=1e9, t_stop=540.0)
    mets = [snapshot_from(g, "m0"), snapshot_from(g, "m1")]
    outs = []
    for module_timers in (True, False):
        ens = _ens(ms, g, "init")
        status, cache = driver.run_simulation(ctl, ens, mets, num_devices=4, fused=True,
                                              timers=Sink(), module_timers=module_timers,
                                              sort_every=2)
        assert status == 0
        outs.append(np.stack([ens.lon, ens.lat, ens.p, ens.time, *ens.q, *cache.uvwp]))
        if module_timers:
            timed = list(recs)
    np.testing.assert_array_equal(outs[0], outs[1])
    keys = {(gr, n, s) for gr, n, s, _ in timed}
    for d in range(4):
        scope = f"device{d}"
        for mod in driver.PIPELINE + ("generate_random_nums", "module_timesteps"):
            assert ("PHYSICS", mod, scope) in keys, mod
        assert ("INIT", "ACC_INIT", scope) in keys
        assert ("MEMORY", "DELETE_DATA_REGION", scope) in keys
        fused = sum(ns for gr, n, sc, ns in timed if n == "module_fused_step" and sc == scope)
        split = sum(ns for gr, n, sc, ns in timed
                    if gr == "PHYSICS" and n != "module_fused_step" and sc == scope)
        assert fused > 0 and abs(split - fused) <= 0.01 * fused + 1000
        adv = sum(ns for gr, n, sc, ns in timed if n == "module_advection" and sc == scope)
        assert adv > 0
    assert all(ns >= 0 for *_, ns in timed)


def test_device_image_fields_read_and_write_like_the_reference_image(rt):
    """region.image.ens.<field> behaves like the reference image's arrays
    (device_runtime.py:165-219): the owned range is read from / written to
    HBM, the rest is the image's own copy, and copy-back moves only the
    owned range (acceptance c7, test_acceptance.py:205-220)."""
    dr, _, _, ms, syn = rt
    from paper_2211_12616_b200.partition import partition_all
    ens = syn.particles(100, seed=2)
    host = dr.ModelImage(ctl=ms.Control(), ens=ens, cache=ms.cache_allocate(100),
                         clim=ms.read_clim(), met0=None, met1=None, dt=np.zeros(100), batch=None)
    before = ens.lon.copy()
    with dr.DevicePool(4, debug=True) as pool:
        ranges = partition_all(100, 4)
        region = pool.region_create(1, host, ranges[1], with_batch=False)
        pool.region_update_device(region, host, ("ens", "cache"))
        np.testing.assert_array_equal(np.asarray(region.image.ens.lon), before)
        region.image.ens.lon[:] = 999.0
        assert region.image.ens.lon[30] == 999.0 and region.image.ens.lon[80] == 999.0
        host.ens.lon[0] += 100.0                      # the image is isolated from the host
        assert region.image.ens.lon[0] == 999.0
        region.image.ens.q[2, 26] = 7.0
        pool.region_update_host(region, host, ranges[1])
    inside = slice(ranges[1].start, ranges[1].end)
    assert np.all(host.ens.lon[inside] == 999.0)
    out = np.r_[1:ranges[1].start, ranges[1].end:100]
    np.testing.assert_array_equal(host.ens.lon[out], before[out])
    assert host.ens.q[2, 26] == 7.0 and host.ens.q[2, 80] == 0.0


def test_met_replication_between_devices(rt):
    """A snapshot one device holds reaches another by GPU-to-GPU copy
    (lt_met_copy_slot), not a second host upload; values identical."""
    dr, _, _, ms, syn = rt
    from paper_2211_12616_b200.context import DeviceContext
    m0, m1 = syn.analytic_pair(dlon=10.0, dlat=5.0, nlev=16)
    a, b = DeviceContext(0), DeviceContext(0)
    a.bind_pair(m0, m1)
    loads = []
    orig = b.load_met
    b.load_met = lambda *args, **kw: (loads.append(args), orig(*args, **kw))
    b.bind_pair(m0, m1, donor=lambda key: (a, a.find_slot(key)) if a.find_slot(key) is not None
                else None)
    assert loads == []
    rs = np.random.default_rng(2)
    lon, lat, p = rs.uniform(-180, 180, 5000), rs.uniform(-90, 90, 5000), rs.uniform(5, 1000, 5000)
    np.testing.assert_array_equal(b.interpolate(1800.0, lon, lat, p),
                                  a.interpolate(1800.0, lon, lat, p))
    a.close()
    b.close()
    # the pool wires the donor in: the second device's image copies from the first
    host = dr.ModelImage(ctl=ms.Control(), ens=syn.particles(10), cache=ms.cache_allocate(10),
                         clim=ms.read_clim(), met0=m0, met1=m1, dt=np.zeros(10), batch=None)
    with dr.DevicePool(2) as pool:
        r0 = pool.region_create(0, host, None, with_batch=False)
        pool.region_update_device(r0, host, ("met0", "met1"))
        r1 = pool.region_create(1, host, None, with_batch=False)
        c1 = r1.image.engine.ctx
        seen = []
        orig1 = c1.copy_slot_from
        c1.copy_slot_from = lambda *args, **kw: (seen.append(args), orig1(*args, **kw))
        pool.region_update_device(r1, host, ("met0", "met1"))
        assert len(seen) == 2


def test_met_broadcast_replicates_slot(rt):
    """lt_met_broadcast: the root's packed slot lands in each other
    context's chosen slot (here all contexts share GPU 0, so the transfer is
    the device-local leg; distinct GPUs take one NCCL broadcast group), with
    the time level, in stream order after the root's upload; values equal a
    direct upload's.  Argument errors map onto the reference's exceptions."""
    _, _, _, ms, syn = rt
    from paper_2211_12616_b200 import _capi as capi
    from paper_2211_12616_b200.context import DeviceContext, met_broadcast
    m0, m1 = syn.analytic_pair(dlon=10.0, dlat=5.0, nlev=16, t0=0.0, t1=3600.0)
    a, b, c, ref = (DeviceContext(0) for _ in range(4))
    for x in (a, b, c, ref):
        x.set_grid(m0.lons, m0.lats, m0.levs)
    a.load_met(0, m0, key="k0")
    a.load_met(2, m1, key="k1")
    ref.load_met(0, m0)
    ref.load_met(1, m1)
    met_broadcast([b, a, c], 1, [1, 0, 2])      # root a: slot 0 -> b slot 1, c slot 2
    met_broadcast([a, b, c], 0, [2, 0, 1])      # slot 2 (m1) -> b slot 0, c slot 1
    assert b.slot_key(1) == "k0" and c.slot_key(1) == "k1"
    b.use_met(1, 0)
    c.use_met(2, 1)
    ref.use_met(0, 1)
    rs = np.random.default_rng(4)
    lon, lat, p = rs.uniform(-180, 180, 4000), rs.uniform(-90, 90, 4000), rs.uniform(5, 1000, 4000)
    want = ref.interpolate(1234.0, lon, lat, p)
    np.testing.assert_array_equal(b.interpolate(1234.0, lon, lat, p), want)
    np.testing.assert_array_equal(c.interpolate(1234.0, lon, lat, p), want)
    import ctypes as C
    t = C.c_double()
    capi.check(b.lib.lt_met_slot_time(b.h, 0, C.byref(t)))
    assert t.value == 3600.0
    with pytest.raises(ValueError):
        met_broadcast([a, b], 0, [2, 3])             # slot out of range
    with pytest.raises(ValueError):
        met_broadcast([a, a], 0, [2, 1])             # context twice
    with pytest.raises(capi.LifecycleError):
        met_broadcast([a, b], 0, [1, 0])             # root slot never loaded
    d = DeviceContext(0)
    d.set_grid(m0.lons[:-2], m0.lats, m0.levs)
    with pytest.raises(ValueError):
        met_broadcast([a, d], 0, [0, 0])             # grid differs
    for x in (a, b, c, ref, d):
        x.close()


def test_nccl_selftest_on_this_box(rt):
    """NCCL itself on the box: a communicator over every GPU present
    (ncclCommInitAll) and one broadcast group from device 0 into a separate
    buffer on each device, checked byte for byte (lt_nccl_selftest) — the
    collective the met broadcast issues between distinct GPUs."""
    from paper_2211_12616_b200 import _capi as capi
    from paper_2211_12616_b200.context import nccl_info
    lib = capi.load()
    n = capi.device_count()
    capi.check(lib.lt_nccl_selftest(n, 3 << 20))
    info = nccl_info()
    assert info["version"] >= 22700 and info["ranks"] >= n
    with pytest.raises(ValueError):
        capi.check(lib.lt_nccl_selftest(n + 1, 16))


def test_driver_rotations_broadcast_met(rt):
    """driver.run_simulation (fused) on 3 devices with hourly snapshots: each
    rotation's next snapshot is uploaded once and broadcast (MET_BROADCAST
    timer rows), and the result equals the one-device run bit for bit."""
    _, driver, engine, ms, syn = rt
    lons, lats, levs = syn.grid(10.0, 5.0, 16)
    mets = [syn.snapshot(3600.0 * k, lons, lats, levs,
                         syn.era5_like(lons, lats, levs, 7.0 * k, periodic=True))
            for k in range(4)]
    ctl = ms.Control(t_stop=3 * 3600.0, dt_model=600.0, met_dt=3600.0, rng_mode="counter",
                     rng_seed_global=7, output_dt=1e9)

    class Rec:
        def __init__(self):
            self.rows = []

        def record(self, name, group, scope, ns):
            self.rows.append((name, group, scope))
    outs = []
    for nd in (1, 3):
        ens = syn.particles(5000, seed=8)
        timers = Rec()
        status, cache = driver.run_simulation(ctl, ens, mets, num_devices=nd, fused=True,
                                              timers=timers, sort_every=4)
        assert status == 0
        outs.append(np.stack([ens.lon, ens.lat, ens.p, ens.time, *cache.uvwp]))
        n_bc = sum(1 for r in timers.rows if r[0] == "MET_BROADCAST")
        assert n_bc == (0 if nd == 1 else 2)   # snapshots 2 and 3 are prefetched + broadcast
    np.testing.assert_array_equal(outs[1], outs[0])


def test_faithful_rng_fused_equals_module_path_with_sorts(rt, golden_chain):
    """Faithful mode (the reference default, rng.py:105-126): per-device
    streams seeded rank + 83*device, draws indexed by position in the
    device's range.  The fused kernel (draws in-kernel, keyed through the
    id row, box sorts between steps) reproduces the module-by-module path
    bit for bit on 3 devices."""
    _, driver, _, ms, _ = rt
    g = golden_chain
    mets = [snapshot_from(g, "m0"), snapshot_from(g, "m1")]
    ctl = _ctl(ms, output_dt=1e9, t_stop=1800.0, rng_mode="faithful", mpi_rank=1)
    outs = []
    for fused in (True, False):
        ens = _ens(ms, g, "init")
        status, cache = driver.run_simulation(ctl, ens, mets, num_devices=3, fused=fused,
                                              sort_every=2 if fused else 0)
        assert status == 0
        outs.append(np.stack([ens.lon, ens.lat, ens.p, ens.time, *ens.q, *cache.uvwp]))
    np.testing.assert_array_equal(outs[0], outs[1])
