"""GPU: edge cases of the boundary — empty ranges and ensembles, regional
(non-periodic) grids with out-of-hull particles, error mapping of bad
arguments — against the oracle and the reference's exception types."""

import numpy as np
import pytest

from oracle import lagtrans_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    from paper_2211_12616_b200 import _capi, engine, model_state, physics, rng, synthetic
    from paper_2211_12616_b200.partition import WorkRange
    return dict(capi=_capi, engine=engine, ms=model_state, phys=physics, rng=rng,
                syn=synthetic, WorkRange=WorkRange)


def test_empty_work_ranges_are_no_ops(m):
    ms, phys, rng, syn, WR = m["ms"], m["phys"], m["rng"], m["syn"], m["WorkRange"]
    m0, m1 = syn.analytic_pair(dlon=30.0, dlat=30.0, nlev=6)
    ens = syn.particles(10, seed=1)
    before = {k: getattr(ens, k).copy() for k in ("time", "lon", "lat", "p")}
    ctl = ms.Control(rng_mode="counter")
    dt = np.full(10, 180.0)
    w = WR(0, 4, 4)
    b = rng.batch_allocate(10)
    rng.generate_random_nums(rng.module_rng_init(ctl, 1), 0, w, 0, b)
    phys.module_timesteps(ctl, ens, 0.0, w, dt)
    phys.module_advection(ctl, ens, m0, m1, dt, w)
    phys.module_diffusion_turb(ctl, ens, m0, m1, dt, b, w)
    phys.module_position(ctl, ens, w)
    for k, v in before.items():
        np.testing.assert_array_equal(getattr(ens, k), v)
    with pytest.raises(IndexError):
        rng.generate_random_nums(rng.module_rng_init(ctl, 1), 0, WR(0, 5, 11), 0, b)


def test_empty_engine(m):
    engine, syn = m["engine"], m["syn"]
    m0, m1 = syn.analytic_pair(dlon=30.0, dlat=30.0, nlev=6)
    e = engine.Engine(device=0)
    e.upload(syn.particles(0))
    e.bind_met(m0, m1)
    e.sort()
    e.step(m["ms"].Control(rng_mode="counter"), 0, engine.ADV_DIFF)
    out = e.download()
    assert out.np == 0 and out.lon.size == 0
    e.close()


def test_regional_grid_clamps_like_the_reference(m):
    """No met_periodic closure on a regional grid: particles outside the
    hull use the boundary cell (physics.py:31-37 clamp), bit-exact."""
    ms, phys = m["ms"], m["phys"]
    rs = np.random.default_rng(3)
    lons = np.arange(0.0, 91.0, 3.0)
    lats = np.arange(-30.0, 31.0, 2.0)
    levs = np.geomspace(1000.0, 50.0, 9).astype(np.float32).astype(np.float64)
    shape = (lons.size, lats.size, levs.size)
    f = lambda: rs.uniform(-10, 10, shape).astype(np.float32).astype(np.float64)
    temp = lambda: (250.0 + f()).astype(np.float32).astype(np.float64)  # fp32-exact met
    m0 = ms.MeteoField(0.0, lons, lats, levs, f(), f(), f(), temp())
    m1 = ms.MeteoField(600.0, lons, lats, levs, f(), f(), f(), temp())
    n = 5000
    lon = rs.uniform(-40, 130, n)
    lat = rs.uniform(-60, 60, n)
    p = rs.uniform(10, 1100, n)
    t = rs.uniform(-50, 700, n)
    got = np.stack(phys.interpolate_met(m0, m1, t, lon, lat, p))
    ref = np.stack(orc.sample(orc.Snapshot.like(m0), orc.Snapshot.like(m1), t, lon, lat, p,
                              ("u", "v", "w", "T")))
    np.testing.assert_array_equal(got, ref)


def test_bad_arguments_raise_reference_types(m):
    capi, ms, syn = m["capi"], m["ms"], m["syn"]
    from paper_2211_12616_b200.context import DeviceContext
    ctx = DeviceContext(0)
    ctx.alloc(100, 5)
    with pytest.raises(IndexError):
        ctx.h2d(capi.F_LON, 0, 90, np.zeros(20))               # beyond the store
    with pytest.raises(ValueError):
        ctx.h2d(capi.F_Q, 7, 0, np.zeros(10))                  # no q row 7
    with pytest.raises(ValueError):
        ctx.h2d(99, 0, 0, np.zeros(10))                        # unknown field
    with pytest.raises(capi.LifecycleError):
        ctx.run(ms.Control(), capi.MOD_ADVECTION, 0, 10)       # no met selected
    with pytest.raises(IndexError):
        ctx.run(ms.Control(), capi.MOD_POSITION, 0, 101)       # range beyond the store
    with pytest.raises(ValueError):
        ctx.set_grid([0.0, 1.0], [0.0, 1.0], [10.0, 20.0])     # levels must decrease
    with pytest.raises(capi.LifecycleError):
        ctx.sort_by_box(0, 10)                                 # sort needs met
    ctx.close()


def test_run_steps_arguments(m):
    """lt_run_steps: nsteps < 1 and faithful draws (whose stream state is per
    step on the host) are argument errors; a non-production chain runs as
    single steps and matches them."""
    capi, ms, syn, engine = m["capi"], m["ms"], m["syn"], m["engine"]
    m0, m1 = syn.analytic_pair(dlon=30.0, dlat=30.0, nlev=6)
    ens = syn.particles(500, seed=2)
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(m0, m1)
    with pytest.raises(ValueError):
        e.ctx.run_steps(ms.Control(rng_mode="counter"), engine.ADV_DIFF, 0, 500, 0, 0,
                        flags=capi.RUN_RNG_INKERNEL)
    with pytest.raises(ValueError):
        e.ctx.run_steps(ms.Control(rng_mode="faithful"), engine.ADV_DIFF, 0, 500, 0, 3,
                        flags=capi.RUN_RNG_INKERNEL)
    ctl = ms.Control(rng_mode="counter")
    adv = engine.modules_mask(["advection", "position"])
    e.ctx.run_steps(ctl, adv, 0, 500, 0, 4)
    got = e.download()
    e.close()
    f = engine.Engine(device=0)
    f.upload(ens)
    f.bind_met(m0, m1)
    for k in range(4):
        f.ctx.run(ctl, adv, 0, 500, step=k)
    ref = f.download()
    f.close()
    for k in ("lon", "lat", "p", "time"):
        np.testing.assert_array_equal(getattr(got, k), getattr(ref, k))
