"""CPU: host-side rules of the path, restated from the reference's own
tests — partition (test_partition.py, acceptance c3), per-device seeds
(acceptance c4), control validation (test_model_state.py), met_periodic
(ingest.py:195-207) — against the drop-in's modules."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import lagtrans_oracle as orc


def test_partition_coverage_disjoint_balanced_ordered():
    """Acceptance c3 (test_acceptance.py:121-138)."""
    from paper_2211_12616_b200.partition import partition_all

    def check(n, d):
        ranges = partition_all(n, d)
        assert ranges[0].start == 0 and ranges[-1].end == n
        for a, b in zip(ranges, ranges[1:]):
            assert a.end == b.start
        sizes = [r.size for r in ranges]
        assert max(sizes) - min(sizes) <= 1
        assert [r.device_id for r in ranges] == list(range(d))

    for n in range(0, 300):
        for d in range(1, 9):
            check(n, d)
    rs = np.random.default_rng(0)
    for _ in range(300):
        check(int(rs.integers(0, 10 ** 6)), int(rs.integers(1, 65)))


@settings(max_examples=200, deadline=None)
@given(n=st.integers(0, 10 ** 7), d=st.integers(1, 64))
def test_partition_matches_oracle(n, d):
    from paper_2211_12616_b200.partition import calc_device_workload_range
    for dev in {0, d // 2, d - 1}:
        w = calc_device_workload_range(n, d, dev)
        assert (w.start, w.end) == orc.split_range(n, d, dev)


def test_partition_rejects_bad_arguments():
    from paper_2211_12616_b200.partition import calc_device_workload_range
    with pytest.raises(ValueError):
        calc_device_workload_range(10, 0, 0)
    with pytest.raises(ValueError):
        calc_device_workload_range(10, 2, 2)


def test_seed_formula_and_injectivity():
    """Acceptance c4 (test_acceptance.py:141-148)."""
    from paper_2211_12616_b200.rng import rng_seed_for
    assert rng_seed_for(0, 0) == 0
    assert rng_seed_for(0, 1) == 83
    assert rng_seed_for(2, 3) == 251
    for rank in range(11):
        seeds = [rng_seed_for(rank, d) for d in range(8)]
        assert len(set(seeds)) == len(seeds)


def test_rng_init_and_faithful_advance():
    from paper_2211_12616_b200 import rng
    from paper_2211_12616_b200.model_state import Control
    r = rng.module_rng_init(Control(rng_mode="faithful", mpi_rank=2), 3)
    assert r.device_states == [2, 85, 168]
    r = rng.module_rng_init(Control(rng_mode="counter", rng_seed_global=-1), 2)
    assert r.seed_global == 0xFFFFFFFFFFFFFFFF
    with pytest.raises(ValueError):
        rng.module_rng_init(Control(), 0)
    # seven draws per particle per fill (rng.py:125)
    assert rng.advance_faithful(5, 3) == (5 + 21 * rng.GAMMA) & rng.MASK64
    assert rng.splitmix64_next(0)[0] == 0xE220A8397B1DCDAF


def test_validate_control_rules():
    from paper_2211_12616_b200.model_state import Control, validate_control
    assert validate_control(Control()) == []
    bad = Control(dt_model=0.0, turb_meso=1.5, p_top=2000.0, isosurf_mode="x",
                  rng_mode="y", nq=4, decay_tau=-1.0, precision="half")
    msgs = validate_control(bad)
    for frag in ("dt_model", "turb_meso", "p_top", "isosurf_mode", "rng_mode", "nq",
                 "decay_tau", "precision"):
        assert any(frag in m for m in msgs), frag


def test_met_periodic_rule():
    from paper_2211_12616_b200 import synthetic
    from paper_2211_12616_b200.model_state import MeteoField, met_periodic
    lons, lats, levs = synthetic.grid(30.0, 30.0, 4)
    f = synthetic.era5_like(lons, lats, levs)
    met = MeteoField(0.0, lons, lats, levs, f["u"], f["v"], f["w"], f["T"])
    closed = met_periodic(met)
    assert closed.lons[-1] == lons[0] + 360.0 and closed.u.shape[0] == lons.size + 1
    np.testing.assert_array_equal(closed.u[-1], closed.u[0])
    part = MeteoField(0.0, lons[:5], lats, levs, f["u"][:5], f["v"][:5], f["w"][:5], f["T"][:5])
    assert met_periodic(part) is part
    ref = orc.close_longitudes(orc.Snapshot.like(met))
    np.testing.assert_array_equal(ref.lons, closed.lons)


def test_box_keys_order_columns_then_level_pairs():
    """The sort key (Morton lon/lat column, then the pair of level cells k//2
    — two consecutive 32-byte records) is injective over such boxes, equal
    inside one, and orders columns in Z order, level boxes ascending inside a
    column."""
    from paper_2211_12616_b200 import synthetic
    lons, lats, levs = synthetic.grid(30.0, 20.0, 6)
    f = synthetic.era5_like(lons, lats, levs)
    snap = orc.close_longitudes(orc.Snapshot(0.0, lons, lats, levs, f["u"], f["v"], f["w"],
                                             f["T"]))
    nx, ny, nz = snap.lons.size, snap.lats.size, snap.levs.size
    ii, jj, kk = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1), np.arange(nz - 1), indexing="ij")
    # cell centres -> (i, j, k) through the reference locate, then keys
    lon = (snap.lons[ii] + snap.lons[ii + 1]) / 2
    lat = (snap.lats[jj] + snap.lats[jj + 1]) / 2
    rev = snap.levs[::-1]
    p = (rev[kk] + rev[kk + 1]) / 2
    keys = orc.box_keys(snap, lon.ravel(), lat.ravel(), p.ravel())
    i, j, k, *_ = orc.cell_of(snap, lon.ravel(), lat.ravel(), p.ravel())
    boxes = np.stack([i, j, k // orc.BOX_LEVELS], axis=1)
    assert np.unique(keys).size == np.unique(boxes, axis=0).shape[0]

    def morton(a, b):
        return sum(((a >> t) & 1) << (2 * t + 1) | ((b >> t) & 1) << (2 * t) for t in range(16))
    nb = (nz - 2) // orc.BOX_LEVELS + 1
    brute = np.array([morton(int(a), int(b)) * nb + int(c) // orc.BOX_LEVELS
                      for a, b, c in zip(i, j, k)])
    np.testing.assert_array_equal(keys, brute)


def test_clim_hno3_and_tropopause_lookups():
    """ClimData.hno3 / p_trop (model_state.py:165-180) against the oracle's
    restatement, including clamped coordinates and grid nodes."""
    import numpy as np
    from oracle import lagtrans_oracle as orc
    from paper_2211_12616_b200.model_state import read_clim
    clim = read_clim()
    lg, pg, tab, pt = orc.climatology_tables()
    rs = np.random.default_rng(4)
    lat = np.concatenate([rs.uniform(-100, 100, 5000), lg, [-90.0, 90.0]])
    p = np.concatenate([rs.uniform(0, 1200, 5000), pg[:lg.size], [10.0, 1000.0]])
    np.testing.assert_allclose(clim.hno3(lat, p), orc.hno3_lookup(lg, pg, tab, lat, p),
                               rtol=1e-15, atol=0)
    np.testing.assert_array_equal(clim.p_trop(lat), np.interp(lat, lg, pt))
    assert clim.hno3(90.0, 50.0) == 0.5e-8
