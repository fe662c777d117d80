"""GPU: output-side statistics (write_grid / write_ens, output.py:28-64)
reduced in HBM, against the reference's own CSV output (golden) and the
oracle."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import lagtrans_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    from paper_2211_12616_b200 import model_state as ms
    g = load_golden("output")
    ens = ms.ParticleEnsemble(np=g["ens_p"].size, time=g["ens_time"].copy(), p=g["ens_p"].copy(),
                              zeta=g["ens_zeta"].copy(), lon=g["ens_lon"].copy(),
                              lat=g["ens_lat"].copy(), q=g["ens_q"].copy())
    ctl = ms.Control(grid_nx=int(g["grid_nx"]), grid_ny=int(g["grid_ny"]),
                     ens_group_slot=int(g["slot"]), nq=6)
    return g, ens, ctl


def test_write_grid_byte_identical_to_reference(gold, tmp_path):
    from paper_2211_12616_b200 import output
    g, ens, ctl = gold
    output.write_grid(ctl, ens, tmp_path / "grid.csv")
    assert (tmp_path / "grid.csv").read_text() == str(g["grid_csv"])


def test_group_stats_match_reference(gold, tmp_path):
    from paper_2211_12616_b200 import output
    g, ens, ctl = gold
    gids, cnts, means, stds = output.group_stats(ctl, ens)
    og, oc, om, osd = orc.grouped_moments(ens.q[5], ens.lon, ens.lat, ens.p)
    np.testing.assert_array_equal(gids, og)
    np.testing.assert_array_equal(cnts, oc)
    np.testing.assert_allclose(means, om, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(stds, osd, rtol=1e-10, atol=1e-12)
    point = list(gids).index(7)                 # ten particles at one point
    assert stds[:, point].tolist() == [0.0, 0.0, 0.0]
    assert means[:, point].tolist() == [5.0, 6.0, 700.0]
    output.write_ens(ctl, ens, tmp_path / "ens.csv")
    got = [r.split(",") for r in (tmp_path / "ens.csv").read_text().splitlines()]
    ref = [r.split(",") for r in str(g["ens_csv"]).splitlines()]
    assert got[0] == ref[0] and [r[:2] for r in got] == [r[:2] for r in ref]
    np.testing.assert_allclose(np.array([r[2:] for r in got[1:]], float),
                               np.array([r[2:] for r in ref[1:]], float), rtol=1e-10, atol=1e-12)


def test_errors_follow_reference(gold):
    from paper_2211_12616_b200 import output
    g, ens, ctl = gold
    bad = type(ctl)(**{**vars(ctl), "ens_group_slot": -1})
    with pytest.raises(ValueError):
        output.group_stats(bad, ens)
    q = ens.q.copy()
    q[5, 3] = -2.0
    ens2 = type(ens)(ens.np, ens.time, ens.p, ens.zeta, ens.lon, ens.lat, q)
    with pytest.raises(ValueError):
        output.group_stats(ctl, ens2)


def test_statistics_invariant_to_box_sort_and_sharding(gold):
    """Device images: a sorted shard gives the same counts and bitwise the
    same moments (groups reduced in particle-id order); 3 shards merge to
    the single-shard numbers."""
    from paper_2211_12616_b200 import device_runtime as dr
    from paper_2211_12616_b200 import model_state as ms
    from paper_2211_12616_b200 import output, synthetic
    from paper_2211_12616_b200.partition import partition_all
    g, ens, ctl = gold
    m0, m1 = synthetic.analytic_pair(dlon=10.0, dlat=5.0, nlev=12)
    host = dr.ModelImage(ctl=ctl, ens=ens, cache=ms.cache_allocate(ens.np), clim=ms.read_clim(),
                         met0=m0, met1=m1, dt=np.zeros(ens.np), batch=None)
    with dr.DevicePool(1) as pool:
        r = pool.region_create(0, host, None, with_batch=False)
        pool.region_update_device(r, host, ("ens", "met0", "met1"))
        before = output.group_stats(ctl, r.image.ens)
        counts0 = output.grid_counts(ctl, r.image.ens)
        pool.dispatch(0, r.image.engine.sort).result()
        after = output.group_stats(ctl, r.image.ens)
        for a, b in zip(before, after):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(output.grid_counts(ctl, r.image.ens), counts0)
    ranges = partition_all(ens.np, 3)
    with dr.DevicePool(3) as pool:
        for d in range(3):
            rr = pool.region_create(d, host, ranges[d], with_batch=False)
            pool.region_update_device(rr, host, ("ens",))
        np.testing.assert_array_equal(output.pool_grid_counts(ctl, pool), counts0)
        gids, cnts, means, stds = output.pool_group_stats(ctl, pool)
    np.testing.assert_array_equal(gids, before[0])
    np.testing.assert_array_equal(cnts, before[1])
    np.testing.assert_allclose(means, before[2], rtol=1e-12)
    np.testing.assert_allclose(stds, before[3], rtol=1e-9, atol=1e-12)


def test_grid_counts_large_grid_uses_global_bins():
    """0.1 deg bins (3600 x 1800 > shared memory) through the global-atomic kernel."""
    from paper_2211_12616_b200 import model_state as ms
    from paper_2211_12616_b200 import output, synthetic
    ens = synthetic.particles(200_000, seed=8, lat_span=90.0)
    ctl = ms.Control(grid_nx=3600, grid_ny=1800)
    np.testing.assert_array_equal(output.grid_counts(ctl, ens),
                                  orc.bin_counts(ens.lon, ens.lat, 3600, 1800))
