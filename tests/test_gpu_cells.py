"""Box-index audit: the met cell (i, j, k) every kernel uses must be the
reference's _locate cell bit for bit (physics.py:31-47 — searchsorted
(side='left') - 1, clipped, on the reversed levels), for the exact kernels
AND the fast (mixed-precision) kernels the benchmark headline runs, on the
headline 0.25 deg x 137-level grid (where the fast kernels take their
geographic-grid lookups: computed lon/lat cells, log2-guessed levels down to
0.01 hPa) and on the other grids the parity fixtures use.

The points are chosen to break a sloppy lookup: every kind of node hit
(exact node, one ulp either side, 1e-9 .. 3e-6 of a cell either side),
hull clamps, the poles, the +360 seam, plus a uniform cloud.  The oracle's
cell_of is numpy searchsorted itself (pinned in test_oracle_golden.py)."""

import numpy as np
import pytest

from oracle import lagtrans_oracle as orc

pytestmark = pytest.mark.gpu


def grid(dlon, dlat, nlev, pmin, periodic=True):
    from paper_2211_12616_b200 import synthetic
    lons, lats, levs = synthetic.grid(dlon, dlat, nlev, pmin)
    if periodic:
        lons = np.append(lons, lons[0] + 360.0)
    return lons, lats, levs


def near_nodes(axis, rs, n):
    """n coordinates on or next to random nodes of `axis`."""
    nodes = axis[rs.integers(0, axis.size, n)]
    cell = np.abs(np.diff(axis)).max()
    kind = rs.integers(0, 12, n)
    off = np.choose(kind % 6, [0.0 * nodes, 1e-9 * cell + 0 * nodes, 1e-7 * cell + 0 * nodes,
                               1e-6 * cell + 0 * nodes, 3e-6 * cell + 0 * nodes,
                               2e-5 * cell + 0 * nodes])
    sign = np.where(kind < 6, 1.0, -1.0)
    x = nodes + sign * off
    ulp = rs.integers(0, 3, n)   # also one ulp below / above the node itself
    x = np.where(ulp == 1, np.nextafter(nodes, -np.inf), x)
    x = np.where(ulp == 2, np.nextafter(nodes, np.inf), x)
    return x


def audit_points(lons, lats, levs, n=400_000, seed=12616):
    rs = np.random.default_rng(seed)
    k = n // 4
    lon = np.concatenate([rs.uniform(-180.5, 180.5, k), near_nodes(lons, rs, k),
                          near_nodes(lons, rs, k), rs.uniform(-180, 180, k)])
    lat = np.concatenate([rs.uniform(-90.5, 90.5, k), near_nodes(lats, rs, k),
                          rs.uniform(-90, 90, k), near_nodes(lats, rs, k)])
    p = np.concatenate([np.exp(rs.uniform(np.log(levs[-1] * 0.5), np.log(levs[0] * 1.1), k)),
                        near_nodes(levs, rs, k), near_nodes(levs, rs, k),
                        near_nodes(levs, rs, k)])
    # fixed edge cases: seam, poles, hull, top and bottom levels
    edge_lon = np.array([-180.0, 180.0, np.nextafter(180.0, 0), -179.75, 179.75, 0.0, -200.0, 200.0])
    edge_lat = np.array([-90.0, 90.0, np.nextafter(90.0, 0), np.nextafter(-90.0, 0), 0.0, 89.9,
                         -95.0, 95.0])
    edge_p = np.array([levs[0], levs[-1], levs[0] * 1.5, levs[-1] * 0.5, levs[1], levs[-2],
                       500.0, np.nextafter(levs[-1], 1.0)])
    lon = np.concatenate([lon, np.repeat(edge_lon, 64)])
    lat = np.concatenate([lat, np.tile(edge_lat, 64)])
    p = np.concatenate([p, np.tile(np.repeat(edge_p, 8), 8)])
    return lon, lat, p


GRIDS = {
    "0.25deg_x137 (cfg3 headline)": (0.25, 0.25, 137, 0.01),
    "1deg_x60 (cfg1/cfg2)": (1.0, 1.0, 60, 1.0),
    "10x5deg_x20 (golden fixtures)": (10.0, 5.0, 20, 1.0),
}


@pytest.fixture(scope="module")
def ctx():
    from paper_2211_12616_b200.context import DeviceContext
    c = DeviceContext(0)
    yield c
    c.close()


@pytest.mark.parametrize("name", list(GRIDS))
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_cells_bit_exact(ctx, name, precision):
    lons, lats, levs = grid(*GRIDS[name])
    ctx.set_grid(lons, lats, levs)
    lon, lat, p = audit_points(lons, lats, levs)
    snap = orc.Snapshot(0.0, lons, lats, levs, *(np.zeros((1, 1, 1)),) * 4)
    i, j, k, _, _, _ = orc.cell_of(snap, lon, lat, p)
    got = ctx.locate_cells(lon, lat, p, precision)
    bad = (got[0] != i) | (got[1] != j) | (got[2] != k)
    assert not bad.any(), (
        f"{bad.sum()} of {bad.size} cells differ from searchsorted, e.g. "
        f"lon={lon[bad][:3]}, lat={lat[bad][:3]}, p={p[bad][:3]} -> got "
        f"{got[:, bad][:, :3].T.tolist()}, want "
        f"{np.stack([i, j, k])[:, bad][:, :3].T.tolist()}")


def test_cells_non_geographic_grid(ctx):
    """Stretched lon/lat axes and linear levels: the fast kernels' general
    lookup (FAST = 1: guessed cells checked by fp32 fractions)."""
    rs = np.random.default_rng(5)
    lons = np.sort(np.unique(np.round(rs.uniform(-180, 180, 300), 3)))
    lats = np.sort(np.unique(np.round(np.sin(np.linspace(-1.5, 1.5, 151)) * 90, 4)))
    levs = np.linspace(1000.0, 5.0, 48)
    ctx.set_grid(lons, lats, levs)
    lon, lat, p = audit_points(lons, lats, levs, n=200_000, seed=9)
    snap = orc.Snapshot(0.0, lons, lats, levs, *(np.zeros((1, 1, 1)),) * 4)
    i, j, k, _, _, _ = orc.cell_of(snap, lon, lat, p)
    for precision in ("exact", "fast"):
        got = ctx.locate_cells(lon, lat, p, precision)
        bad = (got[0] != i) | (got[1] != j) | (got[2] != k)
        assert not bad.any(), f"{precision}: {bad.sum()} cells differ"
