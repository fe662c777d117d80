"""CPU: the native write_atm (lt_write_atm) reproduces the reference's
output.write_atm bytes (output.py:17-25): Python repr() of every double."""

import math
import struct

import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def out():
    from paper_2211_12616_b200 import output
    return output


def test_format_double_matches_repr(out):
    rs = np.random.default_rng(5)
    special = [0.0, -0.0, 1e-5, 1e-4, 0.0001, 9.999e-5, 1e15, 1e16, 9999999999999998.0,
               1.2345678901234568e+17, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
               0.1, 0.3, 100.0, 123456.0, 1.5, -2.5e-7, float("inf"), float("-inf"),
               float("nan"), 86400.0, 180.0, -179.99999, 1013.25]
    bits = rs.integers(0, 2 ** 63, 20000, dtype=np.uint64) | \
        (rs.integers(0, 2, 20000, dtype=np.uint64) << np.uint64(63))
    randoms = [struct.unpack("<d", struct.pack("<Q", int(b)))[0] for b in bits]
    scaled = list(rs.standard_normal(20000) * 10.0 ** rs.integers(-30, 30, 20000))
    for x in special + randoms + scaled:
        assert out.format_double(x) == repr(float(x)), x


def test_write_atm_byte_identical_to_reference(out, tmp_path):
    from paper_2211_12616_b200 import model_state as ms
    g = load_golden("output")
    ens = ms.ParticleEnsemble(g["ens_p"].size, g["ens_time"], g["ens_p"], g["ens_zeta"],
                              g["ens_lon"], g["ens_lat"], g["ens_q"])
    out.write_atm(ens, tmp_path / "atm.csv", threads=3)
    assert (tmp_path / "atm.csv").read_text() == str(g["atm_csv"])


def test_write_atm_large_and_edge_shapes(out, tmp_path):
    from paper_2211_12616_b200 import model_state as ms
    rs = np.random.default_rng(9)
    for n, nq in ((0, 5), (1, 0), (200_003, 2)):
        f = lambda: rs.standard_normal(n) * 1e3
        ens = ms.ParticleEnsemble(n, f(), f(), f(), f(), f(), rs.standard_normal((nq, n)))
        out.write_atm(ens, tmp_path / "a.csv")
        lines = (tmp_path / "a.csv").read_text().splitlines()
        assert lines[0] == "time,p,zeta,lon,lat" + "".join(f",q{k}" for k in range(nq))
        assert len(lines) == n + 1
        for i in (0, n // 2, n - 1) if n else ():
            vals = [ens.time[i], ens.p[i], ens.zeta[i], ens.lon[i], ens.lat[i], *ens.q[:, i]]
            assert lines[1 + i] == ",".join(repr(float(v)) for v in vals)
