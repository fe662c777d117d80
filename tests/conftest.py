"""Shared fixtures: golden-vector loading and reference-shaped inputs.

Nothing here reads /root/reference — the golden vectors under
tests/golden/ were produced there once (tests/golden/make_golden.py)."""

from __future__ import annotations

import os
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

from oracle import lagtrans_oracle as orc  # noqa: E402


def _ensure_library():
    """Build liblagtrans_b200.so in-tree when a fresh checkout lacks it (it
    is git-ignored); nvcc cross-compiles for sm_100a without a GPU."""
    lib = ROOT / "paper_2211_12616_b200" / "_lib" / "liblagtrans_b200.so"
    if lib.exists():
        return
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_lt_build", ROOT / "paper_2211_12616_b200" / "_build.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()


_ensure_library()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name: str):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def snapshot_from(g, prefix) -> orc.Snapshot:
    f = lambda k: np.asarray(g[f"{prefix}_{k}"], dtype=np.float64)
    return orc.Snapshot(float(g[f"{prefix}_t"]), f("lons"), f("lats"), f("levs"),
                        f("u"), f("v"), f("w"), f("T"))


def control(**kw):
    """A Control-like namespace with the reference defaults
    (model_state.py:18-45) plus the decay extension."""
    base = dict(np_max=100000, nq=5, t_start=0.0, t_stop=86400.0, dt_model=180.0,
                met_dt=21600.0, turb_dx=50.0, turb_dz=0.1, turb_meso=0.16,
                conv_prob=0.0, conv_p_top=300.0, p_surf=1013.25, p_top=10.0,
                sedi_radius=0.0, sedi_density=1000.0, isosurf_mode="off",
                mpi_rank=0, num_devices_requested=-1, rng_mode="faithful",
                rng_seed_global=0, output_dt=3600.0, grid_nx=36, grid_ny=18,
                ens_group_slot=-1, decay_tau=0.0, decay_slot=-1)
    base.update(kw)
    return SimpleNamespace(**base)


def modules_ctl():
    """The Control used by make_golden.gen_modules."""
    return control(np_max=10**6, t_stop=9000.0, met_dt=10800.0, turb_dx=50.0,
                   turb_dz=0.1, turb_meso=0.16, conv_prob=0.3, conv_p_top=300.0,
                   sedi_radius=5e-6, sedi_density=2000.0, isosurf_mode="theta",
                   rng_mode="counter", rng_seed_global=12616)


def chain_ctl():
    """The Control used by make_golden.gen_chain."""
    return control(np_max=10**6, t_stop=9000.0, dt_model=180.0, met_dt=10800.0,
                   turb_dx=50.0, turb_dz=0.1, turb_meso=0.16, conv_prob=0.05,
                   sedi_radius=1e-6, isosurf_mode="theta", rng_mode="counter",
                   rng_seed_global=4242)


@pytest.fixture(scope="session")
def golden_modules():
    return load_golden("modules")


@pytest.fixture(scope="session")
def golden_interp():
    return load_golden("interp")


@pytest.fixture(scope="session")
def golden_rng():
    return load_golden("rng")


@pytest.fixture(scope="session")
def golden_chain():
    return load_golden("chain")


@pytest.fixture(scope="session")
def golden_sbr():
    return load_golden("sbr")


def hires_met_pair(g, phases=(0.0, 5.0), lon_scale=20.0, periodic=False):
    """The met of hires.npz (0.25 deg x 137-level window) or deg1.npz (global
    1 deg x 60, closed by met_periodic): rebuilt from the stored axes by
    tests/golden/hires_met.py (the fields are too large to commit), checked
    byte for byte against the digest of the fields the reference ran on."""
    sys.path.insert(0, str(GOLDEN))
    import hires_met as hm
    lons, lats, levs = g["lons"], g["lats"], g["levs"]
    snaps = []
    for t, phase, dig in ((0.0, phases[0], "digest0"), (10800.0, phases[1], "digest1")):
        f = hm.fields(lons, lats, levs, phase, lon_scale=lon_scale)
        assert hm.fields_digest(f) == str(g[dig]), "golden met rebuilt differently"
        snap = orc.Snapshot(t, lons, lats, levs, f["u"], f["v"], f["w"], f["T"])
        snaps.append(orc.close_longitudes(snap) if periodic else snap)
    return snaps


STAGES = ("in", "timesteps", "isoinit", "advection", "turb", "meso", "convection", "sedi",
          "preiso", "isosurf", "preposition", "position", "meteo", "isopressure")


def restore_stages(g):
    """Undo make_golden.dedupe_stages: a stage's missing array is the
    previous stage's."""
    out = dict(g)
    for f in ("time", "p", "zeta", "lon", "lat", "q", "uvwp", "iso", "dt"):
        prev = None
        for tag in STAGES:
            k = f"{tag}_{f}"
            if k in out:
                prev = out[k]
            elif prev is not None:
                out[k] = prev
    return out


def golden_module_set(name):
    """(golden dict, Control, met0, met1) of a module-pairs fixture:
    "modules" (10 x 5 deg x 20, modules.npz), "hires" (the headline
    0.25 deg x 137-level shape, hires.npz) or "deg1" (cfg1/cfg2's global
    1 deg x 60 grid, deg1.npz); keys under "mod_" in the last two."""
    if name == "modules":
        g = load_golden("modules")
        return g, modules_ctl(), snapshot_from(g, "m0"), snapshot_from(g, "m1")
    h = load_golden(name)
    g = restore_stages({k[4:]: v for k, v in h.items() if k.startswith("mod_")})
    if name == "hires":
        m0, m1 = hires_met_pair(h)
    else:   # deg1
        m0, m1 = hires_met_pair(h, phases=(0.0, 7.0), lon_scale=180.0, periodic=True)
    return g, modules_ctl(), m0, m1


def hires_chain_ctl():
    """The Control of make_golden.gen_hires's 20-step production chain."""
    return control(np_max=10**6, t_stop=86400.0, dt_model=180.0, met_dt=10800.0,
                   turb_dx=50.0, turb_dz=0.1, turb_meso=0.16, rng_mode="counter",
                   rng_seed_global=2211)


@pytest.fixture(scope="session")
def golden_hires():
    g = load_golden("hires")
    return g, hires_met_pair(g)


os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
