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


os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
