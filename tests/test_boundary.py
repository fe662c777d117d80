"""CPU: the C-ABI boundary and the host logic around it — no GPU, no
compute calls.

* liblagtrans_b200.so loads and exports every function include/*.h declares;
* the ctypes mirror of lt_control matches the C struct layout;
* the host-side rules (shard partition, device-count resolution, met
  bracketing, step count, control packing) follow the reference."""

import ctypes as C
import re
from pathlib import Path
from types import SimpleNamespace

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "lagtrans_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(lt_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2211_12616_b200 import _capi
    return _capi.load()


def test_header_declares_the_boundary():
    names = declared_functions()
    assert len(names) >= 30
    for must in ("lt_ctx_create", "lt_run", "lt_rng_fill", "lt_met_load", "lt_sort_by_box",
                 "lt_field_d2h_ordered", "lt_interpolate"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    raw = C.CDLL(str(ROOT / "paper_2211_12616_b200" / "_lib" / "liblagtrans_b200.so"))
    missing = [n for n in declared_functions() if not hasattr(raw, n)]
    assert not missing, f"declared in {HEADER.name} but not exported: {missing}"


def test_ctypes_prototypes_cover_the_header(lib):
    from paper_2211_12616_b200 import _capi
    assert set(declared_functions()) == set(_capi.EXPORTED)


def test_nccl_resolves_at_run_time(lib):
    """The met broadcast's NCCL is dlopen'ed (no link-time dependency): the
    library finds a libnccl here too and reports its version; no
    communicator exists before a broadcast."""
    from paper_2211_12616_b200.context import nccl_info
    info = nccl_info()
    assert info["version"] is not None and info["version"] >= 22700
    assert info["ranks"] == 0


def test_abi_version_and_no_gpu_paths(lib):
    assert lib.lt_abi_version() == 1
    n = C.c_int32(-1)
    rc = lib.lt_device_count(C.byref(n))     # no GPU here: an error code and n == 0
    assert (rc == 0 and n.value >= 0) or (rc < 0 and n.value == 0)
    h = C.c_void_p()
    if rc < 0 or n.value == 0:
        assert lib.lt_ctx_create(0, C.byref(h)) == -1          # LT_ERR_ARG
        assert b"out of range" in lib.lt_last_error()
        assert h.value is None


def test_null_context_is_a_lifecycle_error(lib):
    from paper_2211_12616_b200 import _capi
    assert lib.lt_sync(None) == _capi.LT_ERR_STATE
    with pytest.raises(_capi.LifecycleError):
        _capi.check(lib.lt_sync(None))


def test_control_struct_layout():
    from paper_2211_12616_b200 import _capi
    from paper_2211_12616_b200.model_state import Control
    assert C.sizeof(_capi.LtControl) == 13 * 8 + 2 * 4 + 8 + 2 * 4
    c = _capi.control_struct(Control(rng_mode="counter", rng_seed_global=-1, isosurf_mode="theta",
                                     decay_tau=5.0, decay_slot=5, precision="fast"))
    assert c.rng_mode == 1 and c.isosurf_mode == 2 and c.precision == 1
    assert c.rng_seed_global == 0xFFFFFFFFFFFFFFFF and c.decay_slot == 5
    with pytest.raises(ValueError):
        _capi.control_struct(Control(rng_mode="mersenne"))


def test_status_codes_map_to_reference_exceptions(lib):
    from paper_2211_12616_b200 import _capi
    for rc, exc in ((_capi.LT_ERR_ARG, ValueError), (_capi.LT_ERR_RANGE, IndexError),
                    (_capi.LT_ERR_STATE, _capi.LifecycleError),
                    (_capi.LT_ERR_NOMEM, MemoryError), (_capi.LT_ERR_CUDA, _capi.DeviceError)):
        with pytest.raises(exc):
            _capi.check(rc)
    _capi.check(_capi.LT_OK)


def test_enumerate_devices_rules():
    from paper_2211_12616_b200.device_runtime import MAX_DEVICES, enumerate_devices
    with pytest.raises(ValueError):
        enumerate_devices(0, 8)
    assert enumerate_devices(-1, 8) == 8
    assert enumerate_devices(3, 8) == 3
    assert enumerate_devices(1000, 8) == MAX_DEVICES
    assert enumerate_devices(-1, 0) == 1


def test_driver_host_rules():
    from paper_2211_12616_b200 import driver
    ctl = SimpleNamespace(t_start=0.0, t_stop=86400.0, dt_model=180.0)
    assert driver.n_steps_for(ctl) == 480
    ctl.t_stop = 100.0
    assert driver.n_steps_for(ctl) == 1
    ctl.t_stop = 0.0
    assert driver.n_steps_for(ctl) == 0
    mets = [SimpleNamespace(t_met=3600.0 * k) for k in range(4)]
    m0, m1, rest = driver.bracketing(mets, 5000.0)
    assert (m0.t_met, m1.t_met, [m.t_met for m in rest]) == (3600.0, 7200.0, [10800.0])
    m0, m1, rest = driver.bracketing(mets[:1], 0.0)
    assert m0 is m1
    with pytest.raises(ValueError):
        driver.bracketing(mets[1:], 0.0)


def test_modules_mask_order():
    from paper_2211_12616_b200 import _capi, engine
    assert engine.modules_mask(()) == _capi.MOD_TIMESTEPS
    assert engine.ADV_DIFF == engine.modules_mask(("advection", "turb", "meso", "position"))
    with pytest.raises(KeyError):
        engine.modules_mask(("teleport",))
