"""ctypes binding of liblagtrans_b200.so (include/lagtrans_b200.h).

The library is built in-tree (`paper_2211_12616_b200/_lib/`); importing this
module never falls back to a CPU path — if the library is missing the
import fails loudly and tells the caller how to build it.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "liblagtrans_b200.so"

# status codes (include/lagtrans_b200.h)
LT_OK, LT_ERR_ARG, LT_ERR_RANGE, LT_ERR_STATE, LT_ERR_CUDA, LT_ERR_NOMEM = 0, -1, -2, -3, -4, -5

# module bits
MOD_TIMESTEPS = 1 << 0
MOD_ADVECTION = 1 << 1
MOD_TURB = 1 << 2
MOD_MESO = 1 << 3
MOD_CONVECTION = 1 << 4
MOD_SEDI = 1 << 5
MOD_DECAY = 1 << 6
MOD_ISOSURF = 1 << 7
MOD_POSITION = 1 << 8
MOD_METEO = 1 << 9
MOD_ISOSURF_INIT = 1 << 10

RUN_RNG_INKERNEL = 1 << 0
RUN_DT_ARRAY = 1 << 1
RUN_WRITE_DT = 1 << 2
RUN_MODULE_CLOCKS = 1 << 3
RUN_SORT_KEYS = 1 << 4
# lt_module_cycles slots -> the reference's PHYSICS timer names (driver_cli.py:151-183)
MODULE_CLOCK_NAMES = ("module_timesteps", "generate_random_nums", "module_advection",
                      "module_diffusion_turb", "module_diffusion_meso", "module_convection",
                      "module_sedi", "module_decay", "module_isosurf", "module_position",
                      "module_meteo", "module_isosurf_init")

RNG_MODES = {"faithful": 0, "counter": 1, "philox": 2}
ISO_MODES = {"off": 0, "pressure": 1, "theta": 2}
PRECISIONS = {"exact": 0, "fast": 1}

F_TIME, F_P, F_ZETA, F_LON, F_LAT, F_Q, F_UVWP, F_ISO_VAR, F_DT = range(9)
F_RND_CONV, F_RND_TURB, F_RND_MESO, F_ID = 9, 10, 11, 12

HOME_Q, HOME_ZETA, HOME_DT, HOME_ISO = 1, 2, 4, 8

MET_F32, MET_F64 = 4, 8
MET_CLOSE_LON = 1
MET_DEVICE_SRC = 2


class LifecycleError(RuntimeError):
    """Illegal data-region transition (device_runtime.py:26-27)."""


class DeviceError(RuntimeError):
    """A CUDA failure inside liblagtrans_b200."""


class LtControl(C.Structure):
    """lt_control: kernel-relevant Control fields (model_state.py:18-45)."""
    _fields_ = [("t_stop", C.c_double), ("dt_model", C.c_double), ("met_dt", C.c_double),
                ("turb_dx", C.c_double), ("turb_dz", C.c_double), ("turb_meso", C.c_double),
                ("conv_prob", C.c_double), ("conv_p_top", C.c_double), ("p_surf", C.c_double),
                ("p_top", C.c_double), ("sedi_radius", C.c_double),
                ("sedi_density", C.c_double), ("decay_tau", C.c_double),
                ("isosurf_mode", C.c_int32), ("rng_mode", C.c_int32),
                ("rng_seed_global", C.c_uint64), ("decay_slot", C.c_int32),
                ("precision", C.c_int32)]


class LtHostSoa(C.Structure):
    """lt_host_soa: host particle rows for lt_run_host."""
    _fields_ = [("time", C.c_void_p), ("p", C.c_void_p), ("lon", C.c_void_p),
                ("lat", C.c_void_p), ("uvwp", C.c_void_p), ("iso_var", C.c_void_p),
                ("q", C.c_void_p), ("stride", C.c_int64), ("nq", C.c_int32)]


def control_struct(ctl) -> LtControl:
    """Pack any Control-like object (reference or mirror) into lt_control."""
    iso = ctl.isosurf_mode
    if iso not in ISO_MODES:
        raise ValueError(f"isosurf_mode {iso!r} not in {tuple(ISO_MODES)}")
    mode = ctl.rng_mode
    if mode not in RNG_MODES:
        raise ValueError(f"rng_mode {mode!r} not in {tuple(RNG_MODES)}")
    return LtControl(float(ctl.t_stop), float(ctl.dt_model), float(ctl.met_dt),
                     float(ctl.turb_dx), float(ctl.turb_dz), float(ctl.turb_meso),
                     float(ctl.conv_prob), float(ctl.conv_p_top), float(ctl.p_surf),
                     float(ctl.p_top), float(ctl.sedi_radius), float(ctl.sedi_density),
                     float(getattr(ctl, "decay_tau", 0.0)), ISO_MODES[iso], RNG_MODES[mode],
                     int(ctl.rng_seed_global) & 0xFFFFFFFFFFFFFFFF,
                     int(getattr(ctl, "decay_slot", -1)),
                     PRECISIONS[getattr(ctl, "precision", "exact")])


_P = C.c_void_p
_I32, _I64, _U32, _U64, _D = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
_PROTOS = {
    "lt_abi_version": ([], C.c_int),
    "lt_device_count": ([C.POINTER(_I32)], C.c_int),
    "lt_last_error": ([], C.c_char_p),
    "lt_ctx_create": ([_I32, C.POINTER(_P)], C.c_int),
    "lt_ctx_destroy": ([_P], C.c_int),
    "lt_sync": ([_P], C.c_int),
    "lt_stream": ([_P, C.POINTER(_P)], C.c_int),
    "lt_particles_alloc": ([_P, _I64, _I32, _I32], C.c_int),
    "lt_field_h2d": ([_P, _I32, _I32, _I64, _I64, _P], C.c_int),
    "lt_field_d2h": ([_P, _I32, _I32, _I64, _I64, _P], C.c_int),
    "lt_field_fill": ([_P, _I32, _I32, _I64, _I64, _D], C.c_int),
    "lt_field_devptr": ([_P, _I32, _I32, C.POINTER(_P)], C.c_int),
    "lt_ids_reset": ([_P, _I64, _I64, _I64], C.c_int),
    "lt_met_grid": ([_P, _I32, _I32, _I32, _P, _P, _P, _I32], C.c_int),
    "lt_met_load": ([_P, _I32, _D, _I32, _P, _P, _P, _P, _U32], C.c_int),
    "lt_met_load_nodes": ([_P, _I32, _D, _P, _U32], C.c_int),
    "lt_met_use": ([_P, _I32, _I32], C.c_int),
    "lt_met_copy_slot": ([_P, _I32, _P, _I32], C.c_int),
    "lt_met_broadcast": ([C.POINTER(_P), _I32, _I32, C.POINTER(_I32)], C.c_int),
    "lt_nccl_version": ([C.POINTER(_I32)], C.c_int),
    "lt_nccl_ranks": ([C.POINTER(_I32)], C.c_int),
    "lt_nccl_selftest": ([_I32, _I64], C.c_int),
    "lt_met_slot_time": ([_P, _I32, C.POINTER(_D)], C.c_int),
    "lt_clim_load": ([_P, _I32, _I32, _P, _P, _P, _P], C.c_int),
    "lt_locate_cells": ([_P, _I32, _I64, _P, _P, _P, _P], C.c_int),
    "lt_run": ([_P, C.POINTER(LtControl), _U32, _I64, _I64, _I64, _U64, _I64, _U32], C.c_int),
    "lt_run_steps": ([_P, C.POINTER(LtControl), _U32, _I64, _I64, _I64, _I32, _U32], C.c_int),
    "lt_rng_fill": ([_P, _I32, _U64, _I64, _I64, _I64], C.c_int),
    "lt_philox4x32_10": ([_P, _I32, _P, _P, _P], C.c_int),
    "lt_module_cycles": ([_P, _P, _I32], C.c_int),
    "lt_iso_counter": ([_P, C.POINTER(_I64), _I32], C.c_int),
    "lt_sort_by_box": ([_P, _I64, _I64], C.c_int),
    "lt_sort_info": ([_P, C.POINTER(_I64), C.POINTER(_I64)], C.c_int),
    "lt_set_home_rows": ([_P, _U32], C.c_int),
    "lt_field_d2h_ordered": ([_P, _I32, _I32, _I64, _I64, _I64, _P], C.c_int),
    "lt_field_h2d_ordered": ([_P, _I32, _I32, _I64, _I64, _I64, _P], C.c_int),
    "lt_timing": ([_P, _I32], C.c_int),
    "lt_last_elapsed_ms": ([_P, C.POINTER(C.c_float)], C.c_int),
    "lt_host_alloc": ([_I64, C.POINTER(_P)], C.c_int),
    "lt_host_free": ([_P], C.c_int),
    "lt_interpolate": ([_P, _I64, _P, _P, _P, _P, _P], C.c_int),
    "lt_grid_counts": ([_P, _I32, _I32, _I64, _I64, _P], C.c_int),
    "lt_group_stats": ([_P, _I32, _I64, _I64, _I64, C.POINTER(_I64), _P, _P, _P, _P], C.c_int),
    "lt_write_atm": ([C.c_char_p, _I64, _I32, _P, _P, _P, _P, _P, _P, _I64, _I32], C.c_int),
    "lt_format_double": ([_D, C.c_char_p, _I32, C.POINTER(_I32)], C.c_int),
    "lt_run_host": ([_P, C.POINTER(LtControl), _U32, _I64, _I64, _I64, _U64,
                     C.POINTER(LtHostSoa), _I64], C.c_int),
    "lt_run_host_steps": ([_P, C.POINTER(LtControl), _U32, _I64, _I64, _I32, _I64, _U64,
                           C.POINTER(LtHostSoa), _I64], C.c_int),
}
EXPORTED = tuple(_PROTOS)

_lib = None


def load(path: Path | None = None):
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(path or os.environ.get("LAGTRANS_B200_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build the CUDA library first "
            "(python -m paper_2211_12616_b200._build or __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = C.CDLL(str(path))
    variant = "LAGTRANS_B200_LIB" in os.environ   # an A/B build (tools/ab.sh) may predate
    for name, (args, res) in _PROTOS.items():      # newer entry points; the in-tree one may not
        if variant and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.lt_abi_version() != 1:
        raise ImportError("liblagtrans_b200 ABI version mismatch; rebuild the library")
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a status code onto the reference's exception types."""
    if rc == LT_OK:
        return
    msg = (_lib.lt_last_error() or b"").decode(errors="replace")
    if rc == LT_ERR_ARG:
        raise ValueError(msg)
    if rc == LT_ERR_RANGE:
        raise IndexError(msg)
    if rc == LT_ERR_STATE:
        raise LifecycleError(msg)
    if rc == LT_ERR_NOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def device_count() -> int:
    lib = load()
    n = _I32(0)
    rc = lib.lt_device_count(C.byref(n))
    if rc != LT_OK:
        return 0
    return int(n.value)
