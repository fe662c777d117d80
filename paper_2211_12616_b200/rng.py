"""Random numbers for the time step, mirroring `lagtrans.rng`
(/root/reference/pkg/src/lagtrans/rng.py:32-181).

`generate_random_nums` fills a host RandomBatch for a range on the GPU
(liblagtrans_b200 `lt_rng_fill`); the fused device step instead draws the
same numbers inside the step kernel and never materialises a batch.

Modes:
  faithful  per-device splitmix64 stream seeded mpi_rank + 83*device
            (rng.py:54-68,105-126), word k of a fill = mix(state + k*gamma)
  counter   stateless keyed splitmix64 (rng.py:129-153), bit-identical to
            the reference, including its 24-bit particle-index field
  philox    new fast mode: Philox4x32-10 keyed by (seed, step, full 32-bit
            particle id); matches the reference distributionally only
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .partition import WorkRange

GAMMA = 0x9E3779B97F4A7C15
MASK64 = 0xFFFFFFFFFFFFFFFF
STREAM_CONVECTION, STREAM_DIFF_TURB, STREAM_DIFF_MESO = 0, 1, 2


@dataclass
class RandomBatch:
    """Per-step draws, full-ensemble sized (rng.py:32-44)."""

    convection: np.ndarray
    diff_meso: np.ndarray
    diff_turb: np.ndarray


def batch_allocate(n: int) -> RandomBatch:
    return RandomBatch(np.zeros(n), np.zeros(3 * n), np.zeros(3 * n))


@dataclass
class RngState:
    mode: str
    seed_global: int = 0
    device_states: list[int] = field(default_factory=list)


def rng_seed_for(mpi_rank: int, device_id: int) -> int:
    return mpi_rank + 83 * device_id


def module_rng_init(ctl, num_devices: int) -> RngState:
    if num_devices < 1:
        raise ValueError(f"num_devices must be >= 1, got {num_devices}")
    if ctl.rng_mode == "faithful":
        return RngState("faithful", ctl.rng_seed_global,
                        [rng_seed_for(ctl.mpi_rank, d) & MASK64 for d in range(num_devices)])
    return RngState(ctl.rng_mode, ctl.rng_seed_global & MASK64)


def splitmix64_next(state: int) -> tuple[int, int]:
    """Scalar splitmix64 step (rng.py:71-77)."""
    state = (state + GAMMA) & MASK64
    z = ((state ^ (state >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31), state


def advance_faithful(state: int, n: int) -> int:
    """Device state after a faithful fill of n particles (rng.py:125)."""
    return (state + 7 * n * GAMMA) & MASK64


def generate_random_nums(rng: RngState, step_index: int, work: WorkRange, device_id: int,
                         batch: RandomBatch) -> None:
    """Fill batch entries of particles in `work` only (rng.py:156-181), on the GPU."""
    n_total = batch.image.ens.np if getattr(batch, "is_device_resident", False) \
        else len(batch.convection)
    if not (0 <= work.start <= work.end <= n_total):
        raise IndexError(f"range [{work.start}, {work.end}) outside ensemble of "
                         f"{n_total} particles")
    n = work.size
    if n == 0:
        return
    if getattr(batch, "is_device_resident", False):   # a DevicePool image's batch
        seed = rng.device_states[device_id] if rng.mode == "faithful" else rng.seed_global
        batch.image.rng_fill(rng.mode, seed, step_index, work)
        if rng.mode == "faithful":
            rng.device_states[device_id] = advance_faithful(seed, n)
        return
    from .physics import default_context
    ctx = default_context()
    if rng.mode == "faithful":
        seed = rng.device_states[device_id]
        rng.device_states[device_id] = advance_faithful(seed, n)
    else:
        seed = rng.seed_global
    ctx.ensure_capacity(work.end, with_batch=True)
    # key the draws by global index: slots [start, end) hold particles
    # [start, end) on this scratch context (another call may have left ids)
    ctx.ids_reset(work.start, n, work.start)
    ctx.rng_fill(_capi.RNG_MODES[rng.mode], seed, step_index, work.start, work.end)
    s = work.slice
    batch.convection[s] = ctx.d2h(_capi.F_RND_CONV, 0, work.start, n)
    turb = batch.diff_turb.reshape(n_total, 3)
    meso = batch.diff_meso.reshape(n_total, 3)
    turb[s] = ctx.d2h(_capi.F_RND_TURB, 0, 3 * work.start, 3 * n).reshape(n, 3)
    meso[s] = ctx.d2h(_capi.F_RND_MESO, 0, 3 * work.start, 3 * n).reshape(n, 3)
