"""B200-native drop-in for the particle time step of `lagtrans`
(arXiv 2211.12616's multi-GPU MPTRAC design, reference at
/root/reference/pkg).

Submodules mirror the reference package for the hot path:

  physics         module_* and interpolate_met on sm_100a kernels
  rng             RandomBatch / generate_random_nums (GPU fill)
  partition       WorkRange / calc_device_workload_range (shard rule)
  model_state     Control, ParticleEnsemble, MeteoField, CacheState ...
  device_runtime  DevicePool over real GPUs (device-resident images)
  engine          fused device-resident stepping, met streaming, box sort
  context         DeviceContext: one GPU's lt_ctx (C ABI in include/)
"""

__version__ = "0.1.0"

from . import _capi

_capi.load()  # loads liblagtrans_b200.so now; raises ImportError if it was not built
