"""Host-buffer path throughput: copies only (timesteps module) vs the
production chain, pipelined multi-step calls, to see the PCIe ceiling."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_12616_b200 import engine, synthetic  # noqa: E402
from paper_2211_12616_b200 import model_state as ms  # noqa: E402
from paper_2211_12616_b200.context import pinned_empty  # noqa: E402

n = 50_000_000
m0, m1 = synthetic.analytic_pair(1.0, 1.0, 60, 0.0, 10800.0)
ens = synthetic.particles(n, seed=1)
h = ms.ParticleEnsemble(n, pinned_empty(n), pinned_empty(n), np.zeros(1), pinned_empty(n),
                        pinned_empty(n), np.zeros((5, 1)))
for k in ("time", "p", "lon", "lat"):
    getattr(h, k)[:] = getattr(ens, k)
cache = ms.CacheState(uvwp=pinned_empty((3, n)), iso_var=np.zeros(1))
cache.uvwp[:] = 0.0
ctl = ms.Control(t_stop=1e9, dt_model=180.0, met_dt=10800.0, rng_mode="philox", precision="fast")
e = engine.Engine(device=0)
e.bind_met(m0, m1)
for label, mods in (("copies only (timesteps)", engine.modules_mask(()) | engine.capi.MOD_MESO * 0),
                    ("adv+turb+meso", engine.ADV_DIFF)):
    for chunk in (0, 1 << 21):
        e.step_host(ctl, h, cache, 0, mods, chunk=chunk, steps=1)
        t0 = time.perf_counter()
        K = 6
        e.step_host(ctl, h, cache, 1, mods, chunk=chunk, steps=K)
        dt = (time.perf_counter() - t0) / K
        rows = 7 if mods & engine.capi.MOD_MESO else 4
        print(f"{label:26s} chunk {chunk:>8d}: {dt*1e3:7.1f} ms/step, "
              f"{rows * 8 * n / dt / 1e9:5.1f} GB/s per direction, {n / dt:.3e} particle-steps/s")
e.close()
