"""Distribution of fast-vs-exact run differences over 24 h (480 steps):
    python tools/fast_error.py [counter|philox] [cfg2|cfg3]
(cfg2: the test's 1 deg shape; cfg3: the headline 0.25 deg x 137 grid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_12616_b200 import engine, synthetic  # noqa: E402
from paper_2211_12616_b200 import model_state as ms  # noqa: E402


def run(ctl, m0, m1, ens, steps, sort_every=40):
    e = engine.Engine(device=0)
    e.upload(ens)
    e.bind_met(m0, m1)
    for step in range(steps):
        if sort_every and step % sort_every == 0:
            e.sort()
        e.step(ctl, step, engine.ADV_DIFF)
    out = e.download()
    e.close()
    return out


mode = sys.argv[1] if len(sys.argv) > 1 else "counter"
shape = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
if shape == "cfg3":   # the headline grid: 0.25 deg x 137 levels, 1e6 particles
    m0, m1 = synthetic.analytic_pair(0.25, 0.25, 137, 0.0, 10800.0, p_min=0.01)
    ens = synthetic.particles(1_000_000, seed=21)
else:                 # the test's shape: 1 deg x 60 levels, 2e5 particles
    m0, m1 = synthetic.analytic_pair(1.0, 1.0, 60, 0.0, 10800.0)
    ens = synthetic.particles(200_000, seed=21)
kw = dict(t_stop=86400.0, dt_model=180.0, met_dt=10800.0, rng_mode=mode, rng_seed_global=5)
print("rng", mode, "shape", shape)
ex = run(ms.Control(**kw), m0, m1, ens, 480)
fa = run(ms.Control(precision="fast", **kw), m0, m1, ens, 480)
rp = np.abs(fa.p - ex.p) / ex.p
dlon = np.abs((fa.lon - ex.lon + 180.0) % 360.0 - 180.0) / 360.0
dlat = np.abs(fa.lat - ex.lat) / 180.0
for name, a in (("p", rp), ("lon", dlon), ("lat", dlat)):
    print(name, "max %.3e p99.99 %.3e p99 %.3e median %.3e" % (
        a.max(), np.quantile(a, 0.9999), np.quantile(a, 0.99), np.median(a)))
k = int(np.argmax(rp))
print("worst p particle", k, "init", ens.lon[k], ens.lat[k], ens.p[k], "final exact", ex.lon[k],
      ex.lat[k], ex.p[k], "fast", fa.p[k])
