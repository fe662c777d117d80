"""CPU: bench.py's reference arm keeps the driver's contract without any
product code in the process — the oracle port on the host's cores, the
same metric/config keys as the B200 arm, and `product_code_loaded` false
(its inputs come from synthetic.py / model_state.py loaded without the
package __init__ that maps liblagtrans_b200.so)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_line_without_product_code():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1",
                        "--steps", "3", "--warmup", "3", "--cpu-sample", "5000"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["product_code_loaded"] is False
    assert d["metric"].startswith("particle-steps/s")
    assert d["unit"] == "particle-steps/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "cfg1" and d["config"]["particles"] == 100_000
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
