"""Regenerate profiles/ from a tools/gpu_round.sh run in gpurun_out/:
ncu summaries and line tables of the fast and exact step kernels, the
launch list, and profiles/ncu_step_cfg3.json (what bench.py reports as
roofline.traffic / roofline.issue)."""
import collections
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"

for prec in ("fast", "exact"):
    rep = OUT / f"step_{prec}.ncu-rep"
    summ = subprocess.run([sys.executable, str(ROOT / "tools/ncu_summary.py"), str(rep)],
                          capture_output=True, text=True).stdout
    (PROF / f"r02_step_{prec}_cfg3.json").write_text(summ)
    lines = subprocess.run([sys.executable, str(ROOT / "tools/ncu_lines.py"), str(rep), "40"],
                           capture_output=True, text=True).stdout
    (PROF / f"r02_step_{prec}_cfg3_lines.txt").write_text(lines)
shutil.copy(OUT / "launches.csv", PROF / "r02_launches_cfg3.csv")

out = json.loads((PROF / "ncu_step_cfg3.json").read_text())
for prec in ("fast", "exact"):
    d = json.loads((PROF / f"r02_step_{prec}_cfg3.json").read_text())
    g = lambda k: float(str(d[k]).split()[0])
    dram = (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) * 1e9
    out[prec].update(duration_ms=g("gpu__time_duration.sum"), dram_bytes_per_launch=dram,
                     dram_bytes_per_particle_step=dram / out["particles"],
                     l2_hit_rate_pct=g("lts__t_sector_hit_rate.pct"),
                     l1_hit_rate_pct=g("l1tex__t_sector_hit_rate.pct"),
                     issue_active_pct=g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     thread_instructions_per_particle=d["thread_instructions_per_particle"],
                     stalls_pct=d["stalls_pct"])
    o = out[prec]
    print(prec, f"{o['duration_ms']:.3f} ms", f"{o['dram_bytes_per_particle_step']:.1f} B/p",
          f"issue {o['issue_active_pct']:.1f} %", f"{o['thread_instructions_per_particle']} instr/p",
          f"dram {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} %",
          list(o["stalls_pct"].items())[:3])
(PROF / "ncu_step_cfg3.json").write_text(json.dumps(out, indent=1))

rows = list(csv.reader(open(PROF / "r02_launches_cfg3.csv")))
hdr, agg = None, collections.defaultdict(list)
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        e = dict(zip(hdr, r))
        if e.get("Metric Name") == "gpu__time_duration.sum":
            agg[e["Kernel Name"][:70]].append(float(e["Metric Value"].replace(",", "")))
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):4d} {sum(v) / 1e6:9.2f} ms total {sum(v) / len(v) / 1e6:8.3f} ms avg  {k}")
