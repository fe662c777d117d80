"""Summarise an ncu --set full report of the step kernel: key metrics,
stall reasons and the SASS opcode mix per particle.
    python tools/ncu_summary.py gpurun_out/step_fast.ncu-rep [particles]"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
npart = float(sys.argv[2]) if len(sys.argv) > 2 else 1e8


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
m = {k: (v[i], u[i]) for i, k in enumerate(h)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
out = {}
for k in want:
    if k in m:
        out[k] = m[k][0] + " " + m[k][1]
stalls = []
for k, (val, unit) in m.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            stalls.append((float(val.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in stalls) or 1
out["stalls_pct"] = {k: round(100 * x / tot, 1) for x, k in sorted(stalls, reverse=True)[:10]}
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = sass[1]
ops = collections.Counter()
total = 0
for r in sass[2:]:
    d = dict(zip(hh, r))
    toks = d.get("Source", "").strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    n = int(d.get("Instructions Executed") or 0)
    ops[op] += n
    total += n
out["warp_instructions_per_particle"] = round(total / npart, 2)
out["thread_instructions_per_particle"] = round(32 * total / npart, 1)
out["opcode_mix_per_particle"] = {k: round(32 * n / npart, 1) for k, n in ops.most_common(24)}
print(json.dumps(out, indent=1))
