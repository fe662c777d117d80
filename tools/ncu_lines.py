"""Per-source-line stall samples and instructions from an ncu report
(cuda,sass view).  python tools/ncu_lines.py rep.ncu-rep [top] [particles]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
npart = float(sys.argv[3]) if len(sys.argv) > 3 else 1e8
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname = None
recs = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[2] != "-":    # sass rows carry an address; cuda rows have "-"
        continue
    try:
        recs.append((int(r[4]), int(r[7]), fname, r[0], r[1][:90]))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in recs) or 1
print(f"{'stall%':>7} {'instr/p':>8}  line")
for st, ins, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{100*st/tot:7.2f} {32*ins/npart:8.1f}  {f}:{ln}  {src}")
