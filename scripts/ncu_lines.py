"""Aggregate ncu warp-stall samples per CUDA source line (from `ncu -i X --page source --csv
--print-source cuda,sass`).  Usage: python scripts/ncu_lines.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
agg = defaultdict(int)
src = {}
fname = "?"
idx = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        idx = r.index("Warp Stall Sampling (All Samples)")
        continue
    if idx is None or len(r) <= idx:
        continue
    if r[0]:
        line = (fname, r[0])
        src[line] = r[1].strip()[:90]
    try:
        agg[line] += int(r[idx])
    except ValueError:
        pass
tot = sum(agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100.0 * v / tot:5.1f}% {k[0]}:{k[1]:>5}  {src.get(k, '')}")
