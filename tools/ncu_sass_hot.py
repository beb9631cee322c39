"""Hottest CUDA source lines of one kernel in an ncu report, by warp-stall
samples (report captured with --import-source on, library built -lineinfo).

usage: python tools/ncu_sass_hot.py report.ncu-rep kernel-regex [N]
"""
import csv
import io
import os
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{pat}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, si, items, tot = "?", None, [], 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is None or not r[0].isdigit() or len(r) <= si:
        continue
    try:
        v = int(r[si])
    except ValueError:
        continue
    tot += v
    items.append((v, f"{fname}:{r[0]}", r[1].strip()[:100]))
items.sort(reverse=True)
print(f"total samples {tot}")
for v, loc, s in items[:N]:
    print(f"{v / max(tot, 1) * 100:5.1f}%  {loc:22s} {s}")
