"""Per-source-line executed warp instructions of one kernel in an ncu report
(--import-source on, -lineinfo build): where a kernel's instruction budget goes.
usage: python tools/ncu_inst_lines.py report.ncu-rep kernel-regex [N]"""
import csv
import io
import os
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{pat}", "--launch-count", "1"], capture_output=True, text=True).stdout
fname, hdr, items, tot = "?", None, [], 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        n = int(r[hdr["Instructions Executed"]])
    except ValueError:
        continue
    if r[2] != "-":  # sass rows
        continue
    tot += n
    items.append((n, f"{fname}:{r[0]}", r[1][:110]))
items.sort(reverse=True)
print(f"total warp instructions {tot:.3e}")
for n, loc, src in items[:N]:
    print(f"{100 * n / max(tot, 1):5.1f}% {n:10d}  {loc:28s} {src}")

# per file totals (the phases of a fused kernel live in different files / line ranges)
by = {}
for n, loc, _ in items:
    f, ln = loc.rsplit(":", 1)
    key = f
    if f == "unit.cu":
        ln = int(ln)
        key = "unit.cu filter" if ln < 180 else "unit.cu estimate" if ln < 300 else "unit.cu kernel"
    by[key] = by.get(key, 0) + n
print("by file / phase:")
for k, v in sorted(by.items(), key=lambda x: -x[1]):
    print(f"  {100 * v / max(tot, 1):5.1f}%  {v:.3e}  {k}")
