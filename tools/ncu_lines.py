"""Per-CUDA-source-line stall samples of one kernel in an ncu report
(captured with --import-source on, library built with -lineinfo).

usage: python tools/ncu_lines.py report.ncu-rep [kernel-regex] [--top N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if pat:
    args += ["-k", "regex:" + pat]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows, fname, header = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = r
        continue
    if header is None or len(r) < len(header) or r[2] != "-":
        continue
    d = dict(zip(header[4:], r[4:]))
    try:
        samples = int(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    rows.append((samples, f"{fname}:{r[0]}", r[1].strip()[:70], stalls, d.get("Instructions Executed", "")))
tot = sum(r[0] for r in rows) or 1
for s, loc, src, st, ex in sorted(rows, reverse=True)[:top]:
    mix = ", ".join(f"{k}={v * 100 // max(s, 1)}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{100 * s / tot:5.1f}% {loc:18s} inst={ex:>9s} {src:70s} [{mix}]")
if "--by-inst" in sys.argv:
    print("---- by instructions executed")
    tot_i = sum(int(r[4] or 0) for r in rows) or 1
    for s, loc, src, st, ex in sorted(rows, key=lambda r: -int(r[4] or 0))[:top]:
        print(f"{100 * int(ex) / tot_i:5.1f}% {loc:18s} inst={ex:>9s} {src:70s}")
