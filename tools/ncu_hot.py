"""Summarise an ncu --set full report: per kernel, time / DRAM / stall mix and
the hottest SASS lines (needs the report to have been captured with
--import-source on and the library built with -lineinfo).

usage: python tools/ncu_hot.py report.ncu-rep [kernel-regex] [--lines N]
"""
import csv
import io
import re
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "."
    nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 12
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    h, data = rows[0], rows[2:]
    col = {k: i for i, k in enumerate(h)}
    seen = {}
    for idx, d in enumerate(data):
        name = d[col["Kernel Name"]]
        if not re.search(pat, name):
            continue
        short = name.split("(")[0]
        seen.setdefault(short, 0)
        seen[short] += 1
        if seen[short] > 1:
            continue

        def g(k):
            try:
                return float(d[col[k]].replace(",", ""))
            except Exception:
                return float("nan")
        t = g("gpu__time_duration.sum")
        rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        print(f"== {short}")
        print(f"   time {t:.1f} {h and ''}  dram read {rd} write {wr}  "
              f"sm% {g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} "
              f"dram% {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} "
              f"warps_active% {g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} "
              f"regs {g('launch__registers_per_thread'):.0f} grid {g('launch__grid_size'):.0f} "
              f"inst {g('smsp__inst_executed.sum'):.3g}")
        st = []
        for k, i in col.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(d[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except Exception:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("   stalls: " + ", ".join(f"{k}={v / tot * 100:.0f}%" for v, k in sorted(st, reverse=True)[:7]))
        src = ncu([rep, "--page", "source", "--csv", "--print-source", "sass", "-k", short.split()[-1].split("<")[0],
                   "--launch-count", "1"])
        srows = list(csv.reader(io.StringIO(src)))
        hdr_i = [i for i, r in enumerate(srows) if r and r[0] == "Address"]
        if not hdr_i:
            continue
        sh = srows[hdr_i[0]]
        sd = srows[hdr_i[0] + 1:]
        si = sh.index("Warp Stall Sampling (All Samples)")
        ei = sh.index("Instructions Executed")
        tots = sum(int(r[si]) for r in sd if len(r) > si and r[si].isdigit()) or 1
        seen_addr = set()
        top = sorted([r for r in sd if len(r) > si and r[si].isdigit()], key=lambda r: -int(r[si]))
        k = 0
        for r in top:
            if r[0] in seen_addr:
                continue
            seen_addr.add(r[0])
            print(f"     {int(r[si]) / tots * 100:5.1f}% exec={r[ei]:>9s} {r[1].strip()[:100]}")
            k += 1
            if k >= nlines:
                break


if __name__ == "__main__":
    main()
