"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.

usage: python tools/launches.py gpurun_out/launches.csv [--json out.json]
"""
import collections
import csv
import json
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in data:
        per[r[ii]][r[mi]] = r[vi]
        per[r[ii]]["name"] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for v in per.values():
        n = v["name"].split("(")[0]
        t = float(v["gpu__time_duration.sum"].replace(",", ""))
        by = sum(float(v.get(m, "0").replace(",", "")) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        a = agg[n]
        a[0] += 1
        a[1] += t
        a[2] += by
    out = {}
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out[n] = {"launches": c, "avg_us": t / c / 1000, "avg_dram_bytes": b / c, "dram_gbs": b / t if t else 0}
    return out


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    for n, v in s.items():
        print(f"{n[:70]:70s} n={v['launches']:4d} avg_us={v['avg_us']:9.1f} avg_MB={v['avg_dram_bytes']/1e6:9.2f} GB/s={v['dram_gbs']:8.1f}")
    if "--json" in sys.argv:
        json.dump(s, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
