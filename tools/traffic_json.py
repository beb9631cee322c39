"""Per-stage DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum per
launch) from an ncu --set full report, keyed like bench.py's stages; merged
into profiles/ncu_traffic.json (bench.py reads it for roofline.traffic).

usage: python tools/traffic_json.py report.ncu-rep CONFIG"""
import csv
import io
import json
import os
import subprocess
import sys

STAGES = {
    "K1_append": ["append_kernel"],
    "K2_select": ["quest_filter", "quest_select"],
    "K3a_estimate": ["estimate_kernel"],
    "K3bc_topp": ["topp_unit", "topp_head"],
    "K4_attention": ["attn_kernel", "merge_kernel"],
    "K4a_attn_kernel": ["attn_kernel"],
    "K23_unit": ["unit_step"],
}

rep, cfg = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[0], rows[2:]
col = {k: i for i, k in enumerate(h)}
first = {}
for d in data:
    name = d[col["Kernel Name"]]
    if name in first:
        continue
    b = sum(float(d[col[m]].replace(",", "")) * (1e6 if u == "Mbyte" else 1e9 if u == "Gbyte" else 1e3 if u == "Kbyte" else 1)
            for m, u in ((m, rows[1][col[m]]) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum")))
    first[name] = b
res = {}
for st, pats in STAGES.items():
    tot = sum(v for k, v in first.items() if any(p in k for p in pats) and "DENSE" not in k and ", 1>" not in k)
    if tot:
        res[st] = round(tot)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
allres = json.load(open(path)) if os.path.exists(path) else {}
allres[cfg] = res
json.dump(allres, open(path, "w"), indent=1)
print(json.dumps(res))
