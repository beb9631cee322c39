"""Per-CTA phase timestamps of the fused per-unit kernel (csrc/unit.cu) from a
library built with -DTW_UNIT_TRACE:
    tools/build_variant.sh utrace -DTW_UNIT_TRACE
    TW_LIB_PATH=tools/_variants/utrace/libtwilight.so python tools/unit_trace.py --config C2
phases: 0 start, 1 filter done (+ K1), 2 select done, 3 estimate done, 4 top-p done."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, TAUS  # noqa: E402
from paper_2502_02770_b200 import _lib  # noqa: E402
from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for  # noqa: E402
from paper_2502_02770_b200.workload import make_batch, tau_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--json", default=None)
args = ap.parse_args()
cfg = CONFIGS[args.config]
B, H, G, n = cfg["B"], cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
del batch
step = make_batch(B, H, G, 16, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=2)
dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"])
assert dec.unit_path
q = step.q.contiguous()
buf = (ctypes.c_ulonglong * (4096 * 8))()
res = {}
tbuf = (ctypes.c_ulonglong * (1024 * 8))()
sbuf = (ctypes.c_ulonglong * (512 * 16))()
ttrace = hasattr(_lib.lib(), "tw_debug_unit_ttrace")
utrace = hasattr(_lib.lib(), "tw_debug_utrace")  # absent in the normal build (e.g. under ncu)
for rep in range(4):
    dec.select_estimate_topp(q)
    torch.cuda.synchronize()
    if utrace:
        _lib.lib().tw_debug_utrace(buf)
    if ttrace:
        _lib.lib().tw_debug_unit_ttrace(tbuf)
        _lib.lib().tw_debug_unit_strace(sbuf)
if not utrace:
    sys.exit(0)
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)[:, :5]
rows = a[a[:, 0] > 0]
t0 = rows[:, 0].min()
d = np.diff(rows, axis=1) / 1e3
res = {"config": args.config, "ctas": int(len(rows)), "span_us": float((rows[:, 4].max() - t0) / 1e3),
       "start_spread_us": float((rows[:, 0].max() - t0) / 1e3),
       "end_first_us": float((rows[:, 4].min() - t0) / 1e3),
       "phases": ["filter+K1", "select", "estimate", "topp"],
       "phase_mean_us": d.mean(axis=0).round(2).tolist(), "phase_max_us": d.max(axis=0).round(2).tolist(),
       "phase_min_us": d.min(axis=0).round(2).tolist(),
       "cta_total_mean_us": float(((rows[:, 4] - rows[:, 0]) / 1e3).mean())}
if ttrace:  # top-p body stamps TT(0..5): start, pass 1, crossings, pass 2, resolve, compaction
    tt = np.frombuffer(tbuf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)[:, :6]
    tt = tt[(tt[:, :6] > 0).all(axis=1)]
    res["topp_phases"] = ["pass1", "crossing", "pass2", "resolve", "compaction"]
    res["topp_phase_mean_us"] = (np.diff(tt, axis=1) / 1e3).mean(axis=0).round(2).tolist()
    tt8 = np.frombuffer(tbuf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
    row = tt8[0]
    res["topp_cta0_stamps_us"] = ((row - row[0]) / 1e3).round(2).tolist()  # slots 0..7 (6: crossing start, 7: crossing end, head group 0)
    st = np.frombuffer(sbuf, dtype=np.uint64).reshape(512, 16).astype(np.int64)
    st = st[st[:, 0] > 0]
    k = int((st > 0).sum(axis=1).min())
    res["select_phase_mean_us"] = (np.diff(st[:, :k], axis=1) / 1e3).mean(axis=0).round(2).tolist()
print(json.dumps(res))
if args.json:
    with open(args.json, "w") as f:
        json.dump(res, f, indent=1)
