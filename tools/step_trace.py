"""Where one graph-captured decode step's time goes, kernel by kernel, from a
library built with all device stamps:
    nvcc ... -DTW_ATT_TRACE -DTW_EST_TRACE -DTW_TOPP_TRACE  (tools/_variants/strace)
    TW_LIB_PATH=tools/_variants/strace/libtwilight.so python tools/step_trace.py --config C1
Spans (globaltimer, relative to the select's first CTA): select, estimate
items, top-p CTAs, attention items; the gaps between them are launch / PDL /
drain time.  The filter (before the select) and the merge (after the
attention) carry no stamps."""
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
ap.add_argument("--config", default="C1")
args = ap.parse_args()
cfg = CONFIGS[args.config]
B, H, G, n = cfg["B"], cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
lib = _lib.lib()
for f in ("tw_debug_atrace", "tw_debug_etrace", "tw_debug_select_strace", "tw_debug_ttrace"):
    if not hasattr(lib, f):
        sys.exit(f"library built without the trace for {f}")
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
del batch
step = make_batch(B, H, G, 16, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=2)
dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"])
q = step.q.contiguous()
k_new, v_new = step.k_new.contiguous(), step.v_new.contiguous()
positions = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
out = torch.empty(B, H * G, 128, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        dec.step(q, k_new, v_new, positions, out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    dec.step(q, k_new, v_new, positions, out)
A = (ctypes.c_ulonglong * (32768 * 3))()
E = (ctypes.c_ulonglong * (65536 * 3))()
S = (ctypes.c_ulonglong * (512 * 16))()
T = (ctypes.c_ulonglong * (1024 * 8))()
res = {"config": args.config, "steps": []}
for rep in range(4):
    for f, b in (("tw_debug_atrace", A), ("tw_debug_etrace", E), ("tw_debug_select_strace", S),
                 ("tw_debug_ttrace", T)):
        getattr(lib, f)(b)  # clear
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    for f, b in (("tw_debug_atrace", A), ("tw_debug_etrace", E), ("tw_debug_select_strace", S),
                 ("tw_debug_ttrace", T)):
        getattr(lib, f)(b)
    a = np.frombuffer(A, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
    a = a[a[:, 0] > 0]
    e = np.frombuffer(E, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
    e = e[e[:, 0] > 0]
    sl = np.frombuffer(S, dtype=np.uint64).reshape(512, 16).astype(np.int64)
    sl = sl[sl[:, 0] > 0]
    tt = np.frombuffer(T, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
    tt = tt[tt[:, 0] > 0]
    t0 = sl[:, 0].min()
    us = lambda x: round(float(x - t0) / 1e3, 2)  # noqa: E731
    res["steps"].append({
        "graph_us": round(e0.elapsed_time(e1) * 1e3, 2),
        "select": [us(sl[:, 0].min()), us(sl.max())],
        "estimate_items": [us(e[:, 0].min()), us(e[:, 1].max())],
        "topp_ctas": [us(tt[:, 0].min()), us(tt.max())],
        "attention_items": [us(a[:, 0].min()), us(a[:, 1].max())],
    })
print(json.dumps(res))
