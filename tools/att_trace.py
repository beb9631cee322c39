"""Work-item timeline of the sparse attention (K4; or, with --kernel estimate
and -DTW_EST_TRACE, the INT4 estimate K3a) from a library built with
-DTW_ATT_TRACE:
    tools/build_variant.sh atrace -DTW_ATT_TRACE
    TW_LIB_PATH=tools/_variants/atrace/libtwilight.so python tools/att_trace.py --config C2
Reports the span of the attention kernel, when the item queue drained (last
item start), the tail after it, and the number of busy warps over time."""
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
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--json", default=None)
ap.add_argument("--kernel", default="attention", choices=["attention", "estimate"])
args = ap.parse_args()
cfg = CONFIGS[args.config]
B, H, G, n = cfg["B"], cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
del batch
step = make_batch(B, H, G, 16, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=2)
dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"], chunk_tokens=args.chunk or None)
q = step.q.contiguous()
k_new, v_new = step.k_new.contiguous(), step.v_new.contiguous()
positions = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
NMAX = 32768 if args.kernel == "attention" else 65536
buf = (ctypes.c_ulonglong * (NMAX * 3))()
dbg = "tw_debug_atrace" if args.kernel == "attention" else "tw_debug_etrace"
if not hasattr(_lib.lib(), dbg):
    sys.exit("library built without -DTW_ATT_TRACE / -DTW_EST_TRACE")
res = {}
for rep in range(3):
    dec.step(q, k_new, v_new, positions=positions)
    torch.cuda.synchronize()
    getattr(_lib.lib(), dbg)(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(NMAX, 3).astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
span = float(en.max())
grid = np.linspace(0, span, 41)
busy = [int(((st <= t) & (en > t)).sum()) for t in grid]
nwarps = len(np.unique(a[:, 2]))
dur = en - st
res = {"config": args.config, "kernel": args.kernel, "chunk": dec.params.chunk_tokens, "items": int(len(a)),
       "warps": int(len(np.unique(a[:, 2]))), "span_us": round(span, 2),
       "first_start_spread_us": round(float(np.sort(st)[min(len(st) - 1, len(np.unique(a[:, 2])) - 1)]), 2),
       "last_start_us": round(float(st.max()), 2), "tail_us": round(span - float(st.max()), 2),
       "item_us": {"mean": round(float(dur.mean()), 2), "p50": round(float(np.median(dur)), 2),
                   "max": round(float(dur.max()), 2)},
       "busy_warps_over_time": busy}
print(json.dumps(res))
if args.json:
    with open(args.json, "w") as f:
        json.dump(res, f, indent=1)
