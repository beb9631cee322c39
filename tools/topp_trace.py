"""Per-CTA phase timestamps of topp_unit_kernel (library built with
-DTW_TOPP_TRACE by tools/trace_topp.sh):
    TW_LIB_PATH=/tmp/twtrace/libtwilight.so python tools/topp_trace.py --config C2
phases: 0 start, 1 pass-1 bins done, 2 crossings done, 3 pass 2 done, 4 resolve done, 5 compaction done"""
import argparse
import ctypes
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
args = ap.parse_args()
cfg = CONFIGS[args.config]
B, H, G, n = cfg["B"], cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"])
q = batch.q.contiguous()
pos = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
buf = (ctypes.c_ulonglong * (1024 * 8))()
for rep in range(3):
    cache.append(batch.k_new, batch.v_new, pos)
    dec.select(q)
    dec.estimate(q)
    torch.cuda.synchronize()
    _lib.lib().tw_debug_ttrace(buf)
    dec.topp()
    torch.cuda.synchronize()
    _lib.lib().tw_debug_ttrace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
rows = a[a[:, 0] > 0]
t0 = rows[:, 0].min()
print(f"ctas={len(rows)} span={(rows.max() - t0) / 1e3:.2f}us start_spread={(rows[:, 0].max() - t0) / 1e3:.2f}us")
full = rows[(rows > 0).all(axis=1)] if (rows > 0).all(axis=1).any() else None
nph = int((rows > 0).sum(axis=1).min())  # phases every CTA records
order = np.argsort(rows[0, :nph])
d = np.diff(rows[:, :nph][:, order], axis=1) / 1e3
print("slot order", order.tolist())
print("phase means us (all CTAs):", d.mean(axis=0).round(2).tolist(), " max:", d.max(axis=0).round(2).tolist())
nfull = int((rows > 0).sum(axis=1).max())
if nfull > nph:
    last = rows[(rows > 0).sum(axis=1) == nfull][:, :nfull]
    dl = np.diff(np.sort(last, axis=1), axis=1) / 1e3
    print("CTAs with all phases:", len(last), "phase means us:", dl.mean(axis=0).round(2).tolist())
