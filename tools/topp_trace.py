"""Per-CTA phase timestamps of the top-p kernels (library built with
-DTW_TOPP_TRACE, see tools/trace_topp.sh):  TW_LIB_PATH=/tmp/twtrace/libtwilight.so
python tools/topp_trace.py --config C2"""
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
out = torch.empty(B, H * G, 128, device="cuda")
NT = 8192
buf = (ctypes.c_ulonglong * (3 * NT * 8))()
for rep in range(3):
    cache.append(batch.k_new, batch.v_new, pos)
    dec.select(q)
    dec.estimate(q)
    torch.cuda.synchronize()
    _lib.lib().tw_debug_ttrace(buf)  # clear
    dec.topp()
    torch.cuda.synchronize()
    _lib.lib().tw_debug_ttrace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(3, NT, 8).astype(np.int64)
t0 = a[a > 0].min()
for k, name in enumerate(["hist", "union", "resolve"]):
    x = a[k]
    rows = x[x[:, 0] > 0]
    if not len(rows):
        continue
    last = np.array([r[r > 0].max() for r in rows])
    print(f"{name}: ctas={len(rows)} first_start={(rows[:, 0].min() - t0) / 1e3:.2f}us "
          f"last_end={(last.max() - t0) / 1e3:.2f}us  cta_dur mean={(last - rows[:, 0]).mean() / 1e3:.2f} "
          f"max={(last - rows[:, 0]).max() / 1e3:.2f}")
    nph = int((rows > 0).sum(axis=1).max())
    ok = rows[(rows[:, :nph] > 0).all(axis=1)]
    if len(ok):
        order = np.argsort(ok[0, :nph])  # phases in time order (trace slots need not be)
        print("   phase slots in time order:", order.tolist())
        d = np.diff(ok[:, :nph][:, order], axis=1) / 1e3
        print("   phase means us:", d.mean(axis=0).round(2).tolist(), " max:", d.max(axis=0).round(2).tolist(),
              f"(n={len(ok)})")
st = dec.stats()
print("cand tokens/unit", float(st.cand_pages.float().mean()) * 16, "final/unit", float(st.group_b1.float().mean()))
