"""Phase stamps of the standalone Quest select kernel (K2b) from a library
built with -DTW_TOPP_TRACE (tools/build_variant.sh ttrace -DTW_TOPP_TRACE):
group 0 of every CTA stamps: start, then per query head it selects: keys
loaded, k-th found, pages classified, band rescored; then union done,
compaction done.  Also reports the band pages rescored in fp64 (counters[1])."""
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
args = ap.parse_args()
cfg = CONFIGS[args.config]
B, H, G, n = cfg["B"], cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, :n], batch.V[:, :, :n])
del batch
step = make_batch(B, H, G, 16, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=2)
dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"])
q = step.q.contiguous()
if not hasattr(_lib.lib(), "tw_debug_select_strace"):
    sys.exit("library built without -DTW_TOPP_TRACE")
sbuf = (ctypes.c_ulonglong * (512 * 16))()
for rep in range(3):
    _lib.lib().tw_debug_select_strace(sbuf)
    dec.select(q)
    torch.cuda.synchronize()
    band = int(dec.bufs.counters[1])
    _lib.lib().tw_debug_select_strace(sbuf)
st = np.frombuffer(sbuf, dtype=np.uint64).reshape(512, 16).astype(np.int64)
st = st[st[:, 0] > 0]
k = int((st > 0).sum(axis=1).min())
t0 = st[:, 0].min()
res = {"config": args.config, "ctas": int(len(st)), "stamps": k,
       "span_us": round(float((st[:, k - 1].max() - t0) / 1e3), 2),
       "start_spread_us": round(float((st[:, 0].max() - t0) / 1e3), 2),
       "phase_mean_us": (np.diff(st[:, :k], axis=1) / 1e3).mean(axis=0).round(2).tolist(),
       "band_pages_total": band, "band_pages_per_head": round(band / (B * H * G), 1)}
print(json.dumps(res))
