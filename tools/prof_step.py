"""One C2-shaped layer (or --config) run stage by stage, for ncu captures.

    ncu --set full -k regex:attn_kernel -c 2 -o gpurun_out/attn python tools/prof_step.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS, TAUS  # noqa: E402
from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for  # noqa: E402
from paper_2502_02770_b200.workload import make_batch, tau_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--dense", action="store_true")
ap.add_argument("--batch", type=int, default=0)
args = ap.parse_args()
cfg = CONFIGS[args.config]
B = args.batch or cfg["B"]
H, G, n = cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"])
q = batch.q.contiguous()
pos = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
out = torch.empty(B, H * G, 128, device="cuda")
from paper_2502_02770_b200 import _lib as _lib0  # noqa: E402
for _ in range(args.reps):
    cache.append(batch.k_new, batch.v_new, pos)
    if dec.unit_path:
        dec.select_estimate_topp(q)
    else:
        dec.select(q)
        dec.estimate(q)
        dec.topp()
    dec.attend(q, out)
    if args.dense:
        dec.dense(q, out)
    if _ < args.reps - 1 and hasattr(_lib0.lib(), "tw_debug_strace"):  # keep the last (warm) step's trace
        import ctypes
        _lib0.lib().tw_debug_strace((ctypes.c_ulonglong * (512 * 16))())
torch.cuda.synchronize()
if os.environ.get("TW_LIB_PATH") and hasattr(__import__("paper_2502_02770_b200._lib", fromlist=["lib"]).lib(), "tw_debug_strace"):
    import ctypes
    import numpy as np
    from paper_2502_02770_b200 import _lib
    buf2 = (ctypes.c_ulonglong * (512 * 16))()
    _lib.lib().tw_debug_strace(buf2)
    s = np.frombuffer(buf2, dtype=np.uint64).reshape(512, 16).astype(np.int64)
    units = cache.num_seqs * cache.num_kv_heads
    s = s[:units]
    nph = int((s > 0).sum(axis=1).max())
    d = np.diff(s[:, :nph], axis=1)
    print("select phases us (mean):", (d.mean(axis=0) / 1000).round(2).tolist())
    print("select phases us (max):", (d.max(axis=0) / 1000).round(2).tolist())
    print("select span us:", (s[:, nph - 1].max() - s[:, 0].min()) / 1000)
st = dec.stats()
print("cand tokens/unit", float(st.cand_pages.float().mean()) * 16, "final/unit", float(st.group_b1.float().mean()),
      "rescored pages", int(dec.bufs.counters[1]))
