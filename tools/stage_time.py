"""Per-stage µs of one layer step (bench.stage_breakdown) for quick A/B runs of
library variants:  TW_LIB_PATH=/path/libtwilight.so python tools/stage_time.py --config C2"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS, TAUS, stage_breakdown  # noqa: E402
from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for  # noqa: E402
from paper_2502_02770_b200.workload import make_batch, tau_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--chunk", type=int, default=0)
args = ap.parse_args()
cfg = CONFIGS[args.config]
B = args.batch or cfg["B"]
H, G, n = cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
decs = []
shared = None
for layer in range(args.layers):
    cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
    batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1 + layer)
    cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
    dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"], bufs=shared,
                          chunk_tokens=args.chunk or None)
    shared = dec.bufs
    decs.append(dec)
    q, k_new, v_new = batch.q.contiguous(), batch.k_new.contiguous(), batch.v_new.contiguous()
    del batch
pos = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
out = torch.empty(B, H * G, 128, device="cuda")
for d in decs:
    d.step(q, k_new, v_new, pos, out)
torch.cuda.synchronize()
ms = stage_breakdown(decs, q, k_new, v_new, pos, out, args.reps)
print(json.dumps({"lib": os.environ.get("TW_LIB_PATH", "in-tree"), "config": args.config, "B": B,
                  "chunk": decs[0].params.chunk_tokens,
                  "us": {k: round(v * 1e3, 2) for k, v in ms.items()},
                  "total": round(sum(ms.values()) * 1e3, 2)}))
