"""Where does the end-to-end (host buffers) time go?  Variants of the e2e loop."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS, TAUS  # noqa: E402
from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for  # noqa: E402
from paper_2502_02770_b200.workload import make_batch, tau_schedule  # noqa: E402

cfg = CONFIGS["C2"]
B, H, G, n = cfg["B"], cfg["H"], cfg["G"], cfg["n"]
torch.cuda.set_device(0)
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"])
q, k_new, v_new = batch.q.contiguous(), batch.k_new.contiguous(), batch.v_new.contiguous()
pos = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
out = torch.empty(B, H * G, 128, device="cuda")
q_h, k_h, v_h = q.cpu().pin_memory(), k_new.cpu().pin_memory(), v_new.cpu().pin_memory()
out_h = torch.empty(out.shape).pin_memory()
print("pinned:", q_h.is_pinned(), out_h.is_pinned())
q_d, k_d, v_d = torch.empty_like(q), torch.empty_like(k_new), torch.empty_like(v_new)
dec.step(q_d, k_d, v_d, pos, out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    dec.step(q_d, k_d, v_d, pos, out)
s = torch.cuda.current_stream()


def timeit(name, body, steps=20):
    for _ in range(3):
        body()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(steps):
        body()
    e1.record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e6
    print(f"{name:40s} device {e0.elapsed_time(e1) / steps * 1e3:9.1f} us   wall {wall:9.1f} us")


timeit("graph only", lambda: g.replay())
timeit("h2d q only", lambda: q_d.copy_(q_h, non_blocking=True))
timeit("d2h out only", lambda: out_h.copy_(out, non_blocking=True))
timeit("h2d x3 + graph", lambda: (q_d.copy_(q_h, non_blocking=True), k_d.copy_(k_h, non_blocking=True),
                                  v_d.copy_(v_h, non_blocking=True), g.replay()))
timeit("graph + d2h", lambda: (g.replay(), out_h.copy_(out, non_blocking=True)))
timeit("full e2e", lambda: (q_d.copy_(q_h, non_blocking=True), k_d.copy_(k_h, non_blocking=True),
                            v_d.copy_(v_h, non_blocking=True), g.replay(), out_h.copy_(out, non_blocking=True)))
