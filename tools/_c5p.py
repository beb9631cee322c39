import os, sys, torch
sys.path.insert(0, os.getcwd())
from bench import TAUS
from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for
from paper_2502_02770_b200.workload import make_batch, tau_schedule
B, H, G, n = int(sys.argv[1]), 8, 4, int(sys.argv[2])
p = float(sys.argv[3])
cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1)
cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
step = make_batch(B, H, G, 16, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=2)
dec = TwilightDecoder(cache, "quest", budget=n // 4, p=0.9)
pos = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
q = step.q.contiguous()
out = torch.empty(B, H * G, 128, device="cuda")
for pp in (0.9, p):
    dec.params.p = pp
    dec.step(q, step.k_new.contiguous(), step.v_new.contiguous(), pos, out)
    torch.cuda.synchronize()
    print("ok p", pp, dec.stats().b1.float().mean().item(), flush=True)
