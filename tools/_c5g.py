import os, sys, torch
sys.path.insert(0, os.getcwd())
from bench import TAUS
from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for
from paper_2502_02770_b200.workload import make_batch, tau_schedule
B, H, G, n, Lr = int(sys.argv[1]), 8, 4, int(sys.argv[2]), int(sys.argv[3])
decs, shared = [], None
for l in range(Lr):
    cache = PagedKVCache(B, H, G, pages_for(n), dtype=torch.bfloat16)
    batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=1 + l)
    cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
    del batch
    d = TwilightDecoder(cache, "quest", budget=n // 4, p=0.9, bufs=shared)
    shared = d.bufs
    decs.append(d)
step = make_batch(B, H, G, 16, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=99)
q, kn, vn = step.q.contiguous(), step.k_new.contiguous(), step.v_new.contiguous()
pos = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
out = torch.empty(B, H * G, 128, device="cuda")
for p in (0.9, 0.8, 0.85):
    for d in decs:
        d.params.p = p
    for i, d in enumerate(decs):
        d.step(q, kn, vn, pos, out)
        torch.cuda.synchronize()
        print("eager ok", p, i, flush=True)
    gs = []
    for d in decs:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            d.step(q, kn, vn, pos, out)
        gs.append(g)
    for r in range(4):
        gs[r % Lr].replay()
        torch.cuda.synchronize()
        print("replay ok", p, r, flush=True)
