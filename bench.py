"""Benchmark of the B200 Twilight decode-attention path.

Metric (BASELINE.json): sparse decode-attention microseconds per layer and
achieved HBM GB/s.  One "step" = one decode step of ONE attention layer for
the whole batch: K1 append of the new token, K2 Quest selection + GQA union,
K3 INT4 estimate + top-p + group union, K4 sparse attention (+ split-KV merge).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

N>1 is launched by torchrun (one process per GPU, NCCL); C1/C2/C4/C5-style
configs are batch-sharded (weak scaling: every rank owns its own batch, no
data-path collective), C3 is KV-head-sharded with one NCCL all-gather of the
per-head outputs.  Timing: CUDA events on the launching stream, W warm-up
steps, a barrier + synchronize on both sides of exactly K steps, max over
ranks.  Inputs larger than L2: steps rotate over `layers` independent layer
caches (each bigger than the 126 MB L2).  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

# ----------------------------------------------------------------------------- configs
# n = context length attended (after the append), B per GPU, heads, selector, budget (tokens), p
CONFIGS = {
    "C1": dict(desc="single-layer decode, Llama-3.1-8B head shape (32 q / 8 kv, d=128), batch 1, ctx 8k, "
                    "Quest page 16, p=0.95, random K/V", B=1, H=8, G=4, n=8192, selector="quest", budget=2048,
               p=0.95, layers=16, shard="batch"),
    "C2": dict(desc="Llama-3.1-8B layer shape, batch 16, ctx 32k, Quest budget 8192 + top-p p=0.95, bf16",
               B=16, H=8, G=4, n=32768, selector="quest", budget=8192, p=0.95, layers=4, shard="batch"),
    "C3": dict(desc="LongChat-7B MHA shape (32 heads, d=128), batch 8, ctx 128k, full selector + top-p p=0.9, "
                    "head-sharded", B=8, H=32, G=1, n=131072, selector="full", budget=None, p=0.9, layers=2,
               shard="head"),
    "C4": dict(desc="Llama-3.1-8B all 32 layers decode step, global batch 64, ctx 64k, batch-sharded, random-init "
                    "weights; layers 0-1 dense, others Quest n/4 + top-p p=0.95; all layers alias one physical KV "
                    "cache", B=64, H=8, G=4, n=65536, selector="quest", budget=16384, p=0.95, layers=32,
               shard="batch", model=True),
    "C5": dict(desc="Llama-3.1-8B shape, batch 32, ctx 128k, Quest n/4 + top-p (p sweep point 0.9), "
                    "focused vs diffuse heads", B=32, H=8, G=4, n=131072, selector="quest", budget=32768, p=0.9,
               layers=2, shard="batch", p_sweep=(0.8, 0.85, 0.9, 0.95, 0.99)),
}
TAUS = (0.25, 0.5, 1.0, 2.0)  # per-KV-head temperatures, cycled: focused .. diffuse
METRIC = "sparse decode-attn us/layer & achieved HBM GB/s at 32k-128k ctx, 1/2/4/8 GPU"


def load_read_peak():
    """Read-only streaming bandwidth measured by tools/microbench.cu on a B200
    (profiles/microbench_r01.json): the attention/estimate kernels only read,
    and a read stream runs above the copy (read+write) figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "microbench_r01.json")) as f:
            d = json.load(f)
        return max(v for k, v in d.items() if k.startswith("stream_read_gbs"))
    except Exception:
        return None


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json: 1 Gi bf16 copy, read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        rows = []
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:]))
            except Exception:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, flags in rows:
            for nm, fl in zip(names, flags):
                if fl.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [r[0] for r in rows if r[0] > 500] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------- our arm

def dist_setup(gpus: int):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def min_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def algorithmic_bytes(cfg, dec, n, elem=2):
    """HBM bytes one step MUST move, from the step's actual
    candidate pages U and final sets B1 (read back after timing)."""
    H, G, B = cfg["H_local"], cfg["G"], cfg["B"]
    units = B * H
    d = 128
    P = math.ceil(n / 16)
    bl = dec.bufs if isinstance(dec.bufs, list) else [dec.bufs]
    U = sum(b.cand_count.sum().item() for b in bl)  # candidate pages over all units
    F = sum(b.final_count.sum().item() for b in bl)  # surviving tokens over all units
    k1 = units * (2 * 2 * d * elem + d // 2 + 8 + 2 * 2 * d * elem)          # read k,v; write k,v,codes,params; meta RMW
    k2 = units * (P * 2 * d * elem + G * d * elem + 4 * P) if cfg["selector"] == "quest" else 0
    # K3 is unfused (estimate, then top-p): SURVEY 8(d) adds G*|U|*4*2 -- the
    # candidates' fp32 logits written by the estimate and read back by top-p
    # (|U| = U*16 candidate token slots; at C4/C5 ncu sees them reach DRAM)
    logits = G * U * 16 * 4
    k3a = U * 1152 + logits                                                   # INT4 codes + fp32 scale/zero per page, logits out
    k3bc = 4 * F + logits                                                     # logits in, final index list
    k4 = F * (2 * d * elem + 4) + units * G * d * (elem + 4)                  # gathered K,V rows + q + out
    dense = units * n * 2 * d * elem + units * G * d * (elem + 4)
    k23 = k2 + U * 1152 + 4 * F  # the fused per-unit kernel keeps the logits in L2 / on chip
    step = k1 + (k23 if getattr(dec, "unit_path", False) else k2 + k3a + k3bc) + k4
    return {"K1_append": k1, "K2_select": k2, "K3a_estimate": k3a, "K3bc_topp": k3bc, "K4_attention": k4,
            "K4a_attn_kernel": k4, "K23_unit": k23, "step": step, "K5_dense": dense, "cand_pages": U,
            "final_tokens": F, "logits_round_trip": 2 * logits}


STAGE_NAMES = ["K1_append", "K2_select", "K3a_estimate", "K3bc_topp", "K4_attention"]
# the fused per-unit kernel (tw_select_estimate_topp) runs K2 + K3 as one launch
UNIT_STAGE_NAMES = ["K1_append", "K23_unit", "K4_attention"]


def dominant_kernel(stage_ms):
    """The roofline's kernel: the longest stage; for K4 its attention kernel
    alone (K4a_attn_kernel, timed without the split-KV merge) when measured."""
    dom = max((k for k in stage_ms if k != "K4a_attn_kernel"), key=lambda k: stage_ms[k])
    return "K4a_attn_kernel" if dom == "K4_attention" and stage_ms.get("K4a_attn_kernel") else dom


def stage_names(dec):
    return UNIT_STAGE_NAMES if dec.unit_path else STAGE_NAMES


def stage_breakdown(decs, q, k_new, v_new, positions, out, reps):
    """Mean µs of each stage (K1..K4) per step: every stage captured in its own
    CUDA graph, CUDA events between replays, rotating over `decs`.  With the
    fused per-unit kernel the stages are K1, K2+K3 (one launch), K4."""
    stream = torch.cuda.current_stream()
    B = q.shape[0]
    names = stage_names(decs[0])

    def stage_fns(dec):
        if dec.unit_path:
            return [lambda: dec.cache.append(k_new, v_new, positions),
                    lambda: dec.select_estimate_topp(q),
                    lambda: dec.attend(q, out)]
        subs = [(lo, hi, s) for lo, hi, s, _ in dec.waves] if dec.waves else [(0, B, dec)]
        return [lambda: dec.cache.append(k_new, v_new, positions),
                lambda: [s.select(q[lo:hi]) for lo, hi, s in subs],
                lambda: [s.estimate(q[lo:hi]) for lo, hi, s in subs],
                lambda: [s.topp() for lo, hi, s in subs],
                lambda: [s.attend(q[lo:hi], out[lo:hi]) for lo, hi, s in subs]]
    stage_graphs = []
    for dec in decs:
        row = []
        for fn in stage_fns(dec):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            row.append(g)
        stage_graphs.append(row)
    # K4's attention kernel alone (tw_sparse_attention_part 1, no merge), on the
    # state the layer's step just produced: the roofline's kernel.  No L2 flush
    # is needed (the kernel streams ~7x the L2 in the same item order, so
    # nothing it reads early survives in L2); zeroing a flush buffer left dirty
    # lines whose write-back slowed the kernel by ~3%
    attn_graphs = None
    if not decs[0].unit_path and not decs[0].waves:
        attn_graphs = []
        for dec in decs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                dec.attend_part(q, out, 1)
            attn_graphs.append(g)
    stage_ms = {k: 0.0 for k in names}
    attn_ms = 0.0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 3)]
    for i in range(reps + 1):
        ev[0].record(stream)
        for j, g in enumerate(stage_graphs[i % len(decs)]):
            g.replay()
            ev[j + 1].record(stream)
        if attn_graphs is not None:
            ev[len(names) + 1].record(stream)
            attn_graphs[i % len(decs)].replay()
            ev[len(names) + 2].record(stream)
        torch.cuda.synchronize()
        if i == 0:
            continue
        for j, k in enumerate(names):
            stage_ms[k] += ev[j].elapsed_time(ev[j + 1]) / reps
        if attn_graphs is not None:
            attn_ms += ev[len(names) + 1].elapsed_time(ev[len(names) + 2]) / reps
    if attn_graphs is not None:
        stage_ms["K4a_attn_kernel"] = attn_ms
    return stage_ms


def head_taus(cfg, H_local, rank, world):
    """tau of every query head of this rank's decoders, in head_stats order (unit-major)."""
    H = cfg["H"]
    taus = [TAUS[h % len(TAUS)] for h in range(H)]
    if cfg["shard"] == "head":
        taus = taus[rank * H_local:(rank + 1) * H_local]
    per_unit = taus[:H_local]
    return [t for _ in range(cfg["B"]) for t in per_unit for _ in range(cfg["G"])]


def sweep_point(args, cfg, decs, q, k_new, v_new, positions, out, p, world):
    """One point of the C5 p sweep (BASELINE.json configs[4]; reference sweep_p,
    pipeline.py:465-498): µs/layer at this p and the per-head budget skew --
    B1 per head split into focused (tau 0.25) and diffuse (tau 2.0) heads."""
    old = [d.params.p for d in decs]
    for d in decs:
        d.params.p = p
    graphs = []
    for i in range(len(decs)):
        decs[i].step(q, k_new, v_new, positions, out)
    torch.cuda.synchronize()
    for i in range(len(decs)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            decs[i].step(q, k_new, v_new, positions, out)
        graphs.append(g)
    for i in range(args.warmup):
        graphs[i % len(decs)].replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        graphs[i % len(decs)].replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    st = decs[(args.steps - 1) % len(decs)].stats()
    b1 = st.b1.float().cpu()
    taus = torch.tensor(head_taus(cfg, decs[0].cache.num_kv_heads, int(os.environ.get("RANK", "0")), world))
    def summ(x):
        x = x.sort().values
        return {"min": int(x[0]), "p50": int(x[len(x) // 2]), "max": int(x[-1]), "mean": round(float(x.mean()), 1)}
    foc, dif = b1[taus == min(TAUS)], b1[taus == max(TAUS)]
    for d, v in zip(decs, old):
        d.params.p = v
    return {"p": p, "us_per_layer": round(ms * 1e3, 2), "head_b1": summ(b1),
            "focused_b1 (tau 0.25)": summ(foc), "diffuse_b1 (tau 2.0)": summ(dif),
            "skew_diffuse_over_focused_mean": round(float(dif.mean() / max(foc.mean(), 1.0)), 1),
            "group_final_tokens_mean": round(float(st.group_b1.float().mean()), 1),
            "candidate_mass_mean": round(float(st.candidate_mass.float().mean()), 6)}


def run_ours(args, cfg):
    from paper_2502_02770_b200.decode import DecodeBuffers, PagedKVCache, TwilightDecoder, pages_for
    from paper_2502_02770_b200.workload import make_batch, tau_schedule

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local if world > 1 else 0)
    B, H, G, n = cfg["B"], cfg["H"], cfg["G"], cfg["n"]
    if cfg["shard"] == "head":
        assert H % world == 0, "heads must divide over ranks"
        H_local = H // world
    else:
        H_local = H
    cfg = dict(cfg, H_local=H_local)
    dtype = torch.bfloat16
    L = args.layers or cfg["layers"]
    max_pages = pages_for(n)
    taus = tau_schedule(H, TAUS)[rank * H_local:(rank + 1) * H_local] if cfg["shard"] == "head" else tau_schedule(H, TAUS)
    seed0 = 1234 + 7919 * rank

    caches, decs = [], []
    shared = None
    for layer in range(L):
        cache = PagedKVCache(B, H_local, G, max_pages, dtype=dtype, device=dev)
        batch = make_batch(B, H_local, G, n, dtype, tau=taus, seed=seed0 + layer, device=dev)
        cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])  # the step appends token n-1
        del batch
        dec = TwilightDecoder(cache, cfg["selector"], budget=cfg["budget"], p=cfg["p"], bufs=shared,
                              waves=args.waves if B % max(args.waves, 1) == 0 else 1,
                              chunk_tokens=args.chunk or None)
        shared = dec.bufs
        caches.append(cache)
        decs.append(dec)
        torch.cuda.synchronize()
    step_in = make_batch(B, H_local, G, 16, dtype, tau=taus, seed=seed0 + 999, device=dev)
    q, k_new, v_new = step_in.q.contiguous(), step_in.k_new.contiguous(), step_in.v_new.contiguous()
    positions = torch.full((B,), n - 1, dtype=torch.int32, device=dev)
    out = torch.empty(B, H_local * G, 128, dtype=torch.float32, device=dev)
    gathered = torch.empty(world * B, H_local * G, 128, dtype=torch.float32, device=dev) if (
        cfg["shard"] == "head" and world > 1) else None
    full_out = torch.empty(B, world * H_local * G, 128, dtype=torch.float32, device=dev) if gathered is not None \
        else None

    def gather():
        # head-sharded (C3): the step ends with the all-gather of the per-rank heads, permuted
        # back to head order (dist.gather_head_outputs)
        from paper_2502_02770_b200.dist import gather_head_outputs
        gather_head_outputs(out, world, buf=gathered, out=full_out)

    # --- CUDA graphs: one graph per layer for the fused step (launch-bound otherwise)
    graphs = []
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(L):  # warm the launch path (cudaFuncSetAttribute etc.) outside capture
            decs[i].step(q, k_new, v_new, positions, out)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for i in range(L):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            decs[i].step(q, k_new, v_new, positions, out)
        graphs.append(g)
    torch.cuda.synchronize()

    def replay(i):
        graphs[i % L].replay()
        if gathered is not None:
            gather()

    for i in range(args.warmup):
        replay(i)
    torch.cuda.synchronize()
    barrier(world)

    # --- main timed region: exactly K steps
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local if world > 1 else 0) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(args.steps):
            replay(i)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local, world)
    ms_min = min_over_ranks(ms_local, world)  # per-rank imbalance (head sharding: budget skew across heads)
    clocks = clk.summary()

    # --- p sweep (C5): the same caches, one graph set per p, K timed steps each
    p_list = [float(x) for x in args.p.split(",")] if args.p else list(cfg.get("p_sweep", ()))
    sweep = [sweep_point(args, cfg, decs, q, k_new, v_new, positions, out, p, world) for p in p_list] if p_list else None

    # --- per-stage breakdown: each stage captured in its own CUDA graph, events between replays
    stage_ms = stage_breakdown(decs, q, k_new, v_new, positions, out, reps=max(3, min(args.steps, 10)))

    # --- dense decode attention (K5) on the same caches: the speedup baseline
    dense_graphs = []
    for i in range(L):
        decs[i].dense(q, out)
    torch.cuda.synchronize()
    for i in range(L):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            decs[i].dense(q, out)
        dense_graphs.append(g)
    for i in range(args.warmup):
        dense_graphs[i % L].replay()
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(args.steps):
        dense_graphs[i % L].replay()
    e1.record(stream)
    torch.cuda.synchronize()
    dense_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)

    # --- end to end through the C-ABI step with host buffers (pinned), H2D + D2H inside the timed region
    # the step's inputs travel as ONE pinned staging buffer (q | k_new | v_new), one H2D copy per step
    nq, nk = q.numel(), k_new.numel()
    inp_h = torch.cat([q.reshape(-1), k_new.reshape(-1), v_new.reshape(-1)]).cpu().pin_memory()
    inp_d = torch.empty_like(inp_h, device=q.device)
    q_d = inp_d[:nq].view(q.shape)
    k_d = inp_d[nq:nq + nk].view(k_new.shape)
    v_d = inp_d[nq + nk:].view(v_new.shape)
    res_src = full_out if full_out is not None else out  # the step's result: all heads after the gather
    out_h = torch.empty(res_src.shape, dtype=res_src.dtype).pin_memory()
    copies_in_graph = gathered is None
    if copies_in_graph:
        # single GPU: double-buffered staging, as a serving loop does it.  Step i reads input
        # buffer i%2 and writes output buffer i%2; on a copy stream the H2D of step i+1's inputs
        # overlaps step i and the D2H of step i's result overlaps step i+1.  Every step still
        # moves its own inputs in and its own result out inside the timed region.
        inp_d2 = [torch.empty_like(inp_h, device=q.device) for _ in range(2)]
        out_d2 = [torch.empty_like(out) for _ in range(2)]
        out_h2 = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
        views = [(b[:nq].view(q.shape), b[nq:nq + nk].view(k_new.shape), b[nq + nk:].view(v_new.shape))
                 for b in inp_d2]
        for b in inp_d2:
            b.copy_(inp_h)
        torch.cuda.synchronize()
        e2e_graphs = {}
        for i in range(L):
            for par in range(2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    decs[i].step(views[par][0], views[par][1], views[par][2], positions, out_d2[par])
                e2e_graphs[(i, par)] = g
        copy_s = torch.cuda.Stream(device=q.device)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def pipelined(nsteps):
            copy_s.wait_stream(stream)
            with torch.cuda.stream(copy_s):
                inp_d2[0].copy_(inp_h, non_blocking=True)
                ev_in[0].record(copy_s)
            for i in range(nsteps):
                par = i % 2
                if i + 1 < nsteps:  # next step's inputs, once step i-1 is done reading that buffer
                    with torch.cuda.stream(copy_s):
                        if i >= 1:
                            copy_s.wait_event(ev_done[1 - par])
                        inp_d2[1 - par].copy_(inp_h, non_blocking=True)
                        ev_in[1 - par].record(copy_s)
                stream.wait_event(ev_in[par])
                if i >= 2:
                    stream.wait_event(ev_out[par])  # step i-2's result has left this buffer
                e2e_graphs[(i % L, par)].replay()
                ev_done[par].record(stream)
                with torch.cuda.stream(copy_s):
                    copy_s.wait_event(ev_done[par])
                    out_h2[par].copy_(out_d2[par], non_blocking=True)
                    ev_out[par].record(copy_s)
            stream.wait_stream(copy_s)

        pipelined(args.warmup)
        torch.cuda.synchronize()
        barrier(world)
        e0.record(stream)
        pipelined(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        # the same with no overlap (H2D, step, D2H serial in one graph per layer), reported beside it
        ser_graphs = []
        for i in range(L):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                inp_d.copy_(inp_h, non_blocking=True)
                decs[i].step(q_d, k_d, v_d, positions, out)
                out_h.copy_(out, non_blocking=True)
            ser_graphs.append(g)
        for i in range(args.warmup):
            ser_graphs[i % L].replay()
        torch.cuda.synchronize()
        es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es0.record(stream)
        for i in range(args.steps):
            ser_graphs[i % L].replay()
        es1.record(stream)
        torch.cuda.synchronize()
        e2e_serial_ms = es0.elapsed_time(es1) / args.steps
    else:
        e2e_graphs = []
        for i in range(L):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                decs[i].step(q_d, k_d, v_d, positions, out)
            e2e_graphs.append(g)
        for i in range(args.warmup):  # (every input copied: a garbage k_new would poison the |k| bound)
            inp_d.copy_(inp_h, non_blocking=True)
            e2e_graphs[i % L].replay()
        torch.cuda.synchronize()
        barrier(world)
        e0.record(stream)
        for i in range(args.steps):
            inp_d.copy_(inp_h, non_blocking=True)
            e2e_graphs[i % L].replay()
            gather()
            out_h.copy_(res_src, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_serial_ms = None
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    h2d = q.numel() * q.element_size() + k_new.numel() * k_new.element_size() * 2
    d2h = res_src.numel() * res_src.element_size()

    # --- bytes, roofline, stats
    dec0 = decs[(args.steps - 1) % L]
    ab = algorithmic_bytes(cfg, dec0, n)
    peak, peak_src = load_peak()
    kernel_gbs = {k: (ab[k] / (stage_ms[k] * 1e-3) / 1e9 if stage_ms[k] > 0 and ab[k] else None) for k in stage_ms}
    dominant = dominant_kernel(stage_ms)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(args.config, {}).get(dominant)
        except Exception:
            traffic = None
    stats = dec0.stats()
    b1 = stats.b1.float()
    step_bytes_all = sum_over_ranks(ab["step"], world)
    achieved_step = step_bytes_all / world / (ms * 1e-3) / 1e9  # per GPU
    res = {
        "metric": METRIC,
        "value": round(ms * 1e3, 2),
        "unit": "us/layer",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 5),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: K,V iid N(0,1) bf16, q N(0,1)/tau per KV head (tau cycles 0.25,0.5,1,2), seeded",
        "config": {"workload": cfg["desc"], "config_id": args.config, "batch_per_gpu": cfg["B"],
                   "waves": len(decs[0].waves) or 1,
                   "global_batch": cfg["B"] * (world if cfg["shard"] == "batch" else 1), "ctx": n,
                   "kv_heads": H, "kv_heads_per_gpu": H_local, "group_size": G, "selector": cfg["selector"],
                   "budget_tokens": cfg["budget"], "p": cfg["p"],
                   "parallelism": f"{'batch' if cfg['shard'] == 'batch' else 'kv-head'}-sharded x{world}",
                   "l2": f"steps rotate over {L} layer caches of {caches[0].k_cache.numel() * 4 / 1e9:.2f} GB each "
                         "(K+V+INT4+meta >> 126 MB L2)", "cuda_graphs": True},
        "e2e": {"value": round(e2e_ms * 1e3, 2), "unit": "us/layer", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                **({"serial_value": round(e2e_serial_ms * 1e3, 2),
                    "serial_note": "copies and step serialised in one graph per layer (no overlap)"}
                   if e2e_serial_ms is not None else {}),
                "path": "tw_decode_step C-ABI call, q/k_new/v_new H2D from one pinned host buffer and out D2H to "
                        "pinned host every step" + (" (step captured; double-buffered staging: the next step's "
                                                    "H2D and the previous step's D2H on a copy stream overlap "
                                                    "the current step)" if copies_in_graph else
                                                    " (step captured; copies and the all-gather serial)")},
        # quest: filter (+ fused K1 append), select, estimate, top-p, attention, merge;
        # other selectors: append, select, estimate, top-p, attention, merge
        "gpu_launches": (3 if decs[0].unit_path else 6) * args.steps,
        "roofline": {"bound": "hbm", "kernel": dominant,
                     "achieved": round(kernel_gbs[dominant], 1) if kernel_gbs[dominant] else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(kernel_gbs[dominant] / peak, 4) if kernel_gbs[dominant] else None,
                     "read_peak": load_read_peak(),
                     "frac_vs_read_peak": (round(kernel_gbs[dominant] / load_read_peak(), 4)
                                           if kernel_gbs[dominant] and load_read_peak() else None),
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": ab[dominant],
                     **({"note": "the dominant stage is latency-bound (per-unit select/top-p chains at this "
                                 "batch); its HBM fraction is not the limiter"}
                        if dominant in ("K2_select", "K3bc_topp") and kernel_gbs[dominant]
                        and kernel_gbs[dominant] / peak < 0.2 else {})},
        "rank_ms": {"min": round(ms_min, 5), "max": round(ms, 5)},
        "step_roofline": {"algorithmic_bytes": ab["step"], "achieved_gbs_per_gpu": round(achieved_step, 1),
                          "frac": round(achieved_step / peak, 4),
                          **({"logits_round_trip_bytes": ab["logits_round_trip"],
                              "frac_without_logits": round((ab["step"] - ab["logits_round_trip"]) / (ms * 1e-3) / 1e9
                                                           / peak, 4),
                              "note": "K3 is unfused: SURVEY 8(d)'s + G*|U|*4*2 (candidate logits written by the "
                                      "estimate, read back by top-p) is in the step's bytes"}
                             if not decs[0].unit_path else {})},
        "kernels_us": {k: round(v * 1e3, 2) for k, v in stage_ms.items()},
        "kernels_gbs": {k: (round(v, 1) if v else None) for k, v in kernel_gbs.items()},
        "algorithmic_bytes": {k: ab[k] for k in stage_ms},
        "dense_us_per_layer": round(dense_ms * 1e3, 2),
        "dense_gbs": round(ab["K5_dense"] / (dense_ms * 1e-3) / 1e9, 1),
        "speedup_vs_dense": round(dense_ms / ms, 3),
        "budgets": {"cand_tokens_mean_per_unit": round(ab["cand_pages"] * 16 / (B * H_local), 1),
                    "final_tokens_mean_per_unit": round(ab["final_tokens"] / (B * H_local), 1),
                    "head_b1_min": int(b1.min().item()), "head_b1_max": int(b1.max().item()),
                    "head_b1_mean": round(float(b1.mean().item()), 1)},
        "clocks": clocks,
    }
    if sweep:
        res["p_sweep"] = sweep
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(cfg, n, samples=args.cpu_units)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_model(args, cfg):
    """C4: the whole 32-layer Llama-3.1-8B decode step (model.py), global batch
    sharded over ranks (strong scaling, no collective).  value = step / layers."""
    from paper_2502_02770_b200.model import LlamaConfig, LlamaTwilightDecoder
    from paper_2502_02770_b200.workload import make_batch, tau_schedule

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local if world > 1 else 0)
    assert cfg["B"] % world == 0, "global batch must divide over ranks"
    B, H, G, n = cfg["B"] // world, cfg["H"], cfg["G"], cfg["n"]
    cfg = dict(cfg, B=B, H_local=H)
    L = args.layers or cfg["layers"]
    mcfg = LlamaConfig()
    model = LlamaTwilightDecoder(mcfg, batch=B, ctx=n, selector=cfg["selector"], budget=cfg["budget"], p=cfg["p"],
                                 device=dev, seed=11 + rank, n_layers=L, q_taus=TAUS)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    tokens = torch.randint(0, mcfg.vocab, (B,), device=dev, generator=torch.Generator(device=dev).manual_seed(5 + rank))
    next_tok = torch.empty(B, dtype=torch.int64, device=dev)

    def step():
        logits = model.step(tokens)
        torch.argmax(logits, dim=-1, out=next_tok)

    s = torch.cuda.Stream(device=dev)
    s.wait_stream(stream)
    with torch.cuda.stream(s):
        step()
    stream.wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local if world > 1 else 0) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    clocks = clk.summary()

    # e2e: tokens from pinned host, next tokens back to pinned host, every step
    tok_h = tokens.cpu().pin_memory()
    next_h = torch.empty(B, dtype=torch.int64).pin_memory()
    for _ in range(args.warmup):
        tokens.copy_(tok_h, non_blocking=True)
        graph.replay()
        next_h.copy_(next_tok, non_blocking=True)
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        tokens.copy_(tok_h, non_blocking=True)
        graph.replay()
        next_h.copy_(next_tok, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)

    # breakdown: attention of one Twilight layer (its real q/k/v from an eager step) and one dense layer
    tw_layer = next(i for i in range(L) if i not in mcfg.bypass_layers)
    dec = model.decs[tw_layer]
    rec = {}
    model.step(tokens, record=rec)
    q, k_new, v_new = rec[tw_layer]
    positions = model.positions
    out = torch.empty(B, H * G, 128, dtype=torch.float32, device=dev)
    reps = max(3, min(args.steps, 10))
    stage_ms = stage_breakdown([dec], q, k_new, v_new, positions, out, reps)
    ab = algorithmic_bytes(cfg, dec, n)  # candidate pages / final sets of that layer's step
    stats = dec.stats()
    b1 = stats.b1.float()
    dense_dec = model.decs[mcfg.bypass_layers[0]] if mcfg.bypass_layers else dec
    g = torch.cuda.CUDAGraph()
    dense_dec.dense(q, out)
    with torch.cuda.graph(g):
        dense_dec.dense(q, out)
    g.replay()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    dense_ms = e0.elapsed_time(e1) / reps
    n_tw = sum(1 for i in range(L) if i not in mcfg.bypass_layers)
    n_dense = L - n_tw
    attn_ms = sum(stage_ms.values()) * n_tw + dense_ms * n_dense
    peak, peak_src = load_peak()
    kernel_gbs = {k: (ab[k] / (stage_ms[k] * 1e-3) / 1e9 if stage_ms[k] > 0 and ab[k] else None) for k in stage_ms}
    dominant = dominant_kernel(stage_ms)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(args.config, {}).get(dominant)
        except Exception:
            traffic = None
    wbytes = model.weight_bytes()
    step_bytes = wbytes + n_tw * ab["step"] + n_dense * ab["K5_dense"]
    res = {
        "metric": METRIC,
        "value": round(ms * 1e3 / L, 2),
        "unit": "us/layer",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: random-init weights N(0,0.02) (q-projection columns rescaled so q ~ N(0,1/tau^2) per KV "
                "head, tau cycling 0.25,0.5,1,2 as in C2), K,V iid N(0,1) bf16 prefill, seeded tokens",
        "config": {"workload": cfg["desc"], "config_id": args.config, "model": "Llama-3.1-8B shape (random init)",
                   "layers": L, "global_batch": cfg["B"] * world, "batch_per_gpu": B, "seq_len": n, "ctx": n,
                   "selector": cfg["selector"], "budget_tokens": cfg["budget"], "p": cfg["p"],
                   "bypass_layers": list(mcfg.bypass_layers), "parallelism": f"batch-sharded x{world}",
                   "l2": f"weights {wbytes / 1e9:.1f} GB + KV {model.caches[0].k_cache.numel() * 4 / 1e9:.1f} GB "
                         "streamed per step (>> 126 MB L2)", "cuda_graphs": True,
                   "kv_aliasing": "all layers alias one physical paged cache (BASELINE.md §4)"},
        "e2e": {"value": round(e2e_ms * 1e3 / L, 2), "unit": "us/layer", "h2d_bytes_per_step": B * 8,
                "d2h_bytes_per_step": B * 8,
                "path": "LlamaTwilightDecoder.step (captured) with token ids from pinned host, argmax ids to host"},
        "gpu_launches": ((3 if dec.unit_path else 7 if cfg["selector"] == "quest" else 8) * n_tw
                         + 3 * n_dense) * args.steps,
        "roofline": {"bound": "hbm", "kernel": dominant,
                     "achieved": round(kernel_gbs[dominant], 1) if kernel_gbs[dominant] else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(kernel_gbs[dominant] / peak, 4) if kernel_gbs[dominant] else None,
                     "read_peak": load_read_peak(),
                     "frac_vs_read_peak": (round(kernel_gbs[dominant] / load_read_peak(), 4)
                                           if kernel_gbs[dominant] and load_read_peak() else None),
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": ab[dominant]},
        "step_roofline": {"algorithmic_bytes": step_bytes, "weights_bytes": wbytes,
                          "achieved_gbs_per_gpu": round(step_bytes / (ms * 1e-3) / 1e9, 1),
                          "frac": round(step_bytes / (ms * 1e-3) / 1e9 / peak, 4)},
        "step_split_ms": {"attention_twilight_layers": round(sum(stage_ms.values()) * n_tw, 3),
                          "attention_dense_layers": round(dense_ms * n_dense, 3),
                          "gemm_norm_rope_other": round(ms - attn_ms, 3)},
        "kernels_us": {k: round(v * 1e3, 2) for k, v in stage_ms.items()},
        "kernels_gbs": {k: (round(v, 1) if v else None) for k, v in kernel_gbs.items()},
        "dense_layer_attention_us": round(dense_ms * 1e3, 2),
        "all_dense_step_estimate_ms": round(ms - sum(stage_ms.values()) * n_tw + dense_ms * n_tw, 3),
        "budgets": {"cand_tokens_mean_per_unit": round(ab["cand_pages"] * 16 / (B * H), 1),
                    "final_tokens_mean_per_unit": round(ab["final_tokens"] / (B * H), 1),
                    "head_b1_min": int(b1.min().item()), "head_b1_max": int(b1.max().item()),
                    "head_b1_mean": round(float(b1.mean().item()), 1)},
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg, n, samples=max(2, args.cpu_units // 4))
        cb["sample"] += "; attention of one Twilight layer only (the reference has no model / GEMM code)"
        res["cpu_baseline"] = cb
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- CPU legs (oracle port)

def _unit_arrays(cfg, n, h, seed):
    import numpy as np
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((n, 128)).astype(np.float32)
    V = rng.standard_normal((n, 128)).astype(np.float32)
    tau = TAUS[h % len(TAUS)]
    Q = (rng.standard_normal((cfg["G"], 128)) / tau).astype(np.float32)
    # bf16-representable values, as the GPU sees them
    def bf(x):
        a = x.view(np.uint32).astype(np.uint64)
        return (((a + 0x7FFF + ((a >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)).view(np.float32)
    return bf(K), bf(V), bf(Q)


def _cpu_unit(args):
    """One (sequence, kv head) unit of the reference hot path on the CPU
    oracle: append (quantize one row + page bounds update) then
    select -> union -> estimate -> softmax -> threshold search -> union ->
    attention, with the cache prebuilt (pipeline.py:306-360 with cache=)."""
    cfg, n, h, seed, prepared_cache = args
    import numpy as np
    from oracle import twilight_oracle as orc
    K, V, Q, prep = prepared_cache
    t0 = time.perf_counter()
    orc.quantize_rows(K[-1])          # K1 for the appended row
    orc.page_bounds(K[-16:])          # and its page's bounds
    orc.decode_unit(Q, K, V, selector=cfg["selector"], budget=cfg["budget"] or 1.0, p=cfg["p"],
                    prepared=prep)
    return time.perf_counter() - t0


_POOL_STATE = {}


def _pool_init(cfg, n, seed):
    import numpy as np
    os.environ["OMP_NUM_THREADS"] = "1"
    try:  # one BLAS thread per worker process (BLAS was initialised in the parent)
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    from oracle import twilight_oracle as orc
    K, V, Q = _unit_arrays(cfg, n, seed % len(TAUS), seed)
    _POOL_STATE["unit"] = (K, V, Q, orc.prepare_unit(K))
    _POOL_STATE["cfg"] = cfg
    _POOL_STATE["n"] = n


def _pool_task(i):
    cfg, n = _POOL_STATE["cfg"], _POOL_STATE["n"]
    return _cpu_unit((cfg, n, i, 0, _POOL_STATE["unit"]))


def cpu_baseline(cfg, n, samples=8):
    """Oracle port, 1 thread, `samples` units of this workload; extrapolated
    to the whole batch (units = B * H_kv)."""
    import numpy as np
    from oracle import twilight_oracle as orc
    units = cfg["B"] * cfg["H_local"]
    times = []
    for s in range(samples):
        K, V, Q = _unit_arrays(cfg, n, s, 100 + s)
        prep = orc.prepare_unit(K)
        times.append(_cpu_unit((cfg, n, s, 0, (K, V, Q, prep))))
    per_unit = statistics.mean(times)
    return {"value": round(per_unit * units * 1e6, 1), "unit": "us/layer", "cores": 1, "kind": "port",
            "sample": f"{samples} of {units} (sequence, kv-head) units at ctx {n}, oracle/twilight_oracle.py "
                      f"(NumPy restatement of nucleuskv), 1 thread, cache prebuilt, extrapolated x{units / samples:.1f}",
            "seconds_per_unit": round(per_unit, 4)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


REF_PKG = os.path.join(ROOT, "baseline", "_ref")  # nucleuskv, pip-installed --target (git-ignored, travels)
_REF_UNITS = []


def _ref_pkg_available() -> bool:
    if not os.path.isdir(os.path.join(REF_PKG, "nucleuskv")):
        return False
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    try:
        import nucleuskv.pipeline  # noqa: F401
        return True
    except Exception:
        return False


def _ref_build_unit(cfg, n, i, with_pkg):
    """Unit i of the reference arm: KV head h = i (tau = TAUS[h % 4], the GPU
    arm's mix), its cache prebuilt by the oracle and (when installed) by the
    reference package itself (pipeline.py:177-201 with cache=/metadata=)."""
    from oracle import twilight_oracle as orc
    K, V, Q = _unit_arrays(cfg, n, i, 100 + i)
    unit = {"K": K, "V": V, "Q": Q, "prep": orc.prepare_unit(K)}
    if with_pkg:
        from nucleuskv import pipeline as P, quantcache as QC, selectors as S
        from nucleuskv.pruner import BinarySearchConfig
        sel = S.SelectorConfig(kind="quest", budget=int(cfg["budget"])) if cfg["selector"] == "quest" else \
            S.SelectorConfig(kind="full")
        unit["pcfg"] = P.PipelineConfig(selector=sel, prune=BinarySearchConfig(p=cfg["p"]), estimator_bits=4,
                                        group_map=S.GroupMap(cfg["G"]))
        unit["cache"], unit["meta"] = QC.build_cache(K, page_size=16, bits=4)
    return unit


def _ref_task(args):
    """One step's share of one worker: unit i through the oracle port (always)
    or through nucleuskv's own run_grouped / run_head with the prebuilt cache."""
    i, which = args
    cfg, n = _POOL_STATE["cfg"], _POOL_STATE["n"]
    u = _REF_UNITS[i]
    t0 = time.perf_counter()
    if which == "port":
        _cpu_unit((cfg, n, i, 0, (u["K"], u["V"], u["Q"], u["prep"])))
    else:
        from nucleuskv import pipeline as P
        if cfg["G"] == 1:
            P.run_head(u["Q"][0], u["K"], u["V"], u["pcfg"], cache=u["cache"], metadata=u["meta"])
        else:
            P.run_grouped(u["Q"], u["K"], u["V"], u["pcfg"], cache=u["cache"], metadata=u["meta"])
    return time.perf_counter() - t0


def _ref_worker_init():
    os.environ["OMP_NUM_THREADS"] = "1"
    try:  # one BLAS thread per worker process (BLAS was initialised in the parent)
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU path on all host cores, rank 0
    only.  Each step runs `width` (sequence, KV head) units in parallel, one
    per worker process, covering the GPU arm's tau mix, with every cache
    prebuilt (the GPU arm's step appends into a prebuilt cache too):
      * nucleuskv itself (the reference package, pip-installed into
        baseline/_ref) through run_grouped / run_head -- the line's value;
      * the NumPy restatement in oracle/ (hot path only, no report work) --
        reported beside it.
    ms_per_step is the measured wall of one step (the sample); value is that
    wall extrapolated to the whole batch (x units / width)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    n = cfg["n"]
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    H_local = cfg["H"] // world if cfg["shard"] == "head" else cfg["H"]
    cfg = dict(cfg, H_local=H_local)
    units = cfg["B"] * H_local * (world if cfg["shard"] == "batch" and not cfg.get("model") else 1)
    width = max(1, min(cores, 16 if n > 65536 else 32, units))
    with_pkg = _ref_pkg_available()
    _POOL_STATE["cfg"], _POOL_STATE["n"] = cfg, n
    _REF_UNITS.clear()
    for i in range(width):  # built in the parent, shared copy-on-write by the forked workers
        _REF_UNITS.append(_ref_build_unit(cfg, n, i, with_pkg))
    legs = {}
    ctx = mp.get_context("fork")
    with ctx.Pool(width, initializer=_ref_worker_init) as pool:
        for which in (["pkg"] if with_pkg else []) + ["port"]:
            steps = args.steps if which == "port" else max(1, min(args.steps, 5))
            for _ in range(1 if which == "pkg" else args.warmup):
                pool.map(_ref_task, [(i, which) for i in range(width)], chunksize=1)
            walls, per_unit = [], []
            for _ in range(steps):
                t0 = time.perf_counter()
                per_unit += pool.map(_ref_task, [(i, which) for i in range(width)], chunksize=1)
                walls.append(time.perf_counter() - t0)
            wall = statistics.mean(walls)
            legs[which] = {"ms_per_step": round(wall * 1e3, 3), "steps": steps,
                           "value": round(wall * units / width * 1e6, 1),
                           "seconds_per_unit": round(statistics.mean(per_unit), 4)}
    main_leg = "pkg" if with_pkg else "port"
    L = legs[main_leg]
    kind = "reference" if with_pkg else "port"
    what = ("nucleuskv (the reference package, baseline/_ref) run_grouped/run_head with prebuilt cache" if with_pkg
            else "oracle/twilight_oracle.py (NumPy restatement of nucleuskv)")
    res = {"metric": METRIC, "value": L["value"], "unit": "us/layer", "n_gpus": world, "steps": L["steps"],
           "warmup": args.warmup, "ms_per_step": L["ms_per_step"], "higher_is_better": False,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (NumPy)",
           "data": "synthetic, seeded (NumPy): the GPU arm's shapes and per-KV-head tau mix",
           "impl": "reference",
           "config": {"workload": cfg["desc"], "config_id": args.config},
           "extrapolation": {"units_per_layer": units, "units_per_step": width, "factor": round(units / width, 3),
                             "note": "ms_per_step = measured wall of one step (width units in parallel); "
                                     "value = that wall x factor"},
           "cpu": {"model": cpu_model(), "cores_available": cores},
           "cpu_baseline": {"value": L["value"], "unit": "us/layer", "cores": width, "kind": kind,
                            "sample": f"each step: {width} (sequence, kv-head) units at ctx {n} in parallel (one "
                                      f"per core, tau mix {TAUS}), {what}; extrapolated x{units / width:.2f} to "
                                      f"{units} units"},
           "legs": legs,
           "e2e": {"value": L["value"], "unit": "us/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--waves", type=int, default=1, help="sub-batches pipelined on separate streams (1 = off; measured slower at C2)")
    ap.add_argument("--cpu-units", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=0, help="attention work-item tokens (0: auto)")
    ap.add_argument("--ctx", type=int, default=0, help="context length override (budget scaled with it)")
    ap.add_argument("--p", default="", help="comma-separated top-p sweep (default: the config's own, C5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.ctx:  # context override (e.g. the C1 batch-1 sparse/dense crossover); budget scales as n/4
        scale = args.ctx / cfg["n"]
        cfg.update(n=args.ctx, budget=int(cfg["budget"] * scale) if cfg["budget"] else None,
                   desc=cfg["desc"] + f" [ctx override {args.ctx}]")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.get("model"):
        run_model(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
