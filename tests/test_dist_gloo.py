"""Multi-process (world size 2, gloo, CPU) tests of the sharding host logic:
batch and KV-head sharding cover every unit exactly once, and the head-sharded
all-gather reassembles the single-process output (paper_2502_02770_b200/dist.py).

The sharded work is the real decode path, restated by the CPU oracle
(oracle.decode_unit: Quest -> union -> INT4 estimate -> top-p -> attention per
unit, pipeline.py:306-360): each rank decodes only its own units -- its
sequences (batch mode) or its KV heads (head mode) -- and the reassembled
output must equal the unsharded run bit for bit, which is the per-unit
independence the multi-GPU layout relies on (pipeline.py:336-359)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_02770_b200 import dist as twd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


B_, H_, G_, N_, D_ = 4, 4, 2, 320, 128  # sequences, KV heads, group size, context, head dim


def _workload():
    """Seeded K/V per (sequence, KV head) and q [B, H*G, d], bf16-representable."""
    g = torch.Generator().manual_seed(0)
    K = torch.randn(B_, H_, N_, D_, generator=g).bfloat16().float()
    V = torch.randn(B_, H_, N_, D_, generator=g).bfloat16().float()
    q = (torch.randn(B_, H_ * G_, D_, generator=g) * 2.0).bfloat16().float()
    return K, V, q


def _decode(K, V, q, b_lo, b_hi, h_lo, h_hi):
    """Oracle decode of units (b, h) for b in [b_lo, b_hi), h in [h_lo, h_hi): out [b, h*G, d]."""
    from oracle import twilight_oracle as orc
    out = torch.zeros(b_hi - b_lo, (h_hi - h_lo) * G_, D_, dtype=torch.float32)
    for b in range(b_lo, b_hi):
        for h in range(h_lo, h_hi):
            Q = q[b, h * G_:(h + 1) * G_].numpy()
            res = orc.decode_unit(Q, K[b, h].numpy(), V[b, h].numpy(), selector="quest", budget=96, p=0.9)
            out[b - b_lo, (h - h_lo) * G_:(h - h_lo + 1) * G_] = torch.from_numpy(res["out"].astype("float32"))
    return out


def _worker(rank, world, port, mode, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, V, q = _workload()
        ql = twd.local_queries(q, H_, G_, world, rank, mode)
        if mode == "head":
            hs = twd.shard_kv_heads(H_, world, rank)
            out_local = _decode(K, V, q, 0, B_, hs.start, hs.stop)
            full = twd.gather_head_outputs(out_local, world)
            # the bench's allocation-free form: pre-allocated gather buffer + permuted output
            buf = torch.empty(world * B_, out_local.shape[1], D_)
            full2 = torch.empty(B_, H_ * G_, D_)
            twd.gather_head_outputs(out_local, world, buf=buf, out=full2)
            assert torch.equal(full, full2)
        else:
            bs = twd.shard_batch(B_, world, rank)
            out_local = _decode(K, V, q, bs.start, bs.stop, 0, H_)
            full = twd.gather_batch_outputs(out_local, world)
        result_q.put((rank, full.numpy(), tuple(ql.shape), tuple(out_local.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["head", "batch"])
def test_sharded_outputs_reassemble(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = sorted((q.get(timeout=5) for _ in range(world)), key=lambda r: r[0])
    K, V, qq = _workload()
    want = _decode(K, V, qq, 0, B_, 0, H_).numpy()  # the unsharded run
    for rank, full, qshape, oshape in res:
        assert (full == want).all(), f"rank {rank}: reassembled {mode}-sharded output differs from the unsharded run"
        if mode == "head":
            assert qshape == (B_, H_ // world * G_, D_) and oshape == (B_, H_ // world * G_, D_)
        else:
            assert qshape == (B_ // world, H_ * G_, D_) and oshape == (B_ // world, H_ * G_, D_)


def test_shard_ranges_partition():
    for total, world in [(16, 1), (16, 2), (16, 4), (16, 8), (8, 8), (32, 8)]:
        seen = []
        for r in range(world):
            lo, hi = twd.shard_range(total, world, r)
            seen.extend(range(lo, hi))
        assert seen == list(range(total))
    with pytest.raises(ValueError):
        twd.shard_range(10, 4, 0)
