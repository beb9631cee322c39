"""Multi-process (world size 2, gloo, CPU) tests of the sharding host logic:
batch and KV-head sharding cover every unit exactly once, and the head-sharded
all-gather reassembles the single-process output (paper_2502_02770_b200/dist.py)."""

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


def _unit_output(q):
    # stand-in for one unit's attention output: any per-head function of q
    return torch.tanh(q) * 2.0 + q.sum(-1, keepdim=True)


def _worker(rank, world, port, mode, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, G, d = 4, 8, 4, 16
        g = torch.Generator().manual_seed(0)
        q = torch.randn(B, H * G, d, generator=g)
        ql = twd.local_queries(q, H, G, world, rank, mode)
        out_local = _unit_output(ql)
        if mode == "head":
            full = twd.gather_head_outputs(out_local, world)
        else:
            full = twd.gather_batch_outputs(out_local, world)
        ok = torch.allclose(full, _unit_output(q))
        result_q.put((rank, bool(ok), tuple(ql.shape)))
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
        p.join(120)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok, _ in res), res
    shapes = [s for _, _, s in res]
    if mode == "head":
        assert shapes == [(4, 16, 16), (4, 16, 16)]
    else:
        assert shapes == [(2, 32, 16), (2, 32, 16)]


def test_shard_ranges_partition():
    for total, world in [(16, 1), (16, 2), (16, 4), (16, 8), (8, 8), (32, 8)]:
        seen = []
        for r in range(world):
            lo, hi = twd.shard_range(total, world, r)
            seen.extend(range(lo, hi))
        assert seen == list(range(total))
    with pytest.raises(ValueError):
        twd.shard_range(10, 4, 0)
