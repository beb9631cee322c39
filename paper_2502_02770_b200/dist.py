"""Multi-GPU layout of the decode path: one process per GPU (torchrun).

The path shards naturally: every unit (sequence, KV head) is
independent through all stages (pipeline.py:336-359).

* batch-sharded (C2/C4/C5): rank r owns sequences [r*B/N, (r+1)*B/N) with
  their KV pages, INT4 copy, metadata and page table.  No collective touches
  the data path.
* KV-head-sharded (C3): rank r owns KV heads [r*H/N, (r+1)*H/N) (and their G
  query heads) of every sequence and produces out[B, H/N*G, d]; one NCCL
  all-gather assembles out[B, H*G, d].

These helpers are pure host logic (tested with gloo on CPU); the kernels see
a rank-local PagedKVCache only.
"""

from __future__ import annotations

import torch


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) block of `total` items owned by `rank` (total % world == 0)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if total % world:
        raise ValueError(f"{total} items do not split evenly over {world} ranks")
    per = total // world
    return rank * per, (rank + 1) * per


def shard_batch(B: int, world: int, rank: int) -> slice:
    lo, hi = shard_range(B, world, rank)
    return slice(lo, hi)


def shard_kv_heads(H_kv: int, world: int, rank: int) -> slice:
    lo, hi = shard_range(H_kv, world, rank)
    return slice(lo, hi)


def local_queries(q: torch.Tensor, H_kv: int, G: int, world: int, rank: int, mode: str) -> torch.Tensor:
    """The rank's slice of q [B, H_kv*G, d] for `mode` in {"batch", "head"}."""
    if mode == "batch":
        return q[shard_batch(q.shape[0], world, rank)]
    if mode == "head":
        s = shard_kv_heads(H_kv, world, rank)
        return q[:, s.start * G:s.stop * G]
    raise ValueError(mode)


def gather_head_outputs(out_local: torch.Tensor, world: int, group=None, buf: torch.Tensor | None = None,
                        out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather per-rank outputs [B, Hq/N, d] into [B, Hq, d] (head-sharded mode).

    One collective (all_gather_into_tensor) of world * B*Hq/N*d floats into
    `buf` [N*B, Hq/N, d]; the rank-major result is permuted back to head order
    (into `out` [B, Hq, d] when given).  Pre-allocated buffers keep the step
    allocation-free.
    """
    import torch.distributed as dist

    if world == 1:
        return out_local
    B, hq_local, d = out_local.shape
    if buf is None:
        buf = torch.empty(world * B, hq_local, d, dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(buf, out_local.contiguous(), group=group)
    full = buf.view(world, B, hq_local, d).permute(1, 0, 2, 3)
    if out is None:
        return full.reshape(B, world * hq_local, d)
    out.view(B, world, hq_local, d).copy_(full)
    return out


def gather_batch_outputs(out_local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Collect batch-sharded outputs (only for checking: the data path needs no collective)."""
    import torch.distributed as dist

    if world == 1:
        return out_local
    buf = torch.empty((world * out_local.shape[0],) + tuple(out_local.shape[1:]), dtype=out_local.dtype,
                      device=out_local.device)
    dist.all_gather_into_tensor(buf, out_local.contiguous(), group=group)
    return buf
