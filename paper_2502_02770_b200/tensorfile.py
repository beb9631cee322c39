"""`.twlt` tensor files and file workloads: captured q/k/v
run through the B200 decode path.

Format (tensorfile.py:1-14 of the reference, little-endian): the 4-byte magic
``TWLT``, u32 version (1), u32 rank, rank x u64 dims, then the float32
row-major payload.  The reader validates the header before the payload and
raises one exception type per malformation (tensorfile.py:41-58), so callers
can keep the reference's exit-code mapping.

A file workload (workload.py:148-183) is a directory holding ``q.twlt``
(steps, heads, d) and ``k.twlt`` / ``v.twlt`` (kv_heads, n, d); query head h
reads KV head h // (heads / kv_heads).  ``run_file_workload`` decodes every
step of it on the GPU (one sequence, all KV heads as units of one batched
decode) with the same PipelineConfig the reference's ``run_grouped`` takes.
"""

from __future__ import annotations

import os
import struct

import numpy as np
import torch

MAGIC = b"TWLT"
VERSION = 1
MAX_RANK = 32
MAX_ELEMENTS = 1 << 40


class TensorFileError(Exception):
    """A malformed tensor file."""


class BadMagicError(TensorFileError):
    pass


class VersionMismatchError(TensorFileError):
    pass


class TruncatedFileError(TensorFileError):
    pass


class DimOverflowError(TensorFileError):
    pass


def write_tensor(path, array) -> None:
    """Version-1 file, payload as little-endian float32 (tensorfile.py:61-74)."""
    a = np.asarray(array.detach().cpu() if isinstance(array, torch.Tensor) else array, dtype=np.float32)
    a = np.ascontiguousarray(a.reshape(1) if a.ndim == 0 else a)
    if a.ndim > MAX_RANK or a.size > MAX_ELEMENTS:
        raise DimOverflowError(f"shape {a.shape} exceeds the format limits")
    header = MAGIC + struct.pack("<II", VERSION, a.ndim) + struct.pack(f"<{a.ndim}Q", *a.shape)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(a.astype("<f4", copy=False).tobytes())


def read_tensor(path) -> np.ndarray:
    """Header checks in file order, then the payload (tensorfile.py:77-104)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:4] != MAGIC:
        raise BadMagicError(f"{path}: magic mismatch, not a tensor file")
    if len(raw) < 12:
        raise TruncatedFileError(f"{path}: header cut short")
    version, rank = struct.unpack("<II", raw[4:12])
    if version != VERSION:
        raise VersionMismatchError(f"{path}: version {version}, expected {VERSION}")
    if not 1 <= rank <= MAX_RANK:
        raise DimOverflowError(f"{path}: rank {rank} outside [1, {MAX_RANK}]")
    start = 12 + 8 * rank
    if len(raw) < start:
        raise TruncatedFileError(f"{path}: dimension list cut short")
    dims = struct.unpack(f"<{rank}Q", raw[12:start])
    count = 1
    for dim in dims:
        count *= dim
        if count > MAX_ELEMENTS:
            raise DimOverflowError(f"{path}: dims {dims} overflow the format limit")
    if len(raw) != start + 4 * count:
        raise TruncatedFileError(f"{path}: payload of {len(raw) - start} bytes, dims {dims} need {4 * count}")
    return np.frombuffer(raw, dtype="<f4", offset=start).reshape(dims).astype(np.float32)


def load_file_workload(path):
    """(q [steps, heads, d], k [kv_heads, n, d], v) from a workload directory,
    with the reference's shape checks (workload.py:148-166)."""
    q = read_tensor(os.path.join(path, "q.twlt"))
    k = read_tensor(os.path.join(path, "k.twlt"))
    v = read_tensor(os.path.join(path, "v.twlt"))
    if q.ndim != 3 or k.ndim != 3 or v.ndim != 3:
        raise ValueError("file workload tensors must be rank 3")
    heads, d = q.shape[1], q.shape[2]
    kv_heads = k.shape[0]
    if v.shape != k.shape or k.shape[2] != d:
        raise ValueError("q/k/v tensor shapes are inconsistent")
    if heads % kv_heads != 0:
        raise ValueError(f"{heads} query heads do not map onto {kv_heads} KV heads")
    return q, k, v


def run_file_workload(path, cfg, dtype=torch.bfloat16, device="cuda"):
    """Decode every step of a file workload on the GPU path.  Returns the
    attention outputs [steps, heads, d] (float32) and the decoder of the last
    step (its buffers hold the final sets and per-head statistics)."""
    from . import _lib as L
    from .decode import PagedKVCache, TwilightDecoder, pages_for
    from .pipeline import _check_cfg
    from .selectors import resolve_budget

    _check_cfg(cfg)
    q, k, v = load_file_workload(path)
    steps, heads, d = q.shape
    kv_heads, n, _ = k.shape
    if d != L.HEAD_DIM:
        raise ValueError(f"the B200 path is compiled for d = {L.HEAD_DIM}")
    G = heads // kv_heads
    cache = PagedKVCache(1, kv_heads, G, max_pages=pages_for(n), dtype=dtype, device=device)
    cache.prefill(torch.from_numpy(k).to(device)[None], torch.from_numpy(v).to(device)[None])
    sel = cfg.selector
    if sel.kind == "quest":
        if sel.budget is None:
            raise ValueError("selector 'quest' requires a budget")
        dec = TwilightDecoder(cache, "quest", budget=resolve_budget(sel.budget, n), p=cfg.prune.p)
    elif sel.kind == "sink_window":
        dec = TwilightDecoder(cache, "sink_window", p=cfg.prune.p, sink=sel.sink, window=sel.window)
    elif sel.kind == "channel_pruned":
        if sel.budget is None:
            raise ValueError("selector 'channel_pruned' requires a budget")
        dec = TwilightDecoder(cache, "channel_pruned", budget=resolve_budget(sel.budget, n), p=cfg.prune.p,
                              top_channels=sel.top_channels)
    else:
        dec = TwilightDecoder(cache, "full", p=cfg.prune.p)
    qd = torch.from_numpy(q).to(device=device, dtype=dtype)
    outs = torch.empty(steps, heads, d, dtype=torch.float32, device=device)
    for s in range(steps):
        outs[s] = dec.forward(qd[s].reshape(1, heads, d).contiguous())[0]
    return outs, dec
