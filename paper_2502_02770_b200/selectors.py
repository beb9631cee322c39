"""Candidate selectors with the reference signatures (nucleuskv/selectors.py).

``quest_page_scores``, ``select_quest`` and ``group_union`` run on the B200
kernels (tw_quest_scores / tw_select); ``select_full``, ``select_sink_window``
and ``resolve_budget`` are index arithmetic (the decode path runs sink-window
selection inside tw_select / tw_estimate).  ``top_channels_by_magnitude`` and
``select_channel_pruned`` run on the channel-pruned selector kernel
(csrc/channel.cu, tw_select with TW_SELECT_CHANNEL_PRUNED).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable

import torch

from . import _lib as L
from .attention import TokenSelection

SELECTOR_KINDS = ("full", "quest", "channel_pruned", "sink_window")


@dataclass(frozen=True)
class SelectorConfig:
    """selectors.py:35-50."""
    kind: str = "full"
    budget: float | int | None = None
    page_size: int = 16
    top_channels: int | None = None
    sink: int = 4
    window: int = 64

    def __post_init__(self) -> None:
        if self.kind not in SELECTOR_KINDS:
            raise ValueError(f"unknown selector kind {self.kind!r}")
        if self.page_size < 1:
            raise ValueError("page_size must be at least 1")
        if self.sink < 0 or self.window < 0:
            raise ValueError("sink and window must be non-negative")


@dataclass(frozen=True)
class GroupMap:
    """selectors.py:53-69."""
    group_size: int = 1

    def __post_init__(self) -> None:
        if self.group_size < 1:
            raise ValueError("group_size must be at least 1")

    def group_of(self, head: int) -> int:
        return head // self.group_size

    def groups(self, heads: int) -> int:
        if heads % self.group_size != 0:
            raise ValueError(f"{heads} heads not divisible into groups of {self.group_size}")
        return heads // self.group_size


def resolve_budget(budget: float | int, n: int) -> int:
    """selectors.py:72-87: float fraction in (0, 1] (half-even round), int clamped to n."""
    if isinstance(budget, bool):
        raise ValueError("budget must be a number")
    if isinstance(budget, float):
        if not 0.0 < budget <= 1.0:
            raise ValueError(f"fractional budget {budget} outside (0, 1]")
        return max(1, min(n, round(budget * n)))
    b = int(budget)
    if b < 1:
        raise ValueError("budget must select at least one token")
    return min(b, n)


def select_full(n: int, device="cuda") -> TokenSelection:
    """selectors.py:90-94."""
    if n < 1:
        raise ValueError("context must contain at least one token")
    return TokenSelection.from_indices(torch.arange(n, device=device), n)


def quest_page_scores(q, metadata) -> torch.Tensor:
    """fp64 page bounds, bit-identical to the reference (selectors.py:97-109)."""
    from .quantcache import PageMetadataTable
    if not isinstance(metadata, PageMetadataTable):
        raise ValueError("metadata must come from build_page_metadata/build_cache of this package")
    if len(metadata) == 0:
        raise ValueError("no page metadata")
    cache = metadata.cache
    qv = torch.as_tensor(q, device=cache.device).to(cache.dtype).reshape(1, 1, L.HEAD_DIM).contiguous()
    out = torch.empty(1, cache.max_pages, dtype=torch.float64, device=cache.device)
    L.check(L.lib().tw_quest_scores(ctypes.byref(cache.struct()), L.ptr(qv), L.ptr(out), L.stream_handle()),
            "tw_quest_scores")
    return out[0, : len(metadata)]


def select_quest(q, metadata, budget, page_size: int, n: int) -> TokenSelection:
    """selectors.py:112-132 on the tw_select kernel (exact top-k, ties -> lower page)."""
    from .decode import TwilightDecoder
    from .quantcache import PageMetadataTable
    expected = math.ceil(n / page_size)
    if not isinstance(metadata, PageMetadataTable):
        raise ValueError("metadata must come from build_page_metadata/build_cache of this package")
    if len(metadata) and len(metadata) != expected:
        raise ValueError(f"metadata covers {len(metadata)} pages, context of {n} needs {expected}")
    if page_size != L.PAGE_SIZE:
        raise ValueError("the B200 path uses 16-token pages")
    cache = metadata.cache
    b0 = resolve_budget(budget, n)
    dec = TwilightDecoder(cache, "quest", budget=b0, p=1.0, head_page_bits=True)
    qv = torch.as_tensor(q, device=cache.device).to(cache.dtype).reshape(1, 1, L.HEAD_DIM).contiguous()
    dec.select(qv)
    pages = dec.bufs.cand_pages[0, : int(dec.bufs.cand_count[0].item())].long()
    tok = (pages[:, None] * L.PAGE_SIZE + torch.arange(L.PAGE_SIZE, device=pages.device)).reshape(-1)
    return TokenSelection.from_indices(tok[tok < n], n)


def group_union(selections) -> TokenSelection:
    """Sorted union of the heads' selections (selectors.py:178-186)."""
    if not selections:
        raise ValueError("no selections to union")
    n = selections[0].n
    if any(s.n != n for s in selections):
        raise ValueError("selections span different context sizes")
    merged = torch.unique(torch.cat([s.indices for s in selections]))
    return TokenSelection.from_indices(merged, n)


def _channel_unit(keys_full: torch.Tensor):
    """A one-unit cache holding ``keys_full`` [n, 128]."""
    from .decode import PagedKVCache, pages_for
    n = int(keys_full.shape[0])
    if n < 1:
        raise ValueError("context must contain at least one token")
    cache = PagedKVCache(1, 1, 1, max_pages=pages_for(n), dtype=keys_full.dtype, device=keys_full.device)
    cache.prefill(keys_full[None, None], torch.zeros_like(keys_full)[None, None])
    return cache


def _run_channel_select(cache, q, count: int, b0: int, ids=None):
    from .decode import TwilightDecoder
    dec = TwilightDecoder(cache, "channel_pruned", budget=b0, p=1.0, top_channels=count)
    if ids is not None:
        dec.bufs.chan_ids[0, :count] = ids.to(torch.int32)
        dec.params.channels_fixed = 1
    qv = torch.as_tensor(q, device=cache.device).to(cache.dtype).reshape(1, 1, L.HEAD_DIM).contiguous()
    dec.select(qv)
    return dec


def top_channels_by_magnitude(keys, count: int) -> torch.Tensor:
    """selectors.py:135-143: the ``count`` channels with the largest mean |K|
    (fp64, rows summed in token order; ties -> lower channel), ascending.  Runs
    the magnitude pass of the channel-pruned selector kernel."""
    K = torch.as_tensor(keys)
    if K.ndim != 2:
        raise ValueError("keys must be (n, d)")
    if not 1 <= count <= K.shape[1]:
        raise ValueError(f"count {count} outside [1, {K.shape[1]}]")
    if K.shape[1] != L.HEAD_DIM:
        raise ValueError(f"the B200 path is compiled for d = {L.HEAD_DIM}")
    if not K.is_cuda:
        raise ValueError("keys must be a CUDA tensor (the Twilight path has no CPU fallback)")
    K = K if K.dtype in (torch.bfloat16, torch.float32) else K.float()
    cache = _channel_unit(K.contiguous())
    dec = _run_channel_select(cache, torch.zeros(L.HEAD_DIM, device=K.device), count, 1)
    return dec.bufs.chan_ids[0, :count].long()


def select_channel_pruned(q, keys_reduced, channel_ids, budget) -> TokenSelection:
    """selectors.py:146-161: the B0 tokens with the largest approximate logit
    (K[:, ids] @ q[ids]) / sqrt(d), ties -> lower token, sorted.  Tokens whose
    fp64 scores differ only in the last bits may be ordered differently from the
    reference's BLAS reduction order (the kernel adds in ``channel_ids`` order)."""
    qv = torch.as_tensor(q)
    Kr = torch.as_tensor(keys_reduced)
    ids = torch.as_tensor(channel_ids).long().reshape(-1)
    if Kr.ndim != 2 or Kr.shape[1] != ids.numel():
        raise ValueError("keys_reduced must be (n, len(channel_ids))")
    if ids.numel() == 0 or bool((ids < 0).any()) or bool((ids >= qv.numel()).any()):
        raise ValueError("channel ids outside the query dimension")
    if qv.numel() != L.HEAD_DIM:
        raise ValueError(f"the B200 path is compiled for d = {L.HEAD_DIM}")
    if torch.unique(ids).numel() != ids.numel():
        raise ValueError("repeated channel ids are not supported on the B200 path")
    if not Kr.is_cuda:
        raise ValueError("keys must be a CUDA tensor (the Twilight path has no CPU fallback)")
    n = int(Kr.shape[0])
    b0 = resolve_budget(budget, n)
    dt = Kr.dtype if Kr.dtype in (torch.bfloat16, torch.float32) else torch.float32
    full = torch.zeros(n, L.HEAD_DIM, dtype=dt, device=Kr.device)
    full[:, ids.to(Kr.device)] = Kr.to(dt)
    dec = _run_channel_select(_channel_unit(full), qv.to(Kr.device), ids.numel(), b0, ids.to(Kr.device))
    return TokenSelection.from_indices(channel_selection(dec, 0, n), n)


def channel_selection(dec, unit: int, n: int) -> torch.Tensor:
    """Token indices of a unit's channel-pruned selection (tok_mask), ascending."""
    words = dec.bufs.tok_mask[unit, : -(-n // 32)].long() & 0xFFFFFFFF
    bits = (words[:, None] >> torch.arange(32, device=words.device)) & 1
    idx = torch.nonzero(bits.reshape(-1)).reshape(-1)
    return idx[idx < n]


def select_sink_window(n: int, sink: int, window: int, device="cuda") -> TokenSelection:
    """selectors.py:164-175: the first ``sink`` plus the last ``window`` tokens;
    every token when they meet."""
    if n < 1:
        raise ValueError("context must contain at least one token")
    if sink < 0 or window < 0:
        raise ValueError("sink and window must be non-negative")
    if sink + window < 1:
        raise ValueError("sink + window must keep at least one token")
    if sink + window >= n:
        return select_full(n, device)
    idx = torch.cat([torch.arange(sink, device=device), torch.arange(n - window, n, device=device)])
    return TokenSelection.from_indices(idx, n)


def build_selector(cfg: SelectorConfig, keys, metadata=None) -> Callable:
    """selectors.py:189-209."""
    n = int(keys.shape[0])
    dev = keys.device if isinstance(keys, torch.Tensor) else "cuda"
    if cfg.kind == "full":
        return lambda q: select_full(n, dev)
    if cfg.kind == "sink_window":
        return lambda q: select_sink_window(n, cfg.sink, cfg.window, dev)
    if cfg.budget is None:
        raise ValueError(f"selector {cfg.kind!r} requires a budget")
    if cfg.kind == "channel_pruned":  # the channel slice is fixed once per context
        K = torch.as_tensor(keys)
        count = cfg.top_channels if cfg.top_channels is not None else max(1, K.shape[1] // 8)
        ids = top_channels_by_magnitude(K, count)
        reduced = K[:, ids]
        return lambda q: select_channel_pruned(q, reduced, ids, cfg.budget)
    if metadata is None:
        raise ValueError("quest selector requires page metadata")
    return lambda q: select_quest(q, metadata, cfg.budget, cfg.page_size, n)
