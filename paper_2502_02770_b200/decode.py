"""Batched paged decode layer: the B200 Twilight hot path.

``PagedKVCache`` owns one attention layer's paged pool (bf16/fp32 K and V,
the INT4 K copy with per-row scale/zero, per-page channel min/max, page
table, sequence lengths).  ``TwilightDecoder`` runs one decode step per call:

    K1 tw_quant_append     quantize-on-append (quantcache.py:95-114, 163-175)
    K2 tw_select           Quest bounds + exact page top-k + GQA union (selectors.py:97-186)
    K3 tw_estimate/tw_topp INT4 estimate, candidate softmax, top-p, group union
                           (quantcache.py:238-272, pruner.py:57-114, pipeline.py:336-347)
    K4 tw_sparse_attention subset-softmax attention over the surviving rows (attention.py:89-136)

every stage a hand-written sm_100a kernel behind the C ABI (include/twilight.h);
this module only allocates device buffers and enqueues the calls on the
current stream (CUDA-graph capturable: no host synchronisation).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib as L


def pages_for(n_tokens: int) -> int:
    return -(-n_tokens // L.PAGE_SIZE)


class PagedKVCache:
    """One layer's paged KV pool plus the Twilight INT4/metadata side caches.

    Layout (include/twilight.h): k_cache/v_cache [num_phys_pages, H_kv, 16, d],
    kq [num_phys_pages, H_kv, 1152] u8, kmeta [num_phys_pages, H_kv, 2, d],
    kabsmax [B, H_kv] f32, page_table [B, max_pages] i32, seq_lens [B] i32.
    By default sequence b owns physical pages [b*max_pages, (b+1)*max_pages).
    """

    def __init__(self, num_seqs: int, num_kv_heads: int, group_size: int, max_pages: int,
                 dtype: torch.dtype = torch.bfloat16, device: str | torch.device = "cuda",
                 page_table: torch.Tensor | None = None, num_phys_pages: int | None = None, bits: int = 4):
        if bits not in (2, 4, 8):
            raise ValueError(f"bits must be one of (2, 4, 8), got {bits}")
        self.bits = bits
        self.num_seqs, self.num_kv_heads, self.group_size = num_seqs, num_kv_heads, group_size
        self.max_pages = max_pages
        self.dtype = dtype
        self.device = torch.device(device)
        L.dtype_code(dtype)
        d = L.HEAD_DIM
        if page_table is None:
            num_phys_pages = num_seqs * max_pages
            page_table = torch.arange(num_phys_pages, dtype=torch.int32, device=self.device).view(num_seqs, max_pages)
        elif num_phys_pages is None:
            num_phys_pages = int(page_table.max().item()) + 1
        self.num_phys_pages = num_phys_pages
        self.page_table = page_table.to(device=self.device, dtype=torch.int32).contiguous()
        H = num_kv_heads
        self.k_cache = torch.zeros(num_phys_pages, H, L.PAGE_SIZE, d, dtype=dtype, device=self.device)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.kq = torch.zeros(num_phys_pages, H, L.qblock_bytes(bits), dtype=torch.uint8, device=self.device)
        self.kmeta = torch.zeros(num_phys_pages, H, 2, d, dtype=dtype, device=self.device)
        self.kabsmax = torch.zeros(num_seqs, H, dtype=torch.float32, device=self.device)
        self.seq_lens = torch.zeros(num_seqs, dtype=torch.int32, device=self.device)
        self._struct = None

    def view(self, lo: int, hi: int) -> "PagedKVCache":
        """Sequences [lo, hi) as a cache of their own, sharing the physical pool
        (page table, lengths and |k| bounds are row slices)."""
        v = PagedKVCache.__new__(PagedKVCache)
        v.__dict__.update(self.__dict__)
        v.num_seqs = hi - lo
        v.page_table = self.page_table[lo:hi]
        v.seq_lens = self.seq_lens[lo:hi]
        v.kabsmax = self.kabsmax[lo:hi]
        v._struct = None
        return v

    # ------------------------------------------------------------------ ABI view
    def struct(self) -> L.TwPagedKV:
        if self._struct is None:
            s = L.TwPagedKV()
            s.num_seqs, s.num_kv_heads, s.group_size = self.num_seqs, self.num_kv_heads, self.group_size
            s.head_dim, s.max_pages, s.num_phys_pages = L.HEAD_DIM, self.max_pages, self.num_phys_pages
            s.dtype = L.dtype_code(self.dtype)
            s.bits = self.bits
            s.k_cache, s.v_cache = L.ptr(self.k_cache), L.ptr(self.v_cache)
            s.kq, s.kmeta, s.kabsmax = L.ptr(self.kq), L.ptr(self.kmeta), L.ptr(self.kabsmax)
            s.page_table, s.seq_lens = L.ptr(self.page_table), L.ptr(self.seq_lens)
            self._struct = s
        return self._struct

    @property
    def num_q_heads(self) -> int:
        return self.num_kv_heads * self.group_size

    # ------------------------------------------------------------------ filling
    def prefill(self, K: torch.Tensor, V: torch.Tensor, lengths: torch.Tensor | list[int] | None = None) -> None:
        """Write K/V [B, H_kv, n, d] (rows >= lengths[b] ignored) into the pool,
        then quantize everything with K1-bulk (tw_quant_build)."""
        B, H, n, d = K.shape
        assert (B, H, d) == (self.num_seqs, self.num_kv_heads, L.HEAD_DIM), "K shape mismatch"
        P = pages_for(n)
        assert P <= self.max_pages, "context exceeds max_pages"
        if lengths is None:
            lengths = torch.full((B,), n, dtype=torch.int32)
        lengths = torch.as_tensor(lengths, dtype=torch.int32)
        pad = P * L.PAGE_SIZE - n
        for src, dst in ((K, self.k_cache), (V, self.v_cache)):
            x = src.to(self.dtype)
            if pad:
                x = torch.nn.functional.pad(x, (0, 0, 0, pad))
            x = x.reshape(B, H, P, L.PAGE_SIZE, d).permute(0, 2, 1, 3, 4)  # [B, P, H, 16, d]
            phys = self.page_table[:, :P].reshape(-1).long()
            dst[phys] = x.reshape(B * P, H, L.PAGE_SIZE, d)
        self.seq_lens.copy_(lengths.to(self.device))
        self.kabsmax.zero_()
        L.check(L.lib().tw_quant_build(ctypes.byref(self.struct()), L.stream_handle()), "tw_quant_build")

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor, positions: torch.Tensor | None = None) -> None:
        """K1: write one new token per sequence (k_new/v_new [B, H_kv, d]) at
        `positions` (default: the current seq_lens) and quantize it."""
        pos = self.seq_lens if positions is None else positions
        L.check(L.lib().tw_quant_append(ctypes.byref(self.struct()), L.ptr(k_new.contiguous()),
                                        L.ptr(v_new.contiguous()), L.ptr(pos), L.stream_handle()),
                "tw_quant_append")

    # ------------------------------------------------------------------ host views (tests)
    def unit_keys(self, b: int, h: int) -> torch.Tensor:
        n = int(self.seq_lens[b].item())
        P = pages_for(n)
        phys = self.page_table[b, :P].long()
        return self.k_cache[phys, h].reshape(P * L.PAGE_SIZE, L.HEAD_DIM)[:n]

    def unit_values(self, b: int, h: int) -> torch.Tensor:
        n = int(self.seq_lens[b].item())
        P = pages_for(n)
        phys = self.page_table[b, :P].long()
        return self.v_cache[phys, h].reshape(P * L.PAGE_SIZE, L.HEAD_DIM)[:n]

    def unit_quant(self, b: int, h: int):
        """(packed codes [n, d*bits/8] u8, scale [n] f32, zero [n] f32) of one unit."""
        n = int(self.seq_lens[b].item())
        P = pages_for(n)
        cb = L.PAGE_SIZE * L.HEAD_DIM * self.bits // 8
        blk = self.kq[self.page_table[b, :P].long(), h]  # [P, qblock_bytes(bits)]
        packed = blk[:, :cb].reshape(P * L.PAGE_SIZE, L.HEAD_DIM * self.bits // 8)[:n]
        prm = blk[:, cb:].contiguous().view(torch.float32).view(P, 2, L.PAGE_SIZE)
        scale = prm[:, 0].reshape(-1)[:n]
        zero = prm[:, 1].reshape(-1)[:n]
        return packed, scale, zero

    def unit_meta(self, b: int, h: int):
        n = int(self.seq_lens[b].item())
        meta = self.kmeta[self.page_table[b, :pages_for(n)].long(), h]
        return meta[:, 0], meta[:, 1]


@dataclass
class DecodeStats:
    """Per-query-head record read back after a step (the GPU-side subset of
    PruneReport, pipeline.py:69-90)."""
    b0: torch.Tensor          # candidate tokens per head
    b1: torch.Tensor          # tokens the head's own top-p kept
    candidate_mass: torch.Tensor
    threshold_weight: torch.Tensor
    group_b1: torch.Tensor    # final (group-shared) set size per unit
    cand_pages: torch.Tensor  # union pages per unit


MAX_CHUNK = 512        # tokens per attention work item (csrc/attention.cu kMaxChunk)
MAX_UNIT_ITEMS = 1024  # work items of one unit the split-KV merge accepts


def min_chunk(max_pages: int) -> int:
    """Smallest work-item size (multiple of 16) that splits a full context
    of max_pages pages into at most MAX_UNIT_ITEMS items."""
    T = max_pages * L.PAGE_SIZE
    return max(L.PAGE_SIZE, 16 * -(-(-(-T // MAX_UNIT_ITEMS)) // 16))


def check_chunk(chunk: int, max_pages: int) -> int:
    """tw_attn_geometry on the host: raise ValueError before any kernel runs."""
    chunk = int(chunk)
    if chunk % L.PAGE_SIZE or not L.PAGE_SIZE <= chunk <= MAX_CHUNK:
        raise ValueError(f"chunk_tokens {chunk} must be a multiple of 16 in [16, {MAX_CHUNK}]")
    if chunk < min_chunk(max_pages):
        raise ValueError(f"chunk_tokens {chunk} splits a {max_pages}-page context into more than "
                         f"{MAX_UNIT_ITEMS} work items (need >= {min_chunk(max_pages)})")
    return chunk


def auto_chunk(cache: "PagedKVCache", sms: int = 148, warps_per_sm: int = 8) -> int:
    """Attention work-item size: ~4 items per worker warp when half the
    context survives, clamped to [64, 512] tokens (multiple of 16) and never
    below min_chunk (at most 1024 items per unit for the merge)."""
    units = cache.num_seqs * cache.num_kv_heads
    est = units * cache.max_pages * L.PAGE_SIZE * 0.5 / (4 * sms * warps_per_sm)
    c = 512 if est >= 384 else int(max(64, 16 * round(est / 16)))
    c = max(c, min_chunk(cache.max_pages))
    if c > MAX_CHUNK:
        raise ValueError(f"context of {cache.max_pages} pages exceeds {MAX_UNIT_ITEMS} x {MAX_CHUNK} tokens")
    return c


class DecodeBuffers:
    """Caller-owned intermediate buffers of one decode step (tw_decode_buffers)."""

    def __init__(self, cache: PagedKVCache, chunk_tokens: int | None = None, head_page_bits: bool = False):
        chunk_tokens = check_chunk(chunk_tokens, cache.max_pages) if chunk_tokens else auto_chunk(cache)
        dev = cache.device
        U = cache.num_seqs * cache.num_kv_heads
        Hq = U * cache.group_size
        G = cache.group_size
        T = cache.max_pages * L.PAGE_SIZE
        self.page_scores = torch.empty(Hq, cache.max_pages, dtype=torch.float32, device=dev)
        self.cand_pages = torch.empty(U, cache.max_pages, dtype=torch.int32, device=dev)
        self.cand_count = torch.zeros(U, dtype=torch.int32, device=dev)
        self.logits = torch.empty(U, G, T, dtype=torch.float32, device=dev)
        self.head_max = torch.zeros(Hq, dtype=torch.int32, device=dev)
        self.head_thr = torch.zeros(Hq, dtype=torch.int32, device=dev)
        self.head_stats = torch.zeros(Hq, 4, dtype=torch.float32, device=dev)
        self.final_idx = torch.empty(U, T, dtype=torch.int32, device=dev)
        self.final_count = torch.zeros(U, dtype=torch.int32, device=dev)
        self.unit_items = torch.zeros(U, 2, dtype=torch.int32, device=dev)
        self.max_items = int(L.lib().tw_max_work_items(ctypes.byref(cache.struct()), chunk_tokens))
        self.work_items = torch.empty(self.max_items, 2, dtype=torch.int32, device=dev)
        self.counters = torch.zeros(8, dtype=torch.int32, device=dev)
        self.partials = torch.empty(self.max_items, G, L.HEAD_DIM + 2, dtype=torch.float32, device=dev)
        words = -(-cache.max_pages // 32)
        self.head_page_bits = torch.zeros(Hq, words, dtype=torch.int32, device=dev) if head_page_bits else None
        self.sel_bits = torch.zeros(U, -(-T // 32), dtype=torch.int32, device=dev)
        self.topp_done = torch.zeros(U, dtype=torch.int32, device=dev)  # the library leaves it (and sel_bits) zeroed
        self.tok_mask = torch.zeros(U, -(-T // 32), dtype=torch.int32, device=dev)  # channel-pruned selections
        self.chan_ids = torch.zeros(U, L.HEAD_DIM, dtype=torch.int32, device=dev)  # channel-pruned slice
        self.band_idx = torch.empty(Hq, cache.max_pages, dtype=torch.int32, device=dev)
        self.band_scores = torch.empty(Hq, cache.max_pages, dtype=torch.float64, device=dev)
        s = L.TwDecodeBuffers()
        for name in ("page_scores", "cand_pages", "cand_count", "logits", "head_max", "head_thr", "head_stats",
                     "final_idx", "final_count", "unit_items", "work_items", "counters", "partials",
                     "head_page_bits", "sel_bits", "tok_mask", "chan_ids", "topp_done", "band_idx", "band_scores"):
            setattr(s, name, L.ptr(getattr(self, name)))
        s.max_items = self.max_items
        self._struct = s

    def struct(self) -> L.TwDecodeBuffers:
        return self._struct


def budget_pages_for(budget, n: int) -> int:
    """ceil(resolve_budget(budget, n) / 16) (selectors.py:72-87, :127)."""
    from .selectors import resolve_budget
    return -(-resolve_budget(budget, n) // L.PAGE_SIZE)


class TwilightDecoder:
    """Runs the select -> estimate -> prune -> attend path for one layer.

    selector: "quest" (Quest page top-k with budget B0 tokens), "full", or
    "sink_window" (the first ``sink`` + last ``window`` tokens, selectors.py:164-175), or
    "channel_pruned" (per query head the ``budget`` tokens with the largest
    partial logit over the ``top_channels`` channels of largest mean |K|,
    selectors.py:135-161; any context length).  ``estimator`` "int"
    estimates the candidates' logits from the cache's INT codes
    (quantcache.py:238-272), "exact" from the full-precision keys
    (estimator_bits="exact", pipeline.py:212-214).  With
    ``fix_channels`` the channel slice ranked at the first step is kept for the
    following steps (the reference binds it once per context, selectors.py:203);
    otherwise it is re-ranked over the current cache every step.
    """

    def __init__(self, cache: PagedKVCache, selector: str = "quest", budget=None, p: float = 0.95,
                 chunk_tokens: int | None = None, head_page_bits: bool = False,
                 bufs: DecodeBuffers | list | None = None, waves: int = 1, sink: int = 4, window: int = 64,
                 top_channels: int | None = None, fix_channels: bool = False, estimator: str = "int"):
        self.waves = []
        if waves > 1:
            # sub-batches on their own streams: the select/top-p stages of one wave
            # overlap the HBM-bound stages of another (see step()).
            if cache.num_seqs % waves:
                raise ValueError("num_seqs must divide into waves")
            per = cache.num_seqs // waves
            for w in range(waves):
                sub = TwilightDecoder(cache.view(w * per, (w + 1) * per), selector, budget, p, chunk_tokens,
                                      head_page_bits, bufs[w] if isinstance(bufs, list) else None,
                                      sink=sink, window=window, top_channels=top_channels,
                                      fix_channels=fix_channels, estimator=estimator)
                self.waves.append((w * per, (w + 1) * per, sub, torch.cuda.Stream(device=cache.device)))
            self.cache = cache
            self.params = self.waves[0][2].params
            self.bufs = [wv[2].bufs for wv in self.waves]
            return
        chunk_tokens = check_chunk(chunk_tokens, cache.max_pages) if chunk_tokens else auto_chunk(cache)
        if selector not in ("quest", "full", "sink_window", "channel_pruned"):
            raise ValueError(f"selector {selector!r} is not on the accelerated path "
                             "(quest | full | sink_window | channel_pruned)")
        if top_channels is not None and not 1 <= int(top_channels) <= L.HEAD_DIM:
            raise ValueError(f"top_channels {top_channels} outside [1, {L.HEAD_DIM}]")
        if selector == "sink_window" and (sink < 0 or window < 0 or sink + window < 1):
            raise ValueError("sink and window must be non-negative and keep at least one token")
        if not 0.0 <= p <= 1.0:
            raise ValueError(f"p={p} outside [0, 1]")
        if estimator not in ("int", "exact"):
            raise ValueError(f"estimator {estimator!r} must be 'int' (the cache's INT codes) or 'exact'")
        self.cache = cache
        # buffers may be shared by decoders of layers with the same geometry
        self.bufs = bufs if bufs is not None else DecodeBuffers(cache, chunk_tokens, head_page_bits)
        self.params = L.TwDecodeParams()
        self.selector_name = selector
        self.params.selector = {"quest": L.TW_SELECT_QUEST, "full": L.TW_SELECT_FULL,
                                "sink_window": L.TW_SELECT_SINK_WINDOW,
                                "channel_pruned": L.TW_SELECT_CHANNEL_PRUNED}[selector]
        self.params.sink, self.params.window = int(sink), int(window)
        # build_selector (selectors.py:205-207): d // 8 channels unless given
        self.params.top_channels = int(top_channels) if top_channels is not None else max(1, L.HEAD_DIM // 8)
        self.fix_channels = bool(fix_channels)
        self.params.p = float(p)
        # estimator_bits="exact" (pipeline.py:212-214): logits from the full-precision keys
        self.params.estimator = L.TW_ESTIMATE_EXACT if estimator == "exact" else L.TW_ESTIMATE_INT
        self.params.chunk_tokens = chunk_tokens
        self.params.renormalize = 1
        self.set_budget(budget)

    def set_budget(self, budget, n: int | None = None) -> None:
        if self.params.selector in (L.TW_SELECT_FULL, L.TW_SELECT_SINK_WINDOW):
            self.params.budget_pages = self.cache.max_pages
            return
        if budget is None:
            raise ValueError(f"selector {self.selector_name!r} requires a budget")
        if self.params.selector == L.TW_SELECT_CHANNEL_PRUNED:
            from .selectors import resolve_budget
            if isinstance(budget, float) and n is None:
                raise ValueError("a fractional budget needs the context length n")
            self.params.budget_tokens = resolve_budget(budget, n if n is not None else int(budget))
            self.params.budget_pages = self.cache.max_pages
            return
        if isinstance(budget, float):
            if n is None:
                raise ValueError("a fractional budget needs the context length n")
            self.params.budget_pages = budget_pages_for(budget, n)
        else:
            self.params.budget_pages = -(-int(budget) // L.PAGE_SIZE)

    # ------------------------------------------------------------------ stages
    def _args(self):
        return ctypes.byref(self.cache.struct()), ctypes.byref(self.params), ctypes.byref(self.bufs.struct())

    def select(self, q: torch.Tensor) -> None:
        kv, prm, buf = self._args()
        L.check(L.lib().tw_select(kv, L.ptr(q), prm, buf, L.stream_handle()), "tw_select")
        if self.fix_channels and self.params.selector == L.TW_SELECT_CHANNEL_PRUNED:
            self.params.channels_fixed = 1

    @property
    def unit_path(self) -> bool:
        """True when K2 + K3 run as the fused per-unit kernel (tw_select_estimate_topp)."""
        if self.waves:
            return False
        kv, prm, buf = self._args()
        return bool(L.lib().tw_select_estimate_topp_applies(kv, prm, buf))

    def select_estimate_topp(self, q: torch.Tensor, k_new: torch.Tensor | None = None,
                             v_new: torch.Tensor | None = None, positions: torch.Tensor | None = None) -> None:
        """K2 + K3 in one per-unit launch; with positions, K1 (the append of k_new/v_new) too."""
        kv, prm, buf = self._args()
        L.check(L.lib().tw_select_estimate_topp(kv, L.ptr(q), L.ptr(k_new), L.ptr(v_new), L.ptr(positions), prm,
                                                buf, L.stream_handle()), "tw_select_estimate_topp")

    def estimate(self, q: torch.Tensor) -> None:
        kv, prm, buf = self._args()
        L.check(L.lib().tw_estimate(kv, L.ptr(q), prm, buf, L.stream_handle()), "tw_estimate")

    def topp(self) -> None:
        kv, prm, buf = self._args()
        L.check(L.lib().tw_topp(kv, prm, buf, L.stream_handle()), "tw_topp")

    def attend(self, q: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        kv, prm, buf = self._args()
        L.check(L.lib().tw_sparse_attention(kv, L.ptr(q), prm, buf, L.ptr(out), L.stream_handle()),
                "tw_sparse_attention")
        return out

    def attend_part(self, q: torch.Tensor, out: torch.Tensor, part: int) -> torch.Tensor:
        """K4's kernels one at a time (per-kernel timing): 1 the gather / subset
        softmax kernel, 2 the split-KV merge."""
        kv, prm, buf = self._args()
        L.check(L.lib().tw_sparse_attention_part(kv, L.ptr(q), prm, buf, L.ptr(out), int(part),
                                                 L.stream_handle()), "tw_sparse_attention_part")
        return out

    def dense(self, q: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = self._out()
        if self.waves:
            for lo, hi, sub, _ in self.waves:
                sub.dense(q[lo:hi], out[lo:hi])
            return out
        kv, _, buf = self._args()
        L.check(L.lib().tw_dense_attention(kv, L.ptr(q), buf, L.ptr(out), L.stream_handle()),
                "tw_dense_attention")
        return out

    def _out(self) -> torch.Tensor:
        c = self.cache
        return torch.empty(c.num_seqs, c.num_q_heads, L.HEAD_DIM, dtype=torch.float32, device=c.device)

    def check_q(self, q: torch.Tensor) -> torch.Tensor:
        c = self.cache
        if q.shape != (c.num_seqs, c.num_q_heads, L.HEAD_DIM):
            raise ValueError(f"q must be [B={c.num_seqs}, H_q={c.num_q_heads}, d=128], got {tuple(q.shape)}")
        if q.dtype != c.dtype:
            raise ValueError(f"q dtype {q.dtype} must match the cache dtype {c.dtype}")
        return q.contiguous()

    def forward(self, q: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Attend with the cache as is (no append): K2 -> K3 -> K4."""
        q = self.check_q(q)
        out = self._out() if out is None else out
        if self.waves:
            for lo, hi, sub, _ in self.waves:
                sub.forward(q[lo:hi], out[lo:hi])
            return out
        if self.unit_path:
            self.select_estimate_topp(q)
        else:
            self.select(q)
            self.estimate(q)
            self.topp()
        return self.attend(q, out)

    def _step_waves(self, q, k_new, v_new, positions, out):
        """Append for the whole batch, then each wave's K2 -> K4 on its own
        stream; wave w+1 starts once wave w's estimate is done, so its
        HBM-bound select/estimate overlap wave w's top-p and attention."""
        self.cache.append(k_new, v_new, positions)
        cur = torch.cuda.current_stream()
        prev = torch.cuda.Event()
        prev.record(cur)
        done = []
        for lo, hi, sub, stream in self.waves:
            stream.wait_event(prev)
            with torch.cuda.stream(stream):
                qs = q[lo:hi]
                sub.select(qs)
                sub.estimate(qs)
                prev = torch.cuda.Event()
                prev.record(stream)
                sub.topp()
                sub.attend(qs, out[lo:hi])
                ev = torch.cuda.Event()
                ev.record(stream)
                done.append(ev)
        for ev in done:
            cur.wait_event(ev)
        return out

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
             positions: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """One decode step: append (K1) then K2 -> K4, one fused C-ABI call."""
        q = self.check_q(q)
        out = self._out() if out is None else out
        if self.waves:
            return self._step_waves(q, k_new, v_new, positions, out)
        kv, prm, buf = self._args()
        pos = self.cache.seq_lens if positions is None else positions
        L.check(L.lib().tw_decode_step(kv, L.ptr(q), L.ptr(k_new), L.ptr(v_new), L.ptr(pos), prm, buf,
                                       L.ptr(out), L.stream_handle()), "tw_decode_step")
        return out

    def stats(self) -> DecodeStats:
        if self.waves:
            parts = [wv[2].stats() for wv in self.waves]
            return DecodeStats(*[torch.cat([getattr(p, f) for p in parts]) for f in
                                 ("b0", "b1", "candidate_mass", "threshold_weight", "group_b1", "cand_pages")])
        b = self.bufs
        return DecodeStats(b0=b.head_stats[:, 3].clone(), b1=b.head_stats[:, 0].clone(),
                           candidate_mass=b.head_stats[:, 1].clone(), threshold_weight=b.head_stats[:, 2].clone(),
                           group_b1=b.final_count.clone(), cand_pages=b.cand_count.clone())
