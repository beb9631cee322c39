"""Paged INT4 key cache with the reference signatures (nucleuskv/quantcache.py).

``build_cache`` / ``build_page_metadata`` fill a one-unit ``PagedKVCache``
with the K1 bulk kernel (tw_quant_build); ``quantize_row`` runs tw_quant_rows;
``estimate_scores`` runs tw_estimate_tokens.  The returned objects wrap device
tensors; ``PagedQuantKeyCache.pages`` materialises the reference's per-page
view (packed bytes, fp64 scale/zero, valid_len) for inspection and tests.
Caches of 2, 4 and 8 bits (SUPPORTED_BITS) are built and estimated on the
GPU; the decode path defaults to 4.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib as L
from .attention import TokenSelection
from .decode import PagedKVCache, pages_for

SUPPORTED_BITS = (2, 4, 8)  # quantcache.py:38
PARAM_BYTES = 4             # traffic model (quantcache.py:42)

__all__ = ["SUPPORTED_BITS", "PARAM_BYTES", "QuantParams", "QuantPage", "PageMetadata", "PageMetadataTable",
           "PagedQuantKeyCache", "EstimateResult", "quantize_row", "dequantize_row", "pack_codes", "unpack_codes",
           "build_page_metadata", "build_cache", "estimate_scores"]


@dataclass(frozen=True)
class QuantParams:
    scale: float
    zero: float


@dataclass(frozen=True, eq=False)
class QuantPage:
    packed: bytes
    scales: torch.Tensor
    zeros: torch.Tensor
    valid_len: int


@dataclass(frozen=True, eq=False)
class PageMetadata:
    lo: torch.Tensor
    hi: torch.Tensor


class PageMetadataTable:
    """List-like view of the device page metadata (one PageMetadata per page)."""

    def __init__(self, cache: PagedKVCache, n: int):
        self.cache = cache
        self.n = n
        self.lo, self.hi = cache.unit_meta(0, 0)

    def __len__(self) -> int:
        return pages_for(self.n)

    def __getitem__(self, i: int) -> PageMetadata:
        return PageMetadata(lo=self.lo[i], hi=self.hi[i])

    def __iter__(self):
        return (self[i] for i in range(len(self)))


@dataclass(frozen=True, eq=False)
class PagedQuantKeyCache:
    """quantcache.py:74-81, backed by a one-unit device pool."""
    kv: PagedKVCache
    n_tokens: int
    d: int
    bits: int
    page_size: int

    @property
    def page_table(self) -> list[int]:
        return list(range(pages_for(self.n_tokens)))

    @property
    def pages(self) -> list[QuantPage]:
        packed, scale, zero = self.kv.unit_quant(0, 0)
        out = []
        for p in range(pages_for(self.n_tokens)):
            lo, hi = p * 16, min(self.n_tokens, (p + 1) * 16)
            block = torch.zeros(16, self.d * self.bits // 8, dtype=torch.uint8, device=packed.device)
            block[: hi - lo] = packed[lo:hi]
            sc = torch.zeros(16, dtype=torch.float64, device=packed.device)
            zr = torch.zeros(16, dtype=torch.float64, device=packed.device)
            sc[: hi - lo] = scale[lo:hi].double()
            zr[: hi - lo] = zero[lo:hi].double()
            out.append(QuantPage(packed=bytes(block.cpu().numpy().tobytes()), scales=sc, zeros=zr,
                                 valid_len=hi - lo))
        return out


@dataclass(frozen=True)
class EstimateResult:
    scores: torch.Tensor
    bytes_touched: int


def _as_cuda_matrix(keys) -> torch.Tensor:
    K = torch.as_tensor(keys)
    if not K.is_cuda:
        raise ValueError("keys must be a CUDA tensor (the Twilight path has no CPU fallback)")
    return K


def _unit_cache(keys: torch.Tensor, values: torch.Tensor | None = None, group_size: int = 1,
                num_seqs: int = 1, bits: int = 4) -> PagedKVCache:
    """One KV context as a paged pool.  ``num_seqs`` > 1 makes every sequence
    share the same physical pages (the G-groups of run_grouped)."""
    K = _as_cuda_matrix(keys)
    if K.ndim != 2 or K.shape[0] == 0:
        raise ValueError("keys must be a non-empty (n, d) matrix")
    if K.shape[1] != L.HEAD_DIM:
        raise ValueError(f"the B200 path is built for d={L.HEAD_DIM}, got d={K.shape[1]}")
    if not bool(torch.isfinite(K).all()):
        raise ValueError("keys contain non-finite entries")
    dtype = K.dtype if K.dtype in (torch.bfloat16, torch.float32) else None
    if dtype is None:
        raise ValueError(f"keys dtype {K.dtype} not supported (bf16 or float32)")
    n = K.shape[0]
    P = pages_for(n)
    pt = torch.arange(P, dtype=torch.int32, device=K.device).repeat(num_seqs, 1)
    cache = PagedKVCache(num_seqs, 1, group_size, P, dtype=dtype, device=K.device, page_table=pt, num_phys_pages=P,
                         bits=bits)
    V = values if values is not None else torch.zeros_like(K)
    Kp = K.view(1, 1, n, L.HEAD_DIM)
    Vp = torch.as_tensor(V).to(dtype).view(1, 1, n, L.HEAD_DIM)
    # write the shared pages once (sequence 0), then quantize for every sequence row
    cache.prefill(Kp.expand(num_seqs, 1, n, L.HEAD_DIM), Vp.expand(num_seqs, 1, n, L.HEAD_DIM))
    return cache


def _shared_pool(pool: PagedKVCache, values: torch.Tensor, group_size: int, num_seqs: int) -> PagedKVCache:
    """A prebuilt one-context pool (build_cache) reused for ``num_seqs``
    sequence rows of ``group_size`` query heads: the quantized keys, page
    metadata and |k| bound are shared as built (no tw_quant_build), only the
    values are written into the pool's V pages."""
    n = int(pool.seq_lens[0].item())
    V = torch.as_tensor(values).to(device=pool.device, dtype=pool.dtype)
    if V.shape != (n, L.HEAD_DIM):
        raise ValueError(f"values must be ({n}, {L.HEAD_DIM}) to match the cache, got {tuple(V.shape)}")
    P = pages_for(n)
    pad = P * L.PAGE_SIZE - n
    Vp = torch.nn.functional.pad(V, (0, 0, 0, pad)) if pad else V
    phys = pool.page_table[0, :P].long()
    pool.v_cache[phys, 0] = Vp.view(P, L.PAGE_SIZE, L.HEAD_DIM)
    v = PagedKVCache.__new__(PagedKVCache)
    v.__dict__.update(pool.__dict__)
    v.num_seqs, v.group_size = num_seqs, group_size
    v.page_table = pool.page_table[:1].repeat(num_seqs, 1).contiguous()
    v.seq_lens = pool.seq_lens[:1].repeat(num_seqs).contiguous()
    v.kabsmax = pool.kabsmax[:1].repeat(num_seqs, 1).contiguous()
    v._struct = None
    return v


def quantize_row(k, bits: int = 4):
    """quantcache.py:95-114 on tw_quant_rows: (codes uint8 tensor, QuantParams)."""
    if bits not in SUPPORTED_BITS:
        raise ValueError(f"bits must be one of {SUPPORTED_BITS}, got {bits}")
    row = torch.as_tensor(k)
    if not row.is_cuda:
        raise ValueError("k must be a CUDA tensor")
    if row.ndim != 1 or row.numel() == 0:
        raise ValueError("key row must be a non-empty 1-D array")
    if not bool(torch.isfinite(row).all()):
        raise ValueError("key row contains non-finite entries")
    if row.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError(f"dtype {row.dtype} not supported (bf16 or float32)")
    codes, scale, zero = quantize_rows(row.view(1, -1), bits)
    return codes[0], QuantParams(scale=float(scale[0]), zero=float(zero[0]))


def quantize_rows(rows: torch.Tensor, bits: int = 4):
    """Batched quantize_row: (codes [n, d] u8, scale [n] f64, zero [n] f64)."""
    rows = rows.contiguous()
    n, d = rows.shape
    codes = torch.empty(n, d, dtype=torch.uint8, device=rows.device)
    scale = torch.empty(n, dtype=torch.float64, device=rows.device)
    zero = torch.empty(n, dtype=torch.float64, device=rows.device)
    L.check(L.lib().tw_quant_rows(L.ptr(rows), n, d, L.dtype_code(rows.dtype), bits, L.ptr(codes), L.ptr(scale),
                                  L.ptr(zero), L.stream_handle()), "tw_quant_rows")
    return codes, scale, zero


def dequantize_row(codes, params: QuantParams, dtype=torch.float64) -> torch.Tensor:
    """quantcache.py:117-119."""
    c = torch.as_tensor(codes).double()
    return (params.zero + params.scale * c).to(dtype)


def pack_codes(codes) -> bytes:
    """Two 4-bit codes per byte, even index in the low nibble (quantcache.py:142-151)."""
    arr = torch.as_tensor(codes)
    if arr.ndim != 1 or arr.numel() % 2 != 0:
        raise ValueError("codes must be 1-D with even length")
    if arr.numel() == 0:
        raise ValueError("codes must be non-empty")
    if bool((arr < 0).any()) or bool((arr > 15).any()):
        raise ValueError("4-bit codes must lie in [0, 15]")
    a = arr.to(torch.uint8)
    return bytes((a[0::2] | (a[1::2] << 4)).cpu().numpy().tobytes())


def unpack_codes(packed: bytes, d: int, device="cuda") -> torch.Tensor:
    """quantcache.py:154-160."""
    if d <= 0 or d % 2 != 0:
        raise ValueError("d must be a positive even number")
    if len(packed) != d // 2:
        raise ValueError(f"expected {d // 2} packed bytes, got {len(packed)}")
    b = torch.frombuffer(bytearray(packed), dtype=torch.uint8).to(device)
    out = torch.empty(d, dtype=torch.uint8, device=device)
    out[0::2] = b & 0x0F
    out[1::2] = b >> 4
    return out


def build_page_metadata(keys, page_size: int = 16) -> PageMetadataTable:
    """Per-channel page min/max of the real rows (quantcache.py:163-175)."""
    if page_size != L.PAGE_SIZE:
        if page_size < 1:
            raise ValueError("page_size must be at least 1")
        raise ValueError("the B200 path uses 16-token pages")
    K = _as_cuda_matrix(keys)
    return PageMetadataTable(_unit_cache(K), K.shape[0])


def build_cache(keys, page_size: int = 16, bits: int = 4, values=None):
    """quantcache.py:178-235: (PagedQuantKeyCache, PageMetadataTable)."""
    if bits not in SUPPORTED_BITS:
        raise ValueError(f"bits must be one of {SUPPORTED_BITS}, got {bits}")
    if page_size != L.PAGE_SIZE:
        if page_size < 1:
            raise ValueError("page_size must be at least 1")
        raise ValueError("the B200 path uses 16-token pages")
    K = _as_cuda_matrix(keys)
    kv = _unit_cache(K, values, bits=bits)
    n = K.shape[0]
    return (PagedQuantKeyCache(kv=kv, n_tokens=n, d=K.shape[1], bits=bits, page_size=16), PageMetadataTable(kv, n))


def estimate_scores(q, cache: PagedQuantKeyCache, candidates: TokenSelection) -> EstimateResult:
    """q . k_hat / sqrt(d) at the candidate tokens (quantcache.py:238-272)."""
    qv = torch.as_tensor(q)
    if qv.ndim != 1 or qv.shape[0] != cache.d:
        raise ValueError(f"query dimension {tuple(qv.shape)} does not match cache d={cache.d}")
    if candidates.n != cache.n_tokens:
        raise ValueError("candidate set built for a different context size")
    idx = candidates.indices
    if idx.numel() == 0:
        raise ValueError("no candidates to estimate")
    if int(idx[-1]) >= cache.n_tokens:
        raise IndexError("candidate index beyond cached tokens")
    kv = cache.kv
    qd = qv.to(device=kv.device, dtype=kv.dtype).contiguous()
    ids = idx.to(torch.int32).contiguous()
    m = ids.numel()
    out = torch.empty(m, dtype=torch.float32, device=kv.device)
    status = torch.zeros(1, dtype=torch.int32, device=kv.device)
    L.check(L.lib().tw_estimate_tokens(ctypes.byref(kv.struct()), 0, 0, L.ptr(qd), L.ptr(ids), m, L.ptr(out),
                                       L.ptr(status), L.stream_handle()), "tw_estimate_tokens")
    L.check(int(status.item()), "tw_estimate_tokens")
    return EstimateResult(scores=out, bytes_touched=int(m) * (cache.d * cache.bits // 8 + PARAM_BYTES))
