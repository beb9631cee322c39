"""Llama-3.1-8B decode-step harness around the Twilight attention path (C4).

SURVEY.md §8(f2): the reference has no model code ("real model-weight
loading" is a non-goal); config C4 asks for a whole 32-layer
decode step with random-init weights.  Projections and the MLP are plain
library GEMMs (torch.matmul -> cuBLAS); RMSNorm/RoPE/SiLU are torch ops; the
attention of every layer is this repo's path: layers in `bypass_layers`
(default 0 and 1, pipeline.py:59) use dense decode (K5), the
others append + Quest + INT4 estimate + top-p + sparse attention (K1-K4).

Memory: batch 64 x 64k context is 17.2 GB of K/V per layer (550 GB for 32
layers), so by default all layers alias ONE physical paged cache (BASELINE.md
§4) -- every layer still streams its own full set of bytes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from .decode import PagedKVCache, TwilightDecoder, pages_for


@dataclass(frozen=True)
class LlamaConfig:
    hidden: int = 4096
    n_layers: int = 32
    n_heads: int = 32
    n_kv_heads: int = 8
    head_dim: int = 128
    intermediate: int = 14336
    vocab: int = 128256
    rope_theta: float = 500000.0
    eps: float = 1e-5
    bypass_layers: tuple[int, ...] = (0, 1)


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """Rotate-half RoPE for x [B, H, d] with cos/sin [B, 1, d/2]."""
    x1, x2 = x[..., : x.shape[-1] // 2].float(), x[..., x.shape[-1] // 2:].float()
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1).to(x.dtype)


class LlamaTwilightDecoder:
    """One decode step of a random-init Llama-3.1-8B-shaped model."""

    def __init__(self, cfg: LlamaConfig, batch: int, ctx: int, selector: str = "quest", budget=None, p: float = 0.95,
                 dtype=torch.bfloat16, device="cuda", seed: int = 0, share_kv: bool = True,
                 n_layers: int | None = None, q_taus: tuple[float, ...] | None = None):
        self.cfg = cfg
        self.B, self.ctx, self.dtype = batch, ctx, dtype
        self.L = n_layers or cfg.n_layers
        dev = torch.device(device)
        g = torch.Generator(device=dev)
        g.manual_seed(seed)

        def w(*shape, scale=0.02):
            return (torch.randn(*shape, generator=g, device=dev, dtype=torch.float32) * scale).to(dtype)

        H, Hk, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        self.embed = w(cfg.vocab, cfg.hidden)
        self.lm_head = w(cfg.hidden, cfg.vocab)
        self.norm_f = torch.ones(cfg.hidden, device=dev, dtype=dtype)
        self.layers = []
        G = H // Hk
        for _ in range(self.L):
            wqkv = w(cfg.hidden, (H + 2 * Hk) * d)
            if q_taus:  # per-KV-head query scale: q ~ N(0, 1/tau^2) like the synthetic layer workloads
                col = torch.tensor([1.0 / (0.02 * math.sqrt(cfg.hidden) * q_taus[(j // (G * d)) % len(q_taus)])
                                    for j in range(H * d)], device=dev)
                wqkv[:, : H * d] = (wqkv[:, : H * d].float() * col).to(dtype)
            self.layers.append(dict(
                wqkv=wqkv, wo=w(H * d, cfg.hidden),
                wgu=w(cfg.hidden, 2 * cfg.intermediate), wd=w(cfg.intermediate, cfg.hidden),
                n1=torch.ones(cfg.hidden, device=dev, dtype=dtype), n2=torch.ones(cfg.hidden, device=dev, dtype=dtype)))
        # paged KV caches: one shared pool (default) or one per layer
        n_caches = 1 if share_kv else self.L
        self.caches = []
        for c in range(n_caches):
            cache = PagedKVCache(batch, Hk, G, pages_for(ctx), dtype=dtype, device=dev)
            gk = torch.Generator(device=dev)
            gk.manual_seed(seed + 1000 + c)
            for b0 in range(0, batch, 8):  # fill in slices to bound the fp32 temporaries
                b1 = min(batch, b0 + 8)
                K = torch.randn(b1 - b0, Hk, ctx - 1, d, generator=gk, device=dev).to(dtype)
                V = torch.randn(b1 - b0, Hk, ctx - 1, d, generator=gk, device=dev).to(dtype)
                sub = cache.view(b0, b1)
                sub.prefill(K, V)
                del K, V
            self.caches.append(cache)
        self.decs = []
        shared = None  # one set of step buffers for every layer (same geometry)
        for li in range(self.L):
            cache = self.caches[0 if share_kv else li]
            if li in cfg.bypass_layers:
                dec = TwilightDecoder(cache, "full", p=1.0, bufs=shared)
            else:
                dec = TwilightDecoder(cache, selector, budget=budget, p=p, bufs=shared)
            shared = dec.bufs
            self.decs.append(dec)
        self.positions = torch.full((batch,), ctx - 1, dtype=torch.int32, device=dev)
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, d, 2, device=dev, dtype=torch.float32) / d))
        ang = (ctx - 1) * inv
        self.cos = torch.cos(ang).view(1, 1, -1).expand(batch, 1, -1).contiguous()
        self.sin = torch.sin(ang).view(1, 1, -1).expand(batch, 1, -1).contiguous()
        self.attn_out = torch.empty(batch, H, d, dtype=torch.float32, device=dev)

    def step(self, tokens: torch.Tensor, record: dict | None = None) -> torch.Tensor:
        """tokens [B] int64 -> next-token logits [B, vocab] (float32).
        `record`, if given, receives {layer: (q, k, v)} of the attention inputs."""
        cfg = self.cfg
        H, Hk, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        x = self.embed[tokens]
        for li, lw in enumerate(self.layers):
            h = rms_norm(x, lw["n1"], cfg.eps)
            qkv = h @ lw["wqkv"]
            q = qkv[:, : H * d].view(-1, H, d)
            k = qkv[:, H * d:(H + Hk) * d].view(-1, Hk, d)
            v = qkv[:, (H + Hk) * d:].reshape(-1, Hk, d).contiguous()
            q = rope(q, self.cos, self.sin).contiguous()
            k = rope(k, self.cos, self.sin).contiguous()
            dec = self.decs[li]
            if record is not None:
                record[li] = (q.clone(), k.clone(), v.clone())
            if li in cfg.bypass_layers:
                dec.cache.append(k, v, self.positions)
                dec.dense(q, self.attn_out)
            else:
                dec.step(q, k, v, self.positions, self.attn_out)
            x = x + self.attn_out.view(-1, H * d).to(self.dtype) @ lw["wo"]
            h = rms_norm(x, lw["n2"], cfg.eps)
            gu = h @ lw["wgu"]
            gate, up = gu[:, : cfg.intermediate], gu[:, cfg.intermediate:]
            x = x + (torch.nn.functional.silu(gate.float()) * up.float()).to(self.dtype) @ lw["wd"]
        return (rms_norm(x, self.norm_f, cfg.eps) @ self.lm_head).float()

    def weight_bytes(self) -> int:
        """Weight bytes one step streams (embedding rows are gathered, not streamed)."""
        n = self.lm_head.numel()
        for lw in self.layers:
            n += sum(t.numel() for t in lw.values())
        return n * self.embed.element_size()
