"""Seeded synthetic decode workloads, generated on the GPU.

Pattern of the reference's gaussian_qk generator (workload.py:88-111): keys
and values iid N(0, 1), queries N(0, 1) / tau so logits become
K q / (sqrt(d) tau).  K/V are shared by the G query heads of a KV head.
``page_local`` keys follow test_pipeline.py:189-202 (per-page level with
sigma 3 plus jitter 0.3), the regime where Quest page bounds are informative.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

HEAD_DIM = 128


@dataclass
class DecodeBatch:
    K: torch.Tensor      # [B, H_kv, n, d]
    V: torch.Tensor      # [B, H_kv, n, d]
    q: torch.Tensor      # [B, H_kv*G, d]
    k_new: torch.Tensor  # [B, H_kv, d]
    v_new: torch.Tensor  # [B, H_kv, d]


def tau_schedule(num_kv_heads: int, taus=(0.25, 0.5, 1.0, 2.0)) -> torch.Tensor:
    """Per-KV-head temperature: cycles focused .. diffuse heads."""
    return torch.tensor([taus[h % len(taus)] for h in range(num_kv_heads)], dtype=torch.float32)


def make_batch(B: int, H_kv: int, G: int, n: int, dtype=torch.bfloat16, tau=1.0, seed: int = 0,
               device="cuda", page_local: bool = False) -> DecodeBatch:
    """K/V of n cached tokens plus one new token; q for H_kv*G heads.

    `tau` is a float or a per-KV-head tensor [H_kv] (query heads of a KV
    head share its temperature).
    """
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    d = HEAD_DIM
    K = torch.randn(B, H_kv, n, d, generator=g, device=device, dtype=torch.float32)
    if page_local:
        P = -(-n // 16)
        level = torch.randn(B, H_kv, P, 1, d, generator=g, device=device) * 3.0
        K = (level.expand(B, H_kv, P, 16, d).reshape(B, H_kv, P * 16, d)[:, :, :n] + 0.3 * K)
    V = torch.randn(B, H_kv, n, d, generator=g, device=device, dtype=torch.float32)
    q = torch.randn(B, H_kv * G, d, generator=g, device=device, dtype=torch.float32)
    t = torch.as_tensor(tau, dtype=torch.float32, device=device)
    if t.ndim == 1:
        t = t.repeat_interleave(G).view(1, H_kv * G, 1)
    q = q / t
    k_new = torch.randn(B, H_kv, d, generator=g, device=device)
    v_new = torch.randn(B, H_kv, d, generator=g, device=device)
    return DecodeBatch(K=K.to(dtype), V=V.to(dtype), q=q.to(dtype), k_new=k_new.to(dtype), v_new=v_new.to(dtype))
