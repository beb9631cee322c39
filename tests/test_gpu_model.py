"""C4 decode-step harness (paper_2502_02770_b200/model.py) against a plain
PyTorch fp32 reference of the same random-init model with dense attention.
With the dense configuration on every layer (full selector, p = 1 -- the
reference's bypass_config, pipeline.py:129-136) the logits must agree."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2502_02770_b200.model import LlamaConfig, LlamaTwilightDecoder, rms_norm, rope  # noqa: E402


def torch_reference(m: LlamaTwilightDecoder, tokens):
    cfg = m.cfg
    H, Hk, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    G = H // Hk
    x = m.embed[tokens].float()
    cache = m.caches[0]
    for li, lw in enumerate(m.layers):
        h = rms_norm(x.to(m.dtype), lw["n1"], cfg.eps).float()
        qkv = h @ lw["wqkv"].float()
        q = qkv[:, : H * d].view(-1, H, d)
        k = qkv[:, H * d:(H + Hk) * d].view(-1, Hk, d)
        v = qkv[:, (H + Hk) * d:].reshape(-1, Hk, d)
        q = rope(q.to(m.dtype), m.cos, m.sin).float()
        k = rope(k.to(m.dtype), m.cos, m.sin)
        outs = []
        for b in range(m.B):
            ob = []
            for hk in range(Hk):
                K = cache.unit_keys(b, hk).float().clone()
                V = cache.unit_values(b, hk).float().clone()
                K[-1] = k[b, hk].float()
                V[-1] = v[b, hk].to(m.dtype).float()
                for g in range(G):
                    w = torch.softmax(K @ q[b, hk * G + g] / math.sqrt(d), 0)
                    ob.append(w @ V)
            outs.append(torch.stack(ob))
        attn = torch.stack(outs)
        x = x + attn.view(-1, H * d).to(m.dtype).float() @ lw["wo"].float()
        h = rms_norm(x.to(m.dtype), lw["n2"], cfg.eps).float()
        gu = h @ lw["wgu"].float()
        gate, up = gu[:, : cfg.intermediate], gu[:, cfg.intermediate:]
        x = x + (torch.nn.functional.silu(gate) * up).to(m.dtype).float() @ lw["wd"].float()
    return rms_norm(x.to(m.dtype), m.norm_f, cfg.eps).float() @ m.lm_head.float()


def test_dense_configuration_matches_torch_reference():
    cfg = LlamaConfig(hidden=256, n_layers=3, n_heads=8, n_kv_heads=2, intermediate=512, vocab=1000,
                      bypass_layers=(0, 1, 2))
    m = LlamaTwilightDecoder(cfg, batch=2, ctx=300, seed=3)
    tokens = torch.tensor([5, 77], device="cuda")
    got = m.step(tokens)
    torch.cuda.synchronize()
    want = torch_reference(m, tokens)
    rel = (got - want).abs().max() / want.abs().max()
    assert rel < 3e-2, float(rel)


def test_twilight_layers_run_and_stay_close_to_dense():
    cfg = LlamaConfig(hidden=256, n_layers=3, n_heads=8, n_kv_heads=2, intermediate=512, vocab=1000,
                      bypass_layers=(0,))
    m = LlamaTwilightDecoder(cfg, batch=2, ctx=600, selector="full", p=1.0, seed=4)
    tokens = torch.tensor([1, 2], device="cuda")
    got = m.step(tokens)
    torch.cuda.synchronize()
    want = torch_reference(m, tokens)
    rel = (got - want).abs().max() / want.abs().max()
    assert torch.isfinite(got).all() and rel < 3e-2, float(rel)
