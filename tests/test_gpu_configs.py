"""Parity at the BASELINE configurations: the exact geometry bench.py measures.

For C1 (fp32 and bf16), C2 (the bench's own shapes, seeds and tau mix) and a
C5- and a C3-shaped batch at 131,072 tokens, one decode step runs through
TwilightDecoder.step (the fused K1+K2 path the bench times) and a seeded
sample of units covering every tau is checked against the oracle:

  K1   the appended row's INT4 codes / scale / zero and its page's channel
       min/max: bit-exact (quantcache.py:95-114, 163-175)
  K2   every query head's Quest page set and the unit's union: bit-exact
       (selectors.py:112-132, 178-186)
  K3   logits vs the oracle's INT4 estimate (fixed-point q tolerance); per-head
       top-p sets: the oracle's minimal tie-closed set on the GPU logits up to
       threshold ties (pruner.py:57-114); final set = union of the head sets
       (pipeline.py:347)
  K4   outputs vs the oracle's subset attention on the GPU's final set: 1e-4
       relative (fp32) / 2e-2 (bf16) (attention.py:106-136)

and the chained comparison of SURVEY.md 8(c)(ii) -- the GPU chain against the
oracle's own INT4 chain -- is recorded per unit (symmetric-difference size,
attained-mass delta) in the parity report (TW_PARITY_REPORT, default
gpurun_out/parity_report.json).  The top-p kernel variant each config runs is
chosen by shape (csrc/topp.cu launch_unit): C2 -> topp_unit_kernel<4,4,*>,
C5-shaped (units > SMs) -> <4,2,*>, C3-shaped (G = 1) -> <1,4,*>, C1 ->
topp_head_kernel<4>.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import twilight_oracle as orc
from tests.gpu_util import check_unit_topp, to_np

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for  # noqa: E402
from paper_2502_02770_b200.workload import make_batch, tau_schedule  # noqa: E402

TAUS = (0.25, 0.5, 1.0, 2.0)  # bench.py TAUS
REPORT = {}

# name: (B, H, G, n, selector, budget, p, dtype, sampled (b, h) units)
CONFIGS = {
    "C1_bf16": (1, 8, 4, 8192, "quest", 2048, 0.95, torch.bfloat16, [(0, h) for h in range(8)]),
    "C1_fp32": (1, 8, 4, 8192, "quest", 2048, 0.95, torch.float32, [(0, h) for h in range(8)]),
    "C2": (16, 8, 4, 32768, "quest", 8192, 0.95, torch.bfloat16,
           [(0, 0), (0, 1), (3, 2), (5, 3), (7, 4), (9, 5), (12, 6), (15, 7)]),
    # C5 shape (Llama GQA, 128k, Quest n/4) with 160 units > 148 SMs: the narrow top-p kernel
    "C5_shaped": (20, 8, 4, 131072, "quest", 32768, 0.9, torch.bfloat16,
                  [(0, 0), (4, 1), (9, 2), (13, 3), (19, 4), (2, 7)]),
    # C3 shape per GPU (LongChat MHA, G = 1, full selector, 128k): 8 sequences x 4 KV heads
    "C3_shaped": (8, 4, 1, 131072, "full", None, 0.9, torch.bfloat16,
                  [(0, 0), (2, 1), (5, 2), (7, 3), (3, 0), (6, 2)]),
}


def _write_report():
    path = os.environ.get("TW_PARITY_REPORT") or os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "parity_report.json")
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        old = {}
        if os.path.exists(path):
            with open(path) as f:
                old = json.load(f)
        old.update(REPORT)
        with open(path, "w") as f:
            json.dump(old, f, indent=1)
    except OSError:
        pass


def _bench_geometry(B, H, G, n, selector, budget, p, dtype, seed):
    """bench.run_ours' layer: prefill n-1 tokens, then one step appends token n-1."""
    cache = PagedKVCache(B, H, G, pages_for(n), dtype=dtype)
    batch = make_batch(B, H, G, n, dtype, tau=tau_schedule(H, TAUS), seed=seed)
    cache.prefill(batch.K[:, :, : n - 1], batch.V[:, :, : n - 1])
    del batch
    step = make_batch(B, H, G, 16, dtype, tau=tau_schedule(H, TAUS), seed=seed + 999)
    dec = TwilightDecoder(cache, selector, budget=budget, p=p, head_page_bits=True)
    positions = torch.full((B,), n - 1, dtype=torch.int32, device="cuda")
    q = step.q.contiguous()
    out = dec.step(q, step.k_new.contiguous(), step.v_new.contiguous(), positions)
    torch.cuda.synchronize()
    return cache, dec, q, step, out


@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_parity(name):
    B, H, G, n, selector, budget, p, dtype, units = CONFIGS[name]
    cache, dec, q, step, out = _bench_geometry(B, H, G, n, selector, budget, p, dtype, seed=1234)
    assert cache.seq_lens.tolist() == [n] * B
    bufs = dec.bufs
    words = -(-cache.max_pages // 32)
    bits = bufs.head_page_bits.cpu().numpy().view(np.uint32).reshape(-1, words)
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    rows = []
    taus_seen = set()
    for b, h in units:
        u = b * H + h
        taus_seen.add(TAUS[h % len(TAUS)])
        K, V = to_np(cache.unit_keys(b, h)), to_np(cache.unit_values(b, h))
        assert K.shape[0] == n
        # ---- K1: the appended row and its page
        np.testing.assert_array_equal(K[-1], to_np(step.k_new[b, h]))
        codes, scale, zero = orc.quantize_rows(K[-1:])
        packed, sc, zr = cache.unit_quant(b, h)
        np.testing.assert_array_equal(packed[-1].cpu().numpy(), orc.pack_nibbles(codes)[0])
        assert sc[-1].item() == np.float32(scale[0]) and zr[-1].item() == np.float32(zero[0])
        lo, hi = orc.page_bounds(K)
        mlo, mhi = cache.unit_meta(b, h)
        np.testing.assert_array_equal(to_np(mlo[-1]), lo[-1].astype(np.float32))
        np.testing.assert_array_equal(to_np(mhi[-1]), hi[-1].astype(np.float32))
        Qn = to_np(q[b, h * G:(h + 1) * G])
        # ---- K2: per-head pages and the union
        prepared = orc.prepare_unit(K)
        ncand = int(bufs.cand_count[u])
        cand_pages = bufs.cand_pages[u, :ncand].cpu().numpy()
        if selector == "quest":
            heads = []
            for g in range(G):
                want = orc.quest_select_pages(Qn[g], lo, hi, budget, n)
                got = np.flatnonzero(np.unpackbits(bits[u * G + g].view(np.uint8), bitorder="little"))
                np.testing.assert_array_equal(got, want, err_msg=f"{name} unit {u} head {g} pages")
                heads.append(want)
            np.testing.assert_array_equal(cand_pages, orc.union_sorted(heads))
        else:
            np.testing.assert_array_equal(cand_pages, np.arange(pages_for(n)))
        # ---- K3: estimate + isolated pruner on the GPU logits, final = union of the head sets
        cand, z, sels, final, whys = check_unit_topp(bufs, u, G, p)
        np.testing.assert_array_equal(cand, orc.pages_to_tokens(cand_pages, n))
        for g in range(G):
            z_ref = orc.estimate_logits(Qn[g], prepared[2], prepared[3], prepared[4], cand)
            amp = np.abs(Qn[g]).sum() * np.abs(K).max() / np.sqrt(128)
            np.testing.assert_allclose(z[g], z_ref, rtol=0, atol=2e-6 * amp + 1e-6)
        # ---- K4 on the GPU's final set
        for g in range(G):
            w = orc.full_weights(Qn[g], K)
            want = orc.subset_attention(w, V, final, True)
            np.testing.assert_allclose(to_np(out[b, h * G + g]), want, rtol=tol, atol=tol * np.abs(want).max(),
                                       err_msg=f"{name} unit {u} head {g} output")
        # ---- chained: the oracle's own INT4 chain on the same unit
        res = orc.decode_unit(Qn, K, V, selector=selector, budget=budget if budget else 1.0, p=p,
                              prepared=prepared)
        mass_delta = []
        for g in range(G):
            w = orc.full_weights(Qn[g].astype(np.float64), K.astype(np.float64))
            mass_delta.append(float(w[final].sum() - w[res["final"]].sum()))
        rows.append({"unit": u, "tau": TAUS[h % len(TAUS)], "cand_tokens": int(cand.size),
                     "head_b1": [int(s.size) for s in sels], "final": int(final.size),
                     "oracle_chain_final": int(res["final"].size),
                     "symdiff_vs_oracle_chain": int(np.setxor1d(final, res["final"]).size),
                     "attained_true_mass_delta": mass_delta, "isolated_pruner": whys,
                     "max_abs_out_err": float(max(np.abs(to_np(out[b, h * G + g]) - res["out"][g]).max()
                                                  for g in range(G))) if np.array_equal(final, res["final"])
                     else None})
    assert taus_seen == set(TAUS)
    REPORT[name] = {"B": B, "H_kv": H, "G": G, "ctx": n, "selector": selector, "budget": budget, "p": p,
                    "dtype": str(dtype).replace("torch.", ""), "units_checked": rows}
    _write_report()
