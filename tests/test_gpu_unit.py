"""The fused per-unit K1+K2+K3 kernel (csrc/unit.cu, tw_select_estimate_topp)
against the separate kernels it replaces (tw_quant_append / the fused Quest
filter, tw_select, tw_estimate, tw_topp): same inputs, bit-identical cache
state, candidate pages, logits, per-head statistics, final sets and outputs.
The separate path is itself pinned to the oracle (test_gpu_decode.py,
test_gpu_configs.py); test_gpu_configs.py also runs the fused kernel against
the oracle at the C2 and C5 shapes."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for  # noqa: E402
from paper_2502_02770_b200.workload import make_batch, tau_schedule  # noqa: E402

TAUS = (0.25, 0.5, 1.0, 2.0)


def _run(B, H, G, n, selector, budget, p, unit, aliased=False, ragged=False, seed=11):
    os.environ["TW_UNIT"] = "1" if unit else "0"
    try:
        cache = PagedKVCache(B, H, G, pages_for(n + 1), dtype=torch.bfloat16)
        batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=seed)
        # ragged: sequence b holds n - 37 b tokens
        cache.prefill(batch.K, batch.V, [n - 37 * b for b in range(B)] if ragged else None)
        step = make_batch(B, H, G, 16, torch.bfloat16, tau=tau_schedule(H, TAUS), seed=seed + 1)
        dec = TwilightDecoder(cache, selector, budget=budget, p=p)
        assert dec.unit_path == unit
        positions = None if aliased else cache.seq_lens.clone()
        out = dec.step(step.q.contiguous(), step.k_new.contiguous(), step.v_new.contiguous(), positions)
        torch.cuda.synchronize()
        return cache, dec, out
    finally:
        os.environ.pop("TW_UNIT", None)


def _same(a, b, what):
    assert torch.equal(a, b), what


@pytest.mark.parametrize("case", [
    dict(B=16, H=8, G=4, n=4100, selector="quest", budget=1024, p=0.95),      # C2-like, small context
    dict(B=16, H=8, G=4, n=4100, selector="quest", budget=1024, p=0.95, aliased=True),
    dict(B=8, H=8, G=4, n=2000, selector="quest", budget=3000, p=0.9),         # budget above n: every page
    dict(B=32, H=4, G=2, n=3333, selector="quest", budget=700, p=0.8),
    dict(B=16, H=4, G=1, n=5000, selector="full", budget=None, p=0.9),
    dict(B=64, H=1, G=4, n=1024, selector="quest", budget=256, p=0.99),
    dict(B=16, H=8, G=4, n=4100, selector="quest", budget=1024, p=0.0),        # p = 0: nothing kept
    dict(B=16, H=8, G=4, n=4100, selector="quest", budget=1024, p=0.95, ragged=True),
    dict(B=16, H=4, G=1, n=3000, selector="full", budget=None, p=0.95, ragged=True, aliased=True),
    dict(B=16, H=8, G=4, n=32767, selector="quest", budget=8192, p=0.95),      # the C2 bench geometry
])
def test_unit_kernel_matches_separate_kernels(case):
    case = dict(case)
    ca, da, oa = _run(**case, unit=True)
    cb, db, ob = _run(**case, unit=False)
    for f in ("k_cache", "v_cache", "kq", "kmeta", "kabsmax", "seq_lens"):
        _same(getattr(ca, f), getattr(cb, f), f)
    ba, bb = da.bufs, db.bufs
    _same(ba.cand_count, bb.cand_count, "cand_count")
    U = ba.cand_count.numel()
    G = case["G"]
    T = ca.max_pages * 16
    for u in range(U):
        c = int(ba.cand_count[u])
        _same(ba.cand_pages[u, :c], bb.cand_pages[u, :c], f"cand_pages unit {u}")
        _same(ba.logits[u, :, :16 * c], bb.logits[u, :, :16 * c], f"logits unit {u}")
        f = int(ba.final_count[u])
        assert f == int(bb.final_count[u]), f"final_count unit {u}"
        _same(ba.final_idx[u, :f], bb.final_idx[u, :f], f"final_idx unit {u}")
    _same(ba.head_max, bb.head_max, "head_max")
    _same(ba.head_thr, bb.head_thr, "head_thr")
    # B1 and B0 exactly; the masses are fp64 sums of fp32 bin masses whose grouping
    # follows the top-p warp-group size (1024 threads per head here at G = 1, 512 in tw_topp)
    _same(ba.head_stats[:, [0, 3]], bb.head_stats[:, [0, 3]], "head_stats B1/B0")
    torch.testing.assert_close(ba.head_stats[:, 1:3], bb.head_stats[:, 1:3], rtol=1e-6, atol=0)
    # work items may be claimed in a different unit order; outputs are per head and identical
    _same(oa, ob, "attention output")
    assert T > 0
