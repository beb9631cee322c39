"""The CPU oracle (oracle/twilight_oracle.py) reproduces the reference's own
outputs (tests/golden, written by oracle/gen_golden.py running nucleuskv).

Bit-exact: INT4 codes, packed bytes, fp64 params, page metadata, fp64 Quest
scores, selected page/token sets, top-p index sets, thresholds, iteration
counts.  fp32 results that go through BLAS (estimate, attention) are compared
with a tolerance, because the summation order of sgemv is not pinned.
"""

import math

import numpy as np
import pytest

from oracle import twilight_oracle as orc


def test_quantization_matches_reference(golden):
    cases = golden("quant")
    assert bytes(cases["pack"]["arange16"]) == bytes.fromhex("1032547698badcfe")
    for name, c in cases.items():
        if name == "pack":
            continue
        codes, scale, zero = orc.quantize_rows(c["K"])
        np.testing.assert_array_equal(codes, c["codes"], err_msg=name)
        np.testing.assert_array_equal(scale, c["scale"], err_msg=name)
        np.testing.assert_array_equal(zero, c["zero"], err_msg=name)
        np.testing.assert_array_equal(orc.pack_nibbles(codes), c["packed"], err_msg=name)
        np.testing.assert_array_equal(orc.unpack_nibbles(c["packed"]), c["codes"], err_msg=name)
        lo, hi = orc.page_bounds(c["K"])
        np.testing.assert_array_equal(lo, c["lo"], err_msg=name)
        np.testing.assert_array_equal(hi, c["hi"], err_msg=name)
        for r in range(3):
            if f"row{r}_codes" in c:
                rc, rs, rz = orc.quantize_rows(c["K"][r])
                np.testing.assert_array_equal(rc[0], c[f"row{r}_codes"])
                assert rs[0] == c[f"row{r}_params"][0] and rz[0] == c[f"row{r}_params"][1]


def test_quest_matches_reference_bit_exact(golden):
    for name, c in golden("quest").items():
        K, q = c["K"], c["q"]
        n = K.shape[0]
        lo, hi = orc.page_bounds(K)
        scores = orc.quest_scores(q, lo, hi)
        np.testing.assert_array_equal(scores, c["scores"], err_msg=name)
        # the explicit summation-order replay the CUDA refine step implements
        replay = orc.numpy_rowsum_order(np.maximum(q.astype(np.float64) * lo, q.astype(np.float64) * hi))
        np.testing.assert_array_equal(replay / math.sqrt(128), c["scores"], err_msg=name)
        b = c["budget"][0]
        budget = float(b) if c["budget"].dtype == np.float64 else int(b)
        pages = orc.quest_select_pages(q, lo, hi, budget, n)
        np.testing.assert_array_equal(orc.pages_to_tokens(pages, n), c["selected"], err_msg=name)


def test_estimate_matches_reference(golden):
    for name, c in golden("estimate").items():
        codes, scale, zero = orc.quantize_rows(c["K"])
        z = orc.estimate_logits(c["q"], codes, scale, zero, c["idx"])
        assert z.dtype == np.float32
        np.testing.assert_allclose(z, c["scores"], rtol=2e-6, atol=2e-6, err_msg=name)
        assert c["idx"].size * (128 // 2 + orc.PARAM_BYTES) == c["bytes"][0]


def test_threshold_search_matches_reference_exactly(golden):
    for name, c in golden("topp").items():
        eps, mi = c["cfg"]
        idx, thr, it = orc.threshold_top_p(c["w"], float(c["p"][0]), float(eps), int(mi))
        np.testing.assert_array_equal(idx, c["idx"], err_msg=name)
        assert thr == c["threshold"][0] or (math.isinf(thr) and math.isinf(c["threshold"][0]))
        assert it == c["iterations"][0], name


def test_minimal_tie_closed_set_equals_converged_search(golden):
    """The direct characterisation the GPU pruner implements equals the
    reference bisection whenever the defaults let it converge."""
    for name, c in golden("topp").items():
        eps, mi = c["cfg"]
        if eps != 1e-15 or mi != 64:
            continue
        got = orc.minimal_tie_closed_top_p(c["w"], float(c["p"][0]))
        np.testing.assert_array_equal(got, c["idx"], err_msg=name)


def test_sort_oracle_agrees_on_distinct_weights(golden):
    for name, c in golden("topp").items():
        eps, mi = c["cfg"]
        w = c["w"]
        if eps != 1e-15 or mi != 64 or np.unique(w).size != w.size:
            continue
        np.testing.assert_array_equal(orc.sort_top_p(w, float(c["p"][0])), c["idx"], err_msg=name)


def test_attention_matches_reference(golden):
    for name, c in golden("attention").items():
        w = orc.full_weights(c["q"], c["K"])
        np.testing.assert_allclose(w, c["w"], rtol=1e-5, atol=1e-9)
        out = orc.subset_attention(c["w"], c["V"], c["idx"], True)
        np.testing.assert_allclose(out, c["out_renorm"], rtol=1e-5, atol=1e-6)
        out = orc.subset_attention(c["w"], c["V"], c["idx"], False)
        np.testing.assert_allclose(out, c["out_plain"], rtol=1e-5, atol=1e-6)


def test_decode_unit_matches_reference_pipeline(golden):
    for name, c in golden("pipeline").items():
        budget, p, kind, is_frac, sink, window = c["cfg"]
        budget = float(budget) if is_frac else int(budget)
        selector = ("full", "quest", "sink_window")[int(kind)]
        res = orc.decode_unit(c["Q"], c["K"], c["V"], selector=selector, budget=budget, p=float(p),
                              sink=int(sink), window=int(window))
        np.testing.assert_array_equal(res["final"], c["final"], err_msg=name)
        assert res["candidates"].size == c["b0"][0], name
        np.testing.assert_allclose(res["out"], c["out"], rtol=1e-5, atol=1e-6, err_msg=name)


def test_two_and_eight_bit_caches_match_reference(golden):
    """SUPPORTED_BITS (quantcache.py:38): codes, packing (_pack_matrix :122-130),
    params and estimate_scores for the 2- and 8-bit caches."""
    for name, c in golden("quant_bits").items():
        bits = int(name[1])
        codes, scale, zero = orc.quantize_rows(c["K"], bits)
        np.testing.assert_array_equal(codes, c["codes"], err_msg=name)
        np.testing.assert_array_equal(orc.pack_codes_bits(codes, bits), c["packed"], err_msg=name)
        np.testing.assert_array_equal(scale, c["scale"], err_msg=name)
        np.testing.assert_array_equal(zero, c["zero"], err_msg=name)
        z = orc.estimate_logits(c["q"], codes, scale, zero, c["idx"])
        np.testing.assert_allclose(z, c["scores"], rtol=1e-6, atol=1e-6, err_msg=name)


def test_channel_pruned_matches_reference(golden):
    """top_channels_by_magnitude / select_channel_pruned / run_grouped with the
    channel-pruned selector (selectors.py:135-161): bit-exact id and index sets."""
    for name, c in golden("channel").items():
        if name.startswith("m"):
            np.testing.assert_array_equal(orc.top_channels_by_magnitude(c["K"], int(c["count"][0])), c["ids"],
                                          err_msg=name)
        elif name.startswith("s"):
            budget = float(c["budget"][0]) if c["budget"][1] else int(c["budget"][0])
            np.testing.assert_array_equal(orc.channel_pruned_tokens(c["q"], c["K"], c["ids"], budget),
                                          c["indices"], err_msg=name)
        else:
            budget, p, is_frac, top = c["cfg"]
            budget = float(budget) if is_frac else int(budget)
            res = orc.decode_unit(c["Q"], c["K"], c["V"], selector="channel_pruned", budget=budget, p=float(p),
                                  top_channels=None if top < 0 else int(top))
            np.testing.assert_array_equal(res["final"], c["final"], err_msg=name)
            assert res["candidates"].size == c["b0"][0], name
            np.testing.assert_allclose(res["out"], c["out"], rtol=1e-5, atol=1e-6, err_msg=name)


def test_dequantize_unpack_and_exact_estimator_match_reference(golden):
    """dequantize_row / unpack_codes (quantcache.py:117-160) and the exact
    estimator pipelines -- bypass_config and estimator_bits="exact"
    (pipeline.py:129-136, 204-216) -- against the reference's answers."""
    cases = golden("rows")
    for name, c in cases.items():
        if name.startswith("deq"):
            scale, zero = c["params"]
            np.testing.assert_array_equal(orc.dequantize(c["codes"], scale, zero), c["f64"], err_msg=name)
            np.testing.assert_array_equal(orc.dequantize(c["codes"], scale, zero, np.float32), c["f32"], err_msg=name)
        elif name.startswith("unpack"):
            np.testing.assert_array_equal(orc.unpack_nibbles(c["packed"]), c["codes"], err_msg=name)
        else:
            budget, p, is_frac, quest = c["cfg"]
            budget = float(budget) if is_frac else int(budget)
            res = orc.decode_unit(c["Q"], c["K"], c["V"], selector="quest" if quest else "full",
                                  budget=budget, p=float(p), exact=True)
            np.testing.assert_array_equal(res["final"], c["final"], err_msg=name)
            assert res["candidates"].size == c["b0"][0]
            np.testing.assert_allclose(res["out"], c["out"], rtol=1e-5, atol=1e-6, err_msg=name)
