"""Host-side logic of the drop-in API (no GPU): configuration dataclasses and
their validation, budget resolution, the analytic cost model -- each against
the reference's documented behaviour (file:line in the docstrings)."""

import math

import numpy as np
import pytest

import paper_2502_02770_b200 as tw
from oracle import twilight_oracle as orc


def test_resolve_budget_matches_reference_rules():
    # selectors.py:72-87: float fractions use Python's half-even round, ints clamp
    for n in (1, 7, 33, 1000, 32768):
        for b in (0.25, 0.5, 1.0, 0.001, 1, 16, 8192, 10**9):
            assert tw.resolve_budget(b, n) == orc.resolve_budget(b, n)
    assert tw.resolve_budget(0.5, 5) == 2  # round(2.5) == 2 (half-even)
    for bad in (True, 0, -3, 0.0, 1.5):
        with pytest.raises(ValueError):
            tw.resolve_budget(bad, 10)


def test_budget_pages_round_up():
    from paper_2502_02770_b200.decode import budget_pages_for
    assert budget_pages_for(8192, 32768) == 512
    assert budget_pages_for(100, 777) == 7
    assert budget_pages_for(0.25, 1000) == 16


def test_config_validation():
    with pytest.raises(ValueError):
        tw.BinarySearchConfig(p=1.5)
    with pytest.raises(ValueError):
        tw.BinarySearchConfig(p=0.9, epsilon=0.0)
    with pytest.raises(ValueError):
        tw.BinarySearchConfig(p=0.9, max_iters=0)
    with pytest.raises(ValueError):
        tw.SelectorConfig(kind="bogus")
    with pytest.raises(ValueError):
        tw.SelectorConfig(page_size=0)
    with pytest.raises(ValueError):
        tw.GroupMap(0)
    with pytest.raises(ValueError):
        tw.GroupMap(4).groups(6)
    assert tw.GroupMap(4).groups(32) == 8 and tw.GroupMap(4).group_of(5) == 1
    with pytest.raises(ValueError):
        tw.PipelineConfig(estimator_bits=3)
    with pytest.raises(ValueError):
        tw.PipelineConfig(selector_cost_fraction=0.0)


def test_bypass_config_is_dense_exact():
    cfg = tw.PipelineConfig(selector=tw.SelectorConfig(kind="quest", budget=0.25), prune=tw.BinarySearchConfig(p=0.9))
    by = tw.bypass_config(cfg)
    assert by.selector.kind == "full" and by.prune.p == 1.0 and by.estimator_bits == "exact"
    assert by.selector.page_size == 16


def test_cost_model_matches_paper():
    # PAPER.md:324-327 / test_acceptance.py:139-152: B0 = N/4, B1 = N/64 -> 20/9
    n = 4096.0
    assert math.isclose(tw.model_speedup(n, n / 4, n / 64), 20.0 / 9.0)
    assert tw.memory_overhead(4) == 0.125
    with pytest.raises(ValueError):
        tw.model_speedup(10, 5, 6)
    with pytest.raises(ValueError):
        tw.memory_overhead(3)


def test_channel_pruned_validation():
    # selectors.py:135-161 argument checks (raised before any device work), and
    # host tensors are refused: the selector has no CPU fallback
    import torch
    with pytest.raises(ValueError):
        tw.top_channels_by_magnitude(torch.zeros(10, 128), 0)
    with pytest.raises(ValueError):
        tw.top_channels_by_magnitude(torch.zeros(10, 128), 4)
    with pytest.raises(ValueError):
        tw.select_channel_pruned(torch.zeros(128), torch.zeros(10, 3), [1, 2], 5)
    with pytest.raises(ValueError):
        tw.select_channel_pruned(torch.zeros(128), torch.zeros(10, 2), [1, 200], 5)
    with pytest.raises(ValueError):
        tw.select_channel_pruned(torch.zeros(128), torch.zeros(10, 2), [4, 4], 5)
    with pytest.raises(ValueError):
        tw.select_channel_pruned(torch.zeros(128), torch.zeros(10, 2), [4, 5], 5)


def test_select_sink_window_validation():
    # selectors.py:164-175 argument checks (raised before any device work)
    for bad in ((0, 1, 1), (10, -1, 3), (10, 0, 0)):
        with pytest.raises(ValueError):
            tw.select_sink_window(*bad, device="cpu")


def test_pack_codes_known_answers():
    # test_quantcache.py:75-78 -- no device work involved
    assert tw.pack_codes(np.array([0, 15])) == b"\xf0"
    assert tw.pack_codes(np.arange(16)) == bytes.fromhex("1032547698badcfe")
    with pytest.raises(ValueError):
        tw.pack_codes(np.array([7, 3, 12]))
    with pytest.raises(ValueError):
        tw.pack_codes(np.array([16, 0]))


def test_bench_roofline_kernel_choice():
    """bench.py's roofline kernel: the longest stage, and for K4 the attention
    kernel timed alone (the split-KV merge excluded) when it was measured."""
    import bench
    assert bench.dominant_kernel({"K2_select": 5, "K4_attention": 10, "K4a_attn_kernel": 9}) == "K4a_attn_kernel"
    assert bench.dominant_kernel({"K2_select": 20, "K4_attention": 10, "K4a_attn_kernel": 9}) == "K2_select"
    assert bench.dominant_kernel({"K2_select": 5, "K4_attention": 10}) == "K4_attention"
