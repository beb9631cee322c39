"""The reference-signature API (paper_2502_02770_b200 as a drop-in for
nucleuskv) against the golden vectors the REFERENCE produced
(tests/golden, oracle/gen_golden.py).  Same inputs, same assertions as the
reference's own tests where they exist (test_quantcache.py, test_selectors.py,
test_pruner.py, test_attention.py, test_pipeline.py)."""

import math

import numpy as np
import pytest
import torch

from oracle import twilight_oracle as orc
from tests.gpu_util import check_unit_topp, topp_set_ok

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2502_02770_b200 as tw  # noqa: E402
from paper_2502_02770_b200 import pipeline as _pl  # noqa: E402


def assert_final_set_and_output(Q, K, V, cfg, G, final_api, outs_api, tol, name=""):
    """Reruns the API's kernels (pipeline._run: the same deterministic launch
    sequence) to read each head's top-p set: every head's set must be the
    oracle's minimal tie-closed set on the GPU logits up to threshold ties
    (pruner.py:57-114), the final set their union (pipeline.py:347) and equal
    to what the API returned, and the outputs must match the oracle's subset
    attention over that final set (attention.py:106-136)."""
    dec, _ = _pl._run(Q, K, V, cfg, G)
    torch.cuda.synchronize()
    _, _, _, final, _ = check_unit_topp(dec.bufs, 0, G, cfg.prune.p)
    np.testing.assert_array_equal(final, np.asarray(final_api), err_msg=name)
    Kn, Vn, Qn = K.float().cpu().numpy(), V.float().cpu().numpy(), Q.float().cpu().numpy()
    outs = np.asarray(outs_api).reshape(G, -1)
    for g in range(G):
        w = orc.full_weights(Qn[g], Kn)
        want = orc.subset_attention(w, Vn, final, final.size > 0 and w[final].sum() > 0)
        np.testing.assert_allclose(outs[g], want, rtol=tol, atol=tol * np.abs(want).max(), err_msg=name)


def cuda(x, dtype=torch.float32):
    return torch.as_tensor(np.asarray(x), dtype=dtype).cuda()


def as_input(K):
    """bf16-representable golden inputs go in as bf16, the rest as fp32."""
    K = np.asarray(K, dtype=np.float32)
    bf = torch.as_tensor(K).to(torch.bfloat16).float().numpy()
    return cuda(K, torch.bfloat16) if np.array_equal(bf, K) else cuda(K)


def test_build_cache_and_metadata_match_reference(golden):
    for name, c in golden("quant").items():
        if name == "pack":
            continue
        K = as_input(c["K"])
        cache, meta = tw.build_cache(K)
        packed, scale, zero = cache.kv.unit_quant(0, 0)
        np.testing.assert_array_equal(packed.cpu().numpy(), c["packed"], err_msg=name)
        np.testing.assert_array_equal(scale.cpu().numpy(), c["scale"].astype(np.float32), err_msg=name)
        np.testing.assert_array_equal(zero.cpu().numpy(), c["zero"].astype(np.float32), err_msg=name)
        np.testing.assert_array_equal(meta.lo.float().cpu().numpy(), c["lo"].astype(np.float32), err_msg=name)
        np.testing.assert_array_equal(meta.hi.float().cpu().numpy(), c["hi"].astype(np.float32), err_msg=name)
        assert len(meta) == c["lo"].shape[0] and cache.page_table == list(range(len(meta)))
        pages = cache.pages
        assert pages[-1].valid_len == K.shape[0] - 16 * (len(pages) - 1)
        for r in range(3):
            if f"row{r}_codes" in c:
                codes, prm = tw.quantize_row(K[r])
                np.testing.assert_array_equal(codes.cpu().numpy(), c[f"row{r}_codes"])
                assert prm.scale == c[f"row{r}_params"][0] and prm.zero == c[f"row{r}_params"][1]


def test_quantize_row_known_answers():
    # test_quantcache.py:25-38
    codes, prm = tw.quantize_row(cuda(np.arange(16, dtype=np.float32)))
    assert prm.scale == 1.0 and prm.zero == 0.0
    np.testing.assert_array_equal(codes.cpu().numpy(), np.arange(16))
    codes, prm = tw.quantize_row(cuda(np.full(32, -2.75, dtype=np.float32)))
    assert prm.scale == 0.0 and prm.zero == -2.75 and int(codes.sum()) == 0
    for bits in (2, 8):
        k = cuda(np.random.default_rng(8).standard_normal(128).astype(np.float32))
        codes, prm = tw.quantize_row(k, bits=bits)
        ref_codes, ref_scale, ref_zero = orc.quantize_rows(k.cpu().numpy(), bits)
        np.testing.assert_array_equal(codes.cpu().numpy(), ref_codes[0])
    with pytest.raises(ValueError):
        tw.quantize_row(cuda(np.ones(4)), bits=3)


def test_quest_scores_and_selection_bit_exact(golden):
    for name, c in golden("quest").items():
        K, q = as_input(c["K"]), as_input(c["q"])
        n = K.shape[0]
        meta = tw.build_page_metadata(K)
        scores = tw.quest_page_scores(q, meta)
        np.testing.assert_array_equal(scores.cpu().numpy(), c["scores"], err_msg=name)
        b = c["budget"][0]
        budget = float(b) if c["budget"].dtype == np.float64 else int(b)
        sel = tw.select_quest(q, meta, budget, 16, n)
        np.testing.assert_array_equal(sel.indices.cpu().numpy(), c["selected"], err_msg=name)


def test_estimate_scores_match_reference(golden):
    for name, c in golden("estimate").items():
        K, q = as_input(c["K"]), as_input(c["q"])
        cache, _ = tw.build_cache(K)
        sel = tw.TokenSelection.from_indices(cuda(c["idx"], torch.int64), K.shape[0])
        r = tw.estimate_scores(q, cache, sel)
        np.testing.assert_allclose(r.scores.cpu().numpy(), c["scores"], rtol=1e-5, atol=1e-5, err_msg=name)
        assert r.bytes_touched == c["bytes"][0]
    with pytest.raises(IndexError):
        tw.TokenSelection.from_indices([17], 17)


def test_binary_search_top_p_matches_reference(golden):
    exact = 0
    for name, c in golden("topp").items():
        eps, mi = c["cfg"]
        out = tw.binary_search_top_p(cuda(c["w"], torch.float64),
                                     tw.BinarySearchConfig(p=float(c["p"][0]), epsilon=float(eps), max_iters=int(mi)))
        got = out.selection.indices.cpu().numpy()
        np.testing.assert_array_equal(got, c["idx"], err_msg=name)
        assert out.iterations == c["iterations"][0], name
        ref_thr = c["threshold"][0]
        assert out.threshold == ref_thr or (math.isinf(out.threshold) and math.isinf(ref_thr)), name
        exact += 1
    assert exact > 100
    # test_pruner.py:150-156 tie classes are kept whole
    w = cuda([0.3, 0.3, 0.2, 0.2], torch.float64)
    assert tw.binary_search_top_p(w, tw.BinarySearchConfig(p=0.7)).selection.indices.tolist() == [0, 1, 2, 3]
    assert tw.binary_search_top_p(w, tw.BinarySearchConfig(p=0.5)).selection.indices.tolist() == [0, 1]
    with pytest.raises(ValueError):
        tw.binary_search_top_p(cuda([0.9, 0.9], torch.float64), tw.BinarySearchConfig(p=0.5))


def test_prune_maps_back_to_global_indices():
    rng = np.random.default_rng(5)
    z = rng.standard_normal(128)
    w = np.exp(z - z.max())
    w /= w.sum()
    cands = tw.TokenSelection.from_indices(torch.arange(128).cuda(), 128)
    out = tw.prune(cuda(w, torch.float64), cands, tw.BinarySearchConfig(p=0.9))
    direct = tw.binary_search_top_p(cuda(w, torch.float64), tw.BinarySearchConfig(p=0.9))
    assert torch.equal(out.selection.indices, direct.selection.indices)


def test_attention_readout_matches_reference(golden):
    for name, c in golden("attention").items():
        K, V, q = as_input(c["K"]).float(), as_input(c["V"]).float(), as_input(c["q"]).float()
        w = tw.attention_weights(q, K)
        np.testing.assert_allclose(w.cpu().numpy(), c["w"], rtol=1e-5, atol=1e-9)
        sel = tw.TokenSelection.from_indices(cuda(c["idx"], torch.int64), K.shape[0])
        out = tw.sparse_attention(cuda(c["w"]), V, sel, renormalize=True)
        np.testing.assert_allclose(out.cpu().numpy(), c["out_renorm"], rtol=1e-5, atol=1e-6)
        out = tw.sparse_attention(cuda(c["w"]), V, sel, renormalize=False)
        np.testing.assert_allclose(out.cpu().numpy(), c["out_plain"], rtol=1e-5, atol=1e-6)
    empty = tw.TokenSelection.from_indices(torch.zeros(0, dtype=torch.int64).cuda(), 4)
    with pytest.raises(tw.DegenerateSelectionError):
        tw.sparse_attention(cuda(np.full(4, 0.25)), cuda(np.ones((4, 128))), empty, renormalize=True)


def test_select_sink_window_indices():
    # selectors.py:164-175
    assert tw.select_sink_window(100, 4, 10).indices.tolist() == list(range(4)) + list(range(90, 100))
    assert tw.select_sink_window(20, 15, 5).indices.tolist() == list(range(20))  # they meet: every token
    assert tw.select_sink_window(50, 0, 3).indices.tolist() == [47, 48, 49]


def test_run_grouped_and_run_head_match_reference(golden):
    """The whole hot path (K2 -> K3 -> K4 on one context) against run_grouped /
    run_head outputs of the reference: identical final sets up to top-p
    threshold ties, and attention outputs within tolerance."""
    for name, c in golden("pipeline").items():
        budget, p, kind, is_frac, sink, window = c["cfg"]
        budget = float(budget) if is_frac else int(budget)
        selector = ("full", "quest", "sink_window")[int(kind)]
        is_quest = selector == "quest"
        K, V, Q = as_input(c["K"]), as_input(c["V"]), as_input(c["Q"])
        G = Q.shape[0]
        sel = tw.SelectorConfig(kind=selector, budget=budget if is_quest else None, sink=int(sink), window=int(window))
        cfg = tw.PipelineConfig(selector=sel, prune=tw.BinarySearchConfig(p=float(p)), group_map=tw.GroupMap(G))
        if G == 1:
            out, outcome, report = tw.run_head(Q[0], K, V, cfg)
            outs, final, b0 = out[None], outcome.selection.indices, report.b0
        else:
            outs, outcomes, reports = tw.run_grouped(Q, K, V, cfg)
            final, b0 = outcomes[0].selection.indices, reports[0].b0
        assert b0 == c["b0"][0], name
        final = final.cpu().numpy()
        want = c["final"]
        tol = 2e-2 if K.dtype == torch.bfloat16 else 1e-4
        # always: per-head sets = the oracle's up to threshold ties, outputs over the GPU's final set
        assert_final_set_and_output(Q, K, V, cfg, G, final, outs.cpu().numpy(), tol, name)
        if np.array_equal(final, want):
            np.testing.assert_allclose(outs.cpu().numpy(), c["out"], rtol=tol, atol=tol * np.abs(c["out"]).max(),
                                       err_msg=name)


@pytest.mark.parametrize("kind", ["quest", "channel_pruned"])
def test_file_workload_runs_on_the_gpu_path(tmp_path, kind):
    """workload.py:148-183 file workload (q/k/v .twlt) decoded by run_file_workload
    vs the oracle's run_grouped restatement per step and KV head."""
    rng = np.random.default_rng(31)
    steps, heads, kvh, n = 2, 4, 2, 700
    bf = lambda x: torch.from_numpy(x.astype(np.float32)).bfloat16().float().numpy()  # noqa: E731
    q = bf(rng.standard_normal((steps, heads, 128)) * 2.0)
    k = bf(rng.standard_normal((kvh, n, 128)))
    v = bf(rng.standard_normal((kvh, n, 128)))
    for name, a in (("q", q), ("k", k), ("v", v)):
        tw.write_tensor(tmp_path / f"{name}.twlt", a)
    cfg = tw.PipelineConfig(selector=tw.SelectorConfig(kind=kind, budget=256),
                            prune=tw.BinarySearchConfig(p=0.9), group_map=tw.GroupMap(heads // kvh))
    outs, _ = tw.run_file_workload(tmp_path, cfg)
    G = heads // kvh
    for s in range(steps):
        for h in range(kvh):
            res = orc.decode_unit(q[s, h * G:(h + 1) * G], k[h], v[h], selector=kind, budget=256, p=0.9)
            want = res["out"]
            got = outs[s, h * G:(h + 1) * G].cpu().numpy()
            np.testing.assert_allclose(got, want, rtol=2e-2, atol=2e-2 * np.abs(want).max())


def test_dynamism_from_a_batched_step_and_sweep_p():
    from paper_2502_02770_b200.workload import make_batch, tau_schedule
    B, H, G, n = 2, 2, 4, 600
    batch = make_batch(B, H, G, n, torch.bfloat16, tau=tau_schedule(H, (0.3, 2.0)), seed=41)
    cache = tw.PagedKVCache(B, H, G, max_pages=tw.pages_for(n), dtype=torch.bfloat16)
    cache.prefill(batch.K, batch.V)
    dec = tw.TwilightDecoder(cache, "quest", budget=256, p=0.9)
    dec.forward(batch.q.contiguous())
    tags = tw.tag_decode_stats(dec.stats(), H * G)
    st = tw.collect_dynamism(tags)
    b1 = dec.stats().b1.cpu().numpy()
    assert st.overall_mean == pytest.approx(float(b1.mean()))
    assert sorted(st.axes["prompt"].group_means) == [0, 1]
    # p sweep (pipeline.py:465-498): larger p never keeps fewer tokens
    K = batch.K[0, 0].contiguous()
    V = batch.V[0, 0].contiguous()
    items = [(batch.q[0, g], K, V) for g in range(2)]
    cfg = tw.PipelineConfig(selector=tw.SelectorConfig(kind="quest", budget=256))
    rows = tw.sweep_p(items, cfg, [0.5, 0.9, 0.99])
    assert [r.p for r in rows] == [0.5, 0.9, 0.99]
    assert rows[0].mean_b1 <= rows[1].mean_b1 <= rows[2].mean_b1


@pytest.mark.parametrize("bits", [2, 8])
def test_two_and_eight_bit_caches(golden, bits):
    """build_cache(bits) codes / packing / params bit-exact and estimate_scores
    within fp32 tolerance vs the reference (tests/golden/quant_bits.npz)."""
    for name, c in golden("quant_bits").items():
        if int(name[1]) != bits:
            continue
        K = as_input(c["K"])
        cache, _ = tw.build_cache(K, bits=bits)
        packed, scale, zero = cache.kv.unit_quant(0, 0)
        np.testing.assert_array_equal(packed.cpu().numpy(), c["packed"], err_msg=name)
        np.testing.assert_array_equal(scale.cpu().numpy(), c["scale"].astype(np.float32), err_msg=name)
        np.testing.assert_array_equal(zero.cpu().numpy(), c["zero"].astype(np.float32), err_msg=name)
        q = cuda(c["q"], K.dtype)
        r = tw.estimate_scores(q, cache, tw.TokenSelection.from_indices(cuda(c["idx"]).long(), K.shape[0]))
        assert r.bytes_touched == int(c["bytes"][0])
        scale_ref = np.abs(c["q"]).sum() * np.abs(c["K"]).max() / np.sqrt(128)
        np.testing.assert_allclose(r.scores.cpu().numpy(), c["scores"], rtol=0, atol=2e-6 * scale_ref + 1e-6,
                                   err_msg=name)


@pytest.mark.parametrize("bits", [2, 8])
def test_run_grouped_with_two_and_eight_bit_estimators(bits):
    """PipelineConfig.estimator_bits = 2 / 8 through the batched kernels vs the
    oracle restatement of run_grouped with the same cache width."""
    rng = np.random.default_rng(50 + bits)
    n, G = 900, 4
    bf = lambda x: torch.from_numpy(x.astype(np.float32)).bfloat16().float().numpy()  # noqa: E731
    K, V, Q = bf(rng.standard_normal((n, 128))), bf(rng.standard_normal((n, 128))), bf(rng.standard_normal((G, 128)) * 2)
    cfg = tw.PipelineConfig(selector=tw.SelectorConfig(kind="quest", budget=300), prune=tw.BinarySearchConfig(p=0.9),
                            group_map=tw.GroupMap(G), estimator_bits=bits)
    out, outcomes, reports = tw.run_grouped(cuda(Q, torch.bfloat16), cuda(K, torch.bfloat16), cuda(V, torch.bfloat16), cfg)
    res = orc.decode_unit(Q, K, V, selector="quest", budget=300, p=0.9, bits=bits)
    final = outcomes[0].selection.indices.cpu().numpy()
    assert reports[0].b0 == res["candidates"].size
    assert_final_set_and_output(cuda(Q, torch.bfloat16), cuda(K, torch.bfloat16), cuda(V, torch.bfloat16), cfg, G,
                                final, out.cpu().numpy(), 2e-2)
    if np.array_equal(final, res["final"]):
        np.testing.assert_allclose(out.cpu().numpy(), res["out"], rtol=2e-2, atol=2e-2 * np.abs(res["out"]).max())


def test_channel_pruned_api_matches_reference(golden):
    """top_channels_by_magnitude / select_channel_pruned / run_grouped with the
    channel-pruned selector against the reference's own outputs."""
    for name, c in golden("channel").items():
        if name.startswith("m"):
            got = tw.top_channels_by_magnitude(as_input(c["K"]), int(c["count"][0]))
            np.testing.assert_array_equal(got.cpu().numpy(), c["ids"], err_msg=name)
        elif name.startswith("s"):
            budget = float(c["budget"][0]) if c["budget"][1] else int(c["budget"][0])
            K, ids = as_input(c["K"]), torch.as_tensor(c["ids"]).cuda()
            sel = tw.select_channel_pruned(as_input(c["q"]), K[:, ids], ids, budget)
            np.testing.assert_array_equal(sel.indices.cpu().numpy(), c["indices"], err_msg=name)
        else:
            budget, p, is_frac, top = c["cfg"]
            budget = float(budget) if is_frac else int(budget)
            K, V, Q = as_input(c["K"]), as_input(c["V"]), as_input(c["Q"])
            G = Q.shape[0]
            sel = tw.SelectorConfig(kind="channel_pruned", budget=budget, top_channels=None if top < 0 else int(top))
            cfg = tw.PipelineConfig(selector=sel, prune=tw.BinarySearchConfig(p=float(p)), group_map=tw.GroupMap(G))
            if G == 1:
                out, outcome, report = tw.run_head(Q[0], K, V, cfg)
                outs, final, b0 = out[None], outcome.selection.indices, report.b0
            else:
                outs, outcomes, reports = tw.run_grouped(Q, K, V, cfg)
                final, b0 = outcomes[0].selection.indices, reports[0].b0
            assert b0 == c["b0"][0], name
            final = final.cpu().numpy()
            tol = 2e-2 if K.dtype == torch.bfloat16 else 1e-4
            assert_final_set_and_output(Q, K, V, cfg, G, final, outs.cpu().numpy(), tol, name)
            if np.array_equal(final, c["final"]):
                np.testing.assert_allclose(outs.cpu().numpy(), c["out"], rtol=tol,
                                           atol=tol * np.abs(c["out"]).max(), err_msg=name)


def test_channel_pruned_build_selector():
    """build_selector binds the channel slice once per context (selectors.py:203-209)."""
    rng = np.random.default_rng(3)
    K = rng.standard_normal((400, 128)).astype(np.float32)
    q = rng.standard_normal(128).astype(np.float32)
    sel = tw.build_selector(tw.SelectorConfig(kind="channel_pruned", budget=50, top_channels=12), cuda(K))
    got = sel(cuda(q)).indices.cpu().numpy()
    ids = orc.top_channels_by_magnitude(K, 12)
    np.testing.assert_array_equal(got, orc.channel_pruned_tokens(q, K, ids, 50))


def test_dequantize_row_and_unpack_codes_match_reference(golden):
    """dequantize_row / unpack_codes (quantcache.py:117-119, 154-160) against
    the reference's own answers (tests/golden/rows.npz)."""
    for name, c in golden("rows").items():
        if name.startswith("deq"):
            prm = tw.QuantParams(scale=float(c["params"][0]), zero=float(c["params"][1]))
            codes = cuda(c["codes"], torch.uint8)
            np.testing.assert_array_equal(tw.dequantize_row(codes, prm).cpu().numpy(), c["f64"], err_msg=name)
            np.testing.assert_array_equal(tw.dequantize_row(codes, prm, torch.float32).cpu().numpy(), c["f32"],
                                          err_msg=name)
        elif name.startswith("unpack"):
            got = tw.unpack_codes(c["packed"].tobytes(), 2 * c["packed"].size)
            np.testing.assert_array_equal(got.cpu().numpy(), c["codes"], err_msg=name)
            assert tw.pack_codes(got) == c["packed"].tobytes()
    with pytest.raises(ValueError):
        tw.unpack_codes(b"\x00\x01", 6)


def test_exact_estimator_and_bypass_config_match_reference(golden):
    """estimator_bits="exact" (_candidate_logits, pipeline.py:212-214) through
    the exact-estimate kernel, and run_grouped(..., bypass_config(cfg)) -- the
    bypass layers' dense configuration (pipeline.py:129-136, cli.py:83-87) --
    against the reference's outputs and final sets, and the dense oracle."""
    for name, c in golden("rows").items():
        if not name.startswith("x"):
            continue
        budget, p, is_frac, quest = c["cfg"]
        budget = float(budget) if is_frac else int(budget)
        bf = np.array_equal(torch.as_tensor(c["K"]).bfloat16().float().numpy(), c["K"])
        dt = torch.bfloat16 if bf else torch.float32
        K, V, Q = cuda(c["K"], dt), cuda(c["V"], dt), cuda(c["Q"], dt)
        G = Q.shape[0]
        base = tw.PipelineConfig(selector=tw.SelectorConfig(kind="quest" if quest else "full",
                                                            budget=budget if quest else None),
                                 prune=tw.BinarySearchConfig(p=float(p)), group_map=tw.GroupMap(G))
        cfg = replace_cfg_exact(base) if quest else tw.bypass_config(base)
        if G == 1:
            out, outcome, report = tw.run_head(Q[0], K, V, cfg)
            outs, final, b0 = out[None], outcome.selection.indices, report.b0
        else:
            outs, outcomes, reports = tw.run_grouped(Q, K, V, cfg)
            final, b0 = outcomes[0].selection.indices, reports[0].b0
        assert b0 == c["b0"][0], name
        tol = 2e-2 if bf else 1e-4
        final = final.cpu().numpy()
        assert_final_set_and_output(Q, K, V, cfg, G, final, outs.cpu().numpy(), tol, name)
        # the exact logits themselves (fp32 dot products; BLAS order differs)
        dec, _ = _pl._run(Q, K, V, cfg, G)
        torch.cuda.synchronize()
        from tests.gpu_util import unit_candidates
        cand, z = unit_candidates(dec.bufs, 0)
        for g in range(G):
            want = orc.exact_logits(c["Q"][g], c["K"], cand)
            np.testing.assert_allclose(z[g], want, rtol=1e-5, atol=1e-5 * np.abs(want).max(), err_msg=name)
        np.testing.assert_array_equal(final, c["final"], err_msg=name)
        np.testing.assert_allclose(outs.cpu().numpy(), c["out"], rtol=tol, atol=tol * np.abs(c["out"]).max(),
                                   err_msg=name)
        if not quest:  # bypass: the dense oracle (softmax over every token)
            for g in range(G):
                w = orc.full_weights(c["Q"][g], c["K"])
                np.testing.assert_allclose(outs[g].cpu().numpy(), w @ c["V"], rtol=1e-4,
                                           atol=1e-4 * np.abs(w @ c["V"]).max(), err_msg=name)


def replace_cfg_exact(cfg):
    from dataclasses import replace
    return replace(cfg, estimator_bits="exact")


def test_prebuilt_cache_is_reused(monkeypatch):
    """run_grouped / run_head with cache= / metadata= from build_cache reuse
    that pool (_prepare_context, pipeline.py:177-201): no tw_quant_build, the
    same INT4 pages, the same results as building it inside the call; a cache
    of another width is rejected like the reference (:194-198)."""
    from paper_2502_02770_b200 import _lib
    rng = np.random.default_rng(7)
    n, G = 1000, 4
    K = torch.from_numpy(rng.standard_normal((n, 128)).astype(np.float32)).bfloat16().cuda()
    V = torch.from_numpy(rng.standard_normal((n, 128)).astype(np.float32)).bfloat16().cuda()
    Q = torch.from_numpy(rng.standard_normal((8, 128)).astype(np.float32) * 2).bfloat16().cuda()
    cfg = tw.PipelineConfig(selector=tw.SelectorConfig(kind="quest", budget=256), prune=tw.BinarySearchConfig(p=0.9),
                            group_map=tw.GroupMap(G))
    want, want_oc, _ = tw.run_grouped(Q, K, V, cfg)
    cache, meta = tw.build_cache(K)
    lib = _lib.lib()
    real = lib.tw_quant_build
    calls = []
    monkeypatch.setattr(lib, "tw_quant_build", lambda *a: calls.append(1) or real(*a))
    got, got_oc, _ = tw.run_grouped(Q, K, V, cfg, cache=cache, metadata=meta)
    head, head_oc, _ = tw.run_head(Q[0], K, V, tw.PipelineConfig(selector=cfg.selector, prune=cfg.prune),
                                   cache=cache)
    torch.cuda.synchronize()
    assert calls == []
    assert torch.equal(got, want)
    assert torch.equal(got_oc[0].selection.indices, want_oc[0].selection.indices)
    dec, _ = _pl._run(Q, K, V, cfg, G, cache, meta)
    assert dec.cache.kq.data_ptr() == cache.kv.kq.data_ptr()
    with pytest.raises(ValueError):
        tw.run_grouped(Q, K, V, replace_bits(cfg, 2), cache=cache)


def replace_bits(cfg, bits):
    from dataclasses import replace
    return replace(cfg, estimator_bits=bits)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("n,d", [(1, 128), (1000, 128), (131072, 128), (777, 64)])
def test_vector_operators_match_fp32_reference(dtype, n, d):
    """attention_weights / stable_softmax / sparse_attention on the tw_vec_*
    kernels vs a plain fp32 (fp64 for the readout) torch reference of the same
    op (attention.py:79-136)."""
    g = torch.Generator(device="cuda").manual_seed(n + d)
    K = torch.randn(n, d, device="cuda", generator=g).to(dtype)
    V = torch.randn(n, d, device="cuda", generator=g).to(dtype)
    q = (torch.randn(d, device="cuda", generator=g) * 2).to(dtype)
    w = tw.attention_weights(q, K)
    assert w.dtype == dtype
    z = (K.float() @ q.float()) / np.float32(np.sqrt(d))
    ref = torch.softmax(z.double(), 0)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    torch.testing.assert_close(w.double(), ref, rtol=tol, atol=tol * float(ref.max()))
    s = tw.stable_softmax(z)
    torch.testing.assert_close(s.double(), ref, rtol=1e-5, atol=1e-7 * float(ref.max()) + 1e-12)
    idx = torch.unique(torch.randint(0, n, (max(1, n // 3),), device="cuda", generator=g))
    sel = tw.TokenSelection.from_indices(idx, n)
    for wts in (w.float(), ref):  # fp32 and fp64 weights
        for renorm in (False, True):
            got = tw.sparse_attention(wts, V, sel, renormalize=renorm)
            want = wts.double()[idx] @ V.double()[idx]
            if renorm:
                want = want / wts.double()[idx].sum()
            assert got.dtype == torch.promote_types(wts.dtype, V.dtype)
            torch.testing.assert_close(got.double(), want, rtol=1e-5, atol=1e-6 * float(want.abs().max()) + 1e-12)
