"""GPU parity of the batched decode kernels against the CPU oracle.

K1 codes / packed bytes / params / metadata: bit-exact.  K2 page sets and
union: bit-exact (and the fp64 page scores bit-identical to NumPy).  K3
logits: fp32 tolerance; top-p sets: identical up to threshold ties (1e-6).
K4/K5 outputs: 1e-4 relative (fp32) and bf16 inputs with fp32 accumulation.
"""

import math

import numpy as np
import pytest
import torch

from oracle import twilight_oracle as orc
from tests.gpu_util import check_unit_topp, f2key_np, to_np, topp_set_ok

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2502_02770_b200 import _lib  # noqa: E402
from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder, pages_for  # noqa: E402
from paper_2502_02770_b200.workload import make_batch, tau_schedule  # noqa: E402

DTYPES = [torch.float32, torch.bfloat16]


def _cache(B, H, G, n, dtype, lengths, seed=0, tau=1.0, page_local=False, extra_pages=2):
    batch = make_batch(B, H, G, n, dtype, tau=tau, seed=seed, page_local=page_local)
    cache = PagedKVCache(B, H, G, max_pages=pages_for(n) + extra_pages, dtype=dtype)
    cache.prefill(batch.K, batch.V, lengths)
    return cache, batch


@pytest.mark.parametrize("dtype", DTYPES)
def test_k1_bulk_quantization_bit_exact(dtype):
    B, H, G = 2, 3, 1
    cache, _ = _cache(B, H, G, 300, dtype, [300, 177], seed=1)
    for b in range(B):
        for h in range(H):
            K = to_np(cache.unit_keys(b, h))
            codes, scale, zero = orc.quantize_rows(K)
            packed, sc, zr = cache.unit_quant(b, h)
            np.testing.assert_array_equal(packed.cpu().numpy(), orc.pack_nibbles(codes))
            np.testing.assert_array_equal(sc.cpu().numpy(), scale.astype(np.float32))
            np.testing.assert_array_equal(zr.cpu().numpy(), zero.astype(np.float32))
            lo, hi = cache.unit_meta(b, h)
            olo, ohi = orc.page_bounds(K)
            np.testing.assert_array_equal(to_np(lo), olo.astype(np.float32))
            np.testing.assert_array_equal(to_np(hi), ohi.astype(np.float32))
            assert float(cache.kabsmax[b, h]) == float(np.abs(K).max())


@pytest.mark.parametrize("dtype", DTYPES)
def test_k1_append_equals_bulk(dtype):
    B, H, G, n = 2, 2, 4, 300
    lengths = [300, 177]
    full, batch = _cache(B, H, G, n, dtype, lengths, seed=2)
    inc = PagedKVCache(B, H, G, max_pages=full.max_pages, dtype=dtype)
    tail = 21
    inc.prefill(batch.K, batch.V, [l - tail for l in lengths])
    for i in range(tail):
        pos = torch.tensor([l - tail + i for l in lengths], dtype=torch.int32, device="cuda")
        idx = pos.long().view(B, 1, 1, 1).expand(B, H, 1, 128)
        k_new = torch.gather(batch.K, 2, idx).squeeze(2).contiguous()
        v_new = torch.gather(batch.V, 2, idx).squeeze(2).contiguous()
        inc.append(k_new, v_new)
    torch.cuda.synchronize()
    assert inc.seq_lens.tolist() == lengths
    for b in range(B):
        for h in range(H):
            for a, c in zip(inc.unit_quant(b, h), full.unit_quant(b, h)):
                assert torch.equal(a, c)
            for a, c in zip(inc.unit_meta(b, h), full.unit_meta(b, h)):
                assert torch.equal(a, c)
            assert torch.equal(inc.unit_keys(b, h), full.unit_keys(b, h))
            assert torch.equal(inc.unit_values(b, h), full.unit_values(b, h))
    assert torch.equal(inc.kabsmax, full.kabsmax)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("page_local", [False, True])
@pytest.mark.parametrize("B", [2, 20])
def test_k2_quest_pages_bit_exact(dtype, page_local, B):
    """Page sets per head and their union, bit-exact vs the oracle, for a
    small batch and one with more (unit, head) pairs than SMs."""
    H, G, n = 2, 4, 1000
    lengths = [1000, 777] * (B // 2)
    cache, batch = _cache(B, H, G, n, dtype, lengths, seed=3, tau=0.5, page_local=page_local)
    budget = 256
    dec = TwilightDecoder(cache, "quest", budget=budget, p=0.95, head_page_bits=True)
    q = batch.q.contiguous()
    dec.select(q)
    dec.select(q)  # a second step over the same buffers
    # exact fp64 page bounds, bit-identical to NumPy
    import ctypes
    scores = torch.empty(B * H * G, cache.max_pages, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().tw_quest_scores(ctypes.byref(cache.struct()), _lib.ptr(q), _lib.ptr(scores),
                                          _lib.stream_handle()), "tw_quest_scores")
    torch.cuda.synchronize()
    bits = dec.bufs.head_page_bits.cpu().numpy().view(np.uint32)
    for b in range(B):
        for h in range(H):
            K = to_np(cache.unit_keys(b, h))
            lo, hi = orc.page_bounds(K)
            u = b * H + h
            heads = []
            for g in range(G):
                qh = to_np(q[b, h * G + g])
                want = orc.quest_select_pages(qh, lo, hi, budget, lengths[b])
                np.testing.assert_array_equal(scores[u * G + g, : lo.shape[0]].cpu().numpy(),
                                              orc.quest_scores(qh, lo, hi))
                got = np.flatnonzero(np.unpackbits(bits[u * G + g].view(np.uint8), bitorder="little"))
                np.testing.assert_array_equal(got, want)
                heads.append(want)
            cnt = int(dec.bufs.cand_count[u])
            np.testing.assert_array_equal(dec.bufs.cand_pages[u, :cnt].cpu().numpy(), orc.union_sorted(heads))


def test_k2_ties_go_to_the_lower_page():
    B, H, G = 1, 1, 1
    base = make_batch(1, 1, 1, 16, torch.bfloat16, seed=4)
    K = base.K.repeat(1, 1, 8, 1)  # eight identical pages
    cache = PagedKVCache(B, H, G, max_pages=8, dtype=torch.bfloat16)
    cache.prefill(K, K, [128])
    dec = TwilightDecoder(cache, "quest", budget=48, p=0.9)
    dec.select(base.q[:, :1].contiguous())
    assert dec.bufs.cand_pages[0, : int(dec.bufs.cand_count[0])].tolist() == [0, 1, 2]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("G", [1, 4])
def test_k3_estimate_topp_and_k4_attention(dtype, G):
    B, H, n = 2, 2, 1500
    lengths = [1500, 1111]
    tau = tau_schedule(H, (0.3, 1.0))
    cache, batch = _cache(B, H, G, n, dtype, lengths, seed=5 + G, tau=tau)
    p = 0.95
    dec = TwilightDecoder(cache, "quest", budget=512, p=p)
    q = batch.q.contiguous()
    out = dec.forward(q)
    torch.cuda.synchronize()
    bufs = dec.bufs
    T = cache.max_pages * 16
    exact, tolerant = 0, 0
    for b in range(B):
        for h in range(H):
            u = b * H + h
            K = to_np(cache.unit_keys(b, h))
            V = to_np(cache.unit_values(b, h))
            codes, scale, zero = orc.quantize_rows(K)
            ncand = int(bufs.cand_count[u])
            pages = bufs.cand_pages[u, :ncand].cpu().numpy()
            cand = orc.pages_to_tokens(pages, lengths[b])
            pos = (pages[:, None] * 16 + np.arange(16)).reshape(-1)
            valid = pos < lengths[b]
            head_sets = []
            for g in range(G):
                qh = to_np(q[b, h * G + g])
                z_gpu = bufs.logits[u, g, : ncand * 16].cpu().numpy()
                assert np.all(np.isneginf(z_gpu[~valid]))
                z_gpu = z_gpu[valid]
                z_ref = orc.estimate_logits(qh, codes, scale, zero, cand)
                scale_ref = np.abs(qh).sum() * np.abs(K).max() / np.sqrt(128)
                np.testing.assert_allclose(z_gpu, z_ref, rtol=0, atol=2e-6 * scale_ref + 1e-6)
                # isolated pruner: the oracle softmax + search on the GPU's own logits
                thr = np.uint32(bufs.head_thr[u * G + g].item() & 0xFFFFFFFF)
                sel = np.flatnonzero(f2key_np(z_gpu) >= thr)
                w = orc.softmax64(z_gpu)
                ok, why = topp_set_ok(sel, w, p)
                assert ok, f"unit {u} head {g}: {why}"
                exact += why == "equal"
                tolerant += why != "equal"
                head_sets.append(cand[sel])
                assert int(bufs.head_stats[u * G + g, 0]) == sel.size
            final = orc.union_sorted(head_sets)
            cnt = int(bufs.final_count[u])
            np.testing.assert_array_equal(bufs.final_idx[u, :cnt].cpu().numpy(), final)
            # attention over the identical final set (reference: pipeline.py:366-375)
            for g in range(G):
                qh = to_np(q[b, h * G + g])
                w = orc.full_weights(qh, K)
                want = orc.subset_attention(w, V, final, w[final].sum() > 0)
                got = to_np(out[b, h * G + g])
                np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4 * np.abs(want).max())
    assert exact >= tolerant  # near-threshold ties are the exception


@pytest.mark.parametrize("dtype", DTYPES)
def test_k3_full_selector(dtype):
    B, H, G, n = 1, 2, 1, 3000
    cache, batch = _cache(B, H, G, n, dtype, [n], seed=9, tau=0.25)
    dec = TwilightDecoder(cache, "full", p=0.9)
    q = batch.q.contiguous()
    out = dec.forward(q)
    torch.cuda.synchronize()
    for h in range(H):
        assert int(dec.bufs.cand_count[h]) == pages_for(n)
        K, V = to_np(cache.unit_keys(0, h)), to_np(cache.unit_values(0, h))
        cnt = int(dec.bufs.final_count[h])
        final = dec.bufs.final_idx[h, :cnt].cpu().numpy()
        z = dec.bufs.logits[h, 0, :n].cpu().numpy()
        ok, why = topp_set_ok(final, orc.softmax64(z), 0.9)
        assert ok, why
        w = orc.full_weights(to_np(q[0, h]), K)
        want = orc.subset_attention(w, V, final, True)
        np.testing.assert_allclose(to_np(out[0, h]), want, rtol=1e-4, atol=1e-4 * np.abs(want).max())


@pytest.mark.parametrize("dtype", DTYPES)
def test_k5_dense_attention(dtype):
    B, H, G, n = 2, 2, 4, 2100
    lengths = [2100, 1337]
    cache, batch = _cache(B, H, G, n, dtype, lengths, seed=11, tau=0.7)
    dec = TwilightDecoder(cache, "full", p=1.0)
    q = batch.q.contiguous()
    out = dec.dense(q)
    torch.cuda.synchronize()
    for b in range(B):
        for h in range(H):
            K, V = to_np(cache.unit_keys(b, h)), to_np(cache.unit_values(b, h))
            for g in range(G):
                w = orc.full_weights(to_np(q[b, h * G + g]), K)
                want = w @ V
                np.testing.assert_allclose(to_np(out[b, h * G + g]), want, rtol=1e-4,
                                           atol=1e-4 * np.abs(want).max())


def test_decode_step_fused_matches_staged():
    B, H, G, n = 2, 2, 4, 900
    dtype = torch.bfloat16
    a, batch = _cache(B, H, G, n, dtype, [900, 640], seed=13, tau=0.5)
    c, _ = _cache(B, H, G, n, dtype, [900, 640], seed=13, tau=0.5)
    q = batch.q.contiguous()
    da = TwilightDecoder(a, "quest", budget=256, p=0.95)
    dc = TwilightDecoder(c, "quest", budget=256, p=0.95)
    out_a = da.step(q, batch.k_new, batch.v_new)
    c.append(batch.k_new, batch.v_new)
    out_c = dc.forward(q)
    torch.cuda.synchronize()
    assert a.seq_lens.tolist() == [901, 641]
    assert torch.equal(out_a, out_c)


@pytest.mark.parametrize("tau", [0.25, 2.0])
def test_k2_filter_bounds_within_margin_at_32k(tau):
    """The fp32 filter bounds sit within the error bound the select kernel
    assumes, so only a thin band of pages is rescored in fp64."""
    import ctypes
    B, H, G, n = 1, 2, 4, 32768
    cache, batch = _cache(B, H, G, n, torch.bfloat16, [n], seed=21, tau=tau, extra_pages=0)
    dec = TwilightDecoder(cache, "quest", budget=8192, p=0.95)
    q = batch.q.contiguous()
    dec.select(q)
    exact = torch.empty(B * H * G, cache.max_pages, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().tw_quest_scores(ctypes.byref(cache.struct()), _lib.ptr(q), _lib.ptr(exact),
                                          _lib.stream_handle()), "tw_quest_scores")
    torch.cuda.synchronize()
    approx = dec.bufs.page_scores.double() / np.sqrt(128)
    for u in range(B * H):
        amax = float(cache.kabsmax.view(-1)[u])
        for g in range(G):
            qh = q[0, u * G + g].float()
            margin = float(qh.abs().sum()) * amax * 300 / 2**24 / np.sqrt(128)
            err = (approx[u * G + g] - exact[u * G + g]).abs().max().item()
            assert err <= margin, (err, margin)
    rescored = int(dec.bufs.counters[1])
    assert rescored < 0.02 * B * H * G * cache.max_pages, rescored


def test_wave_pipelined_step_matches_single_wave():
    B, H, G, n = 4, 2, 4, 2000
    dtype = torch.bfloat16
    a, batch = _cache(B, H, G, n, dtype, [2000, 1500, 1999, 777], seed=17, tau=tau_schedule(H, (0.3, 1.0)))
    c, _ = _cache(B, H, G, n, dtype, [2000, 1500, 1999, 777], seed=17, tau=tau_schedule(H, (0.3, 1.0)))
    q = batch.q.contiguous()
    d1 = TwilightDecoder(a, "quest", budget=512, p=0.95)
    d2 = TwilightDecoder(c, "quest", budget=512, p=0.95, waves=2)
    o1 = d1.step(q, batch.k_new, batch.v_new)
    o2 = d2.step(q, batch.k_new, batch.v_new)
    torch.cuda.synchronize()
    assert a.seq_lens.tolist() == c.seq_lens.tolist()
    torch.testing.assert_close(o2, o1, rtol=1e-5, atol=1e-6)
    s1, s2 = d1.stats(), d2.stats()
    assert torch.equal(s1.group_b1, s2.group_b1) and torch.equal(s1.cand_pages, s2.cand_pages)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("sink,window", [(4, 64), (0, 100), (37, 1)])
def test_sink_window_selector_batched(dtype, sink, window):
    """select_sink_window (selectors.py:164-175) as the base selector of the
    batched path: candidate tokens, INT4 estimate, top-p and attention vs the
    oracle on every unit (ragged lengths; one unit short enough to keep all)."""
    B, H, G, n = 3, 2, 4, 700
    lengths = [700, 333, 60]
    cache, batch = _cache(B, H, G, n, dtype, lengths, seed=21, tau=tau_schedule(H, (0.4, 1.5)))
    p = 0.9
    dec = TwilightDecoder(cache, "sink_window", p=p, sink=sink, window=window)
    q = batch.q.contiguous()
    out = dec.forward(q)
    torch.cuda.synchronize()
    bufs = dec.bufs
    for b in range(B):
        for h in range(H):
            u = b * H + h
            K, V = to_np(cache.unit_keys(b, h)), to_np(cache.unit_values(b, h))
            want_cand = orc.sink_window_tokens(lengths[b], sink, window)
            ncand = int(bufs.cand_count[u])
            pages = bufs.cand_pages[u, :ncand].cpu().numpy()
            pos = (pages[:, None] * 16 + np.arange(16)).reshape(-1)
            z_all = bufs.logits[u, :, : ncand * 16].cpu().numpy()
            valid = np.isfinite(z_all[0])
            np.testing.assert_array_equal(pos[valid], want_cand)
            Qn = to_np(q[b, h * G:(h + 1) * G])
            _, _, _, final, _ = check_unit_topp(bufs, u, G, p)
            assert np.isin(final, want_cand).all()
            for g in range(G):
                w = orc.full_weights(Qn[g], K)
                want = orc.subset_attention(w, V, final, True)
                np.testing.assert_allclose(to_np(out[b, h * G + g]), want, rtol=1e-4, atol=1e-4 * np.abs(want).max())


@pytest.mark.parametrize("bits", [2, 8])
def test_two_and_eight_bit_cache_build_append_estimate(bits):
    """K1 bulk build and append for 2/8-bit caches bit-exact vs the oracle
    (quantize_rows + _pack_matrix layout), and the batched INT-b estimate."""
    B, H, G, n = 2, 2, 4, 640
    lengths = [640, 401]
    dtype = torch.bfloat16
    batch = make_batch(B, H, G, n, dtype, tau=tau_schedule(H, (0.5, 1.0)), seed=60 + bits)
    cache = PagedKVCache(B, H, G, max_pages=pages_for(n) + 1, dtype=dtype, bits=bits)
    cache.prefill(batch.K, batch.V, lengths)
    pos = torch.tensor(lengths, dtype=torch.int32, device="cuda")
    cache.append(batch.k_new.contiguous(), batch.v_new.contiguous(), pos)  # one appended row per sequence
    dec = TwilightDecoder(cache, "quest", budget=256, p=0.9)
    q = batch.q.contiguous()
    dec.forward(q)
    torch.cuda.synchronize()
    for b in range(B):
        for h in range(H):
            u = b * H + h
            K = to_np(cache.unit_keys(b, h))
            codes, scale, zero = orc.quantize_rows(K, bits)
            packed, sc, zr = cache.unit_quant(b, h)
            np.testing.assert_array_equal(packed.cpu().numpy(), orc.pack_codes_bits(codes, bits))
            np.testing.assert_array_equal(sc.cpu().numpy(), scale.astype(np.float32))
            np.testing.assert_array_equal(zr.cpu().numpy(), zero.astype(np.float32))
            ncand = int(dec.bufs.cand_count[u])
            pages = dec.bufs.cand_pages[u, :ncand].cpu().numpy()
            cand = orc.pages_to_tokens(pages, K.shape[0])
            pos_all = (pages[:, None] * 16 + np.arange(16)).reshape(-1)
            for g in range(G):
                qh = to_np(q[b, h * G + g])
                z = dec.bufs.logits[u, g, : ncand * 16].cpu().numpy()[pos_all < K.shape[0]]
                want = orc.estimate_logits(qh, codes, scale, zero, cand)
                scale_ref = np.abs(qh).sum() * np.abs(K).max() / np.sqrt(128)
                np.testing.assert_allclose(z, want, rtol=0, atol=2e-6 * scale_ref + 1e-6)


def _near_tie_ok(got, want, q, K, ids, budget):
    """Channel-pruned sets may differ from the oracle only where two scores
    tie to fp64 rounding (the reference's BLAS summation order is unpinned)."""
    diff = np.setxor1d(got, want)
    if diff.size == 0:
        return True
    s = (K[:, ids].astype(np.float64) @ np.asarray(q, np.float64)[ids]) / math.sqrt(128)
    kth = np.sort(s)[::-1][orc.resolve_budget(budget, K.shape[0]) - 1]
    return diff.size <= 4 and bool(np.all(np.abs(s[diff] - kth) <= 1e-12 * max(1.0, abs(kth))))


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("top_channels,budget", [(None, 100), (5, 37), (128, 500)])
def test_channel_pruned_selector_batched(dtype, top_channels, budget):
    """The channel-pruned base selector (selectors.py:135-161) on the batched
    path: channel slice, per-head token sets and their group union, then INT4
    estimate / top-p / attention over exactly those tokens vs the oracle
    (ragged lengths; one unit shorter than the budget keeps everything)."""
    B, H, G, n = 3, 2, 4, 900
    lengths = [900, 421, 60]
    cache, batch = _cache(B, H, G, n, dtype, lengths, seed=31, tau=tau_schedule(H, (0.4, 1.5)))
    p = 0.9
    dec = TwilightDecoder(cache, "channel_pruned", budget=budget, p=p, top_channels=top_channels)
    q = batch.q.contiguous()
    out = dec.forward(q)
    torch.cuda.synchronize()
    bufs = dec.bufs
    count = top_channels or 16
    for b in range(B):
        for h in range(H):
            u = b * H + h
            K, V = to_np(cache.unit_keys(b, h)), to_np(cache.unit_values(b, h))
            Qn = to_np(q[b, h * G:(h + 1) * G])
            ids = orc.top_channels_by_magnitude(K, count)
            np.testing.assert_array_equal(bufs.chan_ids[u, :count].cpu().numpy(), ids)
            heads = [orc.channel_pruned_tokens(Qn[g], K, ids, budget) for g in range(G)]
            want_cand = orc.union_sorted(heads)
            ncand = int(bufs.cand_count[u])
            pages = bufs.cand_pages[u, :ncand].cpu().numpy()
            np.testing.assert_array_equal(pages, np.unique(want_cand // 16))
            pos = (pages[:, None] * 16 + np.arange(16)).reshape(-1)
            z_all = bufs.logits[u, :, : ncand * 16].cpu().numpy()
            valid = np.isfinite(z_all[0])
            got = pos[valid]
            if not np.array_equal(got, want_cand):
                assert all(_near_tie_ok(got, want_cand, Qn[g], K, ids, budget) for g in range(G))
                continue
            _, _, _, final, _ = check_unit_topp(bufs, u, G, p)
            assert np.isin(final, want_cand).all()
            for g in range(G):
                w = orc.full_weights(Qn[g], K)
                want = orc.subset_attention(w, V, final, True)
                np.testing.assert_allclose(to_np(out[b, h * G + g]), want, rtol=1e-4, atol=1e-4 * np.abs(want).max())


def test_channel_pruned_selector_long_context():
    """The channel-pruned selector beyond 32k tokens (keys staged in the unit's
    logits rows, not shared memory): slice, per-head token sets and union at a
    131,072-token context (selectors.py:135-161; the reference has no length cap)."""
    B, H, G, n, budget, count = 1, 2, 4, 131072, 8192, 16
    cache, batch = _cache(B, H, G, n, torch.bfloat16, [n], seed=41, tau=tau_schedule(H, (0.4, 1.5)))
    dec = TwilightDecoder(cache, "channel_pruned", budget=budget, p=0.9)
    q = batch.q.contiguous()
    dec.select(q)
    torch.cuda.synchronize()
    bufs = dec.bufs
    for h in range(H):
        K = to_np(cache.unit_keys(0, h))
        Qn = to_np(q[0, h * G:(h + 1) * G])
        ids = orc.top_channels_by_magnitude(K, count)
        np.testing.assert_array_equal(bufs.chan_ids[h, :count].cpu().numpy(), ids)
        heads = [orc.channel_pruned_tokens(Qn[g], K, ids, budget) for g in range(G)]
        want = orc.union_sorted(heads)
        words = bufs.tok_mask[h].cpu().numpy().view(np.uint32)
        got = np.flatnonzero(np.unpackbits(words.view(np.uint8), bitorder="little"))
        if not np.array_equal(got, want):
            assert all(_near_tie_ok(got, want, Qn[g], K, ids, budget) for g in range(G))
        ncand = int(bufs.cand_count[h])
        np.testing.assert_array_equal(bufs.cand_pages[h, :ncand].cpu().numpy(), np.unique(got // 16))


def test_channel_pruned_fixed_slice_survives_appends():
    """fix_channels keeps the slice ranked at the first step (build_selector
    binds it once per context, selectors.py:203); without it every step
    re-ranks the current cache."""
    B, H, G, n = 2, 2, 2, 300
    dtype = torch.float32
    cache, batch = _cache(B, H, G, n, dtype, [300, 250], seed=5, extra_pages=4)
    fixed = TwilightDecoder(cache, "channel_pruned", budget=64, p=0.9, fix_channels=True)
    live = TwilightDecoder(cache, "channel_pruned", budget=64, p=0.9)
    q = batch.q.contiguous()
    fixed.forward(q)
    first = fixed.bufs.chan_ids[:, :16].clone()
    # append large keys on the channels that were NOT selected, until they dominate the magnitudes
    for step in range(40):
        k_new = torch.zeros(B, H, 128, dtype=dtype, device="cuda")
        k_new[..., 100:] = 1e3
        cache.append(k_new, torch.zeros_like(k_new))
    fixed.forward(q)
    live.forward(q)
    torch.cuda.synchronize()
    assert torch.equal(fixed.bufs.chan_ids[:, :16], first)
    for u in range(B * H):
        K = to_np(cache.unit_keys(u // H, u % H))
        np.testing.assert_array_equal(live.bufs.chan_ids[u, :16].cpu().numpy(), orc.top_channels_by_magnitude(K, 16))


@pytest.mark.parametrize("bits", [4, 2, 8])
def test_fused_step_append_matches_separate_append(bits):
    """tw_decode_step fuses K1 into the Quest filter (the warp holding a unit's
    open page appends first): over several steps -- opening new pages -- the
    cache (rows, codes, params, page metadata, |k| bound, lengths) and the
    outputs equal the separate append kernel followed by the staged path."""
    B, H, G, n = 2, 2, 4, 700
    dtype = torch.bfloat16
    lengths = [638, 511]
    batch = make_batch(B, H, G, n, dtype, tau=0.7, seed=77)
    caches = []
    for _ in range(2):
        c = PagedKVCache(B, H, G, max_pages=pages_for(n) + 2, dtype=dtype, bits=bits)
        c.prefill(batch.K, batch.V, lengths)
        caches.append(c)
    fused = TwilightDecoder(caches[0], "quest", budget=160, p=0.9)
    staged = TwilightDecoder(caches[1], "quest", budget=160, p=0.9)
    gen = torch.Generator(device="cuda").manual_seed(3)
    for step in range(20):
        k_new = torch.randn(B, H, 128, device="cuda", generator=gen).to(dtype)
        v_new = torch.randn(B, H, 128, device="cuda", generator=gen).to(dtype)
        q = (torch.randn(B, H * G, 128, device="cuda", generator=gen) * 0.5).to(dtype)
        out_f = fused.step(q, k_new, v_new)
        caches[1].append(k_new, v_new)
        out_s = staged.forward(q)
        torch.cuda.synchronize()
        assert torch.equal(out_f, out_s), step
    a, c = caches
    assert a.seq_lens.tolist() == c.seq_lens.tolist() == [658, 531]
    for name in ("k_cache", "v_cache", "kq", "kmeta", "kabsmax"):
        assert torch.equal(getattr(a, name), getattr(c, name)), name


@pytest.mark.parametrize("selector", ["full", "sink_window", "channel_pruned"])
def test_decode_step_other_selectors_match_staged(selector):
    """tw_decode_step with the non-Quest base selectors (separate K1 append)
    equals append + the staged kernels."""
    B, H, G, n = 2, 2, 4, 600
    dtype = torch.bfloat16
    kw = dict(p=0.9, budget=200) if selector == "channel_pruned" else dict(p=0.9)
    a, batch = _cache(B, H, G, n, dtype, [600, 431], seed=17, tau=0.6)
    c, _ = _cache(B, H, G, n, dtype, [600, 431], seed=17, tau=0.6)
    da, dc = TwilightDecoder(a, selector, **kw), TwilightDecoder(c, selector, **kw)
    q = batch.q.contiguous()
    for _ in range(3):
        out_a = da.step(q, batch.k_new, batch.v_new)
        c.append(batch.k_new, batch.v_new)
        out_c = dc.forward(q)
        torch.cuda.synchronize()
        assert torch.equal(out_a, out_c)
    assert a.seq_lens.tolist() == c.seq_lens.tolist() == [603, 434]


@pytest.mark.parametrize("fused", [False, True])
def test_append_beyond_capacity_is_dropped(fused):
    """A position past the sequence's page table is dropped by K1 (separate
    append kernel and the append fused into the Quest filter): no write, the
    length unchanged; the other sequences append normally."""
    B, H, G = 2, 2, 4
    P = 8
    dtype = torch.bfloat16
    batch = make_batch(B, H, G, P * 16, dtype, seed=91)
    cache = PagedKVCache(B, H, G, max_pages=P, dtype=dtype)
    cache.prefill(batch.K, batch.V, [P * 16, 100])
    before = [t.clone() for t in (cache.k_cache, cache.v_cache, cache.kq, cache.kmeta)]
    pos = torch.tensor([P * 16, 100], dtype=torch.int32, device="cuda")
    if fused:
        TwilightDecoder(cache, "quest", budget=32, p=0.9).step(batch.q.contiguous(), batch.k_new, batch.v_new, pos)
    else:
        cache.append(batch.k_new, batch.v_new, pos)
    torch.cuda.synchronize()
    assert cache.seq_lens.tolist() == [P * 16, 101]
    for t0, t1 in zip(before, (cache.k_cache, cache.v_cache, cache.kq, cache.kmeta)):
        assert torch.equal(t0[:P], t1[:P])  # sequence 0 owns physical pages 0..P-1
    assert torch.equal(cache.unit_keys(1, 0)[100], batch.k_new[1, 0])


def test_step_with_default_positions_many_waves():
    """step() without positions passes cache.seq_lens as the append positions.
    The fused K1+K2 filter writes seq_lens while later filter items still read
    their positions, so the aliased case must take the separate append (ADVICE
    r01): many filter items per unit (B*H well above the SM count) and every
    length a multiple of 16 * 64 tokens (the open page starts a new item)."""
    B, H, G, n = 40, 8, 4, 2048
    dtype = torch.bfloat16
    a, batch = _cache(B, H, G, n, dtype, [n] * B, seed=23, tau=0.6, extra_pages=2)
    c, _ = _cache(B, H, G, n, dtype, [n] * B, seed=23, tau=0.6, extra_pages=2)
    q = batch.q.contiguous()
    da = TwilightDecoder(a, "quest", budget=512, p=0.9)
    dc = TwilightDecoder(c, "quest", budget=512, p=0.9)
    for _ in range(2):
        out_a = da.step(q, batch.k_new, batch.v_new)  # positions = seq_lens (aliased)
        c.append(batch.k_new, batch.v_new)
        out_c = dc.forward(q)
        torch.cuda.synchronize()
        assert torch.equal(out_a, out_c)
    assert a.seq_lens.tolist() == c.seq_lens.tolist() == [n + 2] * B
    for name in ("k_cache", "v_cache", "kq", "kmeta", "kabsmax"):
        assert torch.equal(getattr(a, name), getattr(c, name)), name


def test_chunk_geometry_validated_before_any_kernel():
    """A work-item size the merge cannot take is rejected on the host (and by
    tw_decode_step before K1 appends); auto_chunk never picks one."""
    from paper_2502_02770_b200.decode import auto_chunk, min_chunk
    B, H, G = 1, 8, 4
    cache = PagedKVCache(B, H, G, max_pages=2049, dtype=torch.bfloat16)  # 32k context + one spare page
    assert auto_chunk(cache) >= min_chunk(2049) and auto_chunk(cache) % 16 == 0
    TwilightDecoder(cache, "quest", budget=8192, p=0.95)  # builds: the old 513 * 4 > 2048 limit is gone
    big = PagedKVCache(1, 1, 1, max_pages=8192, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        TwilightDecoder(big, "full", p=0.9, chunk_tokens=64)  # 2048 items per unit
    dec = TwilightDecoder(big, "full", p=0.9)
    dec.params.chunk_tokens = 64  # bypass the host check: the C ABI rejects it before appending
    k = torch.zeros(1, 1, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        dec.step(torch.zeros(1, 1, 128, dtype=torch.bfloat16, device="cuda"), k, k)
    torch.cuda.synchronize()
    assert big.seq_lens.tolist() == [0]


def test_attention_in_parts_equals_whole():
    """tw_sparse_attention_part (the bench's per-kernel timing of K4): the
    attention kernel alone, then the merge alone, reproduce tw_sparse_attention
    bit for bit, and the attention kernel can be re-run on the same state."""
    B, H, G, n = 6, 8, 4, 3000
    dtype = torch.bfloat16
    cache, batch = _cache(B, H, G, n, dtype, [n, 2900, 1500, 3000, 700, 2048], seed=31, tau=0.7)
    q = batch.q.contiguous()
    dec = TwilightDecoder(cache, "quest", budget=1024, p=0.95)
    whole = dec.forward(q).clone()
    out = torch.full_like(whole, float("nan"))
    for _ in range(2):  # re-runnable: the kernel resets its own item counter
        dec.attend_part(q, out, 1)
    dec.attend_part(q, out, 2)
    torch.cuda.synchronize()
    assert torch.equal(out, whole)
    with pytest.raises(ValueError):
        dec.attend_part(q, out, 3)
