"""GPU top-p pruner (tw_topp) on crafted logits vs the oracle's minimal
tie-closed top-p set (binary_search_top_p, pruner.py:57-114, converged), and
the group union (pipeline.py:347).

The logits are written straight into the decode buffers, so the cases can
stress what random K/V never reaches: >8192 logits per head (multi-chunk
histograms), crossing bins with more members than the per-unit list holds
(re-read path), one tie class spanning the whole head, p = 0 / 1, heads with
no valid logit, -inf padding.
"""

import numpy as np
import pytest
import torch

from oracle import twilight_oracle as orc
from tests.gpu_util import f2key_np, topp_set_ok

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2502_02770_b200.decode import PagedKVCache, TwilightDecoder  # noqa: E402


def run_topp(z: np.ndarray, npages: list[int], p: float, seed: int = 0):
    """z: [U, G, T] float32 logits (-inf = invalid).  Returns the decoder."""
    U, G, T = z.shape
    max_pages = T // 16
    cache = PagedKVCache(U, 1, G, max_pages=max_pages, dtype=torch.bfloat16)
    dec = TwilightDecoder(cache, "full", p=p)
    b = dec.bufs
    rng = np.random.default_rng(seed)
    for u in range(U):
        # candidate pages: an increasing subset of the logical pages (exercises the position -> token map)
        pages = np.sort(rng.choice(max_pages, size=npages[u], replace=False)).astype(np.int32)
        b.cand_pages[u, : npages[u]] = torch.from_numpy(pages)
        b.cand_count[u] = npages[u]
    zt = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float32))
    b.logits.copy_(zt.cuda())
    hm = np.zeros(U * G, dtype=np.uint32)
    for u in range(U):
        for g in range(G):
            zz = z[u, g, : npages[u] * 16]
            if np.isfinite(zz).any():
                hm[u * G + g] = f2key_np(np.array([zz[np.isfinite(zz)].max()]))[0]
    b.head_max.copy_(torch.from_numpy(hm.view(np.int32)).cuda())
    b.counters.zero_()
    for _ in range(2):  # the second call checks the library left its scratch zeroed
        b.counters.zero_()
        dec.topp()
    torch.cuda.synchronize()
    return dec


def check(dec, z, npages, p):
    U, G, T = z.shape
    b = dec.bufs
    kinds = []
    for u in range(U):
        npos = npages[u] * 16
        pages = b.cand_pages[u, : npages[u]].cpu().numpy()
        tok = (pages[:, None] * 16 + np.arange(16)).reshape(-1)
        sets = []
        for g in range(G):
            zz = z[u, g, :npos]
            valid = np.isfinite(zz)
            thr = np.uint32(b.head_thr[u * G + g].item() & 0xFFFFFFFF)
            sel = np.flatnonzero(valid & (f2key_np(zz) >= thr))
            if valid.any():
                w = np.zeros(npos)
                w[valid] = orc.softmax64(zz[valid])
                ok, why = topp_set_ok(sel, w, p)
                assert ok, f"unit {u} head {g}: {why}"
                kinds.append(why)
            else:
                assert sel.size == 0
            assert int(b.head_stats[u * G + g, 0]) == sel.size
            sets.append(tok[sel])
        want = orc.union_sorted(sets) if sets else np.zeros(0, np.int64)
        cnt = int(b.final_count[u])
        np.testing.assert_array_equal(b.final_idx[u, :cnt].cpu().numpy(), want)
    return kinds


def _normal(rng, U, G, T, scales):
    z = rng.standard_normal((U, G, T)).astype(np.float32)
    for g in range(G):
        z[:, g] *= scales[g % len(scales)]
    return z


@pytest.mark.parametrize("G", [1, 4])
@pytest.mark.parametrize("p", [0.5, 0.9, 0.95, 0.99])
def test_topp_random_multichunk(G, p):
    rng = np.random.default_rng(int(p * 100) + G)
    U, T = 3, 40960
    z = _normal(rng, U, G, T, (4.0, 2.0, 0.5, 0.25))
    npages = [2560, 1700, 9]
    z[1, :, 1700 * 16 - 5:] = -np.inf  # ragged tail inside the last page
    dec = run_topp(z, npages, p)
    kinds = check(dec, z, npages, p)
    assert kinds.count("equal") >= len(kinds) // 2


def test_topp_single_tie_class_and_flat_heads():
    U, G, T = 2, 4, 32768
    z = np.zeros((U, G, T), np.float32)
    z[0, 1] = 3.25                      # every logit equal: the whole head is one tie class
    z[0, 2, ::2] = 1.0                  # two classes
    z[0, 3] = np.random.default_rng(1).standard_normal(T).astype(np.float32)
    z[1] = -np.inf                      # unit 1 head 0..3: no valid logit at all
    z[1, 2, :100] = 0.5
    npages = [2048, 2048]
    dec = run_topp(z, npages, 0.9)
    check(dec, z, npages, 0.9)
    assert int(dec.bufs.head_stats[1, 0]) == 32768


def test_topp_crossing_bin_overflows_member_list():
    # 30k logits packed inside one 1/120-logit bin -> re-read path, several key levels
    rng = np.random.default_rng(3)
    U, G, T = 1, 4, 65536
    z = np.full((U, G, T), -8.0, np.float32)
    for g in range(G):
        z[0, g, :30000] = (2.0 + rng.uniform(0, 1 / 240, 30000)).astype(np.float32)
        z[0, g, 30000:30010] = 2.5
        z[0, g, 40000:40400:2] = z[0, g, 100]  # duplicates of one member
    npages = [4096]
    for p in (0.3, 0.7):
        dec = run_topp(z, npages, p)
        check(dec, z, npages, p)


@pytest.mark.parametrize("p", [0.0, 1.0])
def test_topp_p_edges(p):
    rng = np.random.default_rng(5)
    U, G, T = 2, 4, 8192
    z = _normal(rng, U, G, T, (1.0, 3.0))
    z[:, :, :7] = -30.0  # weights ~1e-13: p=1 keeps them only if they reach p - 1e-9
    npages = [512, 300]
    dec = run_topp(z, npages, p)
    check(dec, z, npages, p)
    if p == 0.0:
        assert int(dec.bufs.final_count.sum()) == 0


def test_topp_more_units_than_sms():
    # > 148 units selects the two-CTAs-per-SM variant (half the member list)
    rng = np.random.default_rng(11)
    U, G, T = 160, 4, 4096
    z = _normal(rng, U, G, T, (2.0, 0.5, 1.0, 0.25))
    npages = [int(x) for x in rng.integers(1, T // 16 + 1, size=U)]
    dec = run_topp(z, npages, 0.9)
    check(dec, z, npages, 0.9)


@pytest.mark.parametrize("p", [0.2, 0.4, 0.6, 0.8])
def test_topp_bin_boundaries_near_zero(p):
    """Crossing bins whose edges lie near z = 0, where the float guess
    M - b/120 is hundreds of ulps from the exact edge of dbin's bin (the
    rounding of M*120 is ~|M| 3e-8 absolute, the ulp of z ~1e-9): a dense
    cloud of logits on both sides of the edges of the bins around zero, so
    the pass-2 membership interval must equal pass 1's binning exactly (a
    mismatch corrupted the member list on C5 at p = 0.85)."""
    M = np.float32(4.1929)
    vals = [M]
    for b in (504, 505, 506):  # edges at z ~ -0.007, -0.015, -0.024 (M * 120 ~ 503.1)
        e = np.float32(M - np.float32(b) / np.float32(120.0))
        for k in range(-900, 901, 5):
            vals.append(np.float32(e + np.float32(k) * np.spacing(e)))
    v = np.unique(np.asarray(vals, dtype=np.float32))
    z = np.full((1, 1, 16 * (-(-v.size // 16))), -np.inf, dtype=np.float32)
    z[0, 0, : v.size] = np.random.default_rng(3).permutation(v)
    npages = [z.shape[2] // 16]
    dec = run_topp(z, npages, p)
    check(dec, z, npages, p)
