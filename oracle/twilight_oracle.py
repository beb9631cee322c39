"""CPU oracle for the Twilight select-then-prune decode path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2502_02770_b200`` imports this
module; it is used by ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` as the checker
and as the timed CPU baseline -- never as the thing measured or shipped.

It restates, in NumPy, the reference package ``nucleuskv`` (pure
Python/NumPy, /root/reference/pkg/src/nucleuskv) for the functions on the
hot path.  Each function names the reference lines it follows.  Parity of
this restatement is PINNED: ``oracle/gen_golden.py`` runs the reference
itself (importable in the build container) and writes the golden vectors
under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this module
against them (bit-exact for codes, bytes, page ids, fp64 scores and index
sets; fp32 BLAS summation order is the only tolerated difference).

Array conventions: one "unit" is one KV head of one sequence; ``K``/``V``
are (n, d) in the dtype the path computes in (float32 here; bf16 inputs are
passed as their exact float32 upcast), ``Q`` is (G, d) for the G query
heads sharing that KV head.
"""

from __future__ import annotations

import math

import numpy as np

PAGE_SIZE = 16
MASS_SLACK = 1e-9  # attention.py:16
NORMALIZATION_TOLERANCE = 1e-4  # pruner.py:30
PARAM_BYTES = 4  # quantcache.py:42


# --------------------------------------------------------------------------
# stage 1: INT4 key quantization and page metadata


def quantize_rows(K: np.ndarray, bits: int = 4):
    """Per-row asymmetric codes, fp64 arithmetic, half-even rounding.

    Follows quantcache.py:95-114 (row form) and its vectorised twin in
    build_cache, quantcache.py:199-207: scale = (max - min) / (2^bits - 1),
    code = clip(rint((k - min) / scale), 0, levels); a constant row gets
    scale 0, zero = min and all-zero codes.
    Returns (codes uint8 (n, d), scale f64 (n,), zero f64 (n,)).
    """
    X = np.asarray(K, dtype=np.float64)
    if X.ndim == 1:
        X = X[None, :]
    top = (1 << bits) - 1
    rmin = X.min(axis=1)
    rmax = X.max(axis=1)
    width = rmax - rmin
    flat = width == 0.0
    scale = np.where(flat, 0.0, width / top)
    divisor = np.where(flat, 1.0, scale)
    q = np.rint((X - rmin[:, None]) / divisor[:, None])
    q = np.clip(q, 0, top)
    q[flat] = 0
    return q.astype(np.uint8), scale, rmin


def pack_nibbles(codes: np.ndarray) -> np.ndarray:
    """Two 4-bit codes per byte, even channel in the low nibble.

    quantcache.py:122-130 / :142-151 (golden: arange(16) -> 10 32 54 .. fe).
    Works on the last axis; returns uint8 (..., d/2).
    """
    c = np.asarray(codes, dtype=np.uint8)
    return (c[..., 0::2] | (c[..., 1::2] << 4)).astype(np.uint8)


def pack_codes_bits(codes: np.ndarray, bits: int) -> np.ndarray:
    """b-bit codes packed lowest-order field first, 8/b per byte (_pack_matrix,
    quantcache.py:122-130).  Works on the last axis; returns uint8 (..., d*b/8)."""
    c = np.asarray(codes, dtype=np.uint16)
    per = 8 // bits
    g = c.reshape(c.shape[:-1] + (c.shape[-1] // per, per))
    out = np.zeros(g.shape[:-1], dtype=np.uint16)
    for slot in range(per):
        out |= g[..., slot] << (bits * slot)
    return out.astype(np.uint8)


def unpack_nibbles(packed: np.ndarray) -> np.ndarray:
    """Inverse of pack_nibbles (quantcache.py:132-139, :154-160)."""
    b = np.asarray(packed, dtype=np.uint8)
    out = np.empty(b.shape[:-1] + (b.shape[-1] * 2,), dtype=np.uint8)
    out[..., 0::2] = b & 0x0F
    out[..., 1::2] = b >> 4
    return out


def page_bounds(K: np.ndarray, page_size: int = PAGE_SIZE):
    """Per-page, per-channel min and max over the real rows only.

    quantcache.py:163-175; the tail page covers only rows < n
    (test_quantcache.py:125-131).  Returns (lo, hi), each f64 (P, d).
    """
    X = np.asarray(K, dtype=np.float64)
    n, d = X.shape
    P = -(-n // page_size)
    pad = P * page_size - n
    lo_src = np.concatenate([X, np.full((pad, d), np.inf)]) if pad else X
    hi_src = np.concatenate([X, np.full((pad, d), -np.inf)]) if pad else X
    lo = lo_src.reshape(P, page_size, d).min(axis=1)
    hi = hi_src.reshape(P, page_size, d).max(axis=1)
    return lo, hi


# --------------------------------------------------------------------------
# stage 2: Quest page scores, top-k pages, GQA union


def resolve_budget(budget, n: int) -> int:
    """Absolute token budget (selectors.py:72-87): float fraction in (0, 1]
    uses Python's half-even round(); int is clamped to n; bool rejected."""
    if isinstance(budget, bool):
        raise ValueError("budget must be a number")
    if isinstance(budget, float):
        if not 0.0 < budget <= 1.0:
            raise ValueError(f"fractional budget {budget} outside (0, 1]")
        return max(1, min(n, round(budget * n)))
    b = int(budget)
    if b < 1:
        raise ValueError("budget must select at least one token")
    return min(b, n)


def quest_scores(q: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """Upper bound of every in-page logit, in fp64 (selectors.py:97-109).

    Per page: sum_c max(q_c lo_c, q_c hi_c) / sqrt(d).  The row sum is a
    NumPy reduction over the contiguous channel axis, which for d <= 128 is
    NumPy's 8-lane unrolled pairwise sum; the CUDA refine step replays that
    exact order so its fp64 scores are bit-identical.
    """
    qd = np.asarray(q, dtype=np.float64)
    terms = np.maximum(qd * lo, qd * hi)
    return terms.sum(axis=1) / math.sqrt(qd.size)


def numpy_rowsum_order(terms: np.ndarray) -> np.ndarray:
    """Explicit replay of NumPy's float64 row reduction for d <= 128 (8
    strided partial sums, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
    then the d % 8 tail).  Used by tests to prove the summation order the
    CUDA kernel implements is the one NumPy uses."""
    t = np.asarray(terms, dtype=np.float64)
    n = t.shape[-1]
    assert n <= 128, "pairwise blocking above 128 not replayed"
    if n < 8:
        acc = np.zeros(t.shape[:-1])
        # NumPy's short path: -0.0 seeded sequential sum
        acc = acc * 0.0 - 0.0
        for i in range(n):
            acc = acc + t[..., i]
        return acc
    r = [t[..., j].copy() for j in range(8)]
    body = n - (n % 8)
    for i in range(8, body, 8):
        for j in range(8):
            r[j] = r[j] + t[..., i + j]
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    for i in range(body, n):
        res = res + t[..., i]
    return res


def top_pages(scores: np.ndarray, n_pages_wanted: int) -> np.ndarray:
    """Indices of the best pages, ties to the lower page, returned sorted
    (selectors.py:128: stable argsort of -score, first k, then sort)."""
    order = np.argsort(-scores, kind="stable")
    return np.sort(order[:n_pages_wanted])


def quest_select_pages(q, lo, hi, budget, n: int, page_size: int = PAGE_SIZE) -> np.ndarray:
    """select_quest (selectors.py:112-132) at page granularity: the token
    budget is rounded up to whole pages, capped at ceil(n / page_size)."""
    P = -(-n // page_size)
    if lo.shape[0] != P:
        raise ValueError(f"metadata covers {lo.shape[0]} pages, context of {n} needs {P}")
    b0 = resolve_budget(budget, n)
    k = min(P, -(-b0 // page_size))
    return top_pages(quest_scores(q, lo, hi), k)


def pages_to_tokens(pages: np.ndarray, n: int, page_size: int = PAGE_SIZE) -> np.ndarray:
    """Expand sorted page ids to sorted token ids, clipping the tail page
    at n (selectors.py:129-131)."""
    pages = np.asarray(pages, dtype=np.int64)
    if pages.size == 0:
        return np.zeros(0, dtype=np.int64)
    tok = (pages[:, None] * page_size + np.arange(page_size)[None, :]).reshape(-1)
    return tok[tok < n]


def sink_window_tokens(n: int, sink: int, window: int) -> np.ndarray:
    """select_sink_window (selectors.py:164-175): the first ``sink`` plus the
    last ``window`` tokens; every token when they meet (select_full)."""
    if n < 1:
        raise ValueError("context must contain at least one token")
    if sink < 0 or window < 0:
        raise ValueError("sink and window must be non-negative")
    if sink + window < 1:
        raise ValueError("sink + window must keep at least one token")
    if sink + window >= n:
        return np.arange(n, dtype=np.int64)
    return np.unique(np.concatenate([np.arange(sink), np.arange(n - window, n)])).astype(np.int64)


def top_channels_by_magnitude(K: np.ndarray, count: int) -> np.ndarray:
    """selectors.py:135-143: the ``count`` channels of largest mean |K| (fp64;
    NumPy's axis-0 mean adds the rows in order), stable on ties, ascending."""
    K = np.asarray(K, dtype=np.float64)
    if K.ndim != 2:
        raise ValueError("keys must be (n, d)")
    if not 1 <= count <= K.shape[1]:
        raise ValueError(f"count {count} outside [1, {K.shape[1]}]")
    magnitude = np.abs(K).mean(axis=0)
    return np.sort(np.argsort(-magnitude, kind="stable")[:count])


def channel_pruned_tokens(q, K, ids, budget) -> np.ndarray:
    """select_channel_pruned (selectors.py:146-161): the B0 tokens with the
    largest (K[:, ids] @ q[ids]) / sqrt(d) in fp64, ties -> lower token; sorted."""
    q = np.asarray(q, dtype=np.float64)
    ids = np.asarray(ids, dtype=np.int64)
    Kr = np.asarray(K, dtype=np.float64)[:, ids]
    n = Kr.shape[0]
    b0 = resolve_budget(budget, n)
    scores = (Kr @ q[ids]) / math.sqrt(q.size)
    return np.sort(np.argsort(-scores, kind="stable")[:b0])


def union_sorted(index_sets) -> np.ndarray:
    """Sorted union of index arrays (group_union, selectors.py:178-186)."""
    sets = [np.asarray(s, dtype=np.int64) for s in index_sets]
    if not sets:
        raise ValueError("no selections to union")
    return np.unique(np.concatenate(sets))


# --------------------------------------------------------------------------
# stage 3: INT4 estimate + candidate softmax


def estimate_logits(q, codes, scale, zero, token_idx) -> np.ndarray:
    """Approximate logits q . k_hat / sqrt(d) (quantcache.py:238-272).

    k_hat = zero + scale * code is formed in fp64 and cast to q's dtype
    before the dot product (:269); the result is scaled by q.dtype(1/sqrt d)
    (:258, :270).  ``codes``/``scale``/``zero`` are the per-token arrays of
    quantize_rows over the whole context.
    """
    qv = np.asarray(q)
    idx = np.asarray(token_idx, dtype=np.int64)
    if idx.size == 0:
        raise ValueError("no candidates to estimate")
    inv = qv.dtype.type(1.0 / math.sqrt(qv.shape[0]))
    k_hat = zero[idx, None] + scale[idx, None] * codes[idx].astype(np.float64)
    return (k_hat.astype(qv.dtype) @ qv) * inv


def exact_logits(q, K, token_idx) -> np.ndarray:
    """The exact estimator (pipeline.py:212-214): K[idx] @ q divided by
    sqrt(d) in the keys' dtype."""
    Km = np.asarray(K)
    idx = np.asarray(token_idx, dtype=np.int64)
    return (Km[idx] @ np.asarray(q)) / np.asarray(math.sqrt(Km.shape[1]), dtype=Km.dtype)


def dequantize(codes, scale: float, zero: float, dtype=np.float64) -> np.ndarray:
    """dequantize_row (quantcache.py:117-119): zero + scale * code in fp64."""
    return (zero + scale * np.asarray(codes, dtype=np.float64)).astype(dtype)


def softmax64(logits) -> np.ndarray:
    """Max-subtracted softmax in fp64 over the candidates only
    (attention.py:79-86 as called at pipeline.py:236 / :344)."""
    z = np.asarray(logits, dtype=np.float64)
    if z.ndim != 1 or z.size == 0:
        raise ValueError("logits must be a non-empty 1-D array")
    if not np.all(np.isfinite(z)):
        raise ValueError("logits contains non-finite entries")
    e = np.exp(z - z.max())
    return e / e.sum()


# --------------------------------------------------------------------------
# stage 4: top-p threshold search (Algorithm 1) and the sort-based truth


def threshold_top_p(weights, p: float, epsilon: float = 1e-15, max_iters: int = 64):
    """Bracketed threshold bisection of pruner.py:57-114.

    Keeps the invariant mass(w >= lo) >= p_eff; stops when the lowest tie
    class of the current selection cannot be dropped (:99-104), at the
    iteration cap (:105), when the bracket is narrower than epsilon (:107),
    when no weight lies strictly inside the bracket (:109) or the midpoint
    collapses (:112).  Returns (indices of w >= lo, lo, iterations);
    p_eff <= 0 gives (empty, inf, 0) (:80-82).
    """
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or w.size == 0:
        raise ValueError("weights must be a non-empty 1-D array")
    if np.any(w < 0) or not np.all(np.isfinite(w)):
        raise ValueError("weights must be finite and non-negative")
    total = float(w.sum())
    if abs(total - 1.0) > NORMALIZATION_TOLERANCE:
        raise ValueError("weights are not normalized")
    target = min(p, total) - MASS_SLACK
    if target <= 0.0:
        return np.zeros(0, dtype=np.int64), math.inf, 0
    lo_b, hi_b = 0.0, float(w.max())
    it = 0
    alive = w  # w[w >= lo_b] in index order
    while True:
        floor_w = alive.min()
        upper = alive[alive > floor_w]
        if upper.size == 0 or upper.sum() < target:
            break
        if it >= max_iters or hi_b - lo_b < epsilon:
            break
        inside = alive[alive < hi_b]
        if not np.any(inside > lo_b):
            break
        mid = 0.5 * (lo_b + hi_b)
        if not lo_b < mid < hi_b:
            break
        keep = alive[alive >= mid]
        if keep.sum() >= target:
            lo_b, alive = mid, keep
        else:
            hi_b = mid
        it += 1
    return np.flatnonzero(w >= lo_b).astype(np.int64), float(lo_b), it


def sort_top_p(weights, p: float) -> np.ndarray:
    """Minimal-cardinality prefix of the stable descending sort reaching
    min(p, total) - MASS_SLACK (oracle.py:49-62 / :35-46)."""
    w = np.asarray(weights, dtype=np.float64)
    order = np.argsort(-w, kind="stable")
    csum = np.cumsum(w[order])
    target = min(p, float(csum[-1])) - MASS_SLACK
    if target <= 0.0:
        return np.zeros(0, dtype=np.int64)
    k = min(int(np.searchsorted(csum, target, side="left")) + 1, csum.size)
    return np.sort(order[:k])


def minimal_tie_closed_top_p(weights, p: float) -> np.ndarray:
    """The set the converged bisection returns, computed directly: the
    smallest {w >= v} over distinct values v whose mass reaches p_eff.
    (Equivalent to threshold_top_p whenever no early-exit rule fires.)"""
    w = np.asarray(weights, dtype=np.float64)
    target = min(p, float(w.sum())) - MASS_SLACK
    if target <= 0.0:
        return np.zeros(0, dtype=np.int64)
    vals = np.unique(w)[::-1]
    for v in vals:
        if w[w >= v].sum() >= target:
            return np.flatnonzero(w >= v).astype(np.int64)
    return np.arange(w.size, dtype=np.int64)


# --------------------------------------------------------------------------
# stage 5: attention


def full_weights(q, K) -> np.ndarray:
    """softmax(K q / dtype(sqrt d)) over all n tokens, in q's dtype
    (attention.py:89-103)."""
    qv = np.asarray(q)
    Km = np.asarray(K)
    z = (Km @ qv) / np.asarray(np.sqrt(qv.shape[0]), dtype=Km.dtype)
    e = np.exp(z - z.max())
    return e / e.sum()


def subset_attention(w, V, idx, renormalize: bool) -> np.ndarray:
    """w[S] @ V[S], optionally divided by w[S].sum() (attention.py:106-136).
    Empty S: zeros without renormalisation, error with it."""
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size == 0:
        if renormalize:
            raise ValueError("cannot renormalize an empty selection")
        return np.zeros(np.asarray(V).shape[1], dtype=np.result_type(w, V))
    out = w[idx] @ V[idx]
    if renormalize:
        m = w[idx].sum()
        if not m > 0:
            raise ValueError("selected tokens carry no mass")
        out = out / m
    return out


# --------------------------------------------------------------------------
# one unit end to end (the hot half of run_grouped / run_head)


def prepare_unit(K, page_size: int = PAGE_SIZE, bits: int = 4):
    """The cache the reference builds once per context (build_cache,
    quantcache.py:178-235): page bounds + per-row b-bit codes/params."""
    lo, hi = page_bounds(K, page_size)
    codes, scale, zero = quantize_rows(K, bits)
    return lo, hi, codes, scale, zero


def decode_unit(Q, K, V, *, selector: str = "quest", budget=0.25, p: float = 0.95,
                page_size: int = PAGE_SIZE, renormalize: bool = True, logits_override=None, prepared=None,
                sink: int = 4, window: int = 64, bits: int = 4, top_channels=None, exact: bool = False):
    """run_grouped's hot path for one KV head (pipeline.py:306-360):

    per-head Quest (selectors.py:112-132; or select_full :90-94, or
    select_sink_window :164-175, whose token set is the candidates directly) ->
    group union (:338) -> per-head
    INT4 estimate over the union (:342) -> fp64 softmax (:344) -> threshold
    search (:345) -> group set = union of the pruned sets (:347) -> every
    head attends to the group set with renormalised full-context weights
    (:366-375).  With G == 1 this is run_head (pipeline.py:286-303; equal
    per test_pipeline.py:232-241).  ``selector`` is "quest", "full",
    "sink_window" or "channel_pruned" (selectors.py:135-161, channel slice
    fixed per context as build_selector :203-209 does; token sets, not pages).

    ``logits_override`` (G, |union|) replaces the INT4 estimate, so a test
    can feed the GPU's logits to the oracle's softmax + search;
    ``prepared`` = prepare_unit(K) reuses a prebuilt cache (the reference's
    cache=/metadata= arguments); ``exact`` estimates from the keys themselves
    (estimator_bits="exact", pipeline.py:212-214).  Returns a dict with every
    intermediate.
    """
    Q = np.atleast_2d(np.asarray(Q))
    n = K.shape[0]
    G = Q.shape[0]
    lo, hi, codes, scale, zero = prepared if prepared is not None else prepare_unit(K, page_size, bits)
    if selector == "full":
        head_pages = [np.arange(lo.shape[0]) for _ in range(G)]
    elif selector == "quest":
        head_pages = [quest_select_pages(Q[h], lo, hi, budget, n, page_size) for h in range(G)]
    elif selector in ("sink_window", "channel_pruned"):
        head_pages = None
    else:
        raise ValueError(f"selector {selector!r} not on the accelerated path")
    head_tokens = None
    if selector == "sink_window":
        cand = sink_window_tokens(n, sink, window)  # the same for every head: the union is the set itself
        union_pages = np.unique(cand // page_size)
    elif selector == "channel_pruned":
        count = top_channels if top_channels is not None else max(1, K.shape[1] // 8)
        ids = top_channels_by_magnitude(K, count)
        head_tokens = [channel_pruned_tokens(Q[h], K, ids, budget) for h in range(G)]
        cand = union_sorted(head_tokens)
        union_pages = np.unique(cand // page_size)
    else:
        union_pages = union_sorted(head_pages)
        cand = pages_to_tokens(union_pages, n, page_size)
    logits, pruned, thresholds, iters = [], [], [], []
    for h in range(G):
        if logits_override is not None:
            z = np.asarray(logits_override[h])
        elif exact:
            z = exact_logits(Q[h], K, cand)
        else:
            z = estimate_logits(Q[h], codes, scale, zero, cand)
        w = softmax64(z)
        sub, thr, it = threshold_top_p(w, p)
        logits.append(z)
        pruned.append(cand[sub])
        thresholds.append(thr)
        iters.append(it)
    shared = union_sorted(pruned) if pruned else np.zeros(0, dtype=np.int64)
    out = np.empty((G, V.shape[1]), dtype=np.result_type(Q, V))
    for h in range(G):
        w_full = full_weights(Q[h], K)
        ok = renormalize and shared.size > 0 and w_full[shared].sum() > 0
        out[h] = subset_attention(w_full, V, shared, ok)
    return {
        "lo": lo, "hi": hi, "codes": codes, "scale": scale, "zero": zero,
        "head_pages": head_pages, "head_tokens": head_tokens, "union_pages": union_pages, "candidates": cand,
        "logits": logits, "pruned": pruned, "thresholds": thresholds, "iterations": iters,
        "final": shared, "out": out,
    }
