"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python oracle/gen_golden.py

Every vector here is produced by ``nucleuskv`` (the reference), never by
this repo's oracle, so ``tests/test_oracle_golden.py`` pins the oracle to
the reference and the GPU tests pin the CUDA path to the same vectors.
Inputs are seeded; bf16 cases hold bf16-representable float32 values
(the oracle/GPU see exactly these numbers).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16, returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (a + 0x7FFF + ((a >> 16) & 1)) & 0xFFFF0000
    return rounded.astype(np.uint32).view(np.float32)


def main() -> None:
    sys.path.insert(0, REF)
    import nucleuskv as nk
    from nucleuskv.quantcache import _unpack_matrix

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20250204)

    # ---------------------------------------------------------- quantization
    quant = {}
    cases = {
        "gauss_f32": rng.standard_normal((203, 128)).astype(np.float32),
        "gauss_bf16": bf16_round(rng.standard_normal((203, 128)) * 1.7),
        "wide_bf16": bf16_round(rng.standard_normal((64, 128)) * np.exp(rng.standard_normal((64, 1)) * 3)),
        # rows that sit exactly on the 4-bit lattice and rows with .5 ties
        "lattice": np.array([rng.permutation(16).repeat(8) * 0.5 - 3.0 for _ in range(16)], dtype=np.float32),
        "halves": (np.tile(np.arange(128) % 31, (16, 1)) * 0.5).astype(np.float32),
        "constant": np.full((17, 128), -2.75, dtype=np.float32),
    }
    cases["mixed_const"] = np.concatenate([cases["gauss_bf16"][:20], cases["constant"][:5]])
    for name, K in cases.items():
        cache, meta = nk.build_cache(K, page_size=16, bits=4)
        n, d = K.shape
        codes = np.concatenate([_unpack_matrix(pg.packed, 16, d, 4)[: pg.valid_len] for pg in cache.pages])
        packed = np.concatenate([np.frombuffer(pg.packed, dtype=np.uint8).reshape(16, d // 2)[: pg.valid_len] for pg in cache.pages])
        scales = np.concatenate([pg.scales[: pg.valid_len] for pg in cache.pages])
        zeros = np.concatenate([pg.zeros[: pg.valid_len] for pg in cache.pages])
        quant[f"{name}/K"] = K
        quant[f"{name}/codes"] = codes
        quant[f"{name}/packed"] = packed
        quant[f"{name}/scale"] = scales
        quant[f"{name}/zero"] = zeros
        quant[f"{name}/lo"] = np.stack([m.lo for m in meta])
        quant[f"{name}/hi"] = np.stack([m.hi for m in meta])
        # quantize_row on a few rows must agree with the vectorised build
        for r in range(min(3, n)):
            c, prm = nk.quantize_row(K[r])
            quant[f"{name}/row{r}_codes"] = c
            quant[f"{name}/row{r}_params"] = np.array([prm.scale, prm.zero])
    quant["pack/arange16"] = np.frombuffer(nk.pack_codes(np.arange(16)), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "quant.npz"), **quant)

    # ---------------------------------------------------------- quest
    quest = {}
    qi = 0
    for n, budget, dt in [(2048, 512, "f32"), (1000, 0.25, "bf16"), (777, 100, "f32"), (1024, 0.5, "bf16"),
                          (33, 16, "f32"), (20, 64, "bf16"), (1041, 300, "bf16")]:
        K = rng.standard_normal((n, 128)).astype(np.float32)
        q = (rng.standard_normal(128) / 0.5).astype(np.float32)
        if dt == "bf16":
            K, q = bf16_round(K), bf16_round(q)
        meta = nk.build_page_metadata(K, 16)
        scores = nk.quest_page_scores(q, meta)
        sel = nk.select_quest(q, meta, budget, 16, n)
        key = f"c{qi}"
        quest[f"{key}/K"] = K
        quest[f"{key}/q"] = q
        quest[f"{key}/budget"] = np.array([budget], dtype=np.float64 if isinstance(budget, float) else np.int64)
        quest[f"{key}/scores"] = scores
        quest[f"{key}/selected"] = sel.indices
        qi += 1
    # tie handling: identical pages -> lower page wins
    K = np.tile(bf16_round(rng.standard_normal((16, 128))), (8, 1))
    q = bf16_round(rng.standard_normal(128))
    meta = nk.build_page_metadata(K, 16)
    quest["tie/K"] = K
    quest["tie/q"] = q
    quest["tie/budget"] = np.array([48], dtype=np.int64)
    quest["tie/scores"] = nk.quest_page_scores(q, meta)
    quest["tie/selected"] = nk.select_quest(q, meta, 48, 16, K.shape[0]).indices
    np.savez_compressed(os.path.join(OUT, "quest.npz"), **quest)

    # ---------------------------------------------------------- estimate
    est = {}
    for i, (n, dt) in enumerate([(300, "f32"), (512, "bf16"), (77, "f32")]):
        K = rng.standard_normal((n, 128)).astype(np.float32)
        q = (rng.standard_normal(128) * 2).astype(np.float32)
        if dt == "bf16":
            K, q = bf16_round(K), bf16_round(q)
        cache, _ = nk.build_cache(K)
        idx = np.sort(rng.choice(n, size=max(1, n // 3), replace=False))
        sel = nk.TokenSelection.from_indices(idx, n)
        r = nk.estimate_scores(q, cache, sel)
        est[f"e{i}/K"] = K
        est[f"e{i}/q"] = q
        est[f"e{i}/idx"] = idx
        est[f"e{i}/scores"] = r.scores
        est[f"e{i}/bytes"] = np.array([r.bytes_touched])
    np.savez_compressed(os.path.join(OUT, "estimate.npz"), **est)

    # ---------------------------------------------------------- top-p
    topp = {}
    t = 0
    for n in (1, 2, 16, 100, 1000, 2500):
        for spread in (0.3, 1.0, 3.0, 8.0):
            z = rng.standard_normal(n) * spread
            w = np.exp(z - z.max())
            w = w / w.sum()
            for p in (0.0, 0.5, 0.9, 0.95, 0.99, 1.0):
                out = nk.binary_search_top_p(w, nk.BinarySearchConfig(p=p))
                topp[f"t{t}/w"] = w
                topp[f"t{t}/p"] = np.array([p])
                topp[f"t{t}/idx"] = out.selection.indices
                topp[f"t{t}/threshold"] = np.array([out.threshold])
                topp[f"t{t}/iterations"] = np.array([out.iterations])
                topp[f"t{t}/cfg"] = np.array([1e-15, 64.0])
                t += 1
    specials = [
        (np.array([0.3, 0.3, 0.2, 0.2]), 0.7, 1e-15, 64),
        (np.array([0.3, 0.3, 0.2, 0.2]), 0.5, 1e-15, 64),
        (np.array([0.6, 0.0, 0.4]), 1.0, 1e-15, 64),
        (np.full(4, 0.25), 0.0, 1e-15, 64),
        (np.full(8, 0.125), 0.3, 1e-15, 64),
        (np.array([0.5, 0.25, 0.25]), 0.6, 1e-15, 64),
    ]
    z = rng.standard_normal(512)
    w512 = np.exp(z - z.max()); w512 /= w512.sum()
    specials += [(w512, 0.9, 1e-15, 1), (w512, 0.9, 1e6, 64), (w512, 0.9, 1e-4, 64), (w512, 0.99, 1e-15, 5)]
    for w, p, eps, mi in specials:
        out = nk.binary_search_top_p(w, nk.BinarySearchConfig(p=p, epsilon=eps, max_iters=mi))
        topp[f"t{t}/w"] = w
        topp[f"t{t}/p"] = np.array([p])
        topp[f"t{t}/idx"] = out.selection.indices
        topp[f"t{t}/threshold"] = np.array([out.threshold])
        topp[f"t{t}/iterations"] = np.array([out.iterations])
        topp[f"t{t}/cfg"] = np.array([eps, float(mi)])
        t += 1
    np.savez_compressed(os.path.join(OUT, "topp.npz"), **topp)

    # ---------------------------------------------------------- attention
    att = {}
    for i, (n, dt) in enumerate([(500, "f32"), (64, "bf16")]):
        K = rng.standard_normal((n, 128)).astype(np.float32)
        V = rng.standard_normal((n, 128)).astype(np.float32)
        q = (rng.standard_normal(128) * 1.5).astype(np.float32)
        if dt == "bf16":
            K, V, q = bf16_round(K), bf16_round(V), bf16_round(q)
        w = nk.attention_weights(q, K)
        idx = np.sort(rng.choice(n, size=n // 4, replace=False))
        sel = nk.TokenSelection.from_indices(idx, n)
        att[f"a{i}/K"], att[f"a{i}/V"], att[f"a{i}/q"], att[f"a{i}/idx"] = K, V, q, idx
        att[f"a{i}/w"] = w
        att[f"a{i}/out_renorm"] = nk.sparse_attention(w, V, sel, renormalize=True)
        att[f"a{i}/out_plain"] = nk.sparse_attention(w, V, sel, renormalize=False)
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **att)

    # ---------------------------------------------------------- pipeline
    pipe = {}
    configs = [
        # name, n, G, selector, budget, p, tau, dtype
        ("grouped_quest_f32", 1024, 4, "quest", 512, 0.95, 0.5, "f32"),
        ("grouped_quest_bf16", 800, 4, "quest", 0.25, 0.95, 0.35, "bf16"),
        ("head_full_bf16", 600, 1, "full", None, 0.9, 0.4, "bf16"),
        ("head_quest_f32", 777, 1, "quest", 200, 0.8, 1.0, "f32"),
        ("grouped_full_f32", 640, 2, "full", None, 0.99, 2.0, "f32"),
        # sink-window base selector (selectors.py:164-175): sink/window in tokens
        ("grouped_sinkwin_bf16", 900, 4, "sink_window:7:150", None, 0.9, 0.3, "bf16"),
        ("head_sinkwin_f32", 500, 1, "sink_window:0:33", None, 0.95, 0.5, "f32"),
        ("grouped_sinkwin_all_f32", 300, 2, "sink_window:200:120", None, 0.9, 1.0, "f32"),
    ]
    for name, n, G, kind, budget, p, tau, dt in configs:
        sink = window = 0
        if kind.startswith("sink_window"):
            kind, sink, window = kind.split(":")[0], int(kind.split(":")[1]), int(kind.split(":")[2])
        K = rng.standard_normal((n, 128)).astype(np.float32)
        V = rng.standard_normal((n, 128)).astype(np.float32)
        Q = (rng.standard_normal((G, 128)) / tau).astype(np.float32)
        if dt == "bf16":
            K, V, Q = bf16_round(K), bf16_round(V), bf16_round(Q)
        sel = nk.SelectorConfig(kind=kind, budget=budget, page_size=16, **(
            dict(sink=sink, window=window) if kind == "sink_window" else {}))
        cfg = nk.PipelineConfig(selector=sel, prune=nk.BinarySearchConfig(p=p), group_map=nk.GroupMap(G))
        if G == 1:
            out, outcome, report = nk.run_head(Q[0], K, V, cfg)
            outs, finals, b0 = out[None], [outcome.selection.indices], [report.b0]
        else:
            outs, outcomes, reports = nk.run_grouped(Q, K, V, cfg)
            finals, b0 = [o.selection.indices for o in outcomes], [r.b0 for r in reports]
        pipe[f"{name}/K"], pipe[f"{name}/V"], pipe[f"{name}/Q"] = K, V, Q
        # budget, p, selector (0 full, 1 quest, 2 sink_window), budget-is-fraction, sink, window
        pipe[f"{name}/cfg"] = np.array([-1 if budget is None else budget, p,
                                        {"full": 0.0, "quest": 1.0, "sink_window": 2.0}[kind],
                                        1.0 if isinstance(budget, float) else 0.0, sink, window])
        pipe[f"{name}/out"] = np.asarray(outs)
        pipe[f"{name}/final"] = finals[0]
        pipe[f"{name}/b0"] = np.array(b0)
        for h, f in enumerate(finals):
            assert np.array_equal(f, finals[0]) or G == 1
    np.savez_compressed(os.path.join(OUT, "pipeline.npz"), **pipe)

    # ---------------------------------------------------------- 2- and 8-bit caches (SUPPORTED_BITS, quantcache.py:38)
    qb = {}
    rng_b = np.random.default_rng(20250207)
    for bits in (2, 8):
        for name, K in (("gauss_bf16", bf16_round(rng_b.standard_normal((203, 128)) * 1.3)),
                        ("wide_f32", (rng_b.standard_normal((70, 128)) *
                                      np.exp(rng_b.standard_normal((70, 1)) * 2)).astype(np.float32)),
                        ("constant", np.full((19, 128), 0.625, dtype=np.float32))):
            cache, _ = nk.build_cache(K, page_size=16, bits=bits)
            n = K.shape[0]
            per = 128 * bits // 8
            qb[f"b{bits}_{name}/K"] = K
            qb[f"b{bits}_{name}/packed"] = np.concatenate(
                [np.frombuffer(pg.packed, dtype=np.uint8).reshape(16, per)[: pg.valid_len] for pg in cache.pages])
            qb[f"b{bits}_{name}/codes"] = np.concatenate(
                [_unpack_matrix(pg.packed, 16, 128, bits)[: pg.valid_len] for pg in cache.pages])
            qb[f"b{bits}_{name}/scale"] = np.concatenate([pg.scales[: pg.valid_len] for pg in cache.pages])
            qb[f"b{bits}_{name}/zero"] = np.concatenate([pg.zeros[: pg.valid_len] for pg in cache.pages])
            q = bf16_round((rng_b.standard_normal(128) * 1.5).astype(np.float32))
            idx = np.sort(rng_b.choice(n, size=max(1, n // 2), replace=False))
            r = nk.estimate_scores(q.astype(K.dtype), cache, nk.TokenSelection.from_indices(idx, n))
            qb[f"b{bits}_{name}/q"], qb[f"b{bits}_{name}/idx"] = q, idx
            qb[f"b{bits}_{name}/scores"], qb[f"b{bits}_{name}/bytes"] = r.scores, np.array([r.bytes_touched])
    np.savez_compressed(os.path.join(OUT, "quant_bits.npz"), **qb)

    # ---------------------------------------------------------- dynamism summaries (pipeline.py:420-462)
    from nucleuskv.pipeline import PruneReport, TaggedReport, collect_dynamism
    dyn = {}
    tags = [(pr, st, ly, hd) for pr in range(2) for st in range(3) for ly in range(2) for hd in range(4)]
    b1s = rng.integers(0, 5000, size=len(tags))
    fields = {f: 0 for f in PruneReport.__dataclass_fields__}
    reps = [TaggedReport(*t, report=PruneReport(**{**fields, "b1": int(b)})) for t, b in zip(tags, b1s)]
    stats = collect_dynamism(reps, bins=12)
    dyn["tags"], dyn["b1"] = np.array(tags), b1s
    dyn["overall"] = np.array([stats.overall_mean, stats.overall_std])
    for axis, a in stats.axes.items():
        dyn[f"{axis}/summary"] = np.array([a.mean, a.std, a.min, a.max])
        dyn[f"{axis}/groups"] = np.array(sorted(a.group_means.items()), dtype=np.float64)
        dyn[f"{axis}/edges"] = np.array(a.histogram_edges)
        dyn[f"{axis}/counts"] = np.array(a.histogram_counts)
    np.savez_compressed(os.path.join(OUT, "dynamism.npz"), **dyn)

    # ---------------------------------------------------------- .twlt tensor file (tensorfile.py:61-74)
    from nucleuskv.tensorfile import write_tensor
    t = (np.arange(2 * 3 * 5, dtype=np.float32).reshape(2, 3, 5) - 7.25) / 3.0
    write_tensor(os.path.join(OUT, "ref_tensor.twlt"), t)
    np.save(os.path.join(OUT, "ref_tensor.npy"), t)

    # ---------------------------------------------------------- channel-pruned selector (selectors.py:135-161)
    ch = {}
    rng_c = np.random.default_rng(20250311)
    for i, (n, count, dt) in enumerate(((300, 16, "f32"), (1000, 5, "bf16"), (64, 128, "f32"), (40, 1, "f32"))):
        K = (rng_c.standard_normal((n, 128)) * np.exp(rng_c.standard_normal(128))).astype(np.float32)
        if i == 3:  # magnitude ties: equal columns -> lower channel wins
            K[:, 7] = K[:, 3]
            K[:, 90] = -K[:, 3] * 4
            K[:, 91] = K[:, 90]
        if dt == "bf16":
            K = bf16_round(K)
        ch[f"m{i}/K"], ch[f"m{i}/count"] = K, np.array([count])
        ch[f"m{i}/ids"] = nk.selectors.top_channels_by_magnitude(K, count)
    for i, (n, count, budget, dt) in enumerate(((500, 16, 77, "f32"), (333, 9, 0.3, "bf16"),
                                                 (96, 3, 200, "f32"), (50, 16, 1, "bf16"))):
        K = rng_c.standard_normal((n, 128)).astype(np.float32)
        q = rng_c.standard_normal(128).astype(np.float32)
        if dt == "bf16":
            K, q = bf16_round(K), bf16_round(q)
        if i == 2:  # score ties: repeated rows -> lower token first
            K[50:60] = K[10]
        ids = np.sort(rng_c.choice(128, size=count, replace=False))
        sel = nk.selectors.select_channel_pruned(q, K[:, ids].astype(np.float64), ids, budget)
        ch[f"s{i}/K"], ch[f"s{i}/q"], ch[f"s{i}/ids"] = K, q, ids
        ch[f"s{i}/budget"] = np.array([budget, 1.0 if isinstance(budget, float) else 0.0])
        ch[f"s{i}/indices"] = sel.indices
    for i, (n, G, budget, top, p, tau, dt) in enumerate(((700, 4, 96, None, 0.9, 0.4, "bf16"),
                                                         (512, 1, 0.25, 24, 0.95, 0.6, "f32"),
                                                         (900, 2, 300, 8, 0.85, 1.0, "f32"))):
        K = rng_c.standard_normal((n, 128)).astype(np.float32)
        V = rng_c.standard_normal((n, 128)).astype(np.float32)
        Q = (rng_c.standard_normal((G, 128)) / tau).astype(np.float32)
        if dt == "bf16":
            K, V, Q = bf16_round(K), bf16_round(V), bf16_round(Q)
        sel = nk.SelectorConfig(kind="channel_pruned", budget=budget, page_size=16, top_channels=top)
        cfg = nk.PipelineConfig(selector=sel, prune=nk.BinarySearchConfig(p=p), group_map=nk.GroupMap(G))
        if G == 1:
            out, outcome, report = nk.run_head(Q[0], K, V, cfg)
            outs, finals, b0 = out[None], [outcome.selection.indices], [report.b0]
        else:
            outs, outcomes, reports = nk.run_grouped(Q, K, V, cfg)
            finals, b0 = [o.selection.indices for o in outcomes], [r.b0 for r in reports]
        ch[f"p{i}/K"], ch[f"p{i}/V"], ch[f"p{i}/Q"] = K, V, Q
        # budget, p, budget-is-fraction, top_channels (-1: default d // 8)
        ch[f"p{i}/cfg"] = np.array([budget, p, 1.0 if isinstance(budget, float) else 0.0, -1 if top is None else top])
        ch[f"p{i}/out"], ch[f"p{i}/final"], ch[f"p{i}/b0"] = np.asarray(outs), finals[0], np.array(b0)
    np.savez_compressed(os.path.join(OUT, "channel.npz"), **ch)
    rows_and_exact()
    print("golden vectors written to", OUT)


def rows_and_exact() -> None:
    """rows.npz: dequantize_row / unpack_codes answers (quantcache.py:117-160)
    and run_grouped / run_head with the exact estimator -- bypass_config
    (pipeline.py:129-136) and estimator_bits="exact" under Quest -- as the
    reference computes them (pipeline.py:204-216)."""
    sys.path.insert(0, REF)
    import nucleuskv as nk

    rng = np.random.default_rng(20251017)
    out = {}
    for r in range(6):
        bits = (2, 4, 8)[r % 3]
        k = rng.standard_normal(128).astype(np.float32) * (1 + r)
        codes, prm = nk.quantize_row(k, bits=bits)
        out[f"deq{r}/codes"], out[f"deq{r}/params"] = codes, np.array([prm.scale, prm.zero])
        out[f"deq{r}/f64"] = nk.dequantize_row(codes, prm)
        out[f"deq{r}/f32"] = nk.dequantize_row(codes, prm, dtype=np.float32)
    for r in range(4):
        packed = rng.integers(0, 256, size=64 if r else 8, dtype=np.uint8)
        out[f"unpack{r}/packed"] = packed
        out[f"unpack{r}/codes"] = nk.unpack_codes(packed.tobytes(), 2 * packed.size)
    for i, (n, G, kind, budget, p, dt) in enumerate([(700, 4, "full", None, 1.0, "f32"), (513, 1, "full", None, 1.0, "f32"),
                                                     (900, 4, "quest", 256, 0.9, "f32"),
                                                     (640, 2, "quest", 0.3, 0.95, "bf16")]):
        K = rng.standard_normal((n, 128)).astype(np.float32)
        V = rng.standard_normal((n, 128)).astype(np.float32)
        Q = (rng.standard_normal((G, 128)) * 1.5).astype(np.float32)
        if dt == "bf16":
            K, V, Q = bf16_round(K), bf16_round(V), bf16_round(Q)
        base = nk.PipelineConfig(selector=nk.SelectorConfig(kind=kind, budget=budget),
                                 prune=nk.BinarySearchConfig(p=p), group_map=nk.GroupMap(G))
        cfg = nk.bypass_config(base) if kind == "full" else \
            nk.PipelineConfig(selector=base.selector, prune=base.prune, group_map=base.group_map, estimator_bits="exact")
        if G == 1:
            o, oc, rep = nk.run_head(Q[0], K, V, cfg)
            outs, finals, b0 = np.asarray(o)[None], oc.selection.indices, rep.b0
        else:
            o, ocs, reps = nk.run_grouped(Q, K, V, cfg)
            outs, finals, b0 = np.asarray(o), ocs[0].selection.indices, reps[0].b0
        out[f"x{i}/K"], out[f"x{i}/V"], out[f"x{i}/Q"] = K, V, Q
        out[f"x{i}/cfg"] = np.array([-1 if budget is None else budget, p, 1.0 if isinstance(budget, float) else 0.0,
                                     1.0 if kind == "quest" else 0.0])
        out[f"x{i}/out"], out[f"x{i}/final"], out[f"x{i}/b0"] = outs, np.asarray(finals), np.array([b0])
    np.savez_compressed(os.path.join(OUT, "rows.npz"), **out)


if __name__ == "__main__":
    if "--rows" in sys.argv:
        rows_and_exact()
    else:
        main()
