"""Select -> estimate -> prune -> attend with the reference signatures
(nucleuskv/pipeline.py).

``run_head`` / ``run_grouped`` build a one-context paged pool (K1 bulk) --
or reuse the one behind a ``cache=`` / ``metadata=`` from build_cache, as
_prepare_context does (pipeline.py:177-201) -- and run the batched decode
kernels (K2 tw_select, K3 tw_estimate + tw_topp, K4 tw_sparse_attention) for
it: the same code path the batched decoder and the benchmark use.
``estimator_bits="exact"`` (and so bypass_config) estimates from the
full-precision keys (pipeline.py:212-214).  PruneReport fields that need the exact full-context fp64
attention (true mass, residual, Spearman) are instrumentation, not the
decode path; they are computed with device tensor ops after the kernels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import torch

from . import _lib as L
from .attention import TokenSelection
from .decode import TwilightDecoder, pages_for
from .pruner import BinarySearchConfig, PruneOutcome
from .quantcache import PagedQuantKeyCache, PageMetadataTable, _shared_pool, _unit_cache
from .selectors import GroupMap, SelectorConfig, resolve_budget

__all__ = ["PipelineConfig", "PruneReport", "bypass_config", "run_head", "run_grouped", "model_speedup",
           "memory_overhead"]

ESTIMATOR_MODES = (2, 4, 8, "exact")
DEFAULT_SELECTOR_COST_FRACTION = 1.0 / 16.0


@dataclass(frozen=True)
class PipelineConfig:
    """pipeline.py:52-66."""
    selector: SelectorConfig = field(default_factory=SelectorConfig)
    prune: BinarySearchConfig = field(default_factory=lambda: BinarySearchConfig(p=0.95))
    estimator_bits: int | str = 4
    group_map: GroupMap | None = None
    renormalize_output: bool = True
    bypass_layers: tuple[int, ...] = (0, 1)
    selector_cost_fraction: float = DEFAULT_SELECTOR_COST_FRACTION

    def __post_init__(self) -> None:
        if self.estimator_bits not in ESTIMATOR_MODES:
            raise ValueError(f"estimator_bits must be one of {ESTIMATOR_MODES}")
        if not 0.0 < self.selector_cost_fraction <= 1.0:
            raise ValueError("selector_cost_fraction must lie in (0, 1]")


@dataclass(frozen=True)
class PruneReport:
    """pipeline.py:69-90."""
    n: int
    b0: int
    b1: int
    attained_candidate_mass: float
    attained_true_mass: float
    estimator_spearman: float
    threshold: float
    iterations: int
    residual_error: float
    value_norm: float
    error_bound: float
    tokens_selector: int
    tokens_estimator: int
    tokens_attention: int
    estimator_bytes: int
    cost_units: float
    baseline_units: float
    modeled_speedup: float


def bypass_config(cfg: PipelineConfig) -> PipelineConfig:
    """pipeline.py:129-136: full selector, exact estimator, p = 1."""
    return replace(cfg, selector=SelectorConfig(kind="full", page_size=cfg.selector.page_size),
                   prune=replace(cfg.prune, p=1.0), estimator_bits="exact")


def model_speedup(n, b0, b1, selector_cost_fraction=DEFAULT_SELECTOR_COST_FRACTION, estimator_cost_fraction=0.25):
    """pipeline.py:143-164."""
    if not 0 <= b1 <= b0 <= n:
        raise ValueError(f"need 0 <= b1 <= b0 <= n, got n={n}, b0={b0}, b1={b1}")
    if n <= 0:
        raise ValueError("n must be positive")
    scan = n * selector_cost_fraction
    return (scan + b0) / (scan + b0 * estimator_cost_fraction + b1)


def memory_overhead(bits: int) -> float:
    """pipeline.py:167-174."""
    if bits not in (2, 4, 8):
        raise ValueError("bits must be 2, 4, or 8")
    return (bits / 16.0) * 0.5


def _midrank(x: torch.Tensor) -> torch.Tensor:
    order = torch.argsort(x, stable=True)
    xs = x[order]
    _, inv, counts = torch.unique_consecutive(xs, return_inverse=True, return_counts=True)
    ends = torch.cumsum(counts, 0).double()
    avg = ends - (counts.double() - 1.0) / 2.0  # 1-based average rank of each tie block
    ranks = torch.empty_like(xs, dtype=torch.float64)
    ranks[order] = avg[inv]
    return ranks


def _spearman(a: torch.Tensor, b: torch.Tensor) -> float:
    """Midrank Pearson correlation (stats.py:38-60); 0 for constant inputs."""
    if a.numel() < 2:
        return 0.0
    ra, rb = _midrank(a.double()), _midrank(b.double())
    ra, rb = ra - ra.mean(), rb - rb.mean()
    den = float(torch.sqrt((ra * ra).sum() * (rb * rb).sum()))
    return float((ra * rb).sum()) / den if den > 0 else 0.0


def _check_cfg(cfg: PipelineConfig) -> None:
    if cfg.selector.kind not in ("full", "quest", "sink_window", "channel_pruned"):
        raise NotImplementedError(f"selector {cfg.selector.kind!r} is not on the B200 path")
    if cfg.selector.page_size != L.PAGE_SIZE:
        raise ValueError("the B200 path uses 16-token pages")
    if cfg.prune.epsilon != 1e-15 or cfg.prune.max_iters != 64:
        raise NotImplementedError("the decode path implements the converged search (default epsilon/max_iters); "
                                  "use binary_search_top_p for other settings")
    if not cfg.renormalize_output:
        raise NotImplementedError("renormalize_output=False needs the full-context denominator (off the hot path)")


def _prepare_context(keys, values, cfg: PipelineConfig, G: int, groups: int, cache, metadata):
    """_prepare_context (pipeline.py:177-201) on the device pool: reuse the
    pool behind a supplied cache (or metadata table) when it fits the config,
    else build one (K1 bulk).  A cache of the wrong width or page size raises
    like the reference (:194-200)."""
    exact = cfg.estimator_bits == "exact"
    n = keys.shape[0]
    pool = None
    if cache is not None and not exact:
        if cache.bits != cfg.estimator_bits:
            raise ValueError(f"cache quantized at {cache.bits} bits, config wants {cfg.estimator_bits}")
        if cache.page_size != cfg.selector.page_size:
            raise ValueError("cache page size differs from selector page size")
        pool = cache.kv
    elif isinstance(metadata, PageMetadataTable) and (exact or metadata.cache.bits == cfg.estimator_bits):
        pool = metadata.cache
    elif cache is not None and isinstance(cache, PagedQuantKeyCache):
        pool = cache.kv  # exact estimator: only the keys and page metadata of the pool are read
    if pool is not None:
        if int(pool.seq_lens[0].item()) != n or pool.dtype != keys.dtype:
            raise ValueError("the supplied cache was built for different keys")
        return _shared_pool(pool, values, G, groups)
    return _unit_cache(keys, values.to(keys.dtype), group_size=G, num_seqs=groups,
                       bits=4 if exact else cfg.estimator_bits)


def _run(Q: torch.Tensor, keys: torch.Tensor, values: torch.Tensor, cfg: PipelineConfig, G: int, cache=None,
         metadata=None):
    """Run the decode kernels for H = groups*G query heads on one KV context."""
    _check_cfg(cfg)
    if not (Q.is_cuda and keys.is_cuda and values.is_cuda):
        raise ValueError("q, keys and values must be CUDA tensors (the Twilight path has no CPU fallback)")
    n = keys.shape[0]
    H = Q.shape[0]
    groups = H // G
    dt = keys.dtype
    kv = _prepare_context(keys, values, cfg, G, groups, cache, metadata)
    est = "exact" if cfg.estimator_bits == "exact" else "int"
    if cfg.selector.kind == "quest":
        if cfg.selector.budget is None:
            raise ValueError("selector 'quest' requires a budget")
        dec = TwilightDecoder(kv, "quest", budget=resolve_budget(cfg.selector.budget, n), p=cfg.prune.p,
                              estimator=est)
    elif cfg.selector.kind == "sink_window":
        dec = TwilightDecoder(kv, "sink_window", p=cfg.prune.p, sink=cfg.selector.sink, window=cfg.selector.window,
                              estimator=est)
    elif cfg.selector.kind == "channel_pruned":
        if cfg.selector.budget is None:
            raise ValueError("selector 'channel_pruned' requires a budget")
        dec = TwilightDecoder(kv, "channel_pruned", budget=resolve_budget(cfg.selector.budget, n), p=cfg.prune.p,
                              top_channels=cfg.selector.top_channels, estimator=est)
    else:
        dec = TwilightDecoder(kv, "full", p=cfg.prune.p, estimator=est)
    q = Q.to(dt).reshape(groups, G, L.HEAD_DIM).contiguous()
    out = dec.forward(q)
    return dec, out.reshape(H, L.HEAD_DIM)


def _reports(dec: TwilightDecoder, Q, keys, values, cfg: PipelineConfig, G: int):
    """Per-head (final selection, PruneReport), report-only fields in fp64."""
    n = keys.shape[0]
    bufs = dec.bufs
    H = Q.shape[0]
    q64, K64, V64 = Q.double(), keys.double(), values.double()
    w64 = torch.softmax((K64 @ q64.T) / math.sqrt(L.HEAD_DIM), dim=0).T  # [H, n]
    exact_out = w64 @ V64
    value_norm = float(torch.linalg.norm(V64))
    Kd, qd = keys.float(), Q.float()
    w_prod = torch.softmax((Kd @ qd.T) / torch.tensor(float(L.HEAD_DIM)).sqrt(), dim=0).T
    res = []
    for h in range(H):
        u, g = h // G, h % G
        cnt = int(bufs.final_count[u].item())
        final = bufs.final_idx[u, :cnt].long()
        ncand = int(bufs.cand_count[u].item())
        pages = bufs.cand_pages[u, :ncand].long()
        cand = (pages[:, None] * 16 + torch.arange(16, device=pages.device)).reshape(-1)
        logits = bufs.logits[u, g, : ncand * 16]
        valid = (cand < n) & torch.isfinite(logits)  # padding and (sink-window) unselected tokens are -inf
        logits = logits[valid]
        cand = cand[valid]
        est_w = torch.softmax(logits.double(), 0)
        in_final = torch.isin(cand, final)
        cand_mass = float(est_w[in_final].sum())
        sel = TokenSelection(indices=final, n=n, attained_mass=cand_mass)
        attained_true = float(w64[h, final].sum()) if cnt else 0.0
        out_h = dec_out = None  # filled by caller
        true_logits = (K64[cand] @ q64[h]) / math.sqrt(L.HEAD_DIM)
        rho = _spearman(logits.double(), true_logits)
        b0, b1 = int(cand.numel()), cnt
        scan = n * cfg.selector_cost_fraction
        exact = cfg.estimator_bits == "exact"
        cost = scan + b0 * (1.0 if exact else cfg.estimator_bits / 16.0) + b1  # _estimator_fraction
        base = scan + b0
        res.append((sel, exact_out[h], dict(n=n, b0=b0, b1=b1, attained_candidate_mass=cand_mass,
                                            attained_true_mass=attained_true, estimator_spearman=rho,
                                            threshold=float(bufs.head_stats[h, 2].item()), iterations=0,
                                            value_norm=value_norm, tokens_selector=n, tokens_estimator=b0,
                                            tokens_attention=b1,
                                            estimator_bytes=b0 * (2 * L.HEAD_DIM if exact else
                                                                  L.HEAD_DIM * cfg.estimator_bits // 8 + 4),
                                            cost_units=cost, baseline_units=base, modeled_speedup=base / cost)))
    return res


def _assemble(res, outs):
    outcomes, reports = [], []
    for h, (sel, exact_h, rep) in enumerate(res):
        residual = float(torch.linalg.norm(exact_h - outs[h].double()))
        reports.append(PruneReport(residual_error=residual,
                                   error_bound=max(0.0, 1.0 - rep["attained_true_mass"]) * rep["value_norm"], **rep))
        outcomes.append(PruneOutcome(selection=sel, threshold=rep["threshold"], iterations=0))
    return outcomes, reports


def run_head(q, keys, values, cfg: PipelineConfig, *, cache: PagedQuantKeyCache | None = None, metadata=None):
    """pipeline.py:286-303 on the B200 kernels: (output, PruneOutcome, PruneReport).

    A supplied ``cache``/``metadata`` (from build_cache) is reused as built
    (_prepare_context, pipeline.py:177-201): no re-quantization."""
    q = torch.as_tensor(q)
    dec, out = _run(q.reshape(1, -1), torch.as_tensor(keys), torch.as_tensor(values), cfg, 1, cache, metadata)
    res = _reports(dec, q.reshape(1, -1), keys, values, cfg, 1)
    outcomes, reports = _assemble(res, out)
    return out[0], outcomes[0], reports[0]


def run_grouped(queries, keys, values, cfg: PipelineConfig, *, cache: PagedQuantKeyCache | None = None,
                metadata=None):
    """pipeline.py:306-360: per-head Quest -> group union -> per-head INT4
    estimate + top-p over the union -> group set = union of pruned sets ->
    every head attends to it.  Returns (outputs [H, d], outcomes, reports)."""
    Q = torch.as_tensor(queries)
    if Q.ndim != 2:
        raise ValueError("queries must be (heads, d)")
    gm = cfg.group_map or GroupMap(1)
    gm.groups(Q.shape[0])
    G = gm.group_size
    if G not in (1, 2, 4, 8):
        raise NotImplementedError("group sizes 1, 2, 4, 8 are compiled")
    dec, out = _run(Q, torch.as_tensor(keys), torch.as_tensor(values), cfg, G, cache, metadata)
    res = _reports(dec, Q, keys, values, cfg, G)
    outcomes, reports = _assemble(res, out)
    return out, outcomes, reports
