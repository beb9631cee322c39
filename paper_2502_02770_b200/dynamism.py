"""Budget dynamism, p sweeps and per-head run rows.

The reference summarises the final budgets B1 along the prompt / step / layer
/ head axes (collect_dynamism, pipeline.py:420-462), sweeps the mass target
over a fixed workload (sweep_p, pipeline.py:465-498) and writes one CSV row
per head (RUN_COLUMNS / write_csv, reporting.py:35-60).  Here the same
summaries are built either from reference-shaped ``TaggedReport`` lists (the
per-head API) or straight from a batched decode step's device statistics
(``tag_decode_stats``: B1 per query head read back from tw_topp's head_stats),
so a serving run can report the paper's dynamism figures without the per-head
fp64 report path.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, replace
from typing import Iterable, Sequence

import numpy as np

from .pipeline import PipelineConfig, PruneReport, run_head

AXES = ("prompt", "step", "layer", "head")


@dataclass(frozen=True)
class TaggedReport:
    """pipeline.py:93-99."""
    prompt: int
    step: int
    layer: int
    head: int
    report: PruneReport


@dataclass(frozen=True)
class AxisSummary:
    """pipeline.py:102-110."""
    mean: float
    std: float
    min: float
    max: float
    group_means: dict
    histogram_edges: tuple
    histogram_counts: tuple


@dataclass(frozen=True)
class DynamismStats:
    """pipeline.py:113-117."""
    axes: dict
    overall_mean: float
    overall_std: float


@dataclass(frozen=True)
class SweepRow:
    """pipeline.py:120-126."""
    p: float
    mean_b1: float
    mean_attained_true_mass: float
    mean_residual_error: float
    mean_cost_units: float


def collect_dynamism(reports: Iterable[TaggedReport], bins: int = 16) -> DynamismStats:
    """pipeline.py:420-462: for each axis, the per-group mean B1 and the
    spread of those means, with one histogram binning [0, max B1] shared by
    all axes.  Tags must be unique."""
    tagged = list(reports)
    if not tagged:
        raise ValueError("no reports to summarize")
    tags = [(t.prompt, t.step, t.layer, t.head) for t in tagged]
    if len(set(tags)) != len(tags):
        dup = next(k for k in tags if tags.count(k) > 1)
        raise ValueError(f"duplicate report tag {dup}")
    b1 = np.array([t.report.b1 for t in tagged], dtype=np.float64)
    edges = np.linspace(0.0, max(1.0, float(b1.max())), bins + 1)
    axes = {}
    for axis in AXES:
        key = np.array([getattr(t, axis) for t in tagged])
        groups = {int(g): float(b1[key == g].mean()) for g in np.unique(key)}
        means = np.fromiter(groups.values(), dtype=np.float64)
        counts = np.histogram(means, bins=edges)[0]
        axes[axis] = AxisSummary(mean=float(means.mean()), std=float(means.std()), min=float(means.min()),
                                 max=float(means.max()), group_means=groups,
                                 histogram_edges=tuple(float(e) for e in edges),
                                 histogram_counts=tuple(int(c) for c in counts))
    return DynamismStats(axes=axes, overall_mean=float(b1.mean()), overall_std=float(b1.std()))


@dataclass(frozen=True)
class _B1Only:
    b1: int


def tag_decode_stats(stats, heads_per_seq: int, *, step: int = 0, layer: int = 0,
                     first_prompt: int = 0) -> list[TaggedReport]:
    """TaggedReports from a batched decode step (TwilightDecoder.stats(); the
    query heads of sequence b are rows b*heads_per_seq ..): prompt = sequence,
    head = query head.  Only ``report.b1`` is populated -- the quantity
    collect_dynamism summarises."""
    b1 = stats.b1.detach().to("cpu").numpy().astype(np.int64)
    if b1.size % heads_per_seq:
        raise ValueError("heads_per_seq does not divide the number of query heads")
    return [TaggedReport(prompt=first_prompt + i // heads_per_seq, step=step, layer=layer, head=i % heads_per_seq,
                         report=_B1Only(int(v))) for i, v in enumerate(b1)]


def sweep_p(items: Sequence, cfg: PipelineConfig, p_grid: Sequence[float]) -> list[SweepRow]:
    """pipeline.py:465-498 on the GPU path: mean B1 / true mass / residual /
    modelled cost per mass target over (q, keys, values) items."""
    grid = [float(p) for p in p_grid]
    if any(b < a for a, b in zip(grid, grid[1:])):
        raise ValueError("p_grid must be sorted ascending")
    if not items:
        raise ValueError("empty workload")
    rows = []
    for p in grid:
        run_cfg = replace(cfg, prune=replace(cfg.prune, p=p))
        reps = [run_head(q, k, v, run_cfg)[2] for q, k, v in items]
        rows.append(SweepRow(p=p, mean_b1=float(np.mean([r.b1 for r in reps])),
                             mean_attained_true_mass=float(np.mean([r.attained_true_mass for r in reps])),
                             mean_residual_error=float(np.mean([r.residual_error for r in reps])),
                             mean_cost_units=float(np.mean([r.cost_units for r in reps]))))
    return rows


# reporting.py:35-43
RUN_COLUMNS = [
    "prompt", "step", "layer", "head", "group", "bypassed",
    "n", "b0", "b1",
    "candidate_mass", "true_mass", "spearman",
    "threshold", "iterations",
    "residual_error", "value_norm", "error_bound",
    "tokens_selector", "tokens_estimator", "tokens_attention",
    "estimator_bytes", "cost_units", "baseline_units", "modeled_speedup",
]


def format_value(v) -> str:
    """reporting.py:46-51: bools as 0/1, floats with 9 significant digits."""
    if isinstance(v, (bool, np.bool_)):
        return "1" if v else "0"
    if isinstance(v, (float, np.floating)):
        return f"{float(v):.9g}"
    return str(v)


def run_row(t: TaggedReport, group: int, bypassed: bool) -> list:
    r = t.report
    return [t.prompt, t.step, t.layer, t.head, group, bypassed, r.n, r.b0, r.b1, r.attained_candidate_mass,
            r.attained_true_mass, r.estimator_spearman, r.threshold, r.iterations, r.residual_error, r.value_norm,
            r.error_bound, r.tokens_selector, r.tokens_estimator, r.tokens_attention, r.estimator_bytes,
            r.cost_units, r.baseline_units, r.modeled_speedup]


def write_run_csv(path, rows: Iterable[list]) -> None:
    """reporting.py:54-60 layout: header RUN_COLUMNS, one line per head."""
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(RUN_COLUMNS)
        for row in rows:
            w.writerow([format_value(v) for v in row])
