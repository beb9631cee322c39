"""Shared helpers for the GPU parity tests (import only from tests)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import twilight_oracle as orc

MASS_TOL = 1e-6  # top-p tolerance: mass slack and relative weight slack at the threshold


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def f2key_np(z: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(z, dtype=np.float32).view(np.uint32)
    return np.where(b & 0x80000000, ~b, b | 0x80000000).astype(np.uint32)


def tie_closed_top_p(w: np.ndarray, p: float) -> np.ndarray:
    """orc.minimal_tie_closed_top_p in O(n log n): the smallest {w >= v} over
    distinct values v whose mass reaches p_eff.  The descending cumulative sum
    locates v; the candidate (and its successor class) are then re-checked with
    the oracle's own masked sums, so the result is the oracle's set."""
    w = np.asarray(w, dtype=np.float64)
    target = min(p, float(w.sum())) - orc.MASS_SLACK
    if target <= 0.0:
        return np.zeros(0, dtype=np.int64)
    vals = np.unique(w)[::-1]  # distinct values, descending
    order = np.sort(w)[::-1]
    k = int(np.searchsorted(np.cumsum(order), target, side="left"))
    k = min(k, order.size - 1)
    j = int(np.searchsorted(-vals, -order[k], side="left"))  # index of order[k] among the distinct values
    # the cumulative sums are in a different order than the oracle's masked sums: settle the boundary exactly
    while j > 0 and w[w >= vals[j - 1]].sum() >= target:
        j -= 1
    while j + 1 < vals.size and w[w >= vals[j]].sum() < target:
        j += 1
    return np.flatnonzero(w >= vals[j]).astype(np.int64)


def topp_set_ok(sel: np.ndarray, w: np.ndarray, p: float, tol: float = MASS_TOL) -> tuple[bool, str]:
    """Is `sel` (indices into w) the reference's top-p set up to threshold ties?

    Exact equality with the oracle's converged search passes outright.  Else
    the set must be top-closed (nothing heavier than its lightest member by
    more than `tol` relative is left out), reach p_eff - tol, and be minimal:
    dropping its lightest class (within `tol`) must fall below p_eff + tol.
    So the only differences allowed are tokens whose weight lies within `tol`
    (relative) of the threshold -- the north star's "ties within 1e-6".
    """
    ref = tie_closed_top_p(w, p)
    sel = np.sort(np.asarray(sel, dtype=np.int64))
    if np.array_equal(sel, ref):
        return True, "equal"
    target = min(p, float(w.sum())) - orc.MASS_SLACK
    if target <= 0:
        return sel.size == 0, "p_eff <= 0 must select nothing"
    if sel.size == 0:
        return False, "empty selection"
    t = w[sel].min()
    outside = np.setdiff1d(np.arange(w.size), sel)
    if outside.size and w[outside].max() > t * (1 + tol):
        return False, f"not top-closed: left out {w[outside].max():.3e} > threshold {t:.3e}"
    mass = w[sel].sum()
    if mass < target - tol:
        return False, f"mass {mass} < target {target}"
    core = sel[w[sel] > t * (1 + tol)]
    if w[core].sum() >= target + tol:
        return False, f"not minimal: {w[core].sum()} without the threshold class"
    diff = np.setxor1d(sel, ref)
    tref = w[ref].min() if ref.size else t
    if np.all(np.abs(w[diff] - tref) <= tol * tref):
        return True, f"weight tie at the threshold (|diff| {diff.size})"
    # otherwise the two top-closed sets may differ by whole classes only when the
    # smaller one sits on the mass boundary (its mass within tol of p_eff)
    small = sel if sel.size < ref.size else ref
    if abs(float(w[small].sum()) - target) <= tol:
        return True, f"mass tie at p_eff (|diff| {diff.size})"
    return False, "a differing token is neither a weight tie nor a mass tie at the threshold"


def unit_candidates(bufs, u: int):
    """(candidate token ids [m], GPU logits [G, m]) of unit u: the candidate
    pages' positions whose logit is finite (past-the-end slots and tokens a
    sink-window / channel-pruned selection left out are -inf)."""
    ncand = int(bufs.cand_count[u])
    pages = bufs.cand_pages[u, :ncand].cpu().numpy().astype(np.int64)
    pos = (pages[:, None] * 16 + np.arange(16)).reshape(-1)
    z_all = bufs.logits[u, :, : ncand * 16].cpu().numpy()
    valid = np.isfinite(z_all[0])
    return pos[valid], z_all[:, valid]


def check_unit_topp(bufs, u: int, G: int, p: float):
    """The GPU's per-head top-p sets of unit u (logit key >= head_thr) against
    the oracle's fp64 softmax + minimal tie-closed set on the GPU's own logits
    (isolated pruner); the group's final set must be their
    union exactly (pipeline.py:347).  Returns (cand, logits, head sets as
    candidate-local indices, final token ids, [why per head])."""
    cand, z = unit_candidates(bufs, u)
    sels, whys = [], []
    for g in range(G):
        thr = np.uint32(int(bufs.head_thr[u * G + g].item()) & 0xFFFFFFFF)
        sel = np.flatnonzero(f2key_np(z[g]) >= thr)
        ok, why = topp_set_ok(sel, orc.softmax64(z[g]), p)
        assert ok, f"unit {u} head {g}: {why}"
        assert int(bufs.head_stats[u * G + g, 0]) == sel.size
        sels.append(sel)
        whys.append(why)
    final = bufs.final_idx[u, : int(bufs.final_count[u])].cpu().numpy()
    want = orc.union_sorted([cand[s] for s in sels]) if sels else np.zeros(0, np.int64)
    np.testing.assert_array_equal(final, want)
    return cand, z, sels, final, whys
