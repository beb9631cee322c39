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


def topp_set_ok(sel: np.ndarray, w: np.ndarray, p: float, tol: float = MASS_TOL) -> tuple[bool, str]:
    """Is `sel` (indices into w) the reference's top-p set up to threshold ties?

    Exact equality with the oracle's converged search passes outright.  Else
    the set must be top-closed (nothing heavier than its lightest member by
    more than `tol` relative is left out), reach p_eff - tol, and be minimal:
    dropping its lightest class (within `tol`) must fall below p_eff + tol.
    """
    ref = orc.minimal_tie_closed_top_p(w, p)
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
    return True, f"tie-tolerant match (|diff| {np.setxor1d(sel, ref).size})"
