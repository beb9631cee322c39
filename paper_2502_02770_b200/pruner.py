"""Top-p pruning with the reference signatures (nucleuskv/pruner.py).

``binary_search_top_p`` runs Algorithm 1 literally on the GPU
(tw_topp_bisect: the same bracket updates and break rules, so thresholds and
iteration counts follow the reference, any epsilon / max_iters).  The decode
hot path uses the equivalent direct characterisation of the converged search
(minimal tie-closed top set, tw_topp) instead -- see csrc/topp.cu.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib as L
from .attention import TokenSelection

__all__ = ["BinarySearchConfig", "PruneOutcome", "binary_search_top_p", "prune"]

_NORMALIZATION_TOLERANCE = 1e-4  # pruner.py:30


@dataclass(frozen=True)
class BinarySearchConfig:
    """pruner.py:24-45."""
    p: float
    epsilon: float = 1e-15
    max_iters: int = 64

    def __post_init__(self) -> None:
        if not 0.0 <= self.p <= 1.0:
            raise ValueError(f"p={self.p} outside [0, 1]")
        if not self.epsilon > 0.0:
            raise ValueError("epsilon must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")


@dataclass(frozen=True, eq=False)
class PruneOutcome:
    selection: TokenSelection
    threshold: float
    iterations: int


def binary_search_top_p(weights, cfg: BinarySearchConfig) -> PruneOutcome:
    """Smallest tie-closed top-weight set reaching cfg.p (pruner.py:57-114)."""
    w = torch.as_tensor(weights)
    if not w.is_cuda:
        raise ValueError("weights must be a CUDA tensor (the Twilight path has no CPU fallback)")
    w = w.to(torch.float64).contiguous()
    if w.ndim != 1 or w.numel() == 0:
        raise ValueError("weights must be a non-empty 1-D array")
    if bool((w < 0).any()) or not bool(torch.isfinite(w).all()):
        raise ValueError("weights must be finite and non-negative")
    total = float(w.sum())
    if abs(total - 1.0) > _NORMALIZATION_TOLERANCE:
        raise ValueError(f"weights are not normalized (mass {total:.6f}); restrict and renormalize before pruning")
    n = w.numel()
    mask = torch.empty(n, dtype=torch.uint8, device=w.device)
    thr = torch.empty(1, dtype=torch.float64, device=w.device)
    its = torch.empty(1, dtype=torch.int32, device=w.device)
    L.check(L.lib().tw_topp_bisect(L.ptr(w), 1, n, float(cfg.p), float(cfg.epsilon), int(cfg.max_iters),
                                   L.ptr(mask), L.ptr(thr), L.ptr(its), L.stream_handle()), "tw_topp_bisect")
    sel = TokenSelection.from_indices(torch.nonzero(mask, as_tuple=True)[0], n, weights=w)
    return PruneOutcome(selection=sel, threshold=float(thr.item()), iterations=int(its.item()))


def prune(weights_estimate, candidates: TokenSelection, cfg: BinarySearchConfig) -> PruneOutcome:
    """Search over the candidate-restricted renormalised weights (pruner.py:117-147)."""
    w = torch.as_tensor(weights_estimate).to(torch.float64)
    if candidates.n != w.shape[0]:
        raise ValueError("candidate set built for a different context size")
    if len(candidates) == 0:
        raise ValueError("cannot prune an empty candidate set")
    sub = w[candidates.indices]
    mass = float(sub.sum())
    if not mass > 0.0:
        raise ValueError("candidate set carries no weight")
    out = binary_search_top_p(sub / mass, cfg)
    glob = candidates.indices[out.selection.indices]
    sel = TokenSelection(indices=glob, n=w.shape[0], attained_mass=out.selection.attained_mass)
    return PruneOutcome(selection=sel, threshold=out.threshold, iterations=out.iterations)
