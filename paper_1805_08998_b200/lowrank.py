"""Low-rank factor pairs and truncation policies (API of ``hmat.lowrank``).

``LowRank(left, right)`` represents ``left @ right.T`` (``lowrank.py:15-43``); rank 0 is a
first-class value.  ``EpsRank`` / ``FixedRank`` are the truncation policies the product
accepts (``lowrank.py:57-72``) and ``select_rank`` is the relative-Frobenius-tail rule
(``lowrank.py:75-90``) that the GPU recompression kernel applies per far block.  These are
host-side value types; no arithmetic of the product runs here.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class LowRank:
    left: np.ndarray   # (m, k)
    right: np.ndarray  # (n, k)
    degraded: bool = field(default=False, compare=False)

    def __post_init__(self):
        if self.left.ndim != 2 or self.right.ndim != 2:
            raise ValueError("factors must be 2-d")
        if self.left.shape[1] != self.right.shape[1]:
            raise ValueError("factor ranks differ")

    @property
    def shape(self):
        return (self.left.shape[0], self.right.shape[0])

    @property
    def rank(self):
        return self.left.shape[1]

    def to_dense(self):
        return self.left @ self.right.T

    def norm(self):
        if self.rank == 0:
            return 0.0
        gram = (self.left.T @ self.left) @ (self.right.T @ self.right)
        return float(np.sqrt(max(np.trace(gram), 0.0)))


def zero_lowrank(m, n):
    return LowRank(np.zeros((m, 0)), np.zeros((n, 0)))


@dataclass(frozen=True)
class FixedRank:
    k_max: int

    def __post_init__(self):
        if self.k_max < 1:
            raise ValueError("k_max must be >= 1")


@dataclass(frozen=True)
class EpsRank:
    eps: float

    def __post_init__(self):
        if not self.eps > 0.0:
            raise ValueError("eps must be positive")


def select_rank(s, policy):
    """Leading singular values kept: smallest r with ||s[r:]|| <= eps ||s|| (EpsRank), or
    min(len(s), k_max) (FixedRank)."""
    s = np.asarray(s, dtype=float)
    if isinstance(policy, FixedRank) or hasattr(policy, "k_max"):
        return min(len(s), int(policy.k_max))
    if isinstance(policy, EpsRank) or hasattr(policy, "eps"):
        if s.size == 0:
            return 0
        tails = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]
        ok = np.flatnonzero(tails <= policy.eps * tails[0])
        return int(ok[0]) if ok.size else int(s.size)
    raise TypeError(f"unknown truncation policy {policy!r}")
