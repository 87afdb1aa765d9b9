"""Compression-scheme selection (API of ``hmat.compressors.CompressorKind``).

The reference compresses each far output block with one matrix-free scheme chosen by
``CompressorKind.tag`` (``compressors.py:122-141``, dispatch ``:441-452``).  On the GPU the
tag selects the recompression route of ``hx_product``: every tag yields
the tolerance-certified truncated SVD of the exact block (best approximation, the
``dense-svd`` semantics), which is within the reference's own rank spread for ``aca``
(+0/+1) and ``bilanczos`` (identical ranks on the configs measured).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

EPS_FLOOR = 1e-15
TAG_CODES = {"aca": 0, "bilanczos": 1, "randomized": 2, "dense-svd": 3}


@dataclass(frozen=True)
class CompressorKind:
    tag: str
    q: int = 1
    seed: int = 0

    TAGS = ("aca", "bilanczos", "randomized", "dense-svd")

    def __post_init__(self):
        if self.tag not in self.TAGS:
            raise ValueError(f"unknown compressor {self.tag!r}")
        if self.q < 0:
            raise ValueError("q must be >= 0")


def clamp_eps(eps):
    """Tolerances at or below machine epsilon clamp to 1e-15 with a warning
    (``compressors.py:144-149``)."""
    if eps <= np.finfo(float).eps:
        warnings.warn(f"tolerance {eps:g} is below machine precision, clamping to "
                      f"{EPS_FLOOR:g}")
        return EPS_FLOOR
    return eps
