"""Compression-scheme selection (API of ``hmat.compressors.CompressorKind``).

The reference compresses each far output block with one matrix-free scheme chosen by
``CompressorKind.tag`` (``compressors.py:122-141``, dispatch ``:441-452``).  The tag selects
the GPU route of ``hx_product`` (``include/hx.h``, ``csrc/iterative.cuh``):

* ``aca``        partially pivoted ACA on the block's implicit sum (rows / columns of the
                 stacked terms, or of the materialized tile), two-hit stop, then the exact
                 ``truncate(eps / 2)`` (compressors.py:162-247);
* ``bilanczos``  Golub-Kahan-Lanczos with two-pass CGS reorthogonalisation, breakdown
                 probes and the core SVD (:271-365), start vectors from the per-block numpy
                 stream ``default_rng((seed << 24) ^ id)`` (multiply.py:61-63);
* ``randomized`` the vector-at-a-time range finder with the two-hit stop, or with a
                 FixedRank policy the blocked finder with ``q`` subspace iterations
                 (:368-428), same per-block streams;
* ``dense-svd``  the best approximation (sketch + QR + Jacobi SVD certified against the
                 exact tail; :431-438).
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
