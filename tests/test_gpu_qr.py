"""Kernel-level parity of the batched Householder QR of the recompression (register, warp
and CTA kernels, and the TSQR route for panels taller than 256 rows) against NumPy fp64.

Contract (the QR feeds the rank-revealing SVD, which only needs an orthonormal basis of
range(X) and X = Q R): ||Q^T Q - I|| and ||Q R - X|| / ||X|| at the 1e-13 level, R upper
triangular and |R| equal to NumPy's up to column signs on full-rank panels; rank-deficient
sketches (the usual case: sketch wider than the block's rank) keep Q orthonormal.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(panels):
    from paper_1805_08998_b200 import _lib
    p = np.array([x.shape[0] for x in panels], np.int32)
    q = np.array([x.shape[1] for x in panels], np.int32)
    X = np.concatenate([x.T.ravel() for x in panels]).astype(np.float64)
    R = np.zeros(int((q.astype(np.int64) ** 2).sum()))
    _lib.check(_lib.lib().hx_debug_qr(len(panels), _lib.ptr(p, _lib.i32p), _lib.ptr(q, _lib.i32p),
                                      _lib.ptr(X, _lib.f64p), _lib.ptr(R, _lib.f64p)), "hx_debug_qr")
    out, ox, orr = [], 0, 0
    for pi, qi in zip(p, q):
        Q = X[ox:ox + pi * qi].reshape(qi, pi).T
        Rm = R[orr:orr + qi * qi].reshape(qi, qi).T
        out.append((Q, Rm))
        ox += pi * qi
        orr += qi * qi
    return out


SHAPES = [(64, 16), (200, 32), (256, 48), (257, 16), (300, 40), (512, 24), (1000, 56),
          (1024, 48), (4096, 32), (5000, 64), (65536, 16), (20000, 8), (700, 96), (3000, 1)]


def test_qr_shapes_against_numpy():
    rng = np.random.default_rng(7)
    panels = [rng.standard_normal(s) for s in SHAPES]
    for X, (Q, R) in zip(panels, _run(panels)):
        q = X.shape[1]
        assert np.allclose(np.triu(R), R, atol=0), X.shape
        assert np.linalg.norm(Q.T @ Q - np.eye(q)) < 1e-13 * q, X.shape
        assert np.linalg.norm(Q @ R - X) <= 1e-13 * np.linalg.norm(X), X.shape
        Rn = np.linalg.qr(X, mode="r")
        assert np.allclose(np.abs(np.diag(R)), np.abs(np.diag(Rn)), rtol=1e-10), X.shape


def test_rank_deficient_tall_sketches():
    """Y = T Omega with rank(T) < q: Householder (and TSQR) keep Q orthonormal."""
    rng = np.random.default_rng(8)
    panels = []
    for m, q, r in [(4096, 48, 3), (65536, 16, 2), (1500, 40, 0), (800, 32, 31)]:
        T = rng.standard_normal((m, r)) @ rng.standard_normal((r, q)) if r else np.zeros((m, q))
        panels.append(T)
    for X, (Q, R) in zip(panels, _run(panels)):
        q = X.shape[1]
        assert np.linalg.norm(Q.T @ Q - np.eye(q)) < 1e-12 * q, X.shape
        assert np.linalg.norm(Q @ R - X) <= 1e-13 * max(np.linalg.norm(X), 1e-300) + 1e-300
