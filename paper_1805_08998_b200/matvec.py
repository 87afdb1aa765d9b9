"""H-matrix times vectors on the GPU, and the product-error estimator built on it.

``hmat_vec`` / ``hmat_vec_transpose`` keep the reference signatures
(``pkg/src/hmat/hmatrix.py:138-174``: tree-ordered vector of length n in, same out);
``hmat_matmat`` takes an (n, s) block of vectors (``_node_matmat``, hmatrix.py:177-211, at
the root).  All arithmetic is ``hx_hmatvec`` in ``libhx.so``: the stacked cores
V_l^T X[sigma_l] and the row bands of Y as two grouped-GEMM launches.

``product_error`` estimates ||C - A B||_F / ||C||_F with s Gaussian probes,
||M X||_F^2 / s being an unbiased estimate of ||M||_F^2: it is how products too large to
materialize (BASELINE configs 3-5) are checked.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .hmatrix import tree_arrays
from .multiply import Device, _host_directory, operand_directory


def _attach(h, dev, slot, device):
    res = getattr(h, "_hx_device", None)
    if res is not None and res[0] == device:
        _, d = operand_directory(h)
        dev.set_operand(slot, dev_ptr=res[1], n=res[2])
    else:
        pool, d = _host_directory(h)
        try:
            dev.set_operand(slot, pool=pool)
        except MemoryError:  # the last product's workspace still holds the device
            _lib.check(_lib.lib().hx_ctx_trim(dev.h), "hx_ctx_trim")
            aux = Device._aux.get(device)
            if aux is not None:
                _lib.check(_lib.lib().hx_ctx_trim(aux.h), "hx_ctx_trim")
            dev.set_operand(slot, pool=pool)
    return d


def hmat_matmat(h, x, transpose=False, device=0):
    """H @ x (or H.T @ x) for x of shape (n,) or (n, s), tree ordering."""
    x = np.asarray(x, dtype=np.float64)
    vec = x.ndim == 1
    X = np.asfortranarray(x.reshape(h.n, -1))
    if X.shape[0] != h.n:
        raise ValueError(f"expected {h.n} rows, got {x.shape}")
    s = X.shape[1]
    Y = np.zeros((h.n, s), order="F")
    with Device.lock(device):
        dev = Device.get(device)
        d = _attach(h, dev, 0, device)
        tb = _lib.TreeBuf(tree_arrays(h.bct))
        ob = _lib.OperandBuf(d)
        _lib.check(_lib.lib().hx_hmatvec(dev.h, C.byref(tb.st), C.byref(ob.st), 0,
                                         int(bool(transpose)), _lib.ptr(X, _lib.f64p),
                                         _lib.ptr(Y, _lib.f64p), s), "hx_hmatvec")
    return Y[:, 0].copy() if vec else Y


def hmat_vec(h, x, device=0):
    x = np.asarray(x, dtype=float)
    if x.shape != (h.n,):
        raise ValueError(f"expected vector of length {h.n}, got {x.shape}")
    return hmat_matmat(h, x, False, device)


def hmat_vec_transpose(h, x, device=0):
    x = np.asarray(x, dtype=float)
    if x.shape != (h.n,):
        raise ValueError(f"expected vector of length {h.n}, got {x.shape}")
    return hmat_matmat(h, x, True, device)


def product_error(c, a, b, probes=8, seed=0, device=0):
    """Randomized estimate of ||C - A B||_F / ||C||_F (and ||C||_F) from `probes`
    Gaussian vectors: C X against A (B X)."""
    rng = np.random.default_rng(seed)
    X = np.asfortranarray(rng.standard_normal((c.n, probes)))
    cx = hmat_matmat(c, X, device=device)
    abx = hmat_matmat(a, hmat_matmat(b, X, device=device), device=device)
    num = np.linalg.norm(cx - abx)
    den = np.linalg.norm(cx)
    return float(num / den), float(den / np.sqrt(probes))


def estimate_product_error(h, k, l, iters=10, block_size=100, seed=0, device=0):
    """Frobenius estimate of ||L - H K|| by block subspace iteration: the reference's
    ``estimate_product_error`` (``multiply.py:266-294``, same signature and defaults).

    Two-sided subspace iteration on the residual operator x -> L x - H (K x): start from
    the Q factor of an n x b Gaussian block (``default_rng(seed)``), then ``iters`` rounds
    of y = qr(R x), x = qr(R^T y); the value is the root of the summed squared singular
    values of R x (a lower bound of ||R||_F that sharpens with b).  Every H-matrix x block
    product runs on the GPU (``hmat_matmat``); the thin QRs and the final SVD of the
    n x b blocks stay on the host, as in the reference."""
    n = l.n
    b = min(block_size, n)
    rng = np.random.default_rng(seed)

    def resid(x):
        return hmat_matmat(l, x, device=device) - hmat_matmat(
            h, hmat_matmat(k, x, device=device), device=device)

    def resid_t(x):
        return hmat_matmat(l, x, True, device) - hmat_matmat(
            k, hmat_matmat(h, x, True, device), True, device)

    x = np.linalg.qr(rng.standard_normal((n, b)))[0]
    for _ in range(iters):
        y = np.linalg.qr(resid(x))[0]
        x = np.linalg.qr(resid_t(y))[0]
    ritz = np.linalg.svd(resid(x), compute_uv=False)
    return float(np.sqrt(np.sum(ritz ** 2)))
