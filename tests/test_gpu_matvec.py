"""GPU H-matrix x vector block (hx_hmatvec) against the oracle's dense operand, and the
randomized product-error estimator against the exact error (reference behaviour:
hmat_vec / hmat_vec_transpose, pkg/src/hmat/hmatrix.py:138-174)."""

import numpy as np
import pytest

from oracle import hmat_oracle as O
from test_gpu_product import _operands

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["small2d.npz", "cfg1.npz", "ragged3d.npz"])
@pytest.mark.parametrize("s", [1, 5, 64, 70])
def test_hmatvec_parity(golden, name, s):
    from paper_1805_08998_b200.matvec import hmat_matmat

    g = golden(name)
    bct, A, B, oa, ob, tol = _operands(g, name)
    dense = oa.to_dense()
    rng = np.random.default_rng(s)
    X = rng.standard_normal((A.n, s))
    for tr in (False, True):
        Y = hmat_matmat(A, X, transpose=tr)
        ref = (dense.T if tr else dense) @ X
        assert np.linalg.norm(Y - ref) <= 1e-13 * np.linalg.norm(ref), (name, s, tr)


def test_hmat_vec_signature(golden):
    from paper_1805_08998_b200.matvec import hmat_vec, hmat_vec_transpose

    g = golden("small2d.npz")
    bct, A, B, oa, ob, tol = _operands(g, "small2d.npz")
    x = np.random.default_rng(0).standard_normal(A.n)
    d = oa.to_dense()
    assert np.allclose(hmat_vec(A, x), d @ x, rtol=0, atol=1e-12 * np.abs(d @ x).max())
    assert np.allclose(hmat_vec_transpose(A, x), d.T @ x, rtol=0,
                       atol=1e-12 * np.abs(d.T @ x).max())
    with pytest.raises(ValueError):
        hmat_vec(A, np.zeros(A.n + 1))


def test_product_error_estimate(golden):
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200.matvec import product_error

    g = golden("cfg1.npz")
    bct, A, B, oa, ob, tol = _operands(g, "cfg1.npz")
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("dense-svd"), policy=hx.EpsRank(tol))
    C = hx.hmult_new(A, B, cfg)
    exact = oa.to_dense() @ ob.to_dense()
    err = np.linalg.norm(hx.to_dense(C) - exact) / np.linalg.norm(hx.to_dense(C))
    est, cnorm = product_error(C, A, B, probes=32)
    # 32 Gaussian probes: the estimate is within a factor ~1.5 of the true ratio
    assert err / 1.6 <= est <= err * 1.6, (est, err)
    assert abs(cnorm - np.linalg.norm(exact)) <= 0.35 * np.linalg.norm(exact)


def test_estimate_product_error_matches_reference_algorithm(golden):
    """estimate_product_error (multiply.py:266-294) on the GPU against the same algorithm
    on the dense matrices (same seed, same block, same iterations): equal to rounding,
    and a lower bound of the exact ||C - A B||_F that captures most of it."""
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200.matvec import estimate_product_error

    g = golden("cfg1.npz")
    bct, A, B, oa, ob, tol = _operands(g, "cfg1.npz")
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("aca"), policy=hx.EpsRank(tol))
    C = hx.hmult_new(A, B, cfg)
    da, db, dc = oa.to_dense(), ob.to_dense(), hx.to_dense(C)
    est = estimate_product_error(A, B, C, iters=10, block_size=100, seed=0)
    # the reference algorithm on dense operators
    n = dc.shape[0]
    rng = np.random.default_rng(0)
    R = dc - da @ db
    x = np.linalg.qr(rng.standard_normal((n, 100)))[0]
    for _ in range(10):
        y = np.linalg.qr(R @ x)[0]
        x = np.linalg.qr(R.T @ y)[0]
    ref = float(np.sqrt(np.sum(np.linalg.svd(R @ x, compute_uv=False) ** 2)))
    exact = np.linalg.norm(R)
    assert abs(est - ref) <= 1e-6 * ref, (est, ref)
    assert 0 < est <= exact * (1 + 1e-9), (est, exact)
