"""GPU operand assembly (ACA on kernel entries) against the oracle assembly, which is
itself pinned to the reference (tests/test_oracle_golden.py)."""

import numpy as np
import pytest

from oracle import hmat_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kern", [("small2d.npz", "exp"), ("cfg1.npz", "exp")])
def test_assembly_matches_oracle(golden, name, kern):
    import paper_1805_08998_b200 as hx

    g = golden(name)
    n, n_min, eta, eps_a, tol = g["params"]
    pts = g["points"]
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, int(n_min)), eta)
    A = hx.assemble_hmatrix(kern, bct, hx.EpsRank(eps_a), pts)
    ranks_ref = g["A/ranks"]
    ids = g["A/ids"]
    diffs = []
    for b, r in zip(ids, ranks_ref):
        p = A.data[int(b)]
        if r >= 0:
            assert hasattr(p, "left"), b
            diffs.append(p.rank - r)
    diffs = np.array(diffs)
    assert np.all(np.abs(diffs) <= 2)
    assert np.mean(diffs == 0) >= 0.9
    # approximation quality against the exact kernel matrix (tree ordering)
    perm = bct.tree.permutation
    K = O.kernel_matrix(kern, pts[perm], pts[perm])
    err = np.linalg.norm(hx.to_dense(A) - K) / np.linalg.norm(K)
    assert err <= 10 * eps_a, err
    assert not A.degraded


def test_assembled_operands_feed_product(golden):
    import paper_1805_08998_b200 as hx

    g = golden("small2d.npz")
    n, n_min, eta, eps_a, tol = g["params"]
    pts = g["points"]
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, int(n_min)), eta)
    A = hx.assemble_hmatrix("exp", bct, hx.EpsRank(eps_a), pts)
    C = hx.hmult_new(A, A, hx.MultiplyConfig(compressor=hx.CompressorKind("dense-svd"),
                                             policy=hx.EpsRank(tol)))
    da = hx.to_dense(A)
    exact = da @ da
    err = np.linalg.norm(hx.to_dense(C) - exact) / np.linalg.norm(exact)
    assert err <= tol
