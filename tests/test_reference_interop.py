"""The drop-in boundary on CPU: the reference's error paths with the same exception types
and messages, the packed-pool cache following mutations of ``HMatrix.data``, and real
reference ``hmat`` objects (``BlockClusterTree`` / ``HMatrix``) packed and planned by the
library.  The reference itself is imported only when ``/root/reference`` exists (this
build container); those tests skip elsewhere."""

import os
import sys
import warnings

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
needs_ref = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import hmat  # noqa: F401
    from hmat import clustering, compressors, hmatrix, lowrank, multiply
    return clustering, compressors, hmatrix, lowrank, multiply


def _err(fn):
    try:
        fn()
    except Exception as exc:  # noqa: BLE001 - compared below
        return type(exc).__name__, str(exc)
    return None


@needs_ref
def test_config_validation_matches_reference():
    """MultiplyConfig (multiply.py:41-47), CompressorKind (compressors.py:137-141), EpsRank /
    FixedRank (lowrank.py:61-72): same exception class and message for each bad input."""
    _, rcomp, _, rlow, rmul = _ref()
    import paper_1805_08998_b200 as hx

    cases = [
        (lambda m: m[0].MultiplyConfig(mode="bogus", policy=m[1].EpsRank(1e-6))),
        (lambda m: m[0].MultiplyConfig(converter="svd", policy=m[1].EpsRank(1e-6))),
        (lambda m: m[0].MultiplyConfig()),
        (lambda m: m[2].CompressorKind("qr")),
        (lambda m: m[2].CompressorKind("randomized", q=-1)),
        (lambda m: m[1].EpsRank(0.0)),
        (lambda m: m[1].EpsRank(-1e-3)),
        (lambda m: m[1].FixedRank(0)),
    ]
    ref = (rmul, rlow, rcomp)
    ours = (hx, hx, hx)
    for case in cases:
        r = _err(lambda: case(ref))
        o = _err(lambda: case(ours))
        assert r is not None and r == o, (r, o)
    # valid configs construct in both
    assert hx.MultiplyConfig(mode="traditional", policy=hx.FixedRank(3)).mode == "traditional"


def test_hmult_new_rejects_other_modes_and_trees():
    """hmult_new: mode != 'new' -> ValueError (multiply.py:254-255); operands on different
    block trees -> ValueError (sumexpr.py:80-81).  Both raise before any device work."""
    import paper_1805_08998_b200 as hx

    rng = np.random.default_rng(0)
    pts = rng.uniform(0, 1, (64, 2))
    b1 = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, 16), 0.8)
    b2 = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, 16), 0.8)
    h1, h2 = hx.HMatrix(b1, {}), hx.HMatrix(b2, {})
    cfg_t = hx.MultiplyConfig(mode="traditional", policy=hx.EpsRank(1e-6))
    with pytest.raises(ValueError, match="config mode must be 'new'"):
        hx.hmult_new(h1, h1, cfg_t)
    cfg = hx.MultiplyConfig(policy=hx.EpsRank(1e-6))
    with pytest.raises(ValueError, match="factors must live on the same block-cluster tree"):
        hx.hmult_new(h1, h2, cfg)


def test_hmult_traditional_checks():
    """multiply.py:259-263's config check; the matrix-free pair converters are not built
    and say so (before any device work)."""
    import paper_1805_08998_b200 as hx

    rng = np.random.default_rng(0)
    pts = rng.uniform(0, 1, (64, 2))
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, 16), 0.8)
    h = hx.HMatrix(bct, {})
    with pytest.raises(ValueError, match="config mode must be 'traditional'"):
        hx.hmult_traditional(h, h, hx.MultiplyConfig(policy=hx.EpsRank(1e-6)))
    for conv in ("aca", "bilanczos", "randomized"):
        with pytest.raises(NotImplementedError, match="not built"):
            hx.hmult_traditional(h, h, hx.MultiplyConfig(mode="traditional", converter=conv,
                                                         policy=hx.EpsRank(1e-6)))


def test_tiny_eps_warns_and_clamps():
    """compressors.py:144-149: eps <= machine epsilon -> UserWarning, clamp to 1e-15."""
    from paper_1805_08998_b200.compressors import EPS_FLOOR, clamp_eps

    with pytest.warns(UserWarning, match="below machine precision"):
        assert clamp_eps(1e-17) == EPS_FLOOR
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        assert clamp_eps(1e-6) == 1e-6


@needs_ref
def test_tiny_eps_warning_text_matches_reference():
    _, rcomp, _, _, _ = _ref()
    from paper_1805_08998_b200.compressors import clamp_eps

    with pytest.warns(UserWarning) as wr:
        rcomp._clamp_eps(2e-16)
    with pytest.warns(UserWarning) as wo:
        clamp_eps(2e-16)
    assert str(wr[0].message) == str(wo[0].message)


def test_packed_pool_follows_data_mutations():
    """The packed operand cached on an HMatrix is dropped when its payloads change
    (assignment, deletion, replacing .data), and the lazy leaf dicts answer get / copy like
    indexing."""
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import multiply
    from paper_1805_08998_b200.hmatrix import LeafDict, _PoolLeaves, pack_operand

    rng = np.random.default_rng(1)
    pts = rng.uniform(0, 1, (512, 2))
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, 16), 0.8)
    arr = hx.hmatrix.block_arrays(bct)
    lo, hi = arr.tree.lo, arr.tree.hi
    data = {}
    for b in np.flatnonzero(arr.kind_code != 0):
        m = int(hi[arr.tau[b]] - lo[arr.tau[b]])
        n = int(hi[arr.sigma[b]] - lo[arr.sigma[b]])
        if arr.kind_code[b] == 1:
            data[int(b)] = hx.LowRank(rng.standard_normal((m, 2)), rng.standard_normal((n, 2)))
        else:
            data[int(b)] = rng.standard_normal((m, n))
    H = hx.HMatrix(bct, data)
    assert isinstance(H.data, LeafDict)
    pool1, d1 = multiply.operand_directory(H)
    assert multiply.operand_directory(H)[0] is pool1  # cached
    far = next(b for b, p in H.data.items() if hasattr(p, "left"))
    H.data[far] = hx.LowRank(H.data[far].left * 2.0, H.data[far].right)
    pool2, _ = multiply.operand_directory(H)
    assert pool2 is not pool1
    assert np.array_equal(pool2, pack_operand(H)[0])
    assert not np.array_equal(pool1, pool2)
    H.data = dict(H.data)  # replaced wholesale
    assert multiply.operand_directory(H)[0] is not pool2
    # a loaded-style lazy dict: get / copy / contains see unpacked entries
    L = hx.HMatrix(bct, {})
    L._hx_packed = (pool2, d1)  # noqa: SLF001
    L.data = _PoolLeaves(L)
    L._hx_packed = (pool2, d1)
    assert L.data.get(far) is not None
    assert far in L.data and len(L.data.copy()) == len(data)
    assert np.allclose(L.data.get(far).left, 2.0 * data[far].left)
    assert L.data.get(-5, "none") == "none"


@needs_ref
def test_reference_objects_pack_and_plan():
    """Real reference objects: a reference BlockClusterTree and a reference-assembled
    HMatrix (reference aca on point-kernel blocks, the survey's PanelSet adapter) are
    packed by pack_operand and planned by hx_plan_create; the planner's restrict log
    equals the oracle's on the same payloads."""
    rclu, rcomp, rhm, rlow, _ = _ref()
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden import assemble  # the committed point-kernel adapter
    from hmat import geometry
    from oracle import hmat_oracle as O
    from paper_1805_08998_b200 import _lib, hmatrix, multiply

    rng = np.random.default_rng(5)
    pts = rng.uniform(0, 1, (256, 2))
    ps = geometry.PanelSet(centers=pts, areas=np.ones(len(pts)), corners=None, level=0)
    bct = rclu.build_block_cluster_tree(rclu.build_cluster_tree(ps, 16), 0.8)
    H = assemble("exp", bct, 1e-8, pts)
    pool, d = hmatrix.pack_operand(H)
    plan = _lib.Plan(hmatrix.tree_arrays(bct), d, d, tile=multiply.plan_tile(bct),
                     flags=_lib.Plan.LOG)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, 16), 0.8)
    data = {b: (O.LR(p.left, p.right) if hasattr(p, "left") else p) for b, p in H.data.items()}
    log = []
    O.hmult_new_o(O.HMatO(obt, data), O.HMatO(obt, data), O.Eps(1e-6), "dense-svd", log=log)
    kmap = {"FF": 0, "FX": 1, "XF": 2}
    ref = np.array([(c, kmap[k], a, b, r) for (c, k, a, b, r) in log], dtype=np.int64)
    L = plan.term_log()
    mine = np.stack([L["block"], L["kind"], L["a"], L["b"], L["rank"]], axis=1)
    assert len(ref) > 0 and np.array_equal(mine, ref)
    assert plan.info.n_far == sum(1 for x in bct.leaves if x.kind == rclu.FAR)
    plan.close()
