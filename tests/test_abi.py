"""CPU checks of the C-ABI library: it loads, exports every symbol of include/hx.h, and
the planner (pure host code) reproduces the reference's restrict term log."""

import os
import re

import numpy as np
import pytest

from oracle import hmat_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "hx.h")).read()
    return sorted(set(re.findall(r"\b(hx_[a-z_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1805_08998_b200 import _lib

    L = _lib.lib()
    names = _declared()
    assert "hx_product" in names and "hx_plan_create" in names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.hx_version() == 1


def _plan_case(g, n_min_tile=None):
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import _lib, hmatrix, multiply

    n, n_min, eta, eps_a, tol = g["params"]
    pts = g["points"]
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, int(n_min)), eta)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, int(n_min)), eta)
    A = O.assemble_o("exp", obt, O.Eps(eps_a), pts)
    H = hx.HMatrix(bct, A.data)
    pool, d = hmatrix.pack_operand(H)
    plan = _lib.Plan(hmatrix.tree_arrays(bct), d, d, tile=multiply.plan_tile(bct),
                     flags=_lib.Plan.LOG)
    return bct, A, plan, tol


@pytest.mark.parametrize("name", ["small2d.npz", pytest.param("cfg1.npz", marks=pytest.mark.slow)])
def test_plan_term_log_matches_restrict(golden, name):
    g = golden(name)
    bct, A, plan, tol = _plan_case(g)
    log = []
    O.hmult_new_o(A, A, O.Eps(tol), "dense-svd", log=log)
    kmap = {"FF": 0, "FX": 1, "XF": 2}
    ref = np.array([(c, kmap[k], a, b, r) for (c, k, a, b, r) in log], dtype=np.int64)
    L = plan.term_log()
    mine = np.stack([L["block"], L["kind"], L["a"], L["b"], L["rank"]], axis=1)
    assert mine.shape == ref.shape
    assert np.array_equal(mine, ref)
    info = plan.info
    assert info.n_far == int(np.sum(bct.kind_code == 1))
    assert info.n_near == int(np.sum(bct.kind_code == 2))


def test_plan_canonical_model_cfg1(golden):
    # cfg1 term formation 1.98 GFLOP / 1.29 GB, near 1.73 GFLOP / 0.44 GB
    bct, A, plan, tol = _plan_case(golden("cfg1.npz"))
    info = plan.info
    assert abs(info.flops_form / 1e9 - 1.98) < 0.01
    assert abs(info.bytes_form / 1e9 - 1.29) < 0.01
    assert abs(info.flops_near / 1e9 - 1.73) < 0.01
    assert abs(info.bytes_near / 1e9 - 0.44) < 0.01


def test_plan_rejects_bad_arguments():
    from paper_1805_08998_b200 import _lib

    import ctypes as C
    h = C.c_void_p()
    rc = _lib.lib().hx_plan_create(None, None, None, None, 64, 0, C.byref(h))
    assert rc == -1
    assert "null" in _lib.last_error()



def test_plan_term_log_ragged_tree(golden):
    """Ragged cluster tree (n = 200, leaves at different depths), A != B: the planner's log
    equals the reference's restrict log; dense sub-view and H-block x dense pairs are
    planned (no NotImplementedError)."""
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import _lib, hmatrix, multiply

    g = golden("ragged3d.npz")
    n, n_min, eta, eps_a, tol = g["params"]
    pts = g["points"]
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, int(n_min)), eta)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, int(n_min)), eta)
    h = int(n) ** (-1.0 / 3.0)
    oa = O.assemble_o("exp0.5", obt, O.Eps(eps_a), pts, h)
    ob = O.assemble_o("inv", obt, O.Eps(eps_a), pts, h)
    _, da = hmatrix.pack_operand(hx.HMatrix(bct, oa.data))
    _, db = hmatrix.pack_operand(hx.HMatrix(bct, ob.data))
    plan = _lib.Plan(hmatrix.tree_arrays(bct), da, db, tile=multiply.plan_tile(bct),
                     flags=_lib.Plan.LOG)
    log = []
    O.hmult_new_o(oa, ob, O.Eps(float(tol)), "dense-svd", log=log)
    kmap = {"FF": 0, "FX": 1, "XF": 2}
    ref = np.array([(c, kmap[k], a, b, r) for (c, k, a, b, r) in log], dtype=np.int64)
    L = plan.term_log()
    mine = np.stack([L["block"], L["kind"], L["a"], L["b"], L["rank"]], axis=1)
    assert mine.shape == ref.shape
    assert np.array_equal(mine, ref)
    assert plan.info.n_dxd > 0


def test_plan_implicit_route_block_sparse_tsub(golden):
    """Implicit route (HX_PLAN_IMPLICIT): the restrict log does not depend on the route, and
    the materialized part of an implicit leaf is the set of its small sub-block terms' dense
    blocks (block-sparse T_sub), never a leaf-sized buffer: the tile workspace can only
    shrink against the fully materialized plan."""
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import _lib, hmatrix, multiply

    g = golden("small2d.npz")
    n, n_min, eta, eps_a, tol = g["params"]
    pts = g["points"]
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, int(n_min)), eta)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, int(n_min)), eta)
    A = O.assemble_o("exp", obt, O.Eps(eps_a), pts)
    pool, d = hmatrix.pack_operand(hx.HMatrix(bct, A.data))
    ta = hmatrix.tree_arrays(bct)
    tile = multiply.plan_tile(bct)
    dense = _lib.Plan(ta, d, d, tile=tile, flags=_lib.Plan.LOG)
    logs = dense.term_log()
    for impl in (32, 64):
        p = _lib.Plan(ta, d, d, tile=tile, flags=_lib.Plan.LOG | multiply.implicit_flags(impl))
        lg = p.term_log()
        for k in ("block", "kind", "a", "b", "rank"):
            assert np.array_equal(lg[k], logs[k])
        assert p.info.n_far == dense.info.n_far and p.info.n_near == dense.info.n_near
        assert p.info.mat_terms == dense.info.mat_terms
        assert p.info.tile_elems <= dense.info.tile_elems
        lv, lvd = p.leaves(), dense.leaves()
        assert np.array_equal(lv["ids"], lvd["ids"]) and np.array_equal(lv["K"], lvd["K"])
        p.close()
    dense.close()
