"""Host planner timing on CPU (no GPU): a BASELINE config's block tree with synthetic
operand ranks (rank grows with the block size like the ACA ranks of the real operands).

usage: HX_PLAN_VERBOSE=1 python tools/plan_bench.py CFG [--reps N]
"""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1805_08998_b200 import _lib, configs  # noqa: E402
from paper_1805_08998_b200.clustering import build_block_cluster_tree, build_cluster_tree  # noqa: E402
from paper_1805_08998_b200.hmatrix import block_arrays, tree_arrays  # noqa: E402


def synthetic_directory(bct, seed=0):
    arr = block_arrays(bct)
    ta = tree_arrays(bct)
    nn = arr.n_nodes
    kind = arr.kind_code
    lo, hi = arr.tree.lo, arr.tree.hi
    m = hi[arr.tau] - lo[arr.tau]
    rng = np.random.default_rng(seed)
    payload = np.where(kind == 1, 1, np.where(kind == 2, 2, 0)).astype(np.int8)
    rank = np.where(kind == 1, np.minimum(m, 10 + 4 * np.log2(np.maximum(m, 1) / 64.0)
                                          + rng.integers(0, 6, nn)), 0).astype(np.int32)
    u = np.zeros(nn, np.int64)
    v = np.zeros(nn, np.int64)
    d = np.zeros(nn, np.int64)
    tot = np.zeros(1, np.int64)
    tb = _lib.TreeBuf(ta)
    import ctypes as C
    _lib.check(_lib.lib().hx_operand_layout(C.byref(tb.st), _lib.ptr(payload, _lib.i8p),
                                            _lib.ptr(rank, _lib.i32p), _lib.ptr(u, _lib.i64p),
                                            _lib.ptr(v, _lib.i64p), _lib.ptr(d, _lib.i64p),
                                            _lib.ptr(tot, _lib.i64p)), "layout")
    return ta, dict(payload=payload, rank=rank, u_off=u, v_off=v, d_off=d)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fill", action="store_true", help="also fill every batch")
    ap.add_argument("--eager", action="store_true", help="fill the batches in the plan call")
    ap.add_argument("--sizes", action="store_true", help="materialization flops by leaf size")
    ap.add_argument("--chunk", type=int, default=-1, help="plan only this chunk of 3")
    ap.add_argument("--implicit", type=int, default=512, help="implicit-route threshold (0: off)")
    a = ap.parse_args()
    c = configs.CONFIGS[a.cfg]
    t0 = time.time()
    pts = configs.make_points(c)
    bct = build_block_cluster_tree(build_cluster_tree(pts, c["n_min"]), c["eta"])
    ta, d = synthetic_directory(bct)
    print(f"tree {time.time() - t0:.1f}s nodes {bct.n_nodes}", flush=True)
    mask = None
    if a.chunk >= 0:
        from paper_1805_08998_b200 import multiply
        groups = multiply.chunk_groups(bct, 3, first=0.5)
        mask = multiply.group_mask(bct, groups[a.chunk])
    for _ in range(a.reps):
        t0 = time.perf_counter()
        from paper_1805_08998_b200 import multiply as _m
        p = _lib.Plan(ta, d, d, mask, 64, flags=(0 if a.eager else _lib.Plan.DEFER) |
                      _m.implicit_flags(a.implicit))
        t1 = time.perf_counter()
        msg = f"plan {1e3 * (t1 - t0):.1f} ms"
        if a.fill:
            mma = np.zeros(6)
            _lib.check(_lib.lib().hx_plan_mma_flops(p.h, _lib.ptr(mma, _lib.f64p)), "fill")
            msg += f" + fill/count {1e3 * (time.perf_counter() - t1):.1f} ms"
        print(msg, "terms", p.info.n_terms_real, p.info.n_terms_expand, flush=True)
        if a.sizes:
            lv = p.leaves()
            for kind in (1, 2):
                sel = lv["kind"] == kind
                m, n, K, fdd = lv["m"][sel], lv["n"][sel], lv["K"][sel], lv["fdd"][sel]
                for s in np.unique(m):
                    q = m == s
                    mat = (2.0 * m[q] * n[q] * K[q] + fdd[q]).sum()
                    print(f"  {'far' if kind == 1 else 'near'} {s:5d}: {q.sum():6d} leaves "
                          f"K mean {K[q].mean():7.1f} mat {mat / 1e9:8.1f} GF")
            a.sizes = False
        p.close()


if __name__ == "__main__":
    main()
