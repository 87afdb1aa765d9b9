"""Probe: GPU-assembled BASELINE config -> GPU product, timings, exact global error.

usage: python tools/probe.py CFG [--steps N] [--tag TAG] [--check]
"""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1805_08998_b200 as hx  # noqa: E402
from paper_1805_08998_b200 import configs  # noqa: E402


def dense_on_gpu(H, torch):
    from paper_1805_08998_b200.hmatrix import block_arrays
    arr = block_arrays(H.bct)
    lo, hi = arr.tree.lo, arr.tree.hi
    n = H.n
    out = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    for b in np.flatnonzero(arr.kind_code != 0):
        p = H.data[int(b)]
        t, s = arr.tau[b], arr.sigma[b]
        if hasattr(p, "left"):
            if p.left.shape[1] == 0:
                continue
            u = torch.from_numpy(np.ascontiguousarray(p.left)).cuda()
            v = torch.from_numpy(np.ascontiguousarray(p.right)).cuda()
            out[lo[t]:hi[t], lo[s]:hi[s]] = u @ v.T
        else:
            out[lo[t]:hi[t], lo[s]:hi[s]] = torch.from_numpy(np.ascontiguousarray(p)).cuda()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tag", default="dense-svd")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--estimate", type=int, default=0, help="probes of the GPU estimator")
    ap.add_argument("--ref-estimate", action="store_true",
                    help="the reference's estimate_product_error (subspace iteration) on the GPU")
    a = ap.parse_args()
    c = configs.CONFIGS[a.cfg]
    t0 = time.time()
    bct, A, B = configs.build_operands(c)
    print(f"cfg{a.cfg}: n={c['n']} nodes={bct.n_nodes} setup {time.time()-t0:.1f}s "
          f"A max rank {max(int(r) for r in A._hx_packed[1]['rank'])} "
          f"B max rank {max(int(r) for r in B._hx_packed[1]['rank'])} "
          f"degraded A {len(A.degraded)} B {len(B.degraded)}", flush=True)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(a.tag), policy=hx.EpsRank(c["tol"]))
    for it in range(a.steps):
        t0 = time.time()
        C = hx.hmult_new(A, B, cfg)
        r = C.report
        info = C.plan_info
        print(f"wall {time.time()-t0:.3f}s plan {r.plan_ms:.0f}ms dev {r.device_ms:.1f}ms "
              f"form {r.form_ms:.1f} mat {r.materialize_ms:.1f} recomp {r.recompress_ms:.1f} "
              f"rounds {r.sketch_rounds} launches {r.launches} chunks {r.chunks} maxr {r.max_far_rank}",
              flush=True)
    print({f[0]: getattr(info, f[0]) for f in info._fields_ if f[0] != "created"}, flush=True)
    ranks = C.leaf_rank[C.plan_leaves["kind"] == 1]
    ms = C.plan_leaves["m"][C.plan_leaves["kind"] == 1]
    for m in np.unique(ms):
        rr = ranks[ms == m]
        print(f"  far {m}: n={len(rr)} rank {rr.min()}-{rr.max()} mean {rr.mean():.2f}")
    if a.estimate:
        from paper_1805_08998_b200.matvec import product_error
        t0 = time.time()
        est, cn = product_error(C, A, B, probes=a.estimate)
        print(f"estimated ||C - AB||/||C|| = {est:.3e} ({a.estimate} probes, tol {c['tol']}) "
              f"||C|| ~ {cn:.4e} check {time.time()-t0:.1f}s", flush=True)
    if a.ref_estimate:
        from paper_1805_08998_b200.matvec import estimate_product_error
        t0 = time.time()
        est = estimate_product_error(A, B, C)
        fro = hx.frobenius_norm(C)
        print(f"estimate_product_error (10 iterations, block 100): ||C - AB|| ~ {est:.4e}, "
              f"/ ||C||_F = {est / fro:.3e} (tol {c['tol']}) {time.time()-t0:.1f}s", flush=True)
    if a.check:
        import torch
        t0 = time.time()
        da = dense_on_gpu(A, torch)
        db = da if B is A else dense_on_gpu(B, torch)
        dc = dense_on_gpu(C, torch)
        ex = da @ db
        err = (torch.linalg.norm(dc - ex) / torch.linalg.norm(ex)).item()
        print(f"rel err ||C - AB||/||AB|| = {err:.3e} (tol {c['tol']}) check {time.time()-t0:.1f}s")


if __name__ == "__main__":
    main()
