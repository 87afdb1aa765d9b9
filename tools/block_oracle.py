"""Per-block oracle check of a large BASELINE config ("Cfg3-5: per-block oracle").

The GPU product runs on the full config; for a stratified sample of output leaves (every
far size class up to --max-size, the largest included, plus some near leaves) the oracle
restatement rebuilds S(leaf) along its root-to-leaf chain (``leaf_expr``, the reference's
sumexpr_root + restrict, sumexpr.py:78-154), densifies it and takes its best approximation
at the tolerance (dense-svd semantics, compressors.py:431-438 with select_rank,
lowrank.py:75-90).  Blocks larger than --dense-max (the reference's own dense cap is 6144,
compressors.py:31) are checked matrix-free, as SURVEY 8(c) prescribes: the oracle's
restatement of the reference ``bilanczos`` (compressors.py:271-365, which reproduces the
dense-svd ranks) runs on S(leaf) through its matvecs, with the per-block seed, and the
factored results are compared through their Gram matrices (no densification).  Contract
per block: rank within +-1, relative difference <= 10 tol; near blocks exact to 1e-12.

usage: python tools/block_oracle.py CFG [--per-class 8] [--max-size 0] [--near 8]
                                        [--dense-max 4096] [--tag dense-svd]
"""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1805_08998_b200 as hx  # noqa: E402
from oracle import hmat_oracle as O  # noqa: E402
from paper_1805_08998_b200 import configs  # noqa: E402


def oracle_operand(H, obt):
    # views into the downloaded pool, no copies (config 5's operands are ~60 GB)
    data = {}
    for b, p in H.data.items():
        data[b] = O.LR(p.left, p.right) if hasattr(p, "left") else p
    return O.HMatO(obt, data, H.degraded)


def lr_rel_diff(u1, v1, u2, v2):
    """||U1 V1^T - U2 V2^T||_F / ||U2 V2^T||_F from thin QRs of the stacked factors (no
    Gram matrices: their traces cancel catastrophically below tol ~1e-8)."""
    _, rl = np.linalg.qr(np.hstack([u1, -u2]))
    _, rr = np.linalg.qr(np.hstack([v1, v2]))
    _, r2l = np.linalg.qr(u2)
    _, r2r = np.linalg.qr(v2)
    num = np.linalg.norm(rl @ rr.T)
    den = np.linalg.norm(r2l @ r2r.T)
    return float(num / max(den, 1e-300))


def certify(s, U, V, tol, batch):
    """Exact epsilon-rank bracket of a block too large for a dense SVD, from the GPU's
    factors: S is applied to the identity in column batches (exact densification, never
    held whole) to measure ||S||_F and the GPU residual d = ||S - U V^T||_F exactly.
    Upper bound: d <= tol ||S|| means the best rank-r error is <= tol ||S||, so the
    epsilon-rank is <= r.  Lower bound (Weyl): sigma_i(S) >= sigma_i(U V^T) - d, so the
    tail ||s[j:]|| >= sqrt(sum_{i >= j} (sigma_i(U V^T) - d)_+^2); any j whose lower bound
    exceeds tol ||S|| is too small a rank."""
    m, n = s.shape
    fro2 = 0.0
    res2 = 0.0
    for j0 in range(0, n, batch):
        j1 = min(n, j0 + batch)
        E = np.zeros((n, j1 - j0))
        E[np.arange(j0, j1), np.arange(j1 - j0)] = 1.0
        blk = s.mat(E)
        fro2 += float(np.sum(blk * blk))
        blk -= U @ V[j0:j1].T
        res2 += float(np.sum(blk * blk))
    nrm = np.sqrt(fro2)
    d = np.sqrt(res2)
    r = U.shape[1]
    hi = r if d <= tol * nrm else None
    sv = np.linalg.svd(np.linalg.qr(U)[1] @ np.linalg.qr(V)[1].T, compute_uv=False)
    low = np.maximum(sv - d, 0.0)
    tails = np.sqrt(np.cumsum((low ** 2)[::-1])[::-1])
    lo = 0
    for j in range(r):
        if tails[j] > tol * nrm:
            lo = j + 1
    return lo, (hi if hi is not None else r + 10 ** 6), d / nrm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--per-class", type=int, default=8)
    ap.add_argument("--max-size", type=int, default=0, help="skip far sizes above (0: none)")
    ap.add_argument("--min-size", type=int, default=0, help="skip far sizes below")
    ap.add_argument("--dense-max", type=int, default=4096,
                    help="blocks up to this: full SVD of the densified S(leaf)")
    ap.add_argument("--values-max", type=int, default=8192,
                    help="blocks up to this: singular values of the densified S(leaf) and "
                         "the GPU block's own residual; larger: matrix-free Lanczos")
    ap.add_argument("--tag", default="dense-svd")
    ap.add_argument("--certify", action="store_true",
                    help="above --values-max: exact rank bracket from the GPU factors and the "
                         "exactly measured residual, besides the Lanczos comparison")
    ap.add_argument("--batch", type=int, default=2048, help="columns per application of S")
    ap.add_argument("--blocks", default="", help="check exactly these block ids (comma list)")
    ap.add_argument("--near", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    c = configs.CONFIGS[a.cfg]
    tol = c["tol"]
    t0 = time.time()
    bct, A, B = configs.build_operands(c)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(a.tag), policy=hx.EpsRank(tol))
    C = hx.hmult_new(A, B, cfg)
    print(f"cfg{a.cfg}: GPU product {C.report.wall_s:.1f} s (setup {time.time() - t0:.1f} s)",
          flush=True)
    pts = configs.make_points(c)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, c["n_min"]), c["eta"])
    oa = oracle_operand(A, obt)
    ob = oa if B is A else oracle_operand(B, obt)
    rng = np.random.default_rng(a.seed)
    lo, hi = bct.tree.lo, bct.tree.hi
    size = (hi[bct.tau] - lo[bct.tau])
    far = np.flatnonzero(bct.kind_code == 1)
    near = np.flatnonzero(bct.kind_code == 2)
    sample = []
    for m in np.unique(size[far]):
        if (a.max_size and m > a.max_size) or m < a.min_size:
            continue
        ids = far[size[far] == m]
        pick = rng.choice(ids, size=min(a.per_class, len(ids)), replace=False)
        sample += [int(b) for b in pick]
    sample += [int(b) for b in rng.choice(near, size=min(a.near, len(near)), replace=False)]
    if a.blocks:
        sample = [int(x) for x in a.blocks.split(",")]
    worst_rank, worst_far, worst_near = 0, 0.0, 0.0
    t1 = time.time()
    for b in sample:
        s = O.leaf_expr(oa, ob, b)
        m, n = s.shape
        q = C.data[b]
        if bct.kind_code[b] == 1 and a.dense_max < min(m, n) <= a.values_max:
            # exact epsilon-rank from the singular values; block difference bounded by
            # ||C_gpu - S|| + ||S - C_best|| (both measured exactly on the dense S)
            tl = time.time()
            dense = s.mat(np.eye(n))
            sv = np.linalg.svd(dense, compute_uv=False)
            r = O.eps_rank(sv, O.Eps(tol))
            nrm = np.linalg.norm(sv)
            e_best = np.linalg.norm(sv[r:]) / nrm
            e_gpu = np.linalg.norm(dense - q.left @ q.right.T) / nrm
            d = (e_gpu + e_best) / max(np.sqrt(max(nrm ** 2 - np.sum(sv[r:] ** 2), 0.0)) / nrm,
                                       1e-300)
            worst_rank = max(worst_rank, abs(q.rank - r))
            worst_far = max(worst_far, d)
            print(f"  far  {b:8d} {m}x{n}: rank gpu {q.rank} oracle {r} (dense singular values, "
                  f"{time.time() - tl:.0f} s), gpu residual {e_gpu:.2e}, best {e_best:.2e}, "
                  f"rel diff <= {d:.2e}", flush=True)
            del dense
            continue
        if bct.kind_code[b] == 1 and min(m, n) > a.values_max and a.certify:
            tl = time.time()
            lo_r, hi_r, e_gpu = certify(s, q.left, q.right, tol, a.batch)
            ref = O.lanczos_o(s, O.Eps(tol), seed=O.block_seed(0, b))
            dl = lr_rel_diff(q.left, q.right, ref.left, ref.right)
            off = max(q.rank - lo_r, hi_r - q.rank)
            worst_rank = max(worst_rank, off)
            worst_far = max(worst_far, 2 * e_gpu)
            print(f"  far  {b:8d} {m}x{n}: rank gpu {q.rank}, exact epsilon-rank in "
                  f"[{lo_r}, {hi_r}] (certificate: S applied to the identity in column "
                  f"batches), gpu residual {e_gpu:.2e} (rel diff to the best <= "
                  f"{2 * e_gpu:.2e}); reference bilanczos rank {ref.rank}, diff {dl:.2e} "
                  f"({time.time() - tl:.0f} s)", flush=True)
            continue
        if bct.kind_code[b] == 1 and min(m, n) > a.values_max:
            tl = time.time()
            ref = O.lanczos_o(s, O.Eps(tol), seed=O.block_seed(0, b))
            d = lr_rel_diff(q.left, q.right, ref.left, ref.right)
            worst_rank = max(worst_rank, abs(q.rank - ref.rank))
            worst_far = max(worst_far, d)
            print(f"  far  {b:8d} {m}x{n}: rank gpu {q.rank} oracle {ref.rank} (Lanczos, "
                  f"matrix-free, {time.time() - tl:.0f} s), rel diff {d:.2e}", flush=True)
            continue
        dense = s.mat(np.eye(n))
        if bct.kind_code[b] == 2:
            d = np.linalg.norm(q - dense) / max(np.linalg.norm(dense), 1e-300)
            worst_near = max(worst_near, d)
            print(f"  near {b:8d} {m}x{n}: rel diff {d:.2e}", flush=True)
            continue
        if a.tag == "aca":
            # the oracle of the aca tag is the reference's ACA on S(leaf) (with its
            # truncate(eps / 2)); the best approximation is reported beside it
            ref = O.aca_o(O.DenseOp(dense), O.Eps(tol))
            r = ref.rank
            best = ref.dense()
            sv = np.linalg.svd(dense, compute_uv=False)
            extra = f" (epsilon-rank {O.eps_rank(sv, O.Eps(tol))})"
        else:
            u, sv, vt = np.linalg.svd(dense, full_matrices=False)
            r = O.eps_rank(sv, O.Eps(tol))
            best = (u[:, :r] * sv[:r]) @ vt[:r]
            extra = ""
        d = np.linalg.norm(q.to_dense() - best) / max(np.linalg.norm(best), 1e-300)
        worst_rank = max(worst_rank, abs(q.rank - r))
        worst_far = max(worst_far, d)
        print(f"  far  {b:8d} {m}x{n}: rank gpu {q.rank} oracle {r}{extra}, rel diff {d:.2e}",
              flush=True)
    print(f"cfg{a.cfg}: {len(sample)} blocks checked in {time.time() - t1:.0f} s: worst rank "
          f"difference {worst_rank}, worst far rel diff {worst_far:.2e} (10 tol = "
          f"{10 * tol:.0e}), worst near rel diff {worst_near:.2e}", flush=True)
    ok = worst_rank <= 1 and worst_far <= 10 * tol and worst_near <= 1e-12
    print("PASS" if ok else "FAIL", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
