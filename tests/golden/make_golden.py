"""Generate the golden fixtures that pin the oracle (and through it the GPU path).

Runs the UNMODIFIED reference (``/root/reference/pkg/src/hmat``) in the build container;
the GPU box never runs this script (it has no ``/root/reference``).  The reference
geometry only knows sphere panels, so point clouds enter through a duck-typed
``PanelSet`` (``centers`` = points, unit ``areas``), exactly the survey's adapter
(SURVEY 8(c)); far leaves are assembled with the reference ``aca`` on an entry-access
``LinearMap`` whose rows/columns come from the point kernel.

Usage:  python tests/golden/make_golden.py      (writes tests/golden/*.npz)
        python tests/golden/make_golden.py traditional   (only traditional.npz)
"""

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import hmat  # noqa: E402
from hmat import clustering, compressors, geometry, hmatrix, lowrank, multiply  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def kern(name, xr, xc, h=None):
    d = xr[:, None, :] - xc[None, :, :]
    r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
    if name == "exp":
        return np.exp(-r)
    if name == "exp0.5":
        return np.exp(-r / 0.5)
    if name == "gauss0.1":
        return np.exp(-(r * r) / 0.1)
    if name == "inv":
        return 1.0 / (r + h)
    raise ValueError(name)


class PointMap(compressors.LinearMap):
    def __init__(self, name, xr, xc, h):
        self.name, self.xr, self.xc, self.h = name, xr, xc, h
        self.shape = (len(xr), len(xc))

    def row(self, i):
        return kern(self.name, self.xr[i:i + 1], self.xc, self.h)[0]

    def col(self, j):
        return kern(self.name, self.xr, self.xc[j:j + 1], self.h)[:, 0]

    def apply(self, v):
        return kern(self.name, self.xr, self.xc, self.h) @ v

    def apply_transpose(self, w):
        return kern(self.name, self.xr, self.xc, self.h).T @ w


def assemble(name, bct, eps, pts, h=None):
    perm = bct.tree.permutation
    data, bad = {}, set()
    for leaf in bct.leaves:
        xr = pts[perm[leaf.tau.lo:leaf.tau.hi]]
        xc = pts[perm[leaf.sigma.lo:leaf.sigma.hi]]
        if leaf.kind == clustering.NEAR:
            data[leaf.id] = kern(name, xr, xc, h)
        else:
            blk = compressors.aca(PointMap(name, xr, xc, h), lowrank.EpsRank(eps))
            if blk.degraded:
                bad.add(leaf.id)
                data[leaf.id] = kern(name, xr, xc, h)
            else:
                data[leaf.id] = blk
    return hmatrix.HMatrix(bct, data, bad)


def leaf_table(H):
    """Per-leaf (id, kind, rank, fro) arrays in leaf order."""
    ids, kinds, ranks, fros = [], [], [], []
    for leaf in H.bct.leaves:
        p = H.data[leaf.id]
        ids.append(leaf.id)
        if isinstance(p, lowrank.LowRank):
            kinds.append(1)
            ranks.append(p.rank)
            fros.append(p.norm())
        else:
            kinds.append(2)
            ranks.append(-1)
            fros.append(float(np.linalg.norm(p)))
    return (np.array(ids), np.array(kinds), np.array(ranks), np.array(fros))


def product_case(tag, A, B, tol, seed=0, keep_dense=False, sample=()):
    cfg = multiply.MultiplyConfig(mode="new",
                                  compressor=compressors.CompressorKind(tag, seed=seed),
                                  policy=lowrank.EpsRank(tol))
    t0 = time.time()
    C = multiply.hmult_new(A, B, cfg)
    wall = time.time() - t0
    ids, kinds, ranks, fros = leaf_table(C)
    rep = C.report
    out = {
        f"{tag}/ids": ids, f"{tag}/kinds": kinds, f"{tag}/ranks": ranks,
        f"{tag}/fros": fros,
        f"{tag}/report": np.array([rep.degraded_blocks, rep.max_far_rank,
                                   rep.matvec_count, rep.far_leaves, rep.near_leaves]),
    }
    if keep_dense:
        out[f"{tag}/dense"] = hmatrix.to_dense(C)
    for b in sample:
        p = C.data[b]
        out[f"{tag}/blk{b}"] = p.to_dense() if isinstance(p, lowrank.LowRank) else p
    print(f"  {tag}: {wall:.2f}s far={rep.far_leaves} near={rep.near_leaves} "
          f"maxr={rep.max_far_rank} mv={rep.matvec_count}", flush=True)
    return out


def product_setup(n, geom, n_min, eta, ka, kb, eps_a, seed=0):
    rng = np.random.default_rng(seed)
    if geom == "square":
        pts = rng.uniform(0, 1, (n, 2))
    elif geom == "cube":
        pts = rng.uniform(0, 1, (n, 3))
    else:
        g = rng.standard_normal((n, 3))
        pts = g / np.linalg.norm(g, axis=1, keepdims=True)
    ps = geometry.PanelSet(centers=pts, areas=np.ones(n), corners=None, level=0)
    tree = clustering.build_cluster_tree(ps, n_min)
    bct = clustering.build_block_cluster_tree(tree, eta)
    h = n ** (-1.0 / 3.0)
    A = assemble(ka, bct, eps_a, pts, h)
    B = A if kb is None else assemble(kb, bct, eps_a, pts, h)
    return pts, tree, bct, A, B


def save(name, arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def case_products(name, n, geom, n_min, eta, ka, kb, eps_a, tol, tags, dense_tags=(),
                  sample=()):
    print(f"case {name}: n={n} {geom} leaf {n_min} eta {eta} {ka}/{kb}", flush=True)
    pts, tree, bct, A, B = product_setup(n, geom, n_min, eta, ka, kb, eps_a)
    dump = clustering.dump_tree(bct)
    arrays = {
        "points": pts, "perm": tree.permutation,
        "dump_sha": np.frombuffer(hashlib.sha256(dump.encode()).digest(), dtype=np.uint8),
        "params": np.array([n, n_min, eta, eps_a, tol]),
    }
    for lab, H in (("A", A), ("B", B)):
        ids, kinds, ranks, fros = leaf_table(H)
        arrays[f"{lab}/ids"], arrays[f"{lab}/kinds"] = ids, kinds
        arrays[f"{lab}/ranks"], arrays[f"{lab}/fros"] = ranks, fros
        if n <= 512:
            arrays[f"{lab}/dense"] = hmatrix.to_dense(H)
    if n <= 2048:
        da = hmatrix.to_dense(A)
        db = hmatrix.to_dense(B)
        exact = da @ db
        arrays["exact_fro"] = np.array([np.linalg.norm(exact)])
    if sample == "auto":
        picked, seen = [], set()
        for leaf in bct.leaves:
            key = (leaf.kind, leaf.tau.size)
            if key not in seen:
                seen.add(key)
                picked.append(leaf.id)
        picked += [leaf.id for leaf in bct.leaves[::157]]
        sample = tuple(sorted(set(picked)))
    arrays["sample"] = np.array(sample, dtype=np.int64)
    for tag in tags:
        out = product_case(tag, A, B, tol, keep_dense=tag in dense_tags, sample=sample)
        arrays.update(out)
    save(name, arrays)


def case_trees():
    """Sphere meshes of the reference tests (dump text, counts, Csp)."""
    arrays = {}
    for level, n_min, eta in ((1, 6, 2.0), (2, 6, 2.0), (3, 16, 2.0)):
        p = geometry.build_sphere_mesh(level)
        tree = clustering.build_cluster_tree(p, n_min)
        bct = clustering.build_block_cluster_tree(tree, eta)
        key = f"sphere{level}_{n_min}"
        arrays[f"{key}/centers"] = p.centers
        arrays[f"{key}/dump"] = np.frombuffer(clustering.dump_tree(bct).encode(),
                                              dtype=np.uint8)
        arrays[f"{key}/counts"] = np.array([len(bct.far_leaves()), len(bct.near_leaves()),
                                            clustering.sparsity_constant(bct),
                                            tree.depth])
        arrays[f"{key}/perm"] = tree.permutation
    save("trees.npz", arrays)


def case_compressors():
    """Compressor outputs on the reference test suite's synthetic operators."""
    arrays = {}
    rng = np.random.default_rng(1)
    m, n = 60, 45
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    decay = (u * 0.5 ** np.arange(n)) @ v.T
    rng = np.random.default_rng(0)
    lowr = rng.standard_normal((50, 7)) @ rng.standard_normal((7, 40))
    arrays["decay"] = decay
    arrays["lowr"] = lowr
    for mat_name, mat in (("decay", decay), ("lowr", lowr)):
        for pol_name, pol in (("eps1e-6", lowrank.EpsRank(1e-6)),
                              ("eps1e-10", lowrank.EpsRank(1e-10)),
                              ("fixed5", lowrank.FixedRank(5))):
            for tag in compressors.CompressorKind.TAGS:
                cm = compressors.CountingMap(compressors.DenseMap(mat))
                out = compressors.compress(cm, pol, compressors.CompressorKind(tag, seed=7))
                key = f"{mat_name}/{pol_name}/{tag}"
                arrays[f"{key}/left"] = out.left
                arrays[f"{key}/right"] = out.right
                arrays[f"{key}/count"] = np.array([cm.total, int(out.degraded)])
    s = np.array([3.0, 2.0, 1.0, 1e-3, 1e-7, 0.0])
    sel = []
    for eps in (1e-1, 1e-3, 1e-6, 1e-9, 0.5, 2.0):
        sel.append(lowrank.select_rank(s, lowrank.EpsRank(eps)))
    arrays["select/s"] = s
    arrays["select/ranks"] = np.array(sel)
    save("compressors.npz", arrays)


def trad_case(conv, A, B, tol, keep_dense=False, sample=()):
    """The reference's traditional-mode product (``hmult_traditional``) with one pair
    converter: per-leaf ranks / norms, the report and dense or sampled blocks."""
    cfg = multiply.MultiplyConfig(mode="traditional",
                                  compressor=compressors.CompressorKind("aca", seed=0),
                                  policy=lowrank.EpsRank(tol), converter=conv)
    t0 = time.time()
    C = multiply.hmult_traditional(A, B, cfg)
    wall = time.time() - t0
    ids, kinds, ranks, fros = leaf_table(C)
    rep = C.report
    out = {
        f"{conv}/ids": ids, f"{conv}/kinds": kinds, f"{conv}/ranks": ranks,
        f"{conv}/fros": fros,
        f"{conv}/report": np.array([rep.degraded_blocks, rep.max_far_rank,
                                    rep.matvec_count, rep.far_leaves, rep.near_leaves]),
    }
    if keep_dense:
        out[f"{conv}/dense"] = hmatrix.to_dense(C)
    for b in sample:
        p = C.data[b]
        out[f"{conv}/blk{b}"] = p.to_dense() if isinstance(p, lowrank.LowRank) else p
    print(f"  traditional {conv}: {wall:.2f}s far={rep.far_leaves} maxr={rep.max_far_rank} "
          f"mv={rep.matvec_count}", flush=True)
    return out


def case_traditional(specs, convs=("hier-approx", "dense-svd")):
    """traditional.npz: the traditional-mode products of the product cases (same operands
    as small2d / ragged3d / cfg1, keys prefixed by the case name)."""
    arrays = {}
    for name, n, geom, n_min, eta, ka, kb, eps_a, tol, sample in specs:
        print(f"traditional {name}: n={n}", flush=True)
        pts, tree, bct, A, B = product_setup(n, geom, n_min, eta, ka, kb, eps_a)
        if sample == "auto":
            picked, seen = [], set()
            for leaf in bct.leaves:
                key = (leaf.kind, leaf.tau.size)
                if key not in seen:
                    seen.add(key)
                    picked.append(leaf.id)
            picked += [leaf.id for leaf in bct.leaves[::157]]
            sample = tuple(sorted(set(picked)))
        arrays[f"{name}/sample"] = np.array(sample, dtype=np.int64)
        for conv in convs:
            try:
                out = trad_case(conv, A, B, tol, keep_dense=n <= 512, sample=sample)
            except Exception as exc:  # recorded: the reference itself rejects the case
                print(f"  traditional {conv}: reference raised {exc!r}", flush=True)
                arrays[f"{name}/{conv}/error"] = np.frombuffer(repr(exc).encode(), np.uint8)
                continue
            arrays.update({f"{name}/{k}": v for k, v in out.items()})
    save("traditional.npz", arrays)


TRAD_SPECS = (
    ("small2d", 256, "square", 16, 0.8, "exp", None, 1e-8, 1e-6, ()),
    ("ragged3d", 200, "cube", 12, 1.0, "exp0.5", "inv", 1e-8, 1e-8, ()),
    ("cfg1", 2048, "square", 32, 0.8, "exp", None, 1e-8, 1e-6, "auto"),
)


if __name__ == "__main__":
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if sys.argv[1:] == ["traditional"]:
        case_traditional(TRAD_SPECS)
        sys.exit(0)
    case_trees()
    case_compressors()
    all_tags = ("dense-svd", "aca", "bilanczos", "randomized")
    case_products("small2d.npz", 256, "square", 16, 0.8, "exp", None, 1e-8, 1e-6,
                  all_tags, dense_tags=all_tags)
    case_products("ragged3d.npz", 200, "cube", 12, 1.0, "exp0.5", "inv", 1e-8, 1e-8,
                  all_tags, dense_tags=all_tags)
    case_products("cfg1.npz", 2048, "square", 32, 0.8, "exp", None, 1e-8, 1e-6,
                  all_tags, sample="auto")
