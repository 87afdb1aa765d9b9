"""CPU oracle: a NumPy restatement of the reference's tolerance-controlled H x H product.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module, and
only as the checker or as the timed CPU baseline.  The product package
(``paper_1805_08998_b200``) never imports it; the GPU path fails loudly when its CUDA
library is missing instead of falling back here.

What it restates (all citations are ``file:line`` in the reference tree
``/root/reference/pkg/src/hmat``):

* cluster tree by cardinality-balanced bisection along the longest box axis
  (``clustering.py:61-89``), block-cluster tree with the Euclidean-diameter /
  Chebyshev-distance admissibility test and DFS pre-order ids (``clustering.py:92-172``);
* operand assembly: dense near leaves, ACA far leaves with dense fallback when ACA
  cannot certify convergence (``hmatrix.py:97-118``);
* the sum-expression descent: low-rank terms sliced without arithmetic, pending pairs split
  over the middle cluster, thin products for sub-pairs with a factored side
  (``sumexpr.py:93-154``), H-subtree times thin matrix (``hmatrix.py:177-202``);
* the compressors on the implicit operator: ACA (``compressors.py:162-247``),
  Golub-Kahan-Lanczos (``:271-365``), randomized adaptive / fixed (``:368-428``), dense SVD
  (``:431-438``) and the shared epsilon-rank rule (``lowrank.py:75-90``);
* the product driver ``hmult_new`` (``multiply.py:207-256``) with per-block seeds
  (``multiply.py:61-63``) and the report counters (``multiply.py:50-58``);
* the HMX1 operator file format (``hmatrix.py:9-24``, ``save_hmatrix`` / ``load_hmatrix``
  ``:334-388``).

Parity of this restatement is pinned against the reference itself: ``tests/golden`` holds
fixtures produced by importing the reference in the build container
(``tests/golden/make_golden.py``), and ``tests/test_oracle_golden.py`` checks this module
against them.

Block-tree kinds are small ints: ``INNER=0, FAR=1, NEAR=2``.
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

INNER, FAR, NEAR = 0, 1, 2
KIND_NAMES = {INNER: "inner", FAR: "far", NEAR: "near"}
EPS_FLOOR = 1e-15            # compressors.py:28
DENSE_CAP = 6144             # compressors.py:29, sumexpr.py:31


# --------------------------------------------------------------------------- trees


class ClusterTreeO:
    """Array form of the reference cluster tree (``clustering.py:61-89``).

    Cluster ids are creation (pre-order) ids; ``perm[pos]`` is the original point index
    at tree position ``pos``.
    """

    def __init__(self, points, n_min):
        pts = np.asarray(points, dtype=float)
        if n_min < 1:
            raise ValueError("n_min must be >= 1")
        if len(pts) == 0:
            raise ValueError("empty panel set")
        self.n = len(pts)
        self.n_min = n_min
        perm = np.arange(self.n)
        lo, hi, lev, kids, blo, bhi = [], [], [], [], [], []

        def split(a, b, depth):
            cid = len(lo)
            sub = pts[perm[a:b]]
            box_lo, box_hi = sub.min(axis=0), sub.max(axis=0)
            lo.append(a)
            hi.append(b)
            lev.append(depth)
            kids.append([-1, -1])
            blo.append(box_lo)
            bhi.append(box_hi)
            if b - a > n_min:
                ax = int(np.argmax(box_hi - box_lo))
                order = np.argsort(sub[:, ax], kind="stable")
                perm[a:b] = perm[a:b][order]
                m = a + (b - a) // 2
                kids[cid] = [split(a, m, depth + 1), split(m, b, depth + 1)]
            return cid

        split(0, self.n, 0)
        self.lo = np.array(lo, dtype=np.int64)
        self.hi = np.array(hi, dtype=np.int64)
        self.level = np.array(lev, dtype=np.int64)
        self.children = np.array(kids, dtype=np.int64)
        self.box_lo = np.array(blo)
        self.box_hi = np.array(bhi)
        self.perm = perm
        self.depth = int(self.level.max())

    def is_leaf(self, c):
        return self.children[c, 0] < 0


def admissible_o(tree, t, s, eta):
    """``min(diam) <= eta * dist`` with Euclidean diameters, Chebyshev gap
    (``clustering.py:92-107``)."""
    dt = float(np.linalg.norm(tree.box_hi[t] - tree.box_lo[t]))
    ds = float(np.linalg.norm(tree.box_hi[s] - tree.box_lo[s]))
    gap = np.maximum(tree.box_lo[t] - tree.box_hi[s], tree.box_lo[s] - tree.box_hi[t])
    dist = float(max(0.0, gap.max()))
    return min(dt, ds) <= eta * dist


class BlockTreeO:
    """Array form of the reference block-cluster tree (``clustering.py:154-172``)."""

    def __init__(self, tree: ClusterTreeO, eta):
        self.tree = tree
        self.eta = eta
        tau, sig, kind, lev, kids = [], [], [], [], []

        def visit(t, s, depth):
            bid = len(tau)
            tau.append(t)
            sig.append(s)
            kind.append(NEAR)
            lev.append(depth)
            kids.append([-1, -1, -1, -1])
            if admissible_o(tree, t, s, eta):
                kind[bid] = FAR
            elif not tree.is_leaf(t) and not tree.is_leaf(s):
                kind[bid] = INNER
                out = []
                for tc in tree.children[t]:
                    for sc in tree.children[s]:
                        out.append(visit(int(tc), int(sc), depth + 1))
                kids[bid] = out
            return bid

        visit(0, 0, 0)
        self.tau = np.array(tau, dtype=np.int64)
        self.sigma = np.array(sig, dtype=np.int64)
        self.kind = np.array(kind, dtype=np.int64)
        self.level = np.array(lev, dtype=np.int64)
        self.children = np.array(kids, dtype=np.int64)
        self.n_nodes = len(tau)

    @property
    def n(self):
        return self.tree.n

    def rows(self, b):
        t = self.tau[b]
        return int(self.tree.lo[t]), int(self.tree.hi[t])

    def cols(self, b):
        s = self.sigma[b]
        return int(self.tree.lo[s]), int(self.tree.hi[s])

    def shape(self, b):
        r0, r1 = self.rows(b)
        c0, c1 = self.cols(b)
        return r1 - r0, c1 - c0

    def leaves(self):
        return [b for b in range(self.n_nodes) if self.kind[b] != INNER]

    def child_for(self, b, t, s):
        """Child of block ``b`` with row cluster ``t`` and column cluster ``s``."""
        for c in self.children[b]:
            if c >= 0 and self.tau[c] == t and self.sigma[c] == s:
                return int(c)
        raise ValueError("child block not found")

    def dump(self):
        """Same text as the reference ``dump_tree`` (``clustering.py:218-229``)."""
        lines = []
        stack = [0]
        while stack:
            b = stack.pop()
            r0, r1 = self.rows(b)
            c0, c1 = self.cols(b)
            lines.append(f"level {self.level[b]} rows [{r0},{r1}) cols [{c0},{c1}) "
                         f"{KIND_NAMES[int(self.kind[b])]}")
            stack.extend(int(c) for c in self.children[b][::-1] if c >= 0)
        return "\n".join(lines) + "\n"


# --------------------------------------------------------------------------- kernels

def kernel_matrix(name, xr, xc, h=None):
    """Kernel block between row points ``xr`` and column points ``xc`` with unit weights.

    Distances follow the reference's ``kernel_block`` arithmetic (``geometry.py:170-186``:
    coordinate differences, einsum of squares, sqrt), so that ``exp`` matches
    ``kernel_block("exp", ...)`` on a unit-area point set bit for bit.
    """
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
    raise ValueError(f"unknown kernel {name!r}")


# --------------------------------------------------------------------------- low rank

class LR:
    """Factor pair ``left @ right.T`` (``lowrank.py:15-43``); rank 0 allowed."""

    __slots__ = ("left", "right", "degraded")

    def __init__(self, left, right, degraded=False):
        self.left = left
        self.right = right
        self.degraded = degraded

    @property
    def rank(self):
        return self.left.shape[1]

    def dense(self):
        return self.left @ self.right.T


def empty_lr(m, n, degraded=False):
    return LR(np.zeros((m, 0)), np.zeros((n, 0)), degraded)


@dataclass(frozen=True)
class Eps:
    eps: float


@dataclass(frozen=True)
class Fixed:
    k_max: int


def policy_of(p):
    """Accept reference / product policy objects by duck type."""
    if hasattr(p, "k_max"):
        return Fixed(int(p.k_max))
    return Eps(float(p.eps))


def eps_rank(s, policy):
    """``select_rank`` (``lowrank.py:75-90``): smallest r with ||s[r:]|| <= eps*||s||."""
    if isinstance(policy, Fixed):
        return min(len(s), policy.k_max)
    if len(s) == 0:
        return 0
    rev = np.cumsum(np.asarray(s)[::-1] ** 2)
    tails = np.sqrt(rev)[::-1]
    hit = np.flatnonzero(tails <= policy.eps * tails[0])
    return int(hit[0]) if hit.size else len(s)


def clamp_eps(eps):
    """``_clamp_eps`` (``compressors.py:144-149``)."""
    if eps <= np.finfo(float).eps:
        warnings.warn(f"tolerance {eps:g} is below machine precision, clamping to "
                      f"{EPS_FLOOR:g}")
        return EPS_FLOOR
    return eps


def lr_svd(t: LR):
    """``lowrank_svd`` (``lowrank.py:93-104``): QR both factors, SVD of the core."""
    m, n = t.left.shape[0], t.right.shape[0]
    if t.rank == 0:
        return np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0))
    ql, rl = np.linalg.qr(t.left)
    qr_, rr = np.linalg.qr(t.right)
    uu, s, vvt = np.linalg.svd(rl @ rr.T)
    return ql @ uu, s, qr_ @ vvt.T


def lr_truncate(t: LR, policy):
    """``truncate`` (``lowrank.py:107-113``)."""
    if t.rank == 0:
        return t
    u, s, v = lr_svd(t)
    r = eps_rank(s, policy)
    return LR(u[:, :r] * s[:r], v[:, :r])


# --------------------------------------------------------------------------- operators

class Op:
    """Implicit m x n operator: the ``LinearMap`` protocol (``compressors.py:34-67``) with
    the counting of ``CountingMap`` (``compressors.py:88-119``) built in."""

    shape = (0, 0)

    def __init__(self):
        self.count = 0

    def mat(self, v):            # forward product with an (n, q) block
        raise NotImplementedError

    def mat_t(self, w):          # transpose product with an (m, q) block
        raise NotImplementedError

    def fwd(self, v):
        self.count += 1
        return self.mat(v[:, None])[:, 0]

    def adj(self, w):
        self.count += 1
        return self.mat_t(w[:, None])[:, 0]

    def fwd_block(self, v):
        self.count += v.shape[1]
        return self.mat(v)

    def adj_block(self, w):
        self.count += w.shape[1]
        return self.mat_t(w)

    def row(self, i):
        e = np.zeros(self.shape[0])
        e[i] = 1.0
        return self.adj(e)

    def col(self, j):
        e = np.zeros(self.shape[1])
        e[j] = 1.0
        return self.fwd(e)

    def dense(self):
        if self.shape[1] > DENSE_CAP:
            raise ValueError(f"materialization capped at {DENSE_CAP} columns")
        return self.fwd_block(np.eye(self.shape[1]))


class DenseOp(Op):
    def __init__(self, a):
        super().__init__()
        self.a = np.asarray(a, dtype=float)
        self.shape = self.a.shape

    def mat(self, v):
        return self.a @ v

    def mat_t(self, w):
        return self.a.T @ w


class EntryOp(Op):
    """Entry access into a kernel block (``hmatrix.py:68-94``)."""

    def __init__(self, kern, xr, xc, h=None):
        super().__init__()
        self.kern, self.xr, self.xc, self.h = kern, xr, xc, h
        self.shape = (len(xr), len(xc))

    def row(self, i):
        return kernel_matrix(self.kern, self.xr[i:i + 1], self.xc, self.h)[0]

    def col(self, j):
        return kernel_matrix(self.kern, self.xr, self.xc[j:j + 1], self.h)[:, 0]

    def mat(self, v):
        return kernel_matrix(self.kern, self.xr, self.xc, self.h) @ v

    def mat_t(self, w):
        return kernel_matrix(self.kern, self.xr, self.xc, self.h).T @ w


# --------------------------------------------------------------------------- compressors

def _negligible(nl, nu, acc, eps):
    """Shared adaptive stop test (``compressors.py:152-159``)."""
    return nl * nu <= eps * acc


def aca_o(op: Op, policy):
    """Partially pivoted ACA (``compressors.py:162-247``)."""
    m, n = op.shape
    cap = min(m, n)
    eps = clamp_eps(policy.eps) if isinstance(policy, Eps) else None
    kmax = policy.k_max if isinstance(policy, Fixed) else cap
    lcols, ucols = [], []
    row_used = np.zeros(m, dtype=bool)
    col_used = np.zeros(n, dtype=bool)
    fro2 = 0.0
    piv = 0
    zero_rows = 0
    degraded = False
    streak = 0
    while len(lcols) < min(kmax, cap):
        if piv is None or row_used[piv]:
            free = np.flatnonzero(~row_used)
            if free.size == 0:
                degraded = not (len(lcols) == 0 and zero_rows == m)
                break
            piv = int(free[0])
        row_used[piv] = True
        res_row = op.row(piv)
        if lcols:
            res_row = res_row - np.column_stack(ucols) @ np.array([c[piv] for c in lcols])
        else:
            res_row = res_row - 0.0
        mag = np.where(col_used, 0.0, np.abs(res_row))
        jc = int(np.argmax(mag))
        scale = math.sqrt(fro2)
        if mag[jc] <= 1e-14 * scale or mag[jc] == 0.0:
            if lcols:
                break
            zero_rows += 1
            piv = None
            continue
        u = res_row / res_row[jc]
        res_col = op.col(jc)
        if lcols:
            res_col = res_col - np.column_stack(lcols) @ np.array([c[jc] for c in ucols])
        else:
            res_col = res_col - 0.0
        upd = np.linalg.norm(res_col) * np.linalg.norm(u)
        if upd <= 1e-15 * scale or upd == 0.0:
            break
        if eps is not None:
            ref = scale if lcols else upd
            streak = streak + 1 if _negligible(np.linalg.norm(res_col), np.linalg.norm(u),
                                               ref, eps) else 0
        col_used[jc] = True
        mixed = sum(np.dot(lk, res_col) * np.dot(uk, u) for lk, uk in zip(lcols, ucols))
        fro2 += 2.0 * mixed + upd * upd
        lcols.append(res_col)
        ucols.append(u)
        if streak >= 2:
            break
        rest = np.where(row_used, 0.0, np.abs(res_col))
        piv = int(np.argmax(rest)) if rest.any() else None
    if not lcols:
        return empty_lr(m, n, degraded)
    out = LR(np.column_stack(lcols), np.column_stack(ucols))
    if eps is not None and out.rank > 1:
        out = lr_truncate(out, Eps(0.5 * eps))
    return LR(out.left, out.right, degraded)


def _cgs2(basis, v):
    """Two passes of classical Gram-Schmidt (``compressors.py:264-268``)."""
    for _ in range(2):
        v = v - basis @ (basis.T @ v)
    return v


def lanczos_o(op: Op, policy, seed=0):
    """Golub-Kahan-Lanczos bidiagonalization (``compressors.py:271-365``)."""
    m, n = op.shape
    cap = min(m, n)
    eps = clamp_eps(policy.eps) if isinstance(policy, Eps) else None
    kmax = policy.k_max if isinstance(policy, Fixed) else cap
    rng = np.random.default_rng(seed)
    qs, ws, rows = [], [], []
    fro2 = 0.0
    probes = 0
    streak = 0
    w = rng.standard_normal(n)
    w /= np.linalg.norm(w)
    beta_prev = 0.0
    q_prev = np.zeros(m)
    while len(qs) < min(kmax, cap):
        q = op.fwd(w) - beta_prev * q_prev
        if qs:
            q = _cgs2(np.column_stack(qs), q)
        alpha = np.linalg.norm(q)
        if alpha <= 1e-14 * max(math.sqrt(fro2), 1e-300):
            if probes >= 3 or len(ws) >= n:
                break
            probes += 1
            w = rng.standard_normal(n)
            if ws:
                w = _cgs2(np.column_stack(ws), w)
            nw = np.linalg.norm(w)
            if nw == 0.0:
                break
            w /= nw
            beta_prev = 0.0
            continue
        if eps is not None and qs:
            coupling = np.linalg.norm(np.array([np.hypot(alpha, beta_prev)]))
            streak = streak + 1 if _negligible(coupling, np.linalg.norm(np.array([1.0])),
                                               math.sqrt(max(fro2, 0.0)), eps) else 0
        q /= alpha
        qs.append(q)
        ws.append(w)
        probes = 0
        w_next = op.adj(q) - alpha * w
        w_next = _cgs2(np.column_stack(ws), w_next)
        beta = np.linalg.norm(w_next)
        fro2 += alpha * alpha + beta * beta
        if beta <= 1e-14 * math.sqrt(fro2):
            rows.append(alpha * w)
            break
        w_next /= beta
        rows.append(alpha * w + beta * w_next)
        if streak >= 2:
            break
        q_prev = q
        beta_prev = beta
        w = w_next
    if not qs:
        return empty_lr(m, n)
    qmat = np.column_stack(qs)
    rmat = np.vstack(rows)
    uu, s, vvt = np.linalg.svd(rmat, full_matrices=False)
    r = eps_rank(s, policy) if eps is not None else min(len(qs), len(s))
    return LR((qmat @ uu[:, :r]) * s[:r], vvt[:r].T.copy())


def randomized_adaptive_o(op: Op, eps, seed):
    """Vector-at-a-time randomized range finder (``compressors.py:368-408``)."""
    m, n = op.shape
    eps = clamp_eps(eps)
    rng = np.random.default_rng(seed)
    basis = np.zeros((m, 0))
    rows = []
    fro2 = 0.0
    streak = 0
    for _ in range(min(m, n)):
        g = rng.standard_normal(n)
        y = op.fwd(g)
        y_perp = _cgs2(basis, y)
        ny = np.linalg.norm(y_perp)
        if ny <= 1e-14 * max(math.sqrt(fro2), np.linalg.norm(y)):
            break
        qv = y_perp / ny
        u = op.adj(qv)
        basis = np.column_stack([basis, qv])
        rows.append(u)
        fro2 += float(np.dot(u, u))
        if len(rows) > 1 and _negligible(np.linalg.norm(qv), np.linalg.norm(u),
                                         math.sqrt(fro2), eps):
            streak += 1
            if streak >= 2:
                break
        else:
            streak = 0
    if not rows:
        return empty_lr(m, n)
    return LR(basis, np.column_stack(rows))


def randomized_fixed_o(op: Op, k, q=1, seed=0):
    """Blocked fixed-rank range finder with q subspace iterations (``:416-428``)."""
    m, n = op.shape
    if not 1 <= k <= min(m, n):
        raise ValueError(f"rank {k} out of range for shape {op.shape}")
    rng = np.random.default_rng(seed)
    left = np.linalg.qr(op.fwd_block(rng.standard_normal((n, k))))[0]
    for _ in range(q):
        right = np.linalg.qr(op.adj_block(left))[0]
        left = np.linalg.qr(op.fwd_block(right))[0]
    return LR(left, op.adj_block(left))


def dense_svd_o(op: Op, policy):
    """Materialize, SVD, truncate (``compressors.py:431-438``)."""
    a = op.dense()
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    if isinstance(policy, Eps):
        policy = Eps(clamp_eps(policy.eps))
    r = eps_rank(s, policy)
    return LR(u[:, :r] * s[:r], vt[:r].T.copy())


def compress_o(op: Op, policy, tag, q=1, seed=0):
    """Tag dispatch (``compressors.py:441-452``)."""
    if tag == "aca":
        return aca_o(op, policy)
    if tag == "bilanczos":
        return lanczos_o(op, policy, seed=seed)
    if tag == "randomized":
        if isinstance(policy, Fixed):
            return randomized_fixed_o(op, min(policy.k_max, *op.shape), q=q, seed=seed)
        return randomized_adaptive_o(op, policy.eps, seed=seed)
    if tag == "dense-svd":
        return dense_svd_o(op, policy)
    raise ValueError(f"unknown compressor {tag!r}")


# --------------------------------------------------------------------------- H-matrices

class HMatO:
    """Operand: block tree + ``{leaf id: ndarray | LR}`` (``hmatrix.py:48-65``)."""

    def __init__(self, bt: BlockTreeO, data, degraded=()):
        self.bt = bt
        self.data = data
        self.degraded = set(degraded)

    def is_lr(self, b):
        return self.bt.kind[b] == FAR and isinstance(self.data[b], LR)

    def to_dense(self):
        bt = self.bt
        out = np.zeros((bt.n, bt.n))
        for b in bt.leaves():
            r0, r1 = bt.rows(b)
            c0, c1 = bt.cols(b)
            p = self.data[b]
            out[r0:r1, c0:c1] = p.dense() if isinstance(p, LR) else p
        return out

    def fro(self):
        tot = 0.0
        for p in self.data.values():
            if isinstance(p, LR):
                if p.rank:
                    g = (p.left.T @ p.left) @ (p.right.T @ p.right)
                    tot += max(np.trace(g), 0.0)
            else:
                tot += float(np.sum(p * p))
        return math.sqrt(tot)


def assemble_leaf_o(kern, near, xr, xc, pol, h=None):
    """One leaf of ``assemble_hmatrix`` (``hmatrix.py:97-118``): dense near block, or ACA
    with the dense fallback when ACA cannot certify convergence.  Returns (payload,
    degraded)."""
    if near:
        return kernel_matrix(kern, xr, xc, h), False
    blk = aca_o(EntryOp(kern, xr, xc, h), pol)
    if blk.degraded:
        return kernel_matrix(kern, xr, xc, h), True
    return blk, False


def assemble_o(kern, bt: BlockTreeO, policy, points, h=None):
    """``assemble_hmatrix`` (``hmatrix.py:97-118``) for a point kernel."""
    pts = np.asarray(points, dtype=float)
    perm = bt.tree.perm
    data, bad = {}, set()
    pol = policy_of(policy)
    for b in bt.leaves():
        r0, r1 = bt.rows(b)
        c0, c1 = bt.cols(b)
        data[b], deg = assemble_leaf_o(kern, bt.kind[b] == NEAR, pts[perm[r0:r1]],
                                       pts[perm[c0:c1]], pol, h)
        if deg:
            bad.add(b)
    return HMatO(bt, data, bad)


def _assemble_chunk_o(kern, pol, h, pts, jobs):
    """Worker of ``assemble_parallel_o``: jobs = [(id, near, row points, col points)];
    single-threaded BLAS inside (the processes are the parallelism)."""
    from threadpoolctl import threadpool_limits

    out = []
    with threadpool_limits(limits=1):
        for b, near, ir, ic in jobs:
            p, deg = assemble_leaf_o(kern, near, pts[ir], pts[ic], pol, h)
            out.append((b, (p.left, p.right) if isinstance(p, LR) else p, deg))
    return out


def assemble_parallel_o(kern, bt: BlockTreeO, policy, points, h=None, workers=None):
    """``assemble_o`` with the leaves spread over worker processes (spawned, so the
    parent's BLAS thread pool is never forked); the same per-leaf arithmetic, so the same
    operand.  Assembly is setup, outside any timed region (as ``cli.py:150-158``)."""
    import os
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp

    pts = np.asarray(points, dtype=float)
    perm = bt.tree.perm
    pol = policy_of(policy)
    workers = workers or os.cpu_count() or 1
    leaves = bt.leaves()
    # cost-balanced round-robin over leaves ordered by size
    cost = [bt.shape(b)[0] * bt.shape(b)[1] for b in leaves]
    order = np.argsort(cost)[::-1]
    n_jobs = 4 * workers
    jobs = [[] for _ in range(n_jobs)]
    for i, j in enumerate(order):
        b = leaves[j]
        r0, r1 = bt.rows(b)
        c0, c1 = bt.cols(b)
        jobs[i % n_jobs].append((b, bt.kind[b] == NEAR, perm[r0:r1], perm[c0:c1]))
    data, bad = {}, set()
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        futs = [ex.submit(_assemble_chunk_o, kern, pol, h, pts, js) for js in jobs if js]
        for f in futs:
            for b, p, deg in f.result():
                data[b] = LR(p[0], p[1]) if isinstance(p, tuple) else p
                if deg:
                    bad.add(b)
    return HMatO(bt, data, bad)


def subtree_mat(H: HMatO, b, x, trans=False):
    """H-subtree times an (n_b, q) block, block-local indexing (``hmatrix.py:177-202``)."""
    bt = H.bt
    if bt.kind[b] != INNER:
        p = H.data[b]
        if isinstance(p, LR):
            if p.rank == 0:
                m, n = bt.shape(b)
                return np.zeros((n if trans else m, x.shape[1]))
            return p.right @ (p.left.T @ x) if trans else p.left @ (p.right.T @ x)
        return p.T @ x if trans else p @ x
    r0, _ = bt.rows(b)
    c0, _ = bt.cols(b)
    m, n = bt.shape(b)
    out = np.zeros((n if trans else m, x.shape[1]))
    for c in bt.children[b]:
        cr0, cr1 = bt.rows(c)
        cc0, cc1 = bt.cols(c)
        if trans:
            out[cc0 - c0:cc1 - c0] += subtree_mat(H, c, x[cr0 - r0:cr1 - r0], True)
        else:
            out[cr0 - r0:cr1 - r0] += subtree_mat(H, c, x[cc0 - c0:cc1 - c0], False)
    return out


class View:
    """Block of an operand, optionally a dense sub-slice (``hmatrix.py:205-268``)."""

    __slots__ = ("H", "b", "r0", "r1", "c0", "c1")

    def __init__(self, H: HMatO, b, r0=None, r1=None, c0=None, c1=None):
        bt = H.bt
        rr = bt.rows(b)
        cc = bt.cols(b)
        self.H, self.b = H, b
        self.r0 = rr[0] if r0 is None else r0
        self.r1 = rr[1] if r1 is None else r1
        self.c0 = cc[0] if c0 is None else c0
        self.c1 = cc[1] if c1 is None else c1

    @property
    def sliced(self):
        bt = self.H.bt
        return (self.r0, self.r1) != bt.rows(self.b) or (self.c0, self.c1) != bt.cols(self.b)

    @property
    def inner(self):
        return not self.sliced and self.H.bt.kind[self.b] == INNER

    @property
    def lowrank(self):
        return not self.sliced and self.H.is_lr(self.b)

    @property
    def shape(self):
        return self.r1 - self.r0, self.c1 - self.c0

    def dense_block(self):
        p = self.H.data[self.b]
        if isinstance(p, LR):
            return p.dense()
        rr = self.H.bt.rows(self.b)
        cc = self.H.bt.cols(self.b)
        return p[self.r0 - rr[0]:self.r1 - rr[0], self.c0 - cc[0]:self.c1 - cc[0]]

    def mat(self, x):
        if not self.inner and not self.lowrank:
            return self.dense_block() @ x
        return subtree_mat(self.H, self.b, x, False)

    def mat_t(self, x):
        if not self.inner and not self.lowrank:
            return self.dense_block().T @ x
        return subtree_mat(self.H, self.b, x, True)


class SumExprO(Op):
    """Sum-expression ``S(tau, sigma)`` acting as an operator (``sumexpr.py:33-75``)."""

    def __init__(self, bt, b, shape, lrs, pend):
        super().__init__()
        self.bt = bt
        self.b = b
        self.shape = shape
        self.lrs = lrs
        self.pend = pend
        self._stack = None

    def stacked(self):
        if self._stack is None:
            live = [t for t in self.lrs if t.rank > 0]
            self._stack = ((np.hstack([t.left for t in live]),
                            np.hstack([t.right for t in live])) if live else (None, None))
        return self._stack

    def mat(self, v):
        out = np.zeros((self.shape[0], v.shape[1]))
        L, R = self.stacked()
        if L is not None:
            out += L @ (R.T @ v)
        for p, q in self.pend:
            out += p.mat(q.mat(v))
        return out

    def mat_t(self, w):
        out = np.zeros((self.shape[1], w.shape[1]))
        L, R = self.stacked()
        if L is not None:
            out += R @ (L.T @ w)
        for p, q in self.pend:
            out += q.mat_t(p.mat_t(w))
        return out


def thin_product(p: View, q: View):
    """Low-rank product of a sub-pair with a factored side (``sumexpr.py:93-117``).

    Returns ``(LR, kind)`` with kind in {"FF", "FX", "XF"} for the term-list check.
    """
    m, n = p.shape[0], q.shape[1]
    if p.lowrank and q.lowrank:
        a, b = p.H.data[p.b], q.H.data[q.b]
        if min(a.rank, b.rank) == 0:
            return empty_lr(m, n), "FF"
        core = a.right.T @ b.left
        if a.rank <= b.rank:
            return LR(a.left, b.right @ core.T), "FF"
        return LR(a.left @ core, b.right), "FF"
    if p.lowrank:
        a = p.H.data[p.b]
        if a.rank == 0:
            return empty_lr(m, n), "FX"
        return LR(a.left, q.mat_t(a.right)), "FX"
    b = q.H.data[q.b]
    if b.rank == 0:
        return empty_lr(m, n), "XF"
    return LR(p.mat(b.left), b.right), "XF"


def split_pending(p: View, q: View, t_child, s_child):
    """Sub-pairs of a pending pair on one child (``sumexpr.py:120-133``)."""
    bt = p.H.bt
    tree = bt.tree
    if p.inner:
        rho = bt.sigma[p.b]
        out = []
        for rc in tree.children[rho]:
            pc = View(p.H, bt.child_for(p.b, t_child, int(rc)))
            qc = View(q.H, bt.child_for(q.b, int(rc), s_child))
            out.append((pc, qc))
        return out
    return [(View(p.H, p.b, int(tree.lo[t_child]), int(tree.hi[t_child]), p.c0, p.c1),
             View(q.H, q.b, q.r0, q.r1, int(tree.lo[s_child]), int(tree.hi[s_child])))]


def root_expr(A: HMatO, B: HMatO):
    """``sumexpr_root`` (``sumexpr.py:78-83``)."""
    if A.bt is not B.bt:
        raise ValueError("factors must live on the same block-cluster tree")
    return SumExprO(A.bt, 0, A.bt.shape(0), [], [(View(A, 0), View(B, 0))])


def descend(s: SumExprO, child, log=None):
    """``restrict`` (``sumexpr.py:136-154``): exact child expression.

    ``log`` (optional list) receives one record per created term:
    ``(child, kind, A node, B node, rank)``.
    """
    bt = s.bt
    if child not in bt.children[s.b]:
        raise ValueError("not a child of this block")
    pr0, _ = bt.rows(s.b)
    pc0, _ = bt.cols(s.b)
    r0, r1 = bt.rows(child)
    c0, c1 = bt.cols(child)
    lrs = [LR(t.left[r0 - pr0:r1 - pr0], t.right[c0 - pc0:c1 - pc0])
           for t in s.lrs if t.rank > 0]
    pend = []
    for p, q in s.pend:
        for pc, qc in split_pending(p, q, int(bt.tau[child]), int(bt.sigma[child])):
            if pc.lowrank or qc.lowrank:
                term, kind = thin_product(pc, qc)
                if term.rank > 0:
                    lrs.append(term)
                    if log is not None:
                        log.append((child, kind, pc.b, qc.b, term.rank))
            else:
                pend.append((pc, qc))
    return SumExprO(bt, child, (r1 - r0, c1 - c0), lrs, pend)


def dense_eval(s: SumExprO):
    """``evaluate_dense`` (``sumexpr.py:165-170``)."""
    m, n = s.shape
    if m * n > DENSE_CAP ** 2:
        raise ValueError("block too large to materialize")
    return s.mat(np.eye(n))


# --------------------------------------------------------------------------- product

@dataclass
class ReportO:
    """``MultReport`` (``multiply.py:50-58``)."""
    degraded_blocks: int = 0
    max_far_rank: int = 0
    matvec_count: int = 0
    far_leaves: int = 0
    near_leaves: int = 0
    wall_s: float = 0.0
    warnings: list = field(default_factory=list)


def block_seed(seed, node_id):
    """``_block_seed`` (``multiply.py:61-63``)."""
    return (int(seed) << 24) ^ int(node_id)


def far_block(s: SumExprO, b, policy, tag, q=1, seed=0):
    """``_compress_leaf`` (``multiply.py:66-79``) minus the report bookkeeping."""
    s.count = 0
    out = compress_o(s, policy_of(policy), tag, q=q, seed=block_seed(seed, b))
    return out, s.count


def hmult_new_o(A: HMatO, B: HMatO, policy, tag="dense-svd", q=1, seed=0, log=None,
                only=None):
    """``hmult_new`` (``multiply.py:207-256``): DFS over the block tree, compress far
    leaves from their exact sum-expression, evaluate near leaves densely.

    ``only`` (optional set of leaf ids) restricts the work to the listed output leaves
    (their ancestors are still descended): the per-block oracle for large configs.
    """
    bt = A.bt
    rep = ReportO()
    data, bad = {}, set()
    t0 = time.perf_counter()
    need = None
    if only is not None:
        need = set()
        parent = _parents(bt)
        for b in only:
            x = b
            while x >= 0:
                need.add(x)
                x = parent[x]

    def walk(s, b):
        if bt.kind[b] == INNER:
            for c in bt.children[b]:
                if need is None or int(c) in need:
                    walk(descend(s, int(c), log), int(c))
        elif bt.kind[b] == FAR:
            blk, cnt = far_block(s, b, policy, tag, q, seed)
            rep.matvec_count += cnt
            if blk.degraded:
                rep.degraded_blocks += 1
                r0, r1 = bt.rows(b)
                c0, c1 = bt.cols(b)
                rep.warnings.append(f"block {b} rows [{r0},{r1}) cols [{c0},{c1}): "
                                    "compression did not certify convergence")
                bad.add(b)
            rep.far_leaves += 1
            rep.max_far_rank = max(rep.max_far_rank, blk.rank)
            data[b] = blk
        else:
            rep.near_leaves += 1
            data[b] = dense_eval(s)

    walk(root_expr(A, B), 0)
    rep.wall_s = time.perf_counter() - t0
    out = HMatO(bt, data, bad)
    out.report = rep
    return out


# ------------------------------------------------------------- traditional-mode product

def lr_from_dense(a, policy):
    """``from_dense`` (``lowrank.py:50-54``): truncated SVD of a dense block."""
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    r = eps_rank(s, policy)
    return LR(u[:, :r] * s[:r], vt[:r].T.copy())


def lr_norm(t: LR):
    """``LowRank.norm`` (``lowrank.py:38-43``): Frobenius norm by the k x k Gram trick."""
    if t.rank == 0:
        return 0.0
    g = (t.left.T @ t.left) @ (t.right.T @ t.right)
    return float(np.sqrt(max(np.trace(g), 0.0)))


def truncated_sum_o(terms, policy):
    """``fast_truncate_sum`` (``lowrank.py:123-138``): fold each term into a running
    truncated sum (the first two are added before the first truncation)."""
    if not terms:
        raise ValueError("need at least one term")
    if len(terms) == 1:
        return lr_truncate(terms[0], policy)
    acc = lr_truncate(LR(np.hstack([terms[0].left, terms[1].left]),
                         np.hstack([terms[0].right, terms[1].right])), policy)
    for t in terms[2:]:
        acc = lr_truncate(LR(np.hstack([acc.left, t.left]), np.hstack([acc.right, t.right])),
                          policy)
    return acc


def _pad_o(t: LR, r0, r1, c0, c1, m, n):
    """``_pad_child`` (``multiply.py:103-109``): zero-pad a cell's factors to the block."""
    left = np.zeros((m, t.rank))
    right = np.zeros((n, t.rank))
    left[r0:r1] = t.left
    right[c0:c1] = t.right
    return LR(left, right)


def pair_hier_o(p: View, q: View, policy):
    """``_pair_structural_lowrank`` (``multiply.py:140-189``): bottom-up conversion of a
    pending pair on the grid of its children; each cell folds its middle-cluster
    contributions, then the cells are folded in row-child-major order."""
    if not p.inner:
        return lr_from_dense(p.dense_block() @ q.dense_block(), policy)
    bt = p.H.bt
    tree = bt.tree
    taus = tree.children[bt.tau[p.b]]
    sigmas = tree.children[bt.sigma[q.b]]
    rhos = tree.children[bt.sigma[p.b]]
    m, n = p.shape[0], q.shape[1]
    pr0, _ = bt.rows(p.b)
    qc0, _ = bt.cols(q.b)
    cells = []
    for tau in taus:
        for sigma in sigmas:
            contrib = []
            for rho in rhos:
                pc = View(p.H, bt.child_for(p.b, int(tau), int(rho)))
                qc = View(q.H, bt.child_for(q.b, int(rho), int(sigma)))
                if pc.lowrank or qc.lowrank:
                    term, _ = thin_product(pc, qc)
                elif pc.inner:
                    term = pair_hier_o(pc, qc, policy)
                else:
                    term = lr_from_dense(pc.dense_block() @ qc.dense_block(), policy)
                if term.rank > 0:
                    contrib.append(term)
            if contrib:
                cell = truncated_sum_o(contrib, policy)
                t0, t1 = int(tree.lo[tau]) - pr0, int(tree.hi[tau]) - pr0
                s0, s1 = int(tree.lo[sigma]) - qc0, int(tree.hi[sigma]) - qc0
                cells.append(_pad_o(cell, t0, t1, s0, s1, m, n))
    if not cells:
        return empty_lr(m, n)
    return truncated_sum_o(cells, policy)


class PairOpO(Op):
    """``_PairProductMap`` (``multiply.py:82-100``): a pending pair as a linear operator."""

    def __init__(self, p: View, q: View):
        super().__init__()
        self.p, self.q = p, q
        self.shape = (p.shape[0], q.shape[1])

    def mat(self, v):
        return self.p.mat(self.q.mat(v))

    def mat_t(self, w):
        return self.q.mat_t(self.p.mat_t(w))


def convert_pair_o(p: View, q: View, policy, converter, b, seed=0, q_it=1):
    """``_convert_pair`` (``multiply.py:192-204``): ``(LR, matvec count)``."""
    if converter == "hier-approx":
        return pair_hier_o(p, q, policy_of(policy)), 0
    op = PairOpO(p, q)
    op.count = 0
    out = compress_o(op, policy_of(policy), converter, q=q_it, seed=block_seed(seed, b))
    return out, op.count


def hmult_traditional_o(A: HMatO, B: HMatO, policy, converter="hier-approx", seed=0,
                        q=1, only=None):
    """``hmult_traditional`` (``multiply.py:207-263`` with ``leaf_traditional``): every
    pending pair of a far leaf is converted to low rank on its own, then the leaf's terms,
    largest norm first (stable), are combined by ``fast_truncate_sum``.  Near leaves are
    evaluated densely as in ``hmult_new``."""
    bt = A.bt
    pol = policy_of(policy)
    rep = ReportO()
    data, bad = {}, set()
    t0 = time.perf_counter()
    need = None
    if only is not None:
        need = set()
        parent = _parents(bt)
        for b in only:
            x = b
            while x >= 0:
                need.add(x)
                x = parent[x]

    def walk(s, b):
        if bt.kind[b] == INNER:
            for c in bt.children[b]:
                if need is None or int(c) in need:
                    walk(descend(s, int(c)), int(c))
        elif bt.kind[b] == FAR:
            terms = [t for t in s.lrs if t.rank > 0]
            for p, qq in s.pend:
                t, cnt = convert_pair_o(p, qq, pol, converter, b, seed, q)
                rep.matvec_count += cnt
                if t.degraded:
                    rep.degraded_blocks += 1
                    rep.warnings.append(f"pair conversion degraded on block {b}")
                terms.append(t)
            terms = [t for t in terms if t.rank > 0]
            if terms:
                terms.sort(key=lambda t: -lr_norm(t))
                blk = truncated_sum_o(terms, pol)
            else:
                blk = empty_lr(*s.shape)
            rep.far_leaves += 1
            rep.max_far_rank = max(rep.max_far_rank, blk.rank)
            data[b] = blk
        else:
            rep.near_leaves += 1
            data[b] = dense_eval(s)

    walk(root_expr(A, B), 0)
    rep.wall_s = time.perf_counter() - t0
    out = HMatO(bt, data, bad)
    out.report = rep
    return out


def _parents(bt: BlockTreeO):
    par = getattr(bt, "_parents", None)
    if par is None:
        par = np.full(bt.n_nodes, -1, dtype=np.int64)
        for b in range(bt.n_nodes):
            for c in bt.children[b]:
                if c >= 0:
                    par[c] = b
        bt._parents = par
    return par


def leaf_expr(A: HMatO, B: HMatO, leaf):
    """``S(leaf)`` by replaying the descent along the root-to-leaf chain only."""
    bt = A.bt
    par = _parents(bt)
    chain = []
    x = leaf
    while x > 0:
        chain.append(x)
        x = int(par[x])
    s = root_expr(A, B)
    for c in reversed(chain):
        s = descend(s, c)
    return s


# --------------------------------------------------------------------------- configs

def make_points(cfg, seed=0):
    """Seeded point clouds of the five BASELINE configs."""
    rng = np.random.default_rng(seed)
    n, geom = cfg["n"], cfg["geometry"]
    if geom == "square":
        return rng.uniform(0, 1, (n, 2))
    if geom == "cube":
        return rng.uniform(0, 1, (n, 3))
    if geom == "sphere":
        g = rng.standard_normal((n, 3))
        return g / np.linalg.norm(g, axis=1, keepdims=True)
    raise ValueError(geom)


# ------------------------------------------------------------------ HMX1 files
def fingerprint_o(bt: BlockTreeO):
    """``tree_fingerprint`` (``hmatrix.py:334-335``): sha256 of the block-tree dump."""
    import hashlib
    return hashlib.sha256(bt.dump().encode()).digest()


def save_hmatrix_o(H: HMatO, path):
    """``save_hmatrix`` (``hmatrix.py:338-361``): header, then leaf records in ascending id
    with row-major payloads."""
    import struct
    with open(path, "wb") as f:
        f.write(b"HMX1")
        f.write(struct.pack("<IQ", 1, H.bt.n))
        f.write(fingerprint_o(H.bt))
        f.write(struct.pack("<Q", len(H.data)))
        for b in sorted(H.data):
            p = H.data[b]
            flag = 1 if b in H.degraded else 0
            if isinstance(p, LR):
                f.write(struct.pack("<QBBIII", b, 1, flag, p.left.shape[0], p.right.shape[0],
                                    p.rank))
                f.write(np.ascontiguousarray(p.left).tobytes())
                f.write(np.ascontiguousarray(p.right).tobytes())
            else:
                f.write(struct.pack("<QBBII", b, 0, flag, p.shape[0], p.shape[1]))
                f.write(np.ascontiguousarray(p).tobytes())


def load_hmatrix_o(path, bt: BlockTreeO):
    """``load_hmatrix`` (``hmatrix.py:364-388``) with its header checks and messages."""
    import struct
    with open(path, "rb") as f:
        if f.read(4) != b"HMX1":
            raise ValueError("not an H-matrix file")
        version, n = struct.unpack("<IQ", f.read(12))
        if version != 1:
            raise ValueError(f"unsupported version {version}")
        if n != bt.n:
            raise ValueError(f"dimension mismatch: file {n}, tree {bt.n}")
        if f.read(32) != fingerprint_o(bt):
            raise ValueError("block tree does not match the stored operator")
        (count,) = struct.unpack("<Q", f.read(8))
        data, degraded = {}, set()
        for _ in range(count):
            b, kind, flag = struct.unpack("<QBB", f.read(10))
            if flag:
                degraded.add(b)
            if kind == 1:
                m, nn, k = struct.unpack("<III", f.read(12))
                left = np.frombuffer(f.read(8 * m * k)).reshape(m, k).copy()
                right = np.frombuffer(f.read(8 * nn * k)).reshape(nn, k).copy()
                data[b] = LR(left, right)
            else:
                m, nn = struct.unpack("<II", f.read(8))
                data[b] = np.frombuffer(f.read(8 * m * nn)).reshape(m, nn).copy()
    return HMatO(bt, data, degraded)
