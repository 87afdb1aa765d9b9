"""Cluster trees and block-cluster trees (host-side structure of the product).

Same API and the same trees, bit for bit, as the reference ``hmat.clustering``
(``/root/reference/pkg/src/hmat/clustering.py``): cardinality-balanced bisection at the
median of a stable sort along the longest bounding-box axis (``clustering.py:61-89``);
blocks ``tau x sigma`` are far when ``min(diam) <= eta * dist`` with Euclidean box
diameters and the largest per-axis gap as distance (``clustering.py:92-107``), inner when
both clusters split, near otherwise; cluster and block ids in DFS pre-order
(``clustering.py:159-160``).

The construction is level-synchronous and vectorised (the reference recurses per node in
Python), and the trees are kept as flat arrays -- the form the C-ABI planner consumes.
Object views (``Cluster``, ``BlockNode``) with the reference's attribute names are built
lazily on first access.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

INNER = "inner"
FAR = "far"
NEAR = "near"
KIND_CODE = {INNER: 0, FAR: 1, NEAR: 2}
KIND_NAME = {0: INNER, 1: FAR, 2: NEAR}

DEFAULT_NMIN = 16
DEFAULT_ETA = 2.0


@dataclass(eq=False)
class Cluster:
    lo: int
    hi: int
    box_lo: np.ndarray
    box_hi: np.ndarray
    level: int
    id: int
    children: tuple = ()

    @property
    def size(self):
        return self.hi - self.lo

    @property
    def is_leaf(self):
        return not self.children


def _assign_preorder(levels_children, levels_count):
    """Pre-order ids for a level-ordered tree.

    ``levels_children[l]`` is an (n_l, c) int array of child indices into level l+1
    (-1 for none); returns one id array per level.
    """
    nlev = len(levels_count)
    sizes = [np.ones(levels_count[l], dtype=np.int64) for l in range(nlev)]
    for l in range(nlev - 2, -1, -1):
        ch = levels_children[l]
        if ch.size == 0:
            continue
        sub = np.where(ch >= 0, sizes[l + 1][np.maximum(ch, 0)], 0)
        sizes[l] = 1 + sub.sum(axis=1)
    ids = [np.zeros(levels_count[0], dtype=np.int64)]
    for l in range(nlev - 1):
        ch = levels_children[l]
        nxt = np.zeros(levels_count[l + 1], dtype=np.int64)
        if ch.size:
            sub = np.where(ch >= 0, sizes[l + 1][np.maximum(ch, 0)], 0)
            start = ids[l][:, None] + 1 + np.cumsum(sub, axis=1) - sub
            valid = ch >= 0
            nxt[ch[valid]] = start[valid]
        ids.append(nxt)
    return ids


class ClusterTree:
    """Binary cluster tree over point positions (tree ordering = ``permutation``)."""

    def __init__(self, points, n_min=DEFAULT_NMIN):
        centers = np.asarray(getattr(points, "centers", points), dtype=float)
        if n_min < 1:
            raise ValueError("n_min must be >= 1")
        n = len(centers)
        if n == 0:
            raise ValueError("empty panel set")
        if centers.ndim != 2:
            raise ValueError("points must be an (n, d) array")
        self.n_min = int(n_min)
        perm = np.arange(n)
        lvl_lo, lvl_hi, lvl_blo, lvl_bhi, lvl_child = [], [], [], [], []
        lo = np.array([0], dtype=np.int64)
        hi = np.array([n], dtype=np.int64)
        while True:
            xp = centers[perm]
            # segments of this level need not tie up (leaves of earlier levels drop out)
            cuts = np.empty(2 * len(lo), dtype=np.int64)
            cuts[0::2], cuts[1::2] = lo, hi
            if cuts[-1] == n:
                cuts = cuts[:-1]
            blo = np.minimum.reduceat(xp, cuts, axis=0)[0::2]
            bhi = np.maximum.reduceat(xp, cuts, axis=0)[0::2]
            lvl_lo.append(lo)
            lvl_hi.append(hi)
            lvl_blo.append(blo)
            lvl_bhi.append(bhi)
            split = (hi - lo) > self.n_min
            if not split.any():
                lvl_child.append(np.zeros((len(lo), 0), dtype=np.int64))
                break
            axis = np.argmax(bhi - blo, axis=1)
            pos = np.arange(n)
            start = pos.copy()            # positions outside split segments stay put
            key = pos.astype(float)
            for_split = np.flatnonzero(split)
            seg = np.repeat(for_split, (hi - lo)[for_split])
            where = np.concatenate([np.arange(lo[i], hi[i]) for i in for_split])
            start[where] = lo[seg]
            key[where] = xp[where, axis[seg]]
            order = np.lexsort((key, start))
            perm = perm[order]
            mid = lo + (hi - lo) // 2
            s_idx = np.flatnonzero(split)
            child = np.full((len(lo), 2), -1, dtype=np.int64)
            child[s_idx, 0] = 2 * np.arange(len(s_idx))
            child[s_idx, 1] = 2 * np.arange(len(s_idx)) + 1
            lvl_child.append(child)
            nlo = np.empty(2 * len(s_idx), dtype=np.int64)
            nhi = np.empty(2 * len(s_idx), dtype=np.int64)
            nlo[0::2], nhi[0::2] = lo[s_idx], mid[s_idx]
            nlo[1::2], nhi[1::2] = mid[s_idx], hi[s_idx]
            lo, hi = nlo, nhi
        counts = [len(x) for x in lvl_lo]
        ids = _assign_preorder(lvl_child, counts)
        total = sum(counts)
        self.lo = np.empty(total, dtype=np.int64)
        self.hi = np.empty(total, dtype=np.int64)
        self.level = np.empty(total, dtype=np.int64)
        self.box_lo = np.empty((total, centers.shape[1]))
        self.box_hi = np.empty((total, centers.shape[1]))
        self.child = np.full((total, 2), -1, dtype=np.int32)
        for l, idl in enumerate(ids):
            self.lo[idl] = lvl_lo[l]
            self.hi[idl] = lvl_hi[l]
            self.level[idl] = l
            self.box_lo[idl] = lvl_blo[l]
            self.box_hi[idl] = lvl_bhi[l]
            ch = lvl_child[l]
            if ch.size:
                has = ch[:, 0] >= 0
                self.child[idl[has], 0] = ids[l + 1][ch[has, 0]]
                self.child[idl[has], 1] = ids[l + 1][ch[has, 1]]
        self.permutation = perm
        self.depth = int(self.level.max())
        # Euclidean diameters with the reference's scalar arithmetic (clustering.py:92-93)
        ext = self.box_hi - self.box_lo
        self.diam = np.array([float(np.linalg.norm(e)) for e in ext])
        self._clusters = None

    @property
    def n(self):
        return int(self.hi[0] - self.lo[0])

    @property
    def n_clusters(self):
        return len(self.lo)

    @property
    def clusters(self):
        if self._clusters is None:
            objs = [Cluster(int(self.lo[i]), int(self.hi[i]), self.box_lo[i], self.box_hi[i],
                            int(self.level[i]), i) for i in range(self.n_clusters)]
            for i in range(self.n_clusters):
                if self.child[i, 0] >= 0:
                    objs[i].children = (objs[self.child[i, 0]], objs[self.child[i, 1]])
            self._clusters = objs
        return self._clusters

    @property
    def root(self):
        return self.clusters[0]


def build_cluster_tree(panels, n_min=DEFAULT_NMIN):
    """Bisect point/panel centers into a balanced binary cluster tree."""
    return ClusterTree(panels, n_min)


def _box_dist(tree, t, s):
    gaps = np.maximum(tree.box_lo[t] - tree.box_hi[s], tree.box_lo[s] - tree.box_hi[t])
    return np.maximum(0.0, gaps.max(axis=-1))


def admissible(tau, sigma, eta=DEFAULT_ETA):
    """Symmetric admissibility test on two clusters (reference signature)."""
    d = min(float(np.linalg.norm(tau.box_hi - tau.box_lo)),
            float(np.linalg.norm(sigma.box_hi - sigma.box_lo)))
    gaps = np.maximum(tau.box_lo - sigma.box_hi, sigma.box_lo - tau.box_hi)
    return d <= eta * float(max(0.0, gaps.max()))


@dataclass(eq=False)
class BlockNode:
    tau: Cluster
    sigma: Cluster
    kind: str
    level: int
    id: int
    children: tuple = ()

    @property
    def shape(self):
        return (self.tau.size, self.sigma.size)

    @property
    def is_leaf(self):
        return self.kind != INNER


class BlockClusterTree:
    """Block-cluster tree as arrays ``tau, sigma, kind (0/1/2), level, child (n, 4)``."""

    def __init__(self, tree: ClusterTree, eta=DEFAULT_ETA):
        self.tree = tree
        self.eta = float(eta)
        lv_t, lv_s, lv_k, lv_child = [], [], [], []
        t = np.array([0], dtype=np.int64)
        s = np.array([0], dtype=np.int64)
        while len(t):
            dmin = np.minimum(tree.diam[t], tree.diam[s])
            far = dmin <= self.eta * _box_dist(tree, t, s)
            t_split = tree.child[t, 0] >= 0
            s_split = tree.child[s, 0] >= 0
            inner = ~far & t_split & s_split
            kind = np.where(far, 1, np.where(inner, 0, 2))
            lv_t.append(t)
            lv_s.append(s)
            lv_k.append(kind)
            idx = np.flatnonzero(inner)
            child = np.full((len(t), 4), -1, dtype=np.int64)
            child[idx] = 4 * np.arange(len(idx))[:, None] + np.arange(4)[None, :]
            lv_child.append(child)
            tc = tree.child[t[idx]]
            sc = tree.child[s[idx]]
            t = np.stack([tc[:, 0], tc[:, 0], tc[:, 1], tc[:, 1]], axis=1).ravel().astype(np.int64)
            s = np.stack([sc[:, 0], sc[:, 1], sc[:, 0], sc[:, 1]], axis=1).ravel().astype(np.int64)
        counts = [len(x) for x in lv_t]
        ids = _assign_preorder(lv_child, counts)
        total = sum(counts)
        self.tau = np.empty(total, dtype=np.int32)
        self.sigma = np.empty(total, dtype=np.int32)
        self.kind_code = np.empty(total, dtype=np.int8)
        self.level = np.empty(total, dtype=np.int32)
        self.child = np.full((total, 4), -1, dtype=np.int32)
        for l, idl in enumerate(ids):
            self.tau[idl] = lv_t[l]
            self.sigma[idl] = lv_s[l]
            self.kind_code[idl] = lv_k[l]
            self.level[idl] = l
            ch = lv_child[l]
            has = ch[:, 0] >= 0
            if not has.any():
                continue
            for c in range(4):
                self.child[idl[has], c] = ids[l + 1][ch[has, c]]
        self._nodes = None

    # ---- array helpers
    @property
    def n(self):
        return self.tree.n

    @property
    def n_nodes(self):
        return len(self.tau)

    @property
    def depth(self):
        return int(self.level.max())

    def rows(self, b):
        t = self.tau[b]
        return int(self.tree.lo[t]), int(self.tree.hi[t])

    def cols(self, b):
        s = self.sigma[b]
        return int(self.tree.lo[s]), int(self.tree.hi[s])

    def leaf_ids(self):
        return np.flatnonzero(self.kind_code != 0)

    # ---- reference object API
    @property
    def nodes(self):
        if self._nodes is None:
            cl = self.tree.clusters
            objs = [BlockNode(cl[self.tau[i]], cl[self.sigma[i]], KIND_NAME[int(self.kind_code[i])],
                              int(self.level[i]), i) for i in range(self.n_nodes)]
            for i in np.flatnonzero(self.child[:, 0] >= 0):
                objs[i].children = tuple(objs[c] for c in self.child[i])
            self._nodes = objs
        return self._nodes

    @property
    def root(self):
        return self.nodes[0]

    @property
    def leaves(self):
        nodes = self.nodes
        return [nodes[i] for i in self.leaf_ids()]

    def far_leaves(self):
        nodes = self.nodes
        return [nodes[i] for i in np.flatnonzero(self.kind_code == 1)]

    def near_leaves(self):
        nodes = self.nodes
        return [nodes[i] for i in np.flatnonzero(self.kind_code == 2)]


def build_block_cluster_tree(tree, eta=DEFAULT_ETA):
    """Pair clusters level by level, splitting inadmissible blocks."""
    return BlockClusterTree(tree, eta)


def sparsity_constant(bct):
    """Largest number of blocks sharing one row cluster."""
    return int(np.bincount(bct.tau).max())


def dump_tree(bct):
    """Textual block listing, one line per node in DFS pre-order (reference format)."""
    lo, hi = bct.tree.lo, bct.tree.hi
    out = []
    for b in range(bct.n_nodes):   # ids are pre-order, so id order is DFS order
        t, s = bct.tau[b], bct.sigma[b]
        out.append(f"level {bct.level[b]} rows [{lo[t]},{hi[t]}) cols [{lo[s]},{hi[s]}) "
                   f"{KIND_NAME[int(bct.kind_code[b])]}")
    return "\n".join(out) + "\n"


def tree_arrays(bct):
    """Arrays for the C-ABI ``hx_tree`` (cluster lo/hi/children, block tau/sigma/kind/child)."""
    tr = bct.tree
    return dict(c_lo=np.ascontiguousarray(tr.lo, dtype=np.int64),
                c_hi=np.ascontiguousarray(tr.hi, dtype=np.int64),
                c_child=np.ascontiguousarray(tr.child, dtype=np.int32),
                tau=np.ascontiguousarray(bct.tau, dtype=np.int32),
                sigma=np.ascontiguousarray(bct.sigma, dtype=np.int32),
                kind=np.ascontiguousarray(bct.kind_code, dtype=np.int8),
                child=np.ascontiguousarray(bct.child, dtype=np.int32))


def is_uniform(bct):
    """True when every leaf cluster sits at the same depth (no dense sub-views arise)."""
    tr = bct.tree
    leaf = tr.child[:, 0] < 0
    return bool(np.all(tr.level[leaf] == tr.depth))
