"""H-matrix container (API of ``hmat.hmatrix.HMatrix``) and the packed device-pool layout.

``HMatrix(bct, data, degraded)`` keeps one payload per leaf of the block-cluster tree:
an ndarray on near leaves, a ``LowRank`` on far leaves (``hmatrix.py:48-65``).  All
vectors and blocks are in tree ordering (``hmatrix.py:103-108``).

``pack_operand`` lays an operand out the way the GPU consumes it: one float64 pool with,
per leaf, ``left`` (m x k) then ``right`` (n x k) for low-rank leaves or the m x n block for
dense leaves, all column-major and 128-byte aligned, plus a per-node directory (payload
kind, rank, offsets) -- the ``hx_operand`` of ``include/hx.h``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import clustering
from .lowrank import LowRank

MAX_DENSE = 6144


class HMatrix:
    def __init__(self, bct, data, degraded=None):
        self.bct = bct
        self.data = data
        self.degraded = set(degraded or ())
        self.report = None

    @property
    def n(self):
        return self.bct.n

    @property
    def shape(self):
        return (self.n, self.n)

    def max_far_rank(self):
        return max((p.rank for p in self.data.values() if isinstance(p, LowRank)), default=0)


class _RefTreeArrays:
    """Array view of a reference (object) block-cluster tree."""

    def __init__(self, bct):
        clusters = bct.tree.clusters
        nc = len(clusters)
        self.tree = type("T", (), {})()
        self.tree.lo = np.array([c.lo for c in clusters], dtype=np.int64)
        self.tree.hi = np.array([c.hi for c in clusters], dtype=np.int64)
        ch = np.full((nc, 2), -1, dtype=np.int32)
        for c in clusters:
            if c.children:
                ch[c.id] = [c.children[0].id, c.children[1].id]
        self.tree.child = ch
        self.tree.n = bct.n
        nodes = bct.nodes
        nn = len(nodes)
        self.tau = np.array([b.tau.id for b in nodes], dtype=np.int32)
        self.sigma = np.array([b.sigma.id for b in nodes], dtype=np.int32)
        self.kind_code = np.array([clustering.KIND_CODE[b.kind] for b in nodes], dtype=np.int8)
        self.level = np.array([b.level for b in nodes], dtype=np.int32)
        self.child = np.full((nn, 4), -1, dtype=np.int32)
        for b in nodes:
            if b.children:
                self.child[b.id] = [c.id for c in b.children]
        self.n = bct.n
        self.n_nodes = nn


def block_arrays(bct):
    """Array form of any block-cluster tree (ours, or the reference's object tree)."""
    if hasattr(bct, "kind_code"):
        return bct
    cached = getattr(bct, "_hx_arrays", None)
    if cached is None:
        cached = _RefTreeArrays(bct)
        try:
            bct._hx_arrays = cached
        except AttributeError:  # pragma: no cover
            pass
    return cached


def tree_arrays(bct):
    arr = block_arrays(bct)
    tr = arr.tree
    return dict(c_lo=np.ascontiguousarray(tr.lo, dtype=np.int64),
                c_hi=np.ascontiguousarray(tr.hi, dtype=np.int64),
                c_child=np.ascontiguousarray(tr.child, dtype=np.int32),
                tau=np.ascontiguousarray(arr.tau, dtype=np.int32),
                sigma=np.ascontiguousarray(arr.sigma, dtype=np.int32),
                kind=np.ascontiguousarray(arr.kind_code, dtype=np.int8),
                child=np.ascontiguousarray(arr.child, dtype=np.int32))


def _is_lowrank(p):
    return hasattr(p, "left") and hasattr(p, "right")


def pack_operand(h):
    """Pack an operand's leaves into one column-major float64 pool + directory."""
    arr = block_arrays(h.bct)
    nn = arr.n_nodes
    payload = np.zeros(nn, dtype=np.int8)
    rank = np.zeros(nn, dtype=np.int32)
    u_off = np.zeros(nn, dtype=np.int64)
    v_off = np.zeros(nn, dtype=np.int64)
    d_off = np.zeros(nn, dtype=np.int64)
    leaves = np.flatnonzero(arr.kind_code != 0)
    for b in leaves:
        p = h.data[int(b)]
        if _is_lowrank(p):
            payload[b] = 1
            rank[b] = p.left.shape[1]
        else:
            payload[b] = 2
    # panel order of the device pools (hx_operand_layout, include/hx.h)
    from . import _lib
    tb = _lib.TreeBuf(tree_arrays(h.bct))
    total = np.zeros(1, dtype=np.int64)
    _lib.check(_lib.lib().hx_operand_layout(
        C.byref(tb.st), _lib.ptr(payload, _lib.i8p), _lib.ptr(rank, _lib.i32p),
        _lib.ptr(u_off, _lib.i64p), _lib.ptr(v_off, _lib.i64p), _lib.ptr(d_off, _lib.i64p),
        _lib.ptr(total, _lib.i64p)), "hx_operand_layout")
    pos = int(total[0])
    pool = np.zeros(max(pos, 16), dtype=np.float64)
    for b in leaves:
        p = h.data[int(b)]
        if payload[b] == 1:
            k = rank[b]
            if k:
                m, n = p.left.shape[0], p.right.shape[0]
                pool[u_off[b]:u_off[b] + m * k] = np.asarray(p.left, dtype=float).T.ravel()
                pool[v_off[b]:v_off[b] + n * k] = np.asarray(p.right, dtype=float).T.ravel()
        else:
            a = np.asarray(p, dtype=float)
            pool[d_off[b]:d_off[b] + a.size] = a.T.ravel()
    return pool, dict(payload=payload, rank=rank, u_off=u_off, v_off=v_off, d_off=d_off)


def to_dense(h):
    """Materialize the H-matrix in tree ordering (host helper for checks)."""
    if h.n > MAX_DENSE:
        raise ValueError(f"dense conversion capped at {MAX_DENSE}, got {h.n}")
    arr = block_arrays(h.bct)
    lo, hi = arr.tree.lo, arr.tree.hi
    out = np.zeros((h.n, h.n))
    for b in np.flatnonzero(arr.kind_code != 0):
        p = h.data[int(b)]
        blk = p.left @ p.right.T if _is_lowrank(p) else p
        t, s = arr.tau[b], arr.sigma[b]
        out[lo[t]:hi[t], lo[s]:hi[s]] = blk
    return out


def frobenius_norm(h):
    """Blockwise Frobenius norm; low-rank blocks via the k x k Gram trick."""
    total = 0.0
    for p in h.data.values():
        if _is_lowrank(p):
            if p.left.shape[1]:
                g = (p.left.T @ p.left) @ (p.right.T @ p.right)
                total += max(float(np.trace(g)), 0.0)
        else:
            total += float(np.sum(p * p))
    return float(np.sqrt(total))
