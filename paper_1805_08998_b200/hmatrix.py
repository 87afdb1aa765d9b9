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
import hashlib
import os

import numpy as np

from . import clustering
from .lowrank import LowRank

MAX_DENSE = 6144


class LeafDict(dict):
    """The ``data`` dict of an ``HMatrix``: a plain ``{leaf id: payload}`` dict that counts
    its mutations.  The packed operand pool (and a device copy of it) is cached on the
    ``HMatrix`` under the dict's identity and version, so assigning, deleting or updating
    entries -- or replacing ``h.data`` -- makes the next product or ``save_hmatrix`` repack
    instead of using stale payloads.  Lazy subclasses (payloads unpacked from a pool on
    first access) fill themselves before any mutation, and ``get`` / ``copy`` see lazy
    entries like indexing does."""

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        self.version = 0

    def _fill(self):  # lazy subclasses materialize every entry here
        pass

    def __setitem__(self, key, value):
        self._fill()
        super().__setitem__(key, value)
        self.version += 1

    def __delitem__(self, key):
        self._fill()
        super().__delitem__(key)
        self.version += 1

    def update(self, *args, **kw):
        self._fill()
        super().update(*args, **kw)
        self.version += 1

    def pop(self, *args):
        self._fill()
        self.version += 1
        return super().pop(*args)

    def popitem(self):
        self._fill()
        self.version += 1
        return super().popitem()

    def setdefault(self, key, default=None):
        if key in self:
            return self[key]
        self[key] = default
        return default

    def clear(self):
        self._fill()
        super().clear()
        self.version += 1

    def get(self, key, default=None):
        try:
            return self[key]
        except KeyError:
            return default

    def copy(self):
        self._fill()
        return dict(self.items())


class HMatrix:
    def __init__(self, bct, data, degraded=None):
        self.bct = bct
        self.data = data
        self.degraded = set(degraded or ())
        self.report = None

    @property
    def data(self):
        return self._data

    @data.setter
    def data(self, value):
        # a plain dict is taken over as a LeafDict (same entries) so that its mutations
        # invalidate the packed-pool cache
        self._data = value if isinstance(value, LeafDict) else LeafDict(value)

    def _data_key(self):
        return (id(self._data), self._data.version)

    @property
    def _hx_packed(self):
        """(host pool or None, directory) of the packed operand, or None when the payloads
        changed since it was packed (the device copy is dropped with it)."""
        c = self.__dict__.get("_hx_packed_c")
        if c is None:
            return None
        if c[1] != self._data_key():
            for name in ("_hx_packed_c", "_hx_device", "_hx_pool", "_hx_pool_pinned"):
                self.__dict__.pop(name, None)
            return None
        return c[0]

    @_hx_packed.setter
    def _hx_packed(self, value):
        self.__dict__["_hx_packed_c"] = (value, self._data_key())

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


# ------------------------------------------------------------------ HMX1 operator files
class _PoolLeaves(LeafDict):
    """Leaf payloads unpacked on first access from a packed host pool (loaded operands)."""

    def __init__(self, owner):
        super().__init__()
        self._owner = owner
        self._filled = False

    def _fill(self):
        if self._filled:
            return
        self._filled = True
        from .assembly import unpack_leaves
        h = self._owner
        pool, d = h._hx_packed
        dict.update(self, unpack_leaves(h.bct, pool, d))

    def __missing__(self, key):
        self._fill()
        if dict.__contains__(self, key):
            return dict.__getitem__(self, key)
        raise KeyError(key)

    def __contains__(self, key):
        self._fill()
        return super().__contains__(key)

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __len__(self):
        self._fill()
        return super().__len__()

    def keys(self):
        self._fill()
        return super().keys()

    def values(self):
        self._fill()
        return super().values()

    def items(self):
        self._fill()
        return super().items()


def tree_fingerprint(bct):
    """sha256 of the block-tree dump (reference ``tree_fingerprint``, hmatrix.py:334-335)."""
    return hashlib.sha256(clustering.dump_tree(block_arrays(bct)).encode()).digest()


def _packed(h):
    cached = getattr(h, "_hx_packed", None)
    if cached is None:
        return pack_operand(h)
    pool, d = cached
    if pool is None:  # assembled on the device: one download
        from .assembly import host_pool
        pool, d = host_pool(h)
    return pool, d


def save_hmatrix(h, path):
    """Write the leaf payloads in the HMX1 layout (reference ``save_hmatrix``,
    hmatrix.py:338-361), straight from the packed operand pool (``hx_hmx1_write``)."""
    from . import _lib
    arr = block_arrays(h.bct)
    pool, d = _packed(h)
    tb = _lib.TreeBuf(tree_arrays(h.bct))
    ob = _lib.OperandBuf(d)
    deg = np.zeros(arr.n_nodes, np.int8)
    if h.degraded:
        deg[np.fromiter(h.degraded, dtype=np.int64)] = 1
    fp = np.frombuffer(tree_fingerprint(h.bct), dtype=np.uint8).copy()
    pool = np.ascontiguousarray(pool, dtype=np.float64)
    _lib.check(_lib.lib().hx_hmx1_write(os.fsencode(path), C.byref(tb.st), int(h.n),
                                        _lib.ptr(fp, _lib.u8p), C.byref(ob.st),
                                        _lib.ptr(deg, _lib.i8p), _lib.ptr(pool, _lib.f64p)),
               "save_hmatrix")


def load_hmatrix(path, bct):
    """Read an HMX1 file back (reference ``load_hmatrix``, hmatrix.py:364-388): the header
    checks raise ``ValueError`` with the reference's messages; the payloads land directly in
    a packed pool in panel order (``hx_hmx1_scan`` / ``hx_hmx1_read``), ready for upload;
    ``data`` unpacks lazily into ``LowRank`` / ndarray leaves."""
    from . import _lib
    with open(path, "rb"):  # FileNotFoundError / PermissionError as the reference raises
        pass
    arr = block_arrays(bct)
    nn = arr.n_nodes
    tb = _lib.TreeBuf(tree_arrays(bct))
    payload = np.zeros(nn, np.int8)
    rank = np.zeros(nn, np.int32)
    deg = np.zeros(nn, np.int8)
    pos = np.zeros(nn, np.int64)
    fp = np.frombuffer(tree_fingerprint(bct), dtype=np.uint8).copy()
    _lib.check(_lib.lib().hx_hmx1_scan(os.fsencode(path), C.byref(tb.st), int(bct.n),
                                       _lib.ptr(fp, _lib.u8p), _lib.ptr(payload, _lib.i8p),
                                       _lib.ptr(rank, _lib.i32p), _lib.ptr(deg, _lib.i8p),
                                       _lib.ptr(pos, _lib.i64p)), "load_hmatrix")
    u_off = np.zeros(nn, np.int64)
    v_off = np.zeros(nn, np.int64)
    d_off = np.zeros(nn, np.int64)
    total = np.zeros(1, np.int64)
    _lib.check(_lib.lib().hx_operand_layout(
        C.byref(tb.st), _lib.ptr(payload, _lib.i8p), _lib.ptr(rank, _lib.i32p),
        _lib.ptr(u_off, _lib.i64p), _lib.ptr(v_off, _lib.i64p), _lib.ptr(d_off, _lib.i64p),
        _lib.ptr(total, _lib.i64p)), "hx_operand_layout")
    pool = np.zeros(max(int(total[0]), 16), dtype=np.float64)
    d = dict(payload=payload, rank=rank, u_off=u_off, v_off=v_off, d_off=d_off)
    ob = _lib.OperandBuf(d)
    _lib.check(_lib.lib().hx_hmx1_read(os.fsencode(path), C.byref(tb.st), C.byref(ob.st),
                                       _lib.ptr(pos, _lib.i64p), _lib.ptr(pool, _lib.f64p)),
               "load_hmatrix")
    H = HMatrix(bct, {}, set(np.flatnonzero(deg).tolist()))
    H.data = _PoolLeaves(H)
    H._hx_packed = (pool, d)  # keyed to the lazy dict just installed
    return H
