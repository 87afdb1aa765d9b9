"""GPU operand assembly (``assemble_hmatrix``, reference ``hmatrix.py:97-118``).

Near leaves are dense kernel blocks; far leaves are compressed by partially pivoted ACA on
kernel entries with the reference's stopping rules and its eps/2 SVD recompression
(``compressors.py:162-247``); a far block whose ACA cannot certify convergence is stored
dense and flagged degraded.  Everything runs in ``libhx.so`` (``hx_assemble``); the packed
pool stays on the device and is attached to later products without a copy.  The host
``data`` dict is filled lazily (one download) on first access.

Point kernels (unit quadrature weights, the BASELINE configs; the reference's
``kernel_block("exp", ...)`` on a unit-area point set equals ``"exp"`` here):
``exp``: exp(-r), ``exp0.5``: exp(-r/0.5), ``gauss0.1``: exp(-r^2/0.1), ``inv``: 1/(r+h).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .hmatrix import HMatrix, LeafDict, block_arrays, tree_arrays
from .lowrank import LowRank
from .multiply import Device

KERNELS = {"exp": 0, "exp0.5": 1, "gauss0.1": 2, "inv": 3}


class DevicePool:
    """A library-owned device pool (freed with the object)."""

    def __init__(self, dev, ptr, n):
        self.dev, self.ptr, self.n = dev, ptr, n

    def download(self):
        host = np.empty(max(self.n, 1), dtype=np.float64)
        _lib.check(_lib.lib().hx_pool_download(self.dev.h, C.c_void_p(self.ptr),
                                               _lib.ptr(host, _lib.f64p), self.n),
                   "hx_pool_download")
        return host[:self.n]

    def __del__(self):
        try:
            if self.ptr:
                _lib.lib().hx_pool_free(self.dev.h, C.c_void_p(self.ptr))
                self.ptr = 0
        except Exception:  # pragma: no cover
            pass


class _LazyLeaves(LeafDict):
    """Leaf payload dict filled from the device pool on first access."""

    def __init__(self, owner):
        super().__init__()
        self._owner = owner
        self._filled = False

    def _fill(self):
        if self._filled:
            return
        self._filled = True
        h = self._owner
        pool, d = h._hx_packed
        if pool is None:  # still only on the device: one download
            pool = h._hx_pool.download()
            h._hx_packed = (pool, d)
        dict.update(self, unpack_leaves(h.bct, pool, d))

    def __contains__(self, key):
        self._fill()
        return super().__contains__(key)

    def __missing__(self, key):
        self._fill()
        if dict.__contains__(self, key):
            return dict.__getitem__(self, key)
        raise KeyError(key)

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __len__(self):
        self._fill()
        return super().__len__()

    def values(self):
        self._fill()
        return super().values()

    def items(self):
        self._fill()
        return super().items()

    def keys(self):
        self._fill()
        return super().keys()


def unpack_leaves(bct, pool, d):
    arr = block_arrays(bct)
    lo, hi = arr.tree.lo, arr.tree.hi
    out = {}
    for b in np.flatnonzero(arr.kind_code != 0):
        m = int(hi[arr.tau[b]] - lo[arr.tau[b]])
        n = int(hi[arr.sigma[b]] - lo[arr.sigma[b]])
        if d["payload"][b] == 1:
            r = int(d["rank"][b])
            u, v = int(d["u_off"][b]), int(d["v_off"][b])
            out[int(b)] = LowRank(pool[u:u + m * r].reshape(r, m).T,
                                  pool[v:v + n * r].reshape(r, n).T)
        else:
            o = int(d["d_off"][b])
            out[int(b)] = pool[o:o + m * n].reshape(n, m).T
    return out


def assemble_hmatrix(kind, bct, policy, panels, h=None, device=0):
    """Assemble the kernel H-matrix on the GPU (reference signature plus ``h``/``device``)."""
    if kind not in KERNELS:
        raise ValueError(f"unknown kernel kind {kind!r} (GPU assembly supports {sorted(KERNELS)})")
    if not hasattr(policy, "eps"):
        raise NotImplementedError("GPU assembly supports EpsRank policies")
    eps = float(policy.eps)
    if not eps > 0:
        raise ValueError("eps must be positive")
    pts = np.asarray(getattr(panels, "centers", panels), dtype=np.float64)
    arr = block_arrays(bct)
    perm = bct.tree.permutation
    tree_pts = np.ascontiguousarray(pts[perm])
    if h is None:
        h = len(pts) ** (-1.0 / tree_pts.shape[1]) if kind == "inv" else 0.0
    ta = tree_arrays(bct)
    tb = _lib.TreeBuf(ta)
    nn = arr.n_nodes
    payload = np.zeros(nn, np.int8)
    rank = np.zeros(nn, np.int32)
    u_off = np.zeros(nn, np.int64)
    v_off = np.zeros(nn, np.int64)
    d_off = np.zeros(nn, np.int64)
    degraded = np.zeros(nn, np.int8)
    pool = C.c_void_p()
    n_el = C.c_int64()
    with Device.lock(device):
        dev = Device.get(device)
        _lib.check(_lib.lib().hx_assemble(
            dev.h, C.byref(tb.st), _lib.ptr(tree_pts, _lib.f64p), tree_pts.shape[1],
            KERNELS[kind], float(h), eps, _lib.ptr(payload, _lib.i8p),
            _lib.ptr(rank, _lib.i32p), _lib.ptr(u_off, _lib.i64p), _lib.ptr(v_off, _lib.i64p),
            _lib.ptr(d_off, _lib.i64p), _lib.ptr(degraded, _lib.i8p), C.byref(pool),
            C.byref(n_el)), "hx_assemble")
    H = HMatrix(bct, {}, set(np.flatnonzero(degraded).tolist()))
    H.data = _LazyLeaves(H)
    H._hx_pool = DevicePool(dev, pool.value, int(n_el.value))
    H._hx_device = (device, pool.value, int(n_el.value))
    H._hx_packed = (None, dict(payload=payload, rank=rank, u_off=u_off, v_off=v_off,
                               d_off=d_off))
    return H


def host_pool(H):
    """The packed host copy of an assembled operand (downloads once)."""
    pool, d = H._hx_packed
    if pool is None:
        pool = H._hx_pool.download()
        H._hx_packed = (pool, d)
    return pool, d
