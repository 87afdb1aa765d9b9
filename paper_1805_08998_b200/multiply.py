"""The tolerance-controlled H x H product on the B200 (drop-in for ``hmat.multiply``).

``hmult_new(h, k, cfg)`` keeps the reference signature, checks and errors
(``multiply.py:252-256``, ``sumexpr.py:80-81``, ``multiply.py:41-47``) and returns an
``HMatrix`` on the same block tree whose far leaves are ``LowRank(U S, V)`` and near
leaves dense, with ``.report`` filled like ``MultReport`` (``multiply.py:50-58``).

All arithmetic runs in ``libhx.so`` (``include/hx.h``): the flat term lists are built by
the C++ planner (the ``restrict`` bookkeeping), then term formation, block
materialization and recompression run as sm_100a kernels.  There is no CPU path: a
missing library or GPU raises.

Execution is chunked: the output leaves are split into chunks of whole subtrees rooted at
the first block level that holds a far leaf.  No term is created above that level
(terms come from far operand blocks), so chunks share no work; each chunk's work lists
are planned on a host thread while the device runs the previous chunk, and device
memory is bounded by the largest chunk instead of the whole product.
"""

from __future__ import annotations

import ctypes as C
import os
import collections
import threading
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .compressors import TAG_CODES, CompressorKind, clamp_eps
from .hmatrix import HMatrix, LeafDict, block_arrays, pack_operand, tree_arrays
from .lowrank import EpsRank, FixedRank, LowRank

CONVERTERS = ("hier-approx", "aca", "bilanczos", "randomized", "dense-svd")


@dataclass(frozen=True)
class MultiplyConfig:
    mode: str = "new"
    compressor: CompressorKind = CompressorKind("aca")
    policy: object = None
    converter: str = "hier-approx"

    def __post_init__(self):
        if self.mode not in ("new", "traditional"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.converter not in CONVERTERS:
            raise ValueError(f"unknown converter {self.converter!r}")
        if self.policy is None:
            raise ValueError("a truncation policy is required")


@dataclass
class MultReport:
    degraded_blocks: int = 0
    max_far_rank: int = 0
    matvec_count: int = 0
    far_leaves: int = 0
    near_leaves: int = 0
    wall_s: float = 0.0
    warnings: list = field(default_factory=list)
    # device-side breakdown (milliseconds, CUDA events, summed over chunks) and plan stats
    plan_ms: float = 0.0
    device_ms: float = 0.0
    form_ms: float = 0.0
    materialize_ms: float = 0.0
    recompress_ms: float = 0.0
    upload_ms: float = 0.0
    out_elems: int = 0
    sketch_rounds: int = 0
    launches: int = 0
    chunks: int = 0
    fro2: float = 0.0


class Device:
    """One ``hx_ctx`` per CUDA device, created lazily and reused across products."""

    _cache: dict = {}

    def __init__(self, device=0):
        h = C.c_void_p()
        _lib.check(_lib.lib().hx_ctx_create(int(device), C.byref(h)), "hx_ctx_create")
        self.h = h
        self.device = device

    @classmethod
    def get(cls, device=0):
        if device not in cls._cache:
            cls._cache[device] = Device(device)
        return cls._cache[device]

    _aux: dict = {}
    _locks: dict = {}
    _locks_guard = threading.Lock()

    @classmethod
    def lock(cls, device=0):
        """Per-device re-entrant lock: the contexts of a device (operand slots, streams,
        workspaces) serve one product or H-matrix x block call at a time."""
        with cls._locks_guard:
            if device not in cls._locks:
                cls._locks[device] = threading.RLock()
            return cls._locks[device]

    @classmethod
    def aux(cls, device=0, i=0):
        """Further contexts on the device (own streams and workspace), i = 0, 1, ..."""
        key = device if i == 0 else (device, i)
        if key not in cls._aux:
            cls._aux[key] = Device(device)
        return cls._aux[key]

    def set_operand(self, which, pool=None, dev_ptr=None, n=None):
        if pool is not None:
            pool = np.ascontiguousarray(pool, dtype=np.float64)
            _lib.check(_lib.lib().hx_ctx_operand(self.h, which, _lib.ptr(pool, _lib.f64p), None,
                                                 pool.size), "hx_ctx_operand")
        else:
            _lib.check(_lib.lib().hx_ctx_operand(self.h, which, None, C.c_void_p(dev_ptr),
                                                 int(n)), "hx_ctx_operand")

    def alias_b(self):
        _lib.check(_lib.lib().hx_ctx_operand_alias(self.h), "hx_ctx_operand_alias")


def _policy_args(policy):
    if isinstance(policy, FixedRank) or hasattr(policy, "k_max"):
        return 1, 1.0, int(policy.k_max)
    eps = float(policy.eps)
    if not eps > 0.0:
        raise ValueError("eps must be positive")
    return 0, eps, 0


def operand_directory(h):
    """(pool, directory) of an operand, cached on the object (operands are immutable
    inputs of the product)."""
    cached = getattr(h, "_hx_packed", None)
    if cached is None:
        cached = pack_operand(h)
        try:
            h._hx_packed = cached
        except AttributeError:  # pragma: no cover
            pass
    return cached


def plan_tile(bct):
    arr = block_arrays(bct)
    tr = arr.tree
    leaf = tr.child[:, 0] < 0
    nmin = int((tr.hi - tr.lo)[leaf].max())
    return 32 if nmin <= 32 else 64


def _host_directory(h):
    pool, d = operand_directory(h)
    if pool is None:  # assembled on the device: one download of the packed pool
        pool = h._hx_pool.download()
        h._hx_packed = (pool, d)
    if pool.nbytes >= (64 << 20) and not getattr(h, "_hx_pool_pinned", False):
        # page-locked once: every later upload of this operand is a full-speed DMA
        _lib.pin_host_array(pool)
        try:
            h._hx_pool_pinned = True
        except AttributeError:  # pragma: no cover
            pass
    return pool, d


class _ProductLeaves(LeafDict):
    """Leaf payloads of a product, built on first access from the downloaded result
    buffers (zero-copy views: far leaves LowRank(U*S, V), near leaves m x n arrays)."""

    def __init__(self, chunks):
        super().__init__()
        self._chunks = chunks  # (leaves dict, rank, deg, off, res) per chunk
        self._where = None
        self._filled = False

    def _index(self):
        if self._where is None:
            self._where = {}
            for ci, (lv, rank, deg, off, res) in enumerate(self._chunks):
                for i, b in enumerate(lv["ids"].tolist()):
                    self._where[b] = (ci, i)
        return self._where

    def _make(self, ci, i):
        lv, rank, deg, off, res = self._chunks[ci]
        m, n, o = int(lv["m"][i]), int(lv["n"][i]), int(off[i])
        if lv["kind"][i] == 1:
            r = int(rank[i])
            # column-major views; shapes are the plan's, so LowRank's checks are skipped
            x = object.__new__(LowRank)
            object.__setattr__(x, "left", res[o:o + m * r].reshape(r, m).T)
            object.__setattr__(x, "right", res[o + m * r:o + (m + n) * r].reshape(r, n).T)
            object.__setattr__(x, "degraded", bool(deg[i]))
            return x
        return res[o:o + m * n].reshape(n, m).T

    def __missing__(self, key):
        w = self._index().get(key)
        if w is None:
            raise KeyError(key)
        v = self._make(*w)
        dict.__setitem__(self, key, v)
        return v

    def __contains__(self, key):
        return key in self._index() if not self._filled else dict.__contains__(self, key)

    def _fill(self):
        if self._filled:
            return
        for ci, (lv, *_rest) in enumerate(self._chunks):
            for i, b in enumerate(lv["ids"].tolist()):
                if not dict.__contains__(self, b):
                    dict.__setitem__(self, b, self._make(ci, i))
        self._filled = True

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __len__(self):
        return len(self._index()) if not self._filled else dict.__len__(self)

    def keys(self):
        self._fill()
        return super().keys()

    def values(self):
        self._fill()
        return super().values()

    def items(self):
        self._fill()
        return super().items()


# --------------------------------------------------------------------------- chunks

def _subtree_end(arr):
    """end[b] = one past the last pre-order id of b's subtree."""
    n = arr.n_nodes
    size = np.ones(n, dtype=np.int64)
    child = arr.child
    for b in range(n - 1, -1, -1):
        c = child[b]
        if c[0] >= 0:
            size[b] += size[c].sum()
    return np.arange(n) + size


def _tree_meta(bct, implicit_min=0):
    """(end of each node's subtree in pre-order, cumulative leaf weight).  The weight of a
    leaf is its area -- what its materialized block and most of its term factors scale
    with -- except for far leaves on the implicit route (min(m, n) >= ``implicit_min`` > 0),
    which are never materialized: their workspace is the sketch panels, ~64 (m + n).  Chunks
    sized by plain area put a few huge implicit leaves (config 4: 65536 x 65536) on a par with
    10^6 small blocks and had to be re-planned when they came out ten times too large."""
    arr = block_arrays(bct)
    cache = getattr(arr, "_hx_meta", None)
    if cache is None:
        cache = {}
        try:
            arr._hx_meta = cache
        except AttributeError:  # pragma: no cover
            pass
    meta = cache.get(int(implicit_min))
    if meta is None:
        kind = arr.kind_code
        lo, hi = arr.tree.lo, arr.tree.hi
        m = hi[arr.tau] - lo[arr.tau]
        n = hi[arr.sigma] - lo[arr.sigma]
        area = np.where(kind != 0, m * n, 0)
        if implicit_min > 0:
            impl = (kind == 1) & (np.minimum(m, n) >= implicit_min)
            area = np.where(impl, np.minimum(64 * (m + n), m * n), area)
        end = cache[0][0] if 0 in cache else _subtree_end(arr)
        meta = (end, np.concatenate([[0], np.cumsum(area)]))
        cache[int(implicit_min)] = meta
    return meta


def chunk_units(bct, implicit_min=0):
    """Disjoint pre-order id ranges covering every leaf: the subtrees rooted at the first
    block level holding a far leaf, and the leaves above it; with their leaf weights
    (``_tree_meta``)."""
    arr = block_arrays(bct)
    kind, level = arr.kind_code, arr.level
    far_lv = level[kind == 1]
    lf = int(far_lv.min()) if far_lv.size else int(level.max())
    end, carea = _tree_meta(bct, implicit_min)
    roots = np.flatnonzero((level == lf) | ((level < lf) & (kind != 0)))
    return [(int(b), int(end[b]), float(carea[end[b]] - carea[b])) for b in roots]


def split_chunk(bct, group, implicit_min=0):
    """Halve a chunk (list of units); a single unit splits into its child subtrees (their
    common ancestors' terms are then planned for each part)."""
    if len(group) > 1:
        h = len(group) // 2
        return [group[:h], group[h:]]
    b0, b1, _ = group[0]
    arr = block_arrays(bct)
    end, carea = _tree_meta(bct, implicit_min)
    kids = [int(c) for c in arr.child[b0] if c >= 0]
    if not kids:
        return [group]
    parts = [[(c, int(end[c]), float(carea[end[c]] - carea[c]))] for c in kids]
    return parts


def chunk_groups(bct, n_chunks, first=1.0, weights=None, implicit_min=0):
    """About `n_chunks` chunks of consecutive units; chunk i gets a share of the leaf area
    proportional to weights[i] (default: the first one `first`, the others 1)."""
    units = chunk_units(bct, implicit_min)
    total = sum(u[2] for u in units)
    n_chunks = max(1, n_chunks)
    env = os.environ.get("HX_CHUNK_WEIGHTS")
    if env and len(env.split(",")) == n_chunks:
        weights = [float(x) for x in env.split(",")]
    elif weights is None:
        weights = [first] + [1.0] * (n_chunks - 1)
    bounds = np.cumsum(weights) / sum(weights) * total
    groups, cur, acc = [], [], 0.0
    for u in units:
        cur.append(u)
        acc += u[2]
        if len(groups) < n_chunks - 1 and acc >= bounds[len(groups)]:
            groups.append(cur)
            cur = []
    if cur:
        groups.append(cur)
    return groups


def group_mask(bct, group, base_mask=None):
    arr = block_arrays(bct)
    leaf = arr.kind_code != 0
    m = np.zeros(arr.n_nodes, dtype=np.uint8)
    for b0, b1, _ in group:
        m[b0:b1] = leaf[b0:b1]
    if base_mask is not None:
        m &= (np.asarray(base_mask) != 0).astype(np.uint8)
    return m


def chunk_masks(bct, n_chunks, base_mask=None):
    """Leaf masks of about `n_chunks` chunks (multi-GPU helpers and tests)."""
    out = [group_mask(bct, g, base_mask) for g in chunk_groups(bct, n_chunks)]
    return [m for m in out if m.any()]


def subtree_partition(bct, leaf_cost, world, min_units_per_rank=8, unit_cost=None):
    """Multi-GPU partition of the output leaves: whole subtrees (the chunk
    units: subtrees at the first block level holding a far leaf, split further while
    there are fewer than ``min_units_per_rank`` per rank or one unit outweighs a quarter of
    a rank's share) go to ranks by longest-processing-time greedy on their summed leaf
    cost.  A rank then forms only the terms of its own subtrees (plus the few created at
    the split points), so no term formation is repeated across ranks the way a leaf-wise
    partition would repeat it at every shared ancestor.  ``leaf_cost`` is indexed by node
    id; ``unit_cost(units) -> costs`` (optional) prices the final units for the greedy
    assignment, e.g. from their own plans (``plan_unit_costs``).  Returns (owner rank per
    unit, the units, per-rank load, per-rank leaf masks)."""
    arr = block_arrays(bct)
    leaf = arr.kind_code != 0
    cc = np.concatenate([[0.0], np.cumsum(np.where(leaf, leaf_cost, 0.0))])

    def cost(u):
        return float(cc[u[1]] - cc[u[0]])

    units = [(u[0], u[1]) for u in chunk_units(bct)]
    total = cost((0, arr.n_nodes))
    frozen = set()  # leaf units (nothing to split)
    for _ in range(64 * world):
        cand = [j for j in range(len(units)) if units[j] not in frozen]
        if not cand:
            break
        i = max(cand, key=lambda j: cost(units[j]))
        if len(units) >= min_units_per_rank * world and \
                max(cost(u) for u in units) <= total / (4.0 * world):
            break
        parts = split_chunk(bct, [(units[i][0], units[i][1], 0.0)])
        if len(parts) == 1:
            frozen.add(units[i])
            continue
        # the unit root is an inner block without payload: its children's subtrees cover it
        units[i:i + 1] = [(p[0][0], p[0][1]) for p in parts]
    ucost = np.array([cost(u) for u in units]) if unit_cost is None else \
        np.asarray(unit_cost(units), dtype=float)
    owner = np.zeros(len(units), dtype=np.int64)
    load = np.zeros(world)
    for i in np.argsort(-ucost, kind="stable"):
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += ucost[i]
    masks = []
    for r in range(world):
        m = np.zeros(arr.n_nodes, dtype=np.uint8)
        for (b0, b1), o in zip(units, owner):
            if o == r:
                m[b0:b1] = leaf[b0:b1]
        masks.append(m)
    return owner, units, load, masks


# per-phase rates of one B200 on config 2 (isolated phase times / plan work): term
# formation ~3.8 TB/s of canonical bytes, materialization ~28 TFLOP/s, recompression
# ~2.4 us per far leaf plus its sketch work
FORM_BPS = 3.8e12
MAT_FPS = 28e12
FAR_S = 2.4e-6
SKETCH_BPS = 2.0e12  # gathered sketch products of the implicit leaves
# a rank's wall time is the larger of its device time and its host planning time (the two
# overlap chunk by chunk); the planning time of a unit is measured on its own plan


def plan_unit_costs(h, k, units, tile=None, tag="dense-svd"):
    """Estimated seconds of each unit (a subtree's masked plan): the larger of its device
    time (formation bytes, materialization flops of its near and materialized far leaves,
    the sketch passes of its implicit leaves, a per-far-leaf recompression term) and its
    host planning time (measured: the time its plan took, work lists included).  The plans
    take the route the product of compressor ``tag`` takes (implicit above its threshold).
    For the multi-GPU partition (these plans are made once, outside the timed step)."""
    arr = block_arrays(h.bct)
    leaf = arr.kind_code != 0
    _, da = operand_directory(h)
    _, db = (None, da) if k is h else operand_directory(k)
    ta = tree_arrays(h.bct)
    tile = tile or plan_tile(h.bct)
    iflags = implicit_flags(None, tag)
    imin = (1 << ((iflags >> 8) & 31)) if iflags else 0  # HX_PLAN_IMPLICIT_SHIFT
    out = []
    if units:  # warm-up: the first plan also grows the page-locked plan-array cache
        m = np.zeros(arr.n_nodes, dtype=np.uint8)
        m[units[0][0]:units[0][1]] = leaf[units[0][0]:units[0][1]]
        _lib.Plan(ta, da, db, m, tile, flags=iflags).close()
    for b0, b1 in units:
        m = np.zeros(arr.n_nodes, dtype=np.uint8)
        m[b0:b1] = leaf[b0:b1]
        t0 = time.perf_counter()
        p = _lib.Plan(ta, da, db, m, tile, flags=iflags)  # work lists filled: the host work
        host = time.perf_counter() - t0
        lv = p.leaves()
        far = lv["kind"] == 1
        mm, nn, K = lv["m"].astype(float), lv["n"].astype(float), lv["K"].astype(float)
        impl = far & (np.minimum(lv["m"], lv["n"]) >= imin) if imin else np.zeros(len(far), bool)
        mat = float(np.sum(np.where(impl, 0.0, 2.0 * mm * nn * K + lv["fdd"])))
        # implicit leaves: range and co-range passes stream the stacked factors twice
        sk_bytes = float(np.sum(np.where(impl, 2.0 * 8.0 * K * (mm + nn), 0.0)))
        dev = p.info.bytes_form / FORM_BPS + mat / MAT_FPS + sk_bytes / SKETCH_BPS + \
            8.0 * float(p.info.tile_elems) / FORM_BPS + FAR_S * float(far.sum())
        out.append(max(dev, host))
        p.close()
    return out


def plan_bytes(info):
    """Device workspace a plan needs (the buffers hx_product sizes from it)."""
    return 8.0 * (info.term_elems + info.tile_elems + info.core_elems + info.gather_elems) + \
        48.0 * (info.mat_terms + info.core_terms + info.fac_terms) + \
        40.0 * (info.mat_tiles + info.core_tiles + info.fac_tiles)


def available_bytes(dev):
    """Free device memory plus the workspace both contexts of the device hold for reuse."""
    fb, tb = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().hx_ctx_mem_info(dev.h, C.byref(fb), C.byref(tb)), "hx_ctx_mem_info")
    free = float(fb.value)
    for key, aux in Device._aux.items():
        if (key == dev.device or (isinstance(key, tuple) and key[0] == dev.device)) and \
                aux is not dev:
            free += float(_lib.lib().hx_ctx_held_bytes(aux.h))
    return free


def default_chunks(bct, dev=None, overlap=None, leaf_mask=None):
    """(chunks, overlap): enough chunks to keep one chunk's device workspace (materialized
    blocks plus term factors, ~12x the leaf area on the BASELINE configs) within ~60% of
    free memory.  A large product that fits whole runs instead as 3 chunks alternating
    over two contexts: one chunk's latency-bound recompression overlaps the next chunk's
    term formation (config 2: 427 -> 389 ms).  Memory-bound products overlap too, and
    their chunk sizes adapt (``adaptive``): the first chunk's plan gives the workspace per
    unit of leaf area, and the remaining subtrees are regrouped into chunks that fill the
    per-context budget (config 4: 256 -> ~40 chunks).  Returns (chunks, overlap, adaptive)."""
    env = os.environ.get("HX_CHUNKS")
    if env:
        n = max(1, int(env))
        return n, n > 1 and overlap_default(overlap), False
    if leaf_mask is None:
        area = sum(u[2] for u in chunk_units(bct))
    else:  # a rank's share of a multi-GPU partition
        arr = block_arrays(bct)
        lo, hi = arr.tree.lo, arr.tree.hi
        own = np.flatnonzero(np.asarray(leaf_mask) != 0)
        area = float(np.sum((hi[arr.tau[own]] - lo[arr.tau[own]]) *
                            (hi[arr.sigma[own]] - lo[arr.sigma[own]])))
    free = 60e9
    if dev is not None:
        free = available_bytes(dev)
    need = area * 8.0 * 12.0
    n = max(1, int(np.ceil(need / (0.6 * free))))
    if n == 1:
        if area >= float(os.environ.get("HX_OVERLAP_AREA", 2.5e8)) and overlap_default(overlap):
            return len(OVERLAP_WEIGHTS), True, False
        return 1, False, False
    return n, overlap_default(overlap), os.environ.get("HX_ADAPTIVE_CHUNKS", "1") != "0"


# A product that fits whole runs as 4 chunks on 3 contexts: a small first chunk (its
# planning is the only exposed host work), two full ones, and a half-size last one (its
# recompression tail has nothing left to overlap); config 2: 351 -> 339 ms
OVERLAP_WEIGHTS = (0.2, 1.0, 1.0, 0.5)
OVERLAP_CONTEXTS = 3


def regroup_units(groups, rate, target):
    """Consecutive units of the remaining chunks merged into chunks whose estimated
    workspace (rate x leaf area) stays within target bytes."""
    out, cur, acc = [], [], 0.0
    for u in (u for g in groups for u in g):
        est = rate * u[2]
        if cur and acc + est > target:
            out.append(cur)
            cur, acc = [], 0.0
        cur.append(u)
        acc += est
    if cur:
        out.append(cur)
    return out


# --------------------------------------------------------------------------- product

IMPLICIT_MIN = 512  # far leaves with min(m, n) >= this are sketched without materialization
# The matrix-free tags read rows / columns / matvecs of a block (r + 2 of each for ACA):
# from the stacked terms that costs (r + 2) K (m + n) words against 2 m n K flops for
# materializing the block once, so only very large blocks stay implicit for them.
IMPLICIT_MIN_ITERATIVE = 4096


def implicit_flags(implicit_min=None, tag="dense-svd"):
    """HX_PLAN_IMPLICIT bits for a threshold (power of two; 0 disables; env HX_IMPLICIT)."""
    if implicit_min is None:
        implicit_min = int(os.environ.get("HX_IMPLICIT", IMPLICIT_MIN if tag == "dense-svd"
                                          else IMPLICIT_MIN_ITERATIVE))
    if implicit_min <= 0:
        return 0
    lg = int(np.ceil(np.log2(implicit_min)))
    return (lg & 31) << 8


def overlap_default(overlap=None):
    if overlap is None:
        return os.environ.get("HX_OVERLAP", "1") != "0"
    return bool(overlap)


def multiply_device(h, k, cfg, device=0, leaf_mask=None, sketch0=0, oversample=0,
                    device_operands=True, fetch=True, chunks=None, implicit_min=None,
                    overlap=None, device_pools=None, trad=0):
    """Run the product on one GPU and return the product ``HMatrix``.

    ``device_operands``: attach operand pools already resident on this device (GPU
    assembly) instead of uploading the host copy.  ``leaf_mask`` restricts the product to
    the owned output leaves (multi-GPU partition).  ``fetch=False`` leaves the output
    blocks in device memory (only ranks and the report come back): the device-resident
    measurement of bench.py.  ``chunks``: number of pipelined chunks (default by size).
    ``device_pools``: ((ptr, n) of A, (ptr, n) of B), packed pools already on this device
    (replicas of a multi-GPU product, ``distributed.py``).  Calls on the same device are
    serialized (``Device.lock``).  ``trad``: 0 the new-mode product; 1 / 2 the
    traditional-mode product with the hierarchical / one-truncation pair converter
    (``HX_PLAN_TRAD``)."""
    if h.bct is not k.bct:
        raise ValueError("factors must live on the same block-cluster tree")
    with Device.lock(device):
        return _multiply_device(h, k, cfg, device, leaf_mask, sketch0, oversample,
                                device_operands, fetch, chunks, implicit_min, overlap,
                                device_pools, trad)


def _multiply_device(h, k, cfg, device, leaf_mask, sketch0, oversample, device_operands,
                     fetch, chunks, implicit_min, overlap, device_pools, trad=0):
    if h.bct is not k.bct:
        raise ValueError("factors must live on the same block-cluster tree")
    policy = cfg.policy
    kind, eps, kmax = _policy_args(policy)
    if kind == 0 and eps <= np.finfo(float).eps:
        eps = clamp_eps(eps)
    t_start = time.perf_counter()
    same = k is h

    def resident(x):
        if device_pools is not None:
            p = device_pools[0 if x is h else 1]
            return (device, p[0], p[1])
        d = getattr(x, "_hx_device", None)
        return d if (device_operands and d is not None and d[0] == device) else None

    pool_a, dir_a = operand_directory(h) if resident(h) else _host_directory(h)
    if same:
        pool_b, dir_b = pool_a, dir_a
    else:
        pool_b, dir_b = operand_directory(k) if resident(k) else _host_directory(k)
    dev = Device.get(device)
    for d in [dev] + [a for key, a in Device._aux.items()
                      if key == device or (isinstance(key, tuple) and key[0] == device)]:
        if d is not None:
            _lib.check(_lib.lib().hx_ctx_reset_hints(d.h), "hx_ctx_reset_hints")
    if os.environ.get("HX_TIMING"):
        _lib.lib().hx_timeline_epoch()
    marks = [("start", time.perf_counter())]
    dev_a = resident(h)
    if dev_a is not None:
        dev.set_operand(0, dev_ptr=dev_a[1], n=dev_a[2])
    else:
        dev.set_operand(0, pool=pool_a)
    if same:
        dev.alias_b()
    else:
        dev_b = resident(k)
        if dev_b is not None:
            dev.set_operand(1, dev_ptr=dev_b[1], n=dev_b[2])
        else:
            dev.set_operand(1, pool=pool_b)
    marks.append(("operands", time.perf_counter()))
    comp = cfg.compressor
    pc = _lib.HxProductCfg(kind, eps, kmax, TAG_CODES[comp.tag], int(comp.seed) & (2**64 - 1),
                           int(sketch0), int(oversample), int(getattr(comp, "q", 1)))
    ta = tree_arrays(h.bct)
    tile = plan_tile(h.bct)
    adaptive = False
    if chunks is None:
        nch, use_overlap, adaptive = default_chunks(h.bct, dev, overlap, leaf_mask)
    else:
        nch = max(1, int(chunks))
        use_overlap = nch > 1 and overlap_default(overlap)
    # with overlap the first chunk is small: its planning is the only exposed part
    weights = list(OVERLAP_WEIGHTS) if (chunks is None and use_overlap and not adaptive and
                                        nch == len(OVERLAP_WEIGHTS)) else None
    iflags = implicit_flags(implicit_min, cfg.compressor.tag) if not trad else \
        (int(trad) << TRAD_SHIFT)
    # memory-bound products size their chunks by workspace weight (implicit leaves count by
    # their sketch panels, not their area: _tree_meta); products that fit keep plain areas
    wmin = (1 << ((iflags >> 8) & 31)) if (adaptive and not trad and (iflags >> 8) & 31) else 0
    queue = collections.deque(chunk_groups(h.bct, nch, first=0.2 if use_overlap else 1.0,
                                           weights=weights, implicit_min=wmin))
    budget = 0.8 * available_bytes(dev) - 4e9

    plan_ms = [0.0]
    timeline = []  # (what, host start, host end) for HX_TIMING

    def make_plan(group):
        mask = group_mask(h.bct, group, leaf_mask) if (len(queue_all) > 1 or leaf_mask
                                                       is not None or group_split[0]) else None
        if mask is not None and not mask.any():
            return None
        t0 = time.perf_counter()
        # deferred: the per-batch factor work lists are filled inside hx_product while the
        # device runs the previous batch
        defer = 0 if os.environ.get("HX_PLAN_NODEFER") else _lib.Plan.DEFER
        p = _lib.Plan(ta, dir_a, dir_a if same else dir_b, mask, tile, flags=defer | iflags)
        t1 = time.perf_counter()
        plan_ms[0] += (t1 - t0) * 1e3
        timeline.append(("plan", t0, t1))
        return p

    queue_all = list(queue)
    group_split = [False]
    rep = MultReport()
    # with several chunks, two contexts (two streams) run consecutive chunks concurrently:
    # one chunk's latency-bound recompression overlaps the next chunk's term formation
    ctxs = [dev]
    if len(queue_all) > 1 and use_overlap:
        n_ctx = int(os.environ.get("HX_CONTEXTS", 2 if adaptive else OVERLAP_CONTEXTS))
        n_ctx = max(2, min(n_ctx, len(queue_all)))
        for i in range(n_ctx - 1):
            aux = Device.aux(device, i)
            _lib.check(_lib.lib().hx_ctx_operand_share(aux.h, dev.h), "hx_ctx_operand_share")
            ctxs.append(aux)
        budget = budget / n_ctx

    def run_chunk(plan, ctx, out):
        try:
            st = _lib.HxProductStats()
            t0 = time.perf_counter()
            _lib.check(_lib.lib().hx_product(ctx.h, plan.h, C.byref(pc), C.byref(st)),
                       "hx_product")
            timeline.append(("product", t0, time.perf_counter()))
            t_ret = time.perf_counter()
            if os.environ.get("HX_TIMING"):
                tm = list(st.t_marks)
                print(f"[hx device] ctx {ctxs.index(ctx)}: start {tm[0]:.1f} form-end "
                      f"{tm[1]:.1f} mat-end {tm[2]:.1f} end {tm[3]:.1f} ms", flush=True)
            leaves = plan.leaves()
            nl = len(leaves["ids"])
            rank = np.zeros(nl, np.int32)
            deg = np.zeros(nl, np.int8)
            off = np.zeros(nl, np.int64)
            _lib.check(_lib.lib().hx_result_layout(ctx.h, _lib.ptr(rank, _lib.i32p),
                                                   _lib.ptr(deg, _lib.i8p),
                                                   _lib.ptr(off, _lib.i64p)), "hx_result_layout")
            res = None
            if fetch:
                res = _lib.pinned_empty(max(int(st.out_elems), 1))
                _lib.check(_lib.lib().hx_result_download(ctx.h, _lib.ptr(res, _lib.f64p),
                                                         res.size), "hx_result_download")
            out.update(st=st, leaves=leaves, rank=rank, deg=deg, off=off, res=res,
                       info=plan.info)
            timeline.append(("results", t_ret, time.perf_counter()))
        except BaseException as exc:  # re-raised on the main thread
            out["err"] = exc
        finally:
            t_c = time.perf_counter()
            plan.close()
            timeline.append(("close", t_c, time.perf_counter()))

    chunks_out = []
    seen = [0.0, 0.0]  # planned workspace bytes and leaf area (adaptive chunking)
    last_rate = [0.0]  # workspace rate of the last rejected (too large) plan
    inflight = collections.deque()
    plan = None
    try:
        group = queue.popleft()
        plan = make_plan(group)
        while True:
            # a chunk whose workspace would not fit is split and planned again
            while plan is not None and plan_bytes(plan.info) > budget:
                # split once into as many parts as the measured workspace per leaf area asks
                # for (not by repeated halving: every rejected plan is wasted host time)
                pb = plan_bytes(plan.info)
                area = sum(u[2] for u in group)
                rate = pb / max(area, 1.0)
                last_rate[0] = max(last_rate[0], rate)
                units = group if len(group) > 1 else \
                    [p[0] for p in split_chunk(h.bct, group, wmin)]
                parts = regroup_units([units], rate, 0.7 * budget) if len(units) > 1 \
                    else [units]
                if len(parts) == 1:
                    parts = split_chunk(h.bct, units, wmin)
                if len(parts) == 1:
                    break
                group_split[0] = True
                plan.close()
                group = parts[0]
                queue.extendleft(reversed(parts[1:]))
                plan = make_plan(group)
            if adaptive and plan is not None and queue:
                # workspace per unit of leaf area: the larger of the average over the plans
                # so far and the latest plan's (dense regions are priced by their own rate);
                # the remaining subtrees are regrouped to fill the budget
                pb = plan_bytes(plan.info)
                area = sum(u[2] for u in group)
                seen[0] += pb
                seen[1] += area
                rate = max(seen[0] / max(seen[1], 1.0), pb / max(area, 1.0), last_rate[0])
                last_rate[0] = 0.0
                queue = collections.deque(regroup_units(list(queue), rate, 0.7 * budget))
            if plan is not None:
                if len(inflight) >= len(ctxs):  # chunk i - len(ctxs)'s context must be free
                    t = inflight.popleft()
                    t.join()
                out = {}
                chunks_out.append(out)
                t = threading.Thread(target=run_chunk,
                                     args=(plan, ctxs[(len(chunks_out) - 1) % len(ctxs)], out))
                t.start()
                inflight.append(t)
                plan = None  # owned (and closed) by the chunk thread now
            if not queue:
                break
            # plan the next chunk while the device runs the current one(s)
            group = queue.popleft()
            plan = make_plan(group)
    finally:
        if plan is not None:
            plan.close()
        # every chunk thread is joined, also when planning raised (e.g. MemoryError): no
        # thread may keep running hx_product on this device's contexts after we return
        for t in inflight:
            t.join()
    marks.append(("products", time.perf_counter()))
    degraded = set()
    leaves_all, ranks_all, infos, fetched = [], [], [], []
    n_run = 0
    for out in chunks_out:
        if "err" in out:
            raise out["err"]
        n_run += 1
        st, leaves, rank, deg, off, res = (out[k] for k in ("st", "leaves", "rank", "deg", "off",
                                                            "res"))
        if fetch:
            fetched.append((leaves, rank, deg, off, res))
        far_deg = (leaves["kind"] == 1) & (deg != 0)
        degraded.update(leaves["ids"][far_deg].tolist())
        rep.degraded_blocks += int(st.degraded_blocks)
        rep.max_far_rank = max(rep.max_far_rank, int(st.max_far_rank))
        rep.matvec_count += int(st.matvec_count)
        rep.far_leaves += int(st.far_leaves)
        rep.near_leaves += int(st.near_leaves)
        rep.device_ms += st.ms_total
        rep.form_ms += st.ms_form
        rep.materialize_ms += st.ms_mat
        rep.recompress_ms += st.ms_recompress
        rep.upload_ms += st.ms_upload
        rep.out_elems += int(st.out_elems)
        rep.sketch_rounds = max(rep.sketch_rounds, int(st.sketch_rounds))
        rep.launches += int(st.launches)
        rep.fro2 += float(st.fro2_total)
        leaves_all.append(leaves)
        ranks_all.append(rank)
        infos.append(out["info"])
    marks.append(("unpack", time.perf_counter()))
    if os.environ.get("HX_TIMING"):
        print("[hx timing] " + " ".join(f"{b[0]} {1e3 * (b[1] - a[1]):.1f}ms"
                                        for a, b in zip(marks, marks[1:])), flush=True)
        t00 = marks[0][1]
        print("[hx timeline] " + " ".join(f"{w}:{1e3 * (a - t00):.0f}-{1e3 * (b - t00):.0f}"
                                          for w, a, b in sorted(timeline, key=lambda x: x[1])),
              flush=True)
    if degraded:  # the reference's warning per degraded block (multiply.py:73-78)
        arr = block_arrays(h.bct)
        lo, hi = arr.tree.lo, arr.tree.hi
        for b in sorted(degraded):
            t, sg = arr.tau[b], arr.sigma[b]
            rep.warnings.append(f"block {b} rows [{lo[t]},{hi[t]}) cols [{lo[sg]},{hi[sg]}): "
                                "compression did not certify convergence")
    rep.chunks = n_run
    rep.plan_ms = plan_ms[0]
    rep.wall_s = time.perf_counter() - t_start
    out = HMatrix(h.bct, _ProductLeaves(fetched) if fetch else {}, degraded)
    out.report = rep
    out.plan_info = _sum_info(infos)
    out.plan_leaves = ({key: np.concatenate([lv[key] for lv in leaves_all]) for key in
                        leaves_all[0]} if leaves_all else {})
    out.leaf_rank = np.concatenate(ranks_all) if ranks_all else np.zeros(0, np.int32)
    return out


def _sum_info(infos):
    tot = _lib.HxPlanInfo()
    for inf in infos:
        for name, typ in tot._fields_:
            if name == "created":
                for i in range(3):
                    tot.created[i] += inf.created[i]
            elif name == "max_out_dim":
                tot.max_out_dim = max(tot.max_out_dim, inf.max_out_dim)
            else:
                setattr(tot, name, getattr(tot, name) + getattr(inf, name))
    return tot


def hmult_new(h, k, cfg, devices=None):
    """Product H K with one direct compression per farfield leaf (reference signature,
    ``multiply.py:252-256``).  ``devices`` (optional; default ``HX_DEVICES`` = comma list,
    else GPU 0): with several GPUs the output subtrees are partitioned over them and the
    operand pools replicated by an NCCL broadcast (``distributed.multiply_devices``)."""
    if cfg.mode != "new":
        raise ValueError("config mode must be 'new'")
    if h.bct is not k.bct:
        raise ValueError("factors must live on the same block-cluster tree")
    if devices is None:
        env = os.environ.get("HX_DEVICES", "")
        devices = [int(x) for x in env.split(",") if x.strip()] or [0]
    if len(devices) > 1:
        from .distributed import multiply_devices
        return multiply_devices(h, k, cfg, devices)
    return multiply_device(h, k, cfg, device=int(devices[0]))


# HX_PLAN_TRAD converter codes: hierarchical agglomeration of each pending pair
# (_pair_structural_lowrank, multiply.py:140-189) or one best approximation of the pair
# product (the dense-svd compressor on _PairProductMap, multiply.py:192-204)
TRAD_SHIFT = 4
TRAD_CONVERTERS = {"hier-approx": 1, "dense-svd": 2}


def hmult_traditional(h, k, cfg, device=0):
    """Product H K in the convert-then-truncate discipline (``multiply.py:259-263``): every
    pending pair of a far leaf is converted to low rank on its own, then the leaf's terms
    are combined largest norm first by pairwise truncated summation
    (``fast_truncate_sum``, ``lowrank.py:123-138``); near leaves as in ``hmult_new``.

    Converters ``hier-approx`` (the reference default) and ``dense-svd`` run on the GPU;
    the matrix-free converters (``aca``, ``bilanczos``, ``randomized`` on the pair product)
    are not built and raise ``NotImplementedError``."""
    if cfg.mode != "traditional":
        raise ValueError("config mode must be 'traditional'")
    if h.bct is not k.bct:
        raise ValueError("factors must live on the same block-cluster tree")
    code = TRAD_CONVERTERS.get(cfg.converter)
    if code is None:
        raise NotImplementedError(f"traditional-mode converter {cfg.converter!r} is not built "
                                  f"on the GPU (available: {', '.join(TRAD_CONVERTERS)})")
    return multiply_device(h, k, cfg, device=int(device), trad=code)
