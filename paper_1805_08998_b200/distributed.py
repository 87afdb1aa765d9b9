"""The product on several GPUs: output subtrees partitioned over the GPUs of
one box, operand pools replicated by a broadcast, no reduction.

Output leaves are independent once their terms exist (each far block is compressed from
its own exact sum, ``PAPER.md:4221-4227``), so a GPU owning whole subtrees of the block
tree forms only the terms of its subtrees and compresses only its leaves.  Every output
block is owned by exactly one GPU; the result is the union of the shards.

Two ways in:

* ``multiply_devices(h, k, cfg, devices)`` -- one process driving several GPUs (what
  ``hmult_new(..., devices=[...])`` calls): the packed operand pools go to the first
  device once and are replicated to the others by an NCCL broadcast
  (``torch.cuda.comm.broadcast``), one host thread per device runs its masked product,
  and the shards are merged into one ``HMatrix``.
* ``hmult_new_spmd(h, k, cfg, group)`` -- one process per GPU under ``torchrun``
  (``bench.py``): rank 0 holds the operands; ``broadcast_operand`` replicates the packed
  pool (NCCL for device pools, gloo for host pools), every rank runs its masked product and
  ``gather_product`` collects the shards on rank 0.

The partition is computed once, on one process, and shipped to the others: its unit
prices include measured host planning times, so ranks must not compute it independently.
"""

from __future__ import annotations

import threading

import numpy as np

from .hmatrix import HMatrix, LeafDict, _PoolLeaves, block_arrays, tree_arrays
from .multiply import (MultReport, _host_directory, multiply_device, operand_directory,
                       plan_tile, plan_unit_costs, subtree_partition)


# ------------------------------------------------------------------ partition
def leaf_costs(leaves):
    """Rough device cost per output leaf of a plan (materialization flops plus a far-leaf
    recompression term): the weights that decide where subtrees are split."""
    m = leaves["m"].astype(float)
    n = leaves["n"].astype(float)
    K = leaves["K"].astype(float)
    return 2 * m * n * K + leaves["fdd"] + np.where(leaves["kind"] == 1, 60 * m * n, 0.0)


def partition(h, k, world, measured=True, tag="dense-svd"):
    """Per-rank leaf masks of the output (``multiply.subtree_partition``): units priced by
    their own plans (``plan_unit_costs``, host planning time included) when ``measured``,
    else by the summed leaf costs.  Returns (masks, per-rank load)."""
    from . import _lib

    if world <= 1:
        return [None], np.zeros(1)
    bct = h.bct
    _, da = operand_directory(h) if getattr(h, "_hx_device", None) else _host_directory(h)
    db = da if k is h else (operand_directory(k) if getattr(k, "_hx_device", None)
                            else _host_directory(k))[1]
    full = _lib.Plan(tree_arrays(bct), da, db, None, plan_tile(bct))
    lv = full.leaves()
    full.close()
    cost = np.zeros(block_arrays(bct).n_nodes)
    cost[lv["ids"]] = leaf_costs(lv)
    unit_cost = (lambda us: plan_unit_costs(h, k, us, tag=tag)) if measured else None
    _, _, load, masks = subtree_partition(bct, cost, world, unit_cost=unit_cost)
    return masks, load


# ------------------------------------------------------------------ shards
def merge_reports(reports):
    rep = MultReport()
    for r in reports:
        for name in ("degraded_blocks", "matvec_count", "far_leaves", "near_leaves",
                     "out_elems", "launches", "chunks", "fro2"):
            setattr(rep, name, getattr(rep, name) + getattr(r, name))
        rep.max_far_rank = max(rep.max_far_rank, r.max_far_rank)
        rep.sketch_rounds = max(rep.sketch_rounds, r.sketch_rounds)
        for name in ("wall_s", "plan_ms", "device_ms", "form_ms", "materialize_ms",
                     "recompress_ms", "upload_ms"):  # the slowest shard
            setattr(rep, name, max(getattr(rep, name), getattr(r, name)))
        rep.warnings.extend(r.warnings)
    return rep


def merge_shards(bct, shards):
    """One ``HMatrix`` from per-GPU product shards (disjoint leaf sets)."""
    from .multiply import _ProductLeaves

    if all(isinstance(s.data, _ProductLeaves) for s in shards):
        data = _ProductLeaves([c for s in shards for c in s.data._chunks])
    else:
        data = LeafDict()
        for s in shards:
            for b, p in s.data.items():
                if b in data:
                    raise RuntimeError(f"output leaf {b} computed by two shards")
                dict.__setitem__(data, b, p)
    out = HMatrix(bct, data, set().union(*(s.degraded for s in shards)))
    out.report = merge_reports([s.report for s in shards])
    out.report.warnings.sort()
    return out


# ------------------------------------------------------------------ one process, N GPUs
def _replicate_pool(H, devices):
    """Device pointers of H's packed pool on every device: the pool is placed on the first
    device (its GPU-assembled pool, or one upload of the host pool) and broadcast to the
    others with NCCL (``torch.cuda.comm.broadcast``).  Returns (tensors, [(ptr, n)])."""
    import torch

    res = getattr(H, "_hx_device", None)
    if res is not None and res[0] == devices[0]:
        src = torch.empty(max(res[2], 1), dtype=torch.float64, device=f"cuda:{devices[0]}")
        _copy_device_pool(H, src, res[2])
        n = res[2]
    else:
        pool, _ = _host_directory(H)
        n = int(pool.size)
        src = torch.from_numpy(pool).to(f"cuda:{devices[0]}", non_blocking=False)
    uniq = list(dict.fromkeys(devices))
    outs = torch.cuda.comm.broadcast(src, uniq) if len(uniq) > 1 else [src]
    by_dev = dict(zip(uniq, outs))
    return [by_dev[d] for d in devices], [(by_dev[d].data_ptr(), n) for d in devices]


def _copy_device_pool(H, dst, n):
    import ctypes as C

    from . import _lib

    _lib.check(_lib.lib().hx_pool_download(H._hx_pool.dev.h, C.c_void_p(H._hx_pool.ptr),
                                           C.cast(C.c_void_p(dst.data_ptr()), _lib.f64p), n),
               "hx_pool_download")


def multiply_devices(h, k, cfg, devices, masks=None, fetch=True, **kw):
    """The product on several GPUs of this process (see the module docstring).  A device
    may appear more than once (its shards then run one after the other)."""
    devices = [int(d) for d in devices]
    world = len(devices)
    if masks is None:
        masks, _ = partition(h, k, world, tag=cfg.compressor.tag)
    keep_a, ptr_a = _replicate_pool(h, devices)
    keep_b, ptr_b = (keep_a, ptr_a) if k is h else _replicate_pool(k, devices)
    shards = [None] * world
    errors = []

    def run(i):
        try:
            shards[i] = multiply_device(h, k, cfg, device=devices[i], leaf_mask=masks[i],
                                        fetch=fetch, device_pools=(ptr_a[i], ptr_b[i]), **kw)
        except BaseException as exc:  # re-raised below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    del keep_a, keep_b  # the products are complete: the replicas can go
    if errors:
        raise errors[0]
    out = merge_shards(h.bct, shards)
    out.shards = shards
    return out


# ------------------------------------------------------------------ one process per GPU
def broadcast_operand(H, bct, src=0, group=None, device=None):
    """Replicate an operand from rank ``src`` (which holds ``H``; other ranks pass None):
    the packed pool as one tensor (a CUDA tensor over NCCL when ``device`` is given, else a
    host tensor, e.g. over gloo), the directory and degraded set as objects.  Returns the
    operand on every rank: device-attached (``_hx_device``) or host-packed (lazy leaves)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    if rank == src:
        if device is not None and getattr(H, "_hx_device", None) is not None:
            n = H._hx_device[2]
            _, d = operand_directory(H)
            buf = torch.empty(max(n, 1), dtype=torch.float64, device=f"cuda:{device}")
            _copy_device_pool(H, buf, n)
        else:
            pool, d = _host_directory(H)
            n = int(pool.size)
            buf = torch.from_numpy(np.ascontiguousarray(pool))
            if device is not None:
                buf = buf.to(f"cuda:{device}")
        meta = [n, d, sorted(H.degraded)]
    else:
        meta = [None, None, None]
    dist.broadcast_object_list(meta, src=src, group=group)
    n, d, deg = meta
    if rank != src:
        buf = torch.empty(max(n, 1), dtype=torch.float64,
                          device=f"cuda:{device}" if device is not None else "cpu")
    dist.broadcast(buf, src=src, group=group)
    if rank == src and (device is None or getattr(H, "_hx_device", None) is not None):
        return H
    out = HMatrix(bct, {}, set(deg))
    out._hx_keep = buf
    if device is None:
        out.data = _PoolLeaves(out)
        out._hx_packed = (buf.numpy()[:n], d)
    else:
        from .assembly import _LazyLeaves

        class _Pool:  # host download for the lazy leaves
            def download(self):
                return buf[:n].cpu().numpy()

        out.data = _LazyLeaves(out)
        out._hx_pool = _Pool()
        out._hx_device = (device, buf.data_ptr(), n)
        out._hx_packed = (None, d)
    return out


def gather_product(C, dst=0, group=None):
    """Collect the shards of a partitioned product on rank ``dst`` (every output leaf once);
    other ranks get None.  The payloads travel as pickled numpy arrays."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    mine = (dict(C.data.items()), sorted(C.degraded), C.report)
    parts = [None] * world if rank == dst else None
    dist.gather_object(mine, parts, dst=dst, group=group)
    if rank != dst:
        return None
    shards = []
    for data, deg, rep in parts:
        s = HMatrix(C.bct, data, deg)
        s.report = rep
        shards.append(s)
    return merge_shards(C.bct, shards)


def hmult_new_spmd(h, k, cfg, bct, group=None, device=None, product=None, measured=True):
    """SPMD product under ``torchrun``: every rank calls it with the same block tree
    ``bct`` (built from the same points); rank 0 passes the operands, the other ranks None.

    ``product(h, k, cfg, leaf_mask)`` runs one rank's masked product (default:
    ``multiply_device`` on ``device``); the CPU tests substitute a stand-in.  Returns the
    merged product on rank 0 and None elsewhere."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    if rank == 0 and (h is None or k is None):
        raise ValueError("rank 0 must hold the operands")
    if rank == 0 and (h.bct is not bct or k.bct is not bct):
        raise ValueError("factors must live on the same block-cluster tree")
    same = [k is h if rank == 0 else None]
    dist.broadcast_object_list(same, src=0, group=group)
    A = broadcast_operand(h, bct, 0, group, device)
    B = A if same[0] else broadcast_operand(k, bct, 0, group, device)
    world = dist.get_world_size(group)
    masks = [partition(A, B, world, measured, tag=cfg.compressor.tag)[0] if rank == 0 else None]
    dist.broadcast_object_list(masks, src=0, group=group)
    mask = masks[0][rank]
    if product is None:
        C = multiply_device(A, B, cfg, device=0 if device is None else device, leaf_mask=mask)
    else:
        C = product(A, B, cfg, mask)
    return gather_product(C, 0, group)
