"""Multi-GPU host logic on CPU: LPT partition of output subtrees over ranks and the masked
per-rank plans (world size 2, gloo)."""

import os
import socket

import numpy as np
import pytest


def _cfg1_plan_inputs():
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import hmatrix
    from oracle import hmat_oracle as O

    rng = np.random.default_rng(0)
    pts = rng.uniform(0, 1, (1024, 2))
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, 32), 0.8)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, 32), 0.8)
    A = O.assemble_o("exp", obt, O.Eps(1e-8), pts)
    H = hx.HMatrix(bct, A.data)
    _, d = hmatrix.pack_operand(H)
    return bct, d, H


def test_lpt_partition_balances():
    import bench

    rng = np.random.default_rng(3)
    cost = rng.pareto(1.5, 5000) + 1
    owner, load = bench.lpt_partition(cost, 8)
    assert set(owner.tolist()) == set(range(8))
    assert np.isclose(load.sum(), cost.sum())
    assert load.max() <= load.mean() + cost.max()  # LPT bound


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import bench
    from paper_1805_08998_b200 import _lib, hmatrix, multiply

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bct, d, H = _cfg1_plan_inputs()
    full = _lib.Plan(hmatrix.tree_arrays(bct), d, d, None, multiply.plan_tile(bct))
    lv = full.leaves()
    cost = np.zeros(bct.n_nodes)
    cost[lv["ids"]] = bench.leaf_costs(lv)
    mask = multiply.subtree_partition(bct, cost, world)[3][rank]
    mine = _lib.Plan(hmatrix.tree_arrays(bct), d, d, mask, multiply.plan_tile(bct))
    ml = mine.leaves()
    got = [None] * world
    dist.all_gather_object(got, {"ids": ml["ids"].tolist(), "K": ml["K"].tolist(),
                                 "flops_near": mine.info.flops_near,
                                 "flops_form": mine.info.flops_form})
    if rank == 0:
        out.put((lv["ids"].tolist(), lv["K"].tolist(), full.info.flops_near, got,
                 full.info.flops_form))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_masked_plans_cover_all_leaves_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, K, fnear, got, fform = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    all_ids = sorted(i for g in got for i in g["ids"])
    assert all_ids == sorted(ids)                       # every leaf owned exactly once
    assert len(set(got[0]["ids"]) & set(got[1]["ids"])) == 0
    kfull = dict(zip(ids, K))
    for g in got:                                       # per-leaf term lists unchanged
        for i, k in zip(g["ids"], g["K"]):
            assert kfull[i] == k
    assert np.isclose(sum(g["flops_near"] for g in got), fnear)
    # whole subtrees per rank: term formation is (almost) not repeated across ranks
    assert sum(g["flops_form"] for g in got) <= 1.05 * fform


def test_subtree_partition_covers_and_balances():
    import bench
    from paper_1805_08998_b200 import _lib, hmatrix, multiply

    bct, d, H = _cfg1_plan_inputs()
    full = _lib.Plan(hmatrix.tree_arrays(bct), d, d, None, multiply.plan_tile(bct))
    lv = full.leaves()
    cost = np.zeros(bct.n_nodes)
    cost[lv["ids"]] = bench.leaf_costs(lv)
    for world in (1, 2, 3, 8):
        owner, units, load, masks = multiply.subtree_partition(bct, cost, world)
        tot = np.sum(masks, axis=0)
        leaf = bct.kind_code != 0
        assert np.array_equal(tot, leaf.astype(tot.dtype))   # every leaf exactly once
        assert np.isclose(load.sum(), cost[leaf].sum())
        # units are disjoint subtrees in pre-order
        spans = sorted(units)
        assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
        ucost = [cost[u0:u1].sum() for u0, u1 in units]
        assert load.max() <= load.mean() + max(ucost) + 1e-9


def test_subtree_partition_with_planned_unit_costs():
    from paper_1805_08998_b200 import multiply

    bct, d, H = _cfg1_plan_inputs()
    cost = np.ones(bct.n_nodes)
    seen = []

    def uc(units):
        c = multiply.plan_unit_costs(H, H, units)
        seen.append(c)
        return c

    owner, units, load, masks = multiply.subtree_partition(bct, cost, 4, unit_cost=uc)
    assert len(seen) == 1 and len(seen[0]) == len(units)
    assert all(c > 0 for c in seen[0])
    assert np.isclose(load.sum(), sum(seen[0]))
    tot = np.sum(masks, axis=0)
    assert np.array_equal(tot, (bct.kind_code != 0).astype(tot.dtype))
    assert load.max() <= load.mean() + max(seen[0]) + 1e-12


def _oracle_product(A, B, cfg, mask):
    """CPU stand-in for one rank's masked GPU product: the oracle's hmult_new restricted to
    the rank's leaves, on the operand this rank received (lazy host-pool leaves)."""
    import paper_1805_08998_b200 as hx
    from oracle import hmat_oracle as O

    bct = A.bct
    obt = O.BlockTreeO(O.ClusterTreeO(_points(), 32), 0.8)

    def conv(H):  # C-ordered copies: BLAS rounding depends on the memory layout
        c = np.ascontiguousarray
        return O.HMatO(obt, {b: (O.LR(c(p.left), c(p.right)) if hasattr(p, "left") else c(p))
                             for b, p in H.data.items()})
    oa = conv(A)
    ob = oa if B is A else conv(B)
    only = set(np.flatnonzero(mask).tolist())
    R = O.hmult_new_o(oa, ob, O.Eps(cfg.policy.eps), cfg.compressor.tag, only=only)
    data = {b: (hx.LowRank(p.left, p.right) if isinstance(p, O.LR) else p)
            for b, p in R.data.items()}
    C = hx.HMatrix(bct, data, R.degraded)
    rep = hx.MultReport(far_leaves=R.report.far_leaves, near_leaves=R.report.near_leaves,
                        max_far_rank=R.report.max_far_rank)
    C.report = rep
    return C


def _points():
    return np.random.default_rng(0).uniform(0, 1, (1024, 2))


def _spmd_worker(rank, world, port, out):
    import torch.distributed as dist

    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import distributed, multiply

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pts = _points()
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, 32), 0.8)
    H = None
    if rank == 0:
        _, _, H0 = _cfg1_plan_inputs()
        H = hx.HMatrix(bct, dict(H0.data))
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("aca"), policy=hx.EpsRank(1e-6))
    # the broadcast operand itself: every rank's pool is rank 0's, bit for bit
    A = distributed.broadcast_operand(H, bct)
    pool, _ = multiply._host_directory(A) if rank else multiply.operand_directory(A)
    sums = [None] * world
    dist.all_gather_object(sums, (pool.size, float(np.sum(pool)), pool[::97].tolist()))
    C = distributed.hmult_new_spmd(H, H, cfg, bct, product=_oracle_product)
    if rank == 0:
        out.put((sums, {b: (p.left, p.right) if hasattr(p, "left") else p
                        for b, p in C.data.items()}, C.report.far_leaves,
                 C.report.near_leaves))
    dist.barrier()
    dist.destroy_process_group()


def test_spmd_data_plane_world2():
    """The torchrun data plane end to end on host pools (gloo, world 2): rank 0's packed
    operand is broadcast and attached on rank 1, the partition is shipped from rank 0,
    each rank runs its masked product (the oracle standing in for the GPU), and the shards
    are gathered on rank 0: every output leaf exactly once, bit-identical to world 1."""
    import torch.multiprocessing as mp
    from oracle import hmat_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spmd_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    sums, data, far, near = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert sums[0] == sums[1]
    _, _, H = _cfg1_plan_inputs()
    obt = O.BlockTreeO(O.ClusterTreeO(_points(), 32), 0.8)
    oa = O.HMatO(obt, {b: (O.LR(p.left, p.right) if hasattr(p, "left") else p)
                       for b, p in H.data.items()})
    R = O.hmult_new_o(oa, oa, O.Eps(1e-6), "aca")
    assert sorted(data) == sorted(R.data)
    assert far == R.report.far_leaves and near == R.report.near_leaves
    for b, p in R.data.items():
        q_ = data[b]
        if isinstance(p, O.LR):
            assert np.array_equal(q_[0], p.left) and np.array_equal(q_[1], p.right)
        else:
            assert np.array_equal(q_, p)
