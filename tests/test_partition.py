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
