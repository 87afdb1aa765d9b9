"""The multi-GPU product through the public API, on the one GPU of this run.

``hmult_new(..., devices=[0, 0])`` runs the in-process path (partition, pool replication,
one thread per device entry, merge) with both shards on GPU 0; ``hmult_new_spmd`` runs the
torchrun data plane (NCCL broadcast of the device pool, shipped partition, masked product,
gather) in a world of one.  Both must reproduce the single-GPU product leaf for leaf.
Ranks whose kernels wait on each other are never placed on one GPU: the shards here are
independent products."""

import os
import socket

import numpy as np
import pytest

from test_gpu_product import _check_parity, _operands

pytestmark = pytest.mark.gpu


def _same_product(C1, C2, tol):
    assert sorted(C1.data) == sorted(C2.data)
    for b, p in C1.data.items():
        q = C2.data[b]
        if hasattr(p, "left"):
            assert q.left.shape[1] == p.left.shape[1], b
            d = p.left @ p.right.T
            assert np.linalg.norm(q.left @ q.right.T - d) <= 1e-12 * max(np.linalg.norm(d),
                                                                          1e-300)
        else:
            assert np.array_equal(q, p), b
    assert C2.report.far_leaves == C1.report.far_leaves
    assert C2.report.near_leaves == C1.report.near_leaves


@pytest.mark.parametrize("tag", ["dense-svd", "aca"])
def test_devices_api_matches_single_gpu(golden, tag):
    import paper_1805_08998_b200 as hx

    g = golden("cfg1.npz")
    bct, A, B, oa, ob, tol = _operands(g, "cfg1.npz")
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(tag), policy=hx.EpsRank(tol))
    C1 = hx.hmult_new(A, B, cfg)
    C2 = hx.hmult_new(A, B, cfg, devices=[0, 0])
    assert len(C2.shards) == 2
    own = [set(s.data) for s in C2.shards]
    assert own[0] and own[1] and not (own[0] & own[1])
    _same_product(C1, C2, tol)
    _check_parity(g, tag, bct, C2, oa, ob, tol)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_spmd_nccl_world1_device_pool():
    """GPU-assembled operand (device pool) through broadcast_operand over NCCL, the
    shipped partition, the masked product and the gather."""
    import torch
    import torch.distributed as dist

    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import distributed

    rng = np.random.default_rng(4)
    pts = rng.uniform(0, 1, (4096, 2))
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, 32), 0.8)
    A = hx.assemble_hmatrix("exp", bct, hx.EpsRank(1e-8), pts, device=0)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("aca"), policy=hx.EpsRank(1e-6))
    C1 = hx.hmult_new(A, A, cfg)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        B = distributed.broadcast_operand(A, bct, 0, None, device=0)
        assert B is A
        C2 = distributed.hmult_new_spmd(A, A, cfg, bct, device=0)
    finally:
        dist.destroy_process_group()
    _same_product(C1, C2, 1e-6)
