"""Per-rank product time of a multi-GPU partition, measured one rank at a time on ONE GPU.

Each rank's masked product (its output subtrees; operands resident) runs alone on the
device, so its time is what that rank would take on its own B200 (no rank waits on
another).  The predicted N-GPU step is the max over ranks; speed-up = t(1) / max.
The NCCL operand broadcast is not part of the product step (it happens once, at setup).

usage: python tools/rank_sim.py CFG [--worlds 2,4,8] [--steps 3] [--leafwise] [--tag aca]

A rank's share of the host (16 cores / 8 ranks) is simulated by running the ranks under
`taskset -c 0-1` with OMP_NUM_THREADS=2 (--skip-full), and world 1 separately with the
whole host.
"""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1805_08998_b200 as hx  # noqa: E402
from paper_1805_08998_b200 import _lib, configs, hmatrix, multiply  # noqa: E402


def timed(A, B, cfg, mask, steps, warm=2):
    import torch
    for _ in range(warm):
        multiply.multiply_device(A, B, cfg, leaf_mask=mask, fetch=False)
    ts = []
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        C = multiply.multiply_device(A, B, cfg, leaf_mask=mask, fetch=False)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e3, C.report


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warm", type=int, default=2)
    ap.add_argument("--leafwise", action="store_true", help="old leaf-wise LPT partition")
    ap.add_argument("--leafcost", action="store_true", help="units priced by leaf costs only")
    ap.add_argument("--ranks", default="", help="only these ranks (comma list)")
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--tag", default="dense-svd")
    ap.add_argument("--save-masks", default="", help="write the partition (npz) and exit")
    ap.add_argument("--load-masks", default="", help="use a saved partition (one process per rank)")
    a = ap.parse_args()
    c = configs.CONFIGS[a.cfg]
    bct, A, B = configs.build_operands(c)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(a.tag), policy=hx.EpsRank(c["tol"]))
    _, dA = multiply.operand_directory(A)
    _, dB = multiply.operand_directory(B)
    full = _lib.Plan(hmatrix.tree_arrays(bct), dA, dA if B is A else dB, None,
                     multiply.plan_tile(bct))
    lv = full.leaves()
    cost = np.zeros(bct.n_nodes)
    cost[lv["ids"]] = bench.leaf_costs(lv)
    t1, r1 = (1.0, None) if a.skip_full else timed(A, B, cfg, None, a.steps, a.warm)
    if r1 is not None:
        print(f"cfg{a.cfg} world 1: {t1:.1f} ms (form {r1.form_ms:.1f} "
              f"mat {r1.materialize_ms:.1f} recomp {r1.recompress_ms:.1f})", flush=True)
    only = [int(x) for x in a.ranks.split(",")] if a.ranks else None
    for w in [int(x) for x in a.worlds.split(",")]:
        if a.leafwise:
            owner, load = bench.lpt_partition(bench.leaf_costs(lv), w)
            masks = []
            for r in range(w):
                m = np.zeros(bct.n_nodes, np.uint8)
                m[lv["ids"][owner == r]] = 1
                masks.append(m)
        elif a.load_masks:
            z = np.load(a.load_masks)
            masks, load = list(z["masks"]), z["load"]
        else:
            uc = None if a.leafcost else (lambda us: multiply.plan_unit_costs(A, B, us, tag=a.tag))
            _, units, load, masks = multiply.subtree_partition(bct, cost, w, unit_cost=uc)
        if a.save_masks:
            np.savez_compressed(a.save_masks, masks=np.stack(masks), load=np.asarray(load))
            print(f"partition for world {w} saved to {a.save_masks}", flush=True)
            return
        per = []
        for r in range(w):
            if only is not None and r not in only:
                per.append(0.0)
                continue
            t, rep = timed(A, B, cfg, masks[r], a.steps, a.warm)
            per.append(t)
            print(f"  world {w} rank {r}: {t:.1f} ms (form {rep.form_ms:.1f} "
                  f"mat {rep.materialize_ms:.1f} recomp {rep.recompress_ms:.1f} "
                  f"plan {rep.plan_ms:.1f} chunks {rep.chunks}) "
                  f"load {load[r] / load.sum():.3f}", flush=True)
        print(f"world {w}: max {max(per):.1f} ms mean {np.mean(per):.1f} ms "
              f"speed-up {t1 / max(per):.2f}x (efficiency {t1 / max(per) / w:.2f})", flush=True)


if __name__ == "__main__":
    main()
