"""Per-unit canonical work table of a BASELINE config (input of bench.py's CPU arms).

The CPU reference arm times the reference algorithm (oracle port) on a stratified sample
of the product's *units* -- the subtrees rooted at the first block level that holds a far
leaf (``multiply.chunk_units``).  No low-rank term is created above that level, so the
units share no work and their canonical work adds up to the whole product's.
The table prices every unit once, on this machine, from the GPU product's own plan and
output ranks, so that the CPU arm itself loads no part of the GPU library:

    bench_data/cfg<C>_<tag>_units.npz
        b0, b1        pre-order id range of each unit
        F, B          canonical flops / bytes of the unit (masked plan + product ranks)
        leaves        output leaves per unit
        F_total, B_total, phases   the whole product's figures (for the roofline)

usage (GPU box): python tools/unit_table.py --config 2 --tag aca
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--tag", default="aca")
    args = ap.parse_args()

    import bench
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import _lib, configs, hmatrix, multiply

    c = configs.CONFIGS[args.config]
    bct, A, B = configs.build_operands(c)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(args.tag), policy=hx.EpsRank(c["tol"]))
    C = multiply.multiply_device(A, B, cfg, fetch=False)
    rank_of = dict(zip(C.plan_leaves["ids"].tolist(), C.leaf_rank.tolist()))
    _, dA = multiply.operand_directory(A)
    _, dB = multiply.operand_directory(B)
    ta = hmatrix.tree_arrays(bct)
    tile = multiply.plan_tile(bct)
    full = _lib.Plan(ta, dA, dA if B is A else dB, None, tile)
    lv = full.leaves()
    ph = bench.canonical_phases(full.info, lv, np.array([rank_of[int(b)] for b in lv["ids"]]))
    full.close()
    arr = hmatrix.block_arrays(bct)
    leaf = arr.kind_code != 0
    units = multiply.chunk_units(bct)
    F = np.zeros(len(units))
    Bb = np.zeros(len(units))
    nl = np.zeros(len(units), np.int64)
    for i, (b0, b1, _) in enumerate(units):
        m = np.zeros(arr.n_nodes, np.uint8)
        m[b0:b1] = leaf[b0:b1]
        p = _lib.Plan(ta, dA, dA if B is A else dB, m, tile)
        pl = p.leaves()
        u = bench.canonical_phases(p.info, pl, np.array([rank_of[int(b)] for b in pl["ids"]]))
        F[i], Bb[i], nl[i] = u["F"], u["B"], len(pl["ids"])
        p.close()
    out = os.path.join(ROOT, "bench_data", f"cfg{args.config}_{args.tag}_units.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez(out, b0=np.array([u[0] for u in units]), b1=np.array([u[1] for u in units]),
             F=F, B=Bb, leaves=nl, F_total=ph["F"], B_total=ph["B"],
             phases=np.array([[ph[k]["F"], ph[k]["B"]] for k in ("form", "near", "far")]),
             n_nodes=arr.n_nodes, tag=args.tag, config=args.config)
    print(f"{out}: {len(units)} units, sum F {F.sum() / 1e9:.1f} GFLOP (whole product "
          f"{ph['F'] / 1e9:.1f}), sum B {Bb.sum() / 1e9:.1f} GB (whole {ph['B'] / 1e9:.1f})")


if __name__ == "__main__":
    main()
