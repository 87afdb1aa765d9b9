"""Golden HMX1 operator file written by the UNMODIFIED reference ``save_hmatrix``
(``/root/reference/pkg/src/hmat/hmatrix.py:338-361``), for the HMX1 reader/writer tests.

Operand: n=300 points uniform in [0,1]^2 (seed 3, a ragged tree), leaf 12, eta 0.8,
kernel exp(-r), reference ACA at 1e-6 (the point adapter of make_golden.py).  One far leaf
is replaced by its dense block and flagged degraded, so the file also holds a dense record
on a far node and a set degraded byte, as the reference writes for compression fallbacks.

Usage:  python tests/golden/make_hmx1.py   (writes tests/golden/hmx1_ops300.{hmx,npz})
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as G  # noqa: E402
from hmat import clustering, hmatrix, lowrank  # noqa: E402


def main():
    pts, tree, bct, A, _ = G.product_setup(300, "square", 12, 0.8, "exp", None, 1e-6, seed=3)
    far = [leaf.id for leaf in bct.leaves if leaf.kind == clustering.FAR]
    fb = far[len(far) // 2]
    A.data[fb] = A.data[fb].to_dense()
    A.degraded.add(fb)
    path = os.path.join(HERE, "hmx1_ops300.hmx")
    hmatrix.save_hmatrix(A, path)
    ids, kinds, ranks = [], [], []
    for leaf in bct.leaves:
        p = A.data[leaf.id]
        ids.append(leaf.id)
        kinds.append(1 if isinstance(p, lowrank.LowRank) else 2)
        ranks.append(p.rank if isinstance(p, lowrank.LowRank) else -1)
    np.savez_compressed(os.path.join(HERE, "hmx1_ops300.npz"), points=pts, n_min=12, eta=0.8,
                        ids=np.array(ids), kinds=np.array(kinds), ranks=np.array(ranks),
                        degraded=np.array(sorted(A.degraded)),
                        fingerprint=np.frombuffer(hmatrix.tree_fingerprint(bct), np.uint8))
    print(f"wrote {path} ({os.path.getsize(path)} bytes), far dense leaf {fb}")


if __name__ == "__main__":
    main()
