"""Steady-state wall time of the config-2 product for chunk-count / weight settings
(HX_CHUNKS + HX_CHUNK_WEIGHTS), one process, operands resident.

usage: python tools/chunk_sweep.py [--tag aca]
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1805_08998_b200 as hx  # noqa: E402
from paper_1805_08998_b200 import configs  # noqa: E402

SETTINGS = [
    None,
    (4, "0.2,1,1,0.5"),
    (5, "0.15,1,1,0.6,0.3"),
    (5, "0.2,1,1,1,0.4"),
    (6, "0.15,1,1,1,0.5,0.25"),
    (6, "0.2,0.6,1,1,0.6,0.3"),
    (8, "0.2,0.6,1,1,1,1,0.6,0.3"),
    (3, "0.3,1,0.5"),
]


def main():
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "aca"
    c = configs.CONFIGS[2]
    bct, A, B = configs.build_operands(c)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(tag), policy=hx.EpsRank(c["tol"]))
    for _ in range(3):
        hx.multiply.multiply_device(A, B, cfg, fetch=False)
    for rnd in range(2):
        for st in SETTINGS:
            os.environ.pop("HX_CHUNKS", None)
            os.environ.pop("HX_CHUNK_WEIGHTS", None)
            if st:
                os.environ["HX_CHUNKS"] = str(st[0])
                os.environ["HX_CHUNK_WEIGHTS"] = st[1]
            hx.multiply.multiply_device(A, B, cfg, fetch=False)
            w = []
            for _ in range(5):
                torch.cuda.synchronize()
                w.append(hx.multiply.multiply_device(A, B, cfg, fetch=False).report.wall_s * 1e3)
            print(f"round {rnd} {st}: median {np.median(w):.1f} ms  min {min(w):.1f}  "
                  f"({' '.join(f'{x:.0f}' for x in w)})", flush=True)


if __name__ == "__main__":
    main()
