"""Host/device timeline of device-resident products (HX_TIMING=1): plan and product spans
on the host, per-context device marks (start, formation end, materialization end, end).

usage: HX_TIMING=1 python tools/timeline.py CFG [steps]
"""
import sys

sys.path.insert(0, ".")
import paper_1805_08998_b200 as hx  # noqa: E402
from paper_1805_08998_b200 import configs, multiply  # noqa: E402


def main():
    c = configs.CONFIGS[int(sys.argv[1])]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    bct, A, B = configs.build_operands(c)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("dense-svd"), policy=hx.EpsRank(c["tol"]))
    walls = []
    import gc
    import os
    if os.environ.get("NO_GC"):
        gc.collect()
        gc.disable()
    for _ in range(steps):
        C = multiply.multiply_device(A, B, cfg, fetch=False)
        walls.append(C.report.wall_s * 1e3)
        print(f"-- wall {walls[-1]:.1f} ms", flush=True)
    w = sorted(walls[2:])
    print(f"== median wall of steps 3..{steps}: {w[len(w) // 2]:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
