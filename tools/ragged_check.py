"""Ragged-tree check on the GPU: config 2's geometry and kernel with n not a power of two
(leaves at different depths), exact global error against a dense product.

usage: python tools/ragged_check.py [N]
"""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_1805_08998_b200 as hx  # noqa: E402
from paper_1805_08998_b200 import configs  # noqa: E402
from probe import dense_on_gpu  # noqa: E402


def main():
    import torch

    c = dict(configs.CONFIGS[2])
    c["n"] = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
    bct, A, B = configs.build_operands(c)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("dense-svd"),
                            policy=hx.EpsRank(c["tol"]))
    for _ in range(2):
        t0 = time.time()
        C = hx.hmult_new(A, B, cfg)
        print(f"n={c['n']} wall {time.time() - t0:.3f}s max far rank {C.report.max_far_rank}",
              flush=True)
    da = dense_on_gpu(A, torch)
    dc = dense_on_gpu(C, torch)
    ex = da @ da
    err = (torch.linalg.norm(dc - ex) / torch.linalg.norm(ex)).item()
    print(f"rel err ||C - AB||/||AB|| = {err:.3e} (tol {c['tol']})")


if __name__ == "__main__":
    main()
