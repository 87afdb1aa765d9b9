"""Stage timings of the end-to-end product (host operands in, every block out).

usage: HX_TIMING=1 python tools/e2e_profile.py CFG
"""
import sys
import time

sys.path.insert(0, ".")
import paper_1805_08998_b200 as hx  # noqa: E402
from paper_1805_08998_b200 import configs, multiply  # noqa: E402


def main():
    c = configs.CONFIGS[int(sys.argv[1])]
    bct, A, B = configs.build_operands(c)
    multiply._host_directory(A)
    if B is not A:
        multiply._host_directory(B)
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind("dense-svd"), policy=hx.EpsRank(c["tol"]))
    for _ in range(3):
        t0 = time.perf_counter()
        C = multiply.multiply_device(A, B, cfg, device_operands=False)
        t1 = time.perf_counter()
        n = sum(1 for _ in C.data.values())
        t2 = time.perf_counter()
        print(f"e2e {1e3 * (t1 - t0):.1f} ms (+ touching {n} leaves {1e3 * (t2 - t1):.1f} ms)",
              flush=True)


if __name__ == "__main__":
    main()
