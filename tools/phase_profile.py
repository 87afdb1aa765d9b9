"""One product of a BASELINE config under an ncu range (second product; the first warms up).

usage: ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --csv --log-file out.csv python tools/phase_profile.py CFG [--tag aca]
then:  python tools/phase_profile.py --summarize out.csv
"""
import collections
import csv
import sys

sys.path.insert(0, ".")


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), \
        h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        d = launches.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
        d[r[ni]] = float(r[vi].replace(",", ""))
    runs = []
    for d in launches.values():
        t = d.get("gpu__time_duration.sum", 0.0) / 1e6
        b = (d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)) / 1e9
        if runs and runs[-1][0] == d["name"]:
            runs[-1][1] += 1
            runs[-1][2] += t
            runs[-1][3] += b
        else:
            runs.append([d["name"], 1, t, b])
    tot = sum(r[2] for r in runs)
    for name, n, t, b in runs:
        if t < 0.05:
            continue
        print(f"{t:9.2f} ms x{n:<4d} {b:8.2f} GB {b / max(t, 1e-9):8.1f} GB/s  {name}")
    print(f"{tot:9.2f} ms total")


def main():
    if sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
        return
    import torch
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import configs

    c = configs.CONFIGS[int(sys.argv[1])]
    bct, A, B = configs.build_operands(c)
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "aca"
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(tag), policy=hx.EpsRank(c["tol"]))
    hx.multiply.multiply_device(A, B, cfg, fetch=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    out = hx.multiply.multiply_device(A, B, cfg, fetch=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    r = out.report
    walls = []
    import os
    for _ in range(int(os.environ.get("HX_PP_EXTRA", "3"))):
        walls.append(hx.multiply.multiply_device(A, B, cfg, fetch=False).report.wall_s * 1e3)
    print(f"plan {r.plan_ms:.0f} dev {r.device_ms:.1f} form {r.form_ms:.1f} "
          f"mat {r.materialize_ms:.1f} recomp {r.recompress_ms:.1f} wall(3 more) "
          f"{' '.join(f'{w:.1f}' for w in walls)} ms")
    info = out.plan_info
    print({f[0]: getattr(info, f[0]) for f in info._fields_ if f[0] != "created"})
    if "--flops" in sys.argv:
        import numpy as np
        from paper_1805_08998_b200 import _lib, hmatrix, multiply
        _, dA = multiply.operand_directory(A)
        _, dB = multiply.operand_directory(B)
        wp = _lib.Plan(hmatrix.tree_arrays(bct), dA, dA if B is A else dB, None,
                       multiply.plan_tile(bct))
        mma = np.zeros(6)
        _lib.check(_lib.lib().hx_plan_mma_flops(wp.h, _lib.ptr(mma, _lib.f64p)), "mma")
        print("issued core/fac/mat GF", mma[:3] / 1e9, "useful", mma[3:] / 1e9)


if __name__ == "__main__":
    main()
