"""Build ``libhx.so`` in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

Usage: ``python -m paper_1805_08998_b200.build`` (also called by ``__graft_entry__.build``).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["plan.cpp", "errors.cpp", "hmx1.cpp", "runtime.cu"]
HEADERS = ["hx_types.h", "hx_internal.h", "gemm.cuh", "gemm_ws.cuh", "dense_la.cuh", "dense_la_warp.cuh",
           "qr_rows.cuh", "gather_gemm.cuh", "assemble.cuh", "iterative.cuh",
           "np_random.cuh", "traditional.cuh", "traditional_exec.cuh"]
OUT = os.path.join(HERE, "libhx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2,-fopenmp", "-shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-lgomp"]


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "hx.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _ziggurat_tables():
    """numpy's ziggurat tables for the device normal generator (tools/gen_ziggurat.py)."""
    sys.path.insert(0, os.path.join(HERE, "..", "tools"))
    try:
        import gen_ziggurat
    finally:
        sys.path.pop(0)
    gen_ziggurat.write(os.path.join(CSRC, "zig_tables.inc"))


def build(force=False, verbose=False):
    if not os.path.exists(os.path.join(CSRC, "zig_tables.inc")):
        _ziggurat_tables()
    if not force and not _stale():
        return OUT
    cmd = [NVCC, *FLAGS, *[os.path.join(CSRC, s) for s in SOURCES], "-o", OUT + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libhx.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
