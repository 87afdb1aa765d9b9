#!/bin/bash
# warp-specialized gather GEMM: suite, then A/B on config 2 dense-svd (HEAD build vs new)
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c36_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/c36_tests.log
bash tools/ab_lib.sh dense-svd build/libhx_head.so paper_1805_08998_b200/libhx.so
