#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c34_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c34_tests.log
bash tools/ab_lib.sh aca build/libhx_old.so paper_1805_08998_b200/libhx.so
