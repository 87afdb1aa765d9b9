#!/bin/bash
# block-sparse T_sub of the implicit leaves: suite, config-2 dense-svd A/B, config 4 products
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c42_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/c42_tests.log
bash tools/ab_lib.sh dense-svd build/libhx_head.so paper_1805_08998_b200/libhx.so
for lib in build/libhx_head.so paper_1805_08998_b200/libhx.so; do echo "== cfg4 $lib"; HX_LIB=$PWD/$lib timeout 1200 python tools/probe.py 4 --tag dense-svd --steps 4 2>&1 | grep -E "^wall|^cfg4" ; done
