#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c47_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c47_tests.log
for lib in build/libhx_prev.so paper_1805_08998_b200/libhx.so; do echo "== cfg4 $lib"; HX_LIB=$PWD/$lib timeout 1200 python tools/probe.py 4 --tag dense-svd --steps 5 2>&1 | grep -E "^wall" | tail -3; done
for lib in build/libhx_prev.so paper_1805_08998_b200/libhx.so; do echo "== cfg3 $lib"; HX_LIB=$PWD/$lib timeout 1200 python tools/probe.py 3 --tag aca --steps 5 2>&1 | grep -E "^wall" | tail -3; done
