#!/bin/bash
# WS kernel: branch-free epilogue, arithmetic fragment masks, hull-restricted staging, aligned column staging
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c32_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c32_tests.log
for rep in 1 2; do HX_OVERLAP=0 timeout 600 python tools/phase_profile.py 2 --tag aca 2>&1 | grep "^plan"; done
timeout 900 python bench.py > gpurun_out/c32_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/c32_bench.log | cut -c1-700
