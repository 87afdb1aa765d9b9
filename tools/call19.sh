#!/bin/bash
# GPU session: full GPU tests, A/B of the current build, config-3 measurements
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputests3.log 2>&1; echo rc=$? >> gpurun_out/gputests3.log
HX_OVERLAP=0 bash tools/ab_phases.sh aca "HX_GEMM_WS=1" > gpurun_out/ab_final.log 2>&1
timeout 600 python tools/unit_table.py --config 3 --tag aca > gpurun_out/ut3.log 2>&1
mkdir -p gpurun_out/bench_data; cp bench_data/*.npz gpurun_out/bench_data/ 2>/dev/null
HX_RECOMP_TIMING=1 timeout 900 python tools/probe.py 3 --steps 3 --tag aca > gpurun_out/probe3_recomp.log 2>&1
timeout 1500 python bench.py --config 3 --steps 3 --warmup 3 --alt-tag dense-svd > gpurun_out/bench_cfg3.log 2>&1
timeout 900 python bench.py --impl reference --config 3 --steps 2 --warmup 1 --cpu-budget 20 > gpurun_out/bench_ref_cfg3.log 2>&1
tail -3 gpurun_out/gputests3.log; cat gpurun_out/ab_final.log; tail -2 gpurun_out/ut3.log
