#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/ab_phases.sh aca "HX_WS_RESERVE=0" "HX_WS_RESERVE=8" "HX_WS_RESERVE=16" > gpurun_out/ab_reserve.log 2>&1
timeout 1500 python tools/rank_sim.py 3 --worlds 8 --steps 2 --warm 1 --tag aca > gpurun_out/rank3_full.log 2>&1
OMP_NUM_THREADS=2 timeout 2400 taskset -c 0-1 python tools/rank_sim.py 3 --worlds 8 --steps 2 --warm 1 --tag aca --skip-full > gpurun_out/rank3_2core.log 2>&1
timeout 900 python tools/block_oracle.py 2 --per-class 12 --near 8 --tag aca > gpurun_out/bo2.log 2>&1
timeout 1500 python tools/block_oracle.py 3 --per-class 10 --near 8 --tag aca > gpurun_out/bo3.log 2>&1
tail -2 gpurun_out/rank3_full.log; tail -2 gpurun_out/rank3_2core.log; tail -2 gpurun_out/bo2.log; tail -2 gpurun_out/bo3.log; cat gpurun_out/ab_reserve.log
