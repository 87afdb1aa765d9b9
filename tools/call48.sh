#!/bin/bash
# rank simulations after the planner's compact-key sort
cd "$(dirname "$0")/.."
OMP_NUM_THREADS=2 timeout 1500 taskset -c 0-1 python tools/rank_sim.py 3 --worlds 8 --tag aca --skip-full > gpurun_out/h_rank_sim_cfg3_2c.log 2>&1; tail -10 gpurun_out/h_rank_sim_cfg3_2c.log
timeout 1500 python tools/rank_sim.py 3 --worlds 8 --tag aca > gpurun_out/h_rank_sim_cfg3_full.log 2>&1; tail -10 gpurun_out/h_rank_sim_cfg3_full.log
timeout 2400 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd > gpurun_out/h_rank_sim_cfg4_full.log 2>&1; tail -10 gpurun_out/h_rank_sim_cfg4_full.log
