#!/bin/bash
cd "$(dirname "$0")/.."
timeout 2400 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd > gpurun_out/i_rank_sim_cfg4_full.log 2>&1; tail -10 gpurun_out/i_rank_sim_cfg4_full.log
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q 2>&1 | tail -2
