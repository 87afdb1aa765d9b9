#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --save-masks /tmp/cfg4_w8.npz > gpurun_out/n_part.log 2>&1
HX_TIMING=1 timeout 900 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --skip-full --load-masks /tmp/cfg4_w8.npz --ranks 5 --steps 1 --warm 2 > gpurun_out/n_rank5_timeline.log 2>&1
grep -E "hx timeline|world 8 rank" gpurun_out/n_rank5_timeline.log | tail -3 | cut -c1-1500
