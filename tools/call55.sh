#!/bin/bash
# config 4 at world 8 on the final code: world 1, then one fresh process per rank on a saved partition
cd "$(dirname "$0")/.."
timeout 1500 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --save-masks /tmp/cfg4_w8.npz 2>&1 | grep -E "cfg4 world 1|saved" | tee gpurun_out/p_cfg4_world1.log
for r in 0 1 2 3 4 5 6 7; do timeout 900 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --skip-full --load-masks /tmp/cfg4_w8.npz --ranks $r 2>&1 | grep "world 8 rank $r"; done | tee gpurun_out/p_cfg4_ranks.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/p_bench.log 2>&1; tail -1 gpurun_out/p_bench.log | cut -c1-260
