#!/bin/bash
# config 4 at world 8, one fresh process per rank on a saved partition (no carry-over of device memory state between ranks)
cd "$(dirname "$0")/.."
timeout 1500 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --save-masks /tmp/cfg4_w8.npz > gpurun_out/m_cfg4_partition.log 2>&1; tail -2 gpurun_out/m_cfg4_partition.log
for r in 0 1 2 3 4 5 6 7; do timeout 900 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --skip-full --load-masks /tmp/cfg4_w8.npz --ranks $r 2>&1 | grep "world 8 rank $r"; done | tee gpurun_out/m_cfg4_ranks.log
