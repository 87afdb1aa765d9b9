#!/bin/bash
# chunk sizing by workspace weight: config 4 whole and one rank's timeline, configs 3 and 5 for regressions, suite
cd "$(dirname "$0")/.."
timeout 1200 python tools/probe.py 4 --tag dense-svd --steps 5 2>&1 | grep -E "^wall" | tail -3
timeout 1500 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --save-masks /tmp/cfg4_w8.npz > gpurun_out/o_part.log 2>&1
for r in 5 0 2; do HX_TIMING=1 timeout 900 python tools/rank_sim.py 4 --worlds 8 --tag dense-svd --skip-full --load-masks /tmp/cfg4_w8.npz --ranks $r --steps 3 --warm 2 > gpurun_out/o_rank$r.log 2>&1; grep -E "world 8 rank" gpurun_out/o_rank$r.log; done
grep "hx timeline" gpurun_out/o_rank5.log | tail -1 | cut -c1-900
timeout 1200 python tools/probe.py 3 --tag aca --steps 4 2>&1 | grep -E "^wall" | tail -2
timeout 1200 python tools/probe.py 5 --tag dense-svd --steps 3 2>&1 | grep -E "^wall" | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
