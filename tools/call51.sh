#!/bin/bash
# per-block oracle at full size on the final code (block-sparse T_sub, gather kernel): config 4 implicit sizes, config 5 up to 4096
cd "$(dirname "$0")/.."
timeout 2400 python tools/block_oracle.py 4 --per-class 3 --min-size 512 --near 2 > gpurun_out/k_block_oracle_cfg4.log 2>&1; tail -3 gpurun_out/k_block_oracle_cfg4.log
timeout 2400 python tools/block_oracle.py 5 --per-class 3 --min-size 512 --max-size 4096 --near 2 > gpurun_out/k_block_oracle_cfg5.log 2>&1; tail -3 gpurun_out/k_block_oracle_cfg5.log
