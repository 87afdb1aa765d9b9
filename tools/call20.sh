#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputests4.log 2>&1; echo rc=$? >> gpurun_out/gputests4.log
timeout 900 python bench.py > gpurun_out/bench_final1.log 2>&1
timeout 2400 python tools/block_oracle.py 5 --blocks 350815,352171,85489 --values-max 16384 > gpurun_out/bo5e.log 2>&1
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1
timeout 900 python tools/probe.py 5 --steps 3 > gpurun_out/probe5.log 2>&1
tail -3 gpurun_out/gputests4.log; tail -4 gpurun_out/bo5e.log
