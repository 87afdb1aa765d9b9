#!/bin/bash
# session-4 start: full GPU suite, smoke, config-2 bench (both arms) on the checkpointed state
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gputests.log 2>&1; echo "tests rc=$?" 
timeout 600 python __graft_entry__.py > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/s4_bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/s4_gputests.log; tail -1 gpurun_out/s4_smoke.log; tail -1 gpurun_out/s4_bench.log | cut -c1-1500
