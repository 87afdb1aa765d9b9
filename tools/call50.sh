#!/bin/bash
# round-2 closing evidence on the final code: suite, smoke, bench (both arms), config-3 bench, launch list
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/z_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/z_tests.log
timeout 600 python __graft_entry__.py > gpurun_out/z_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/z_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/z_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/z_bench.log 2>&1; echo "bench rc=$?"
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/z_bench_cfg3.log 2>&1; echo "cfg3 rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/z_launches.csv python tools/phase_profile.py 2 --tag aca > gpurun_out/z_launch_ncu.log 2>&1
tail -1 gpurun_out/z_bench.log | cut -c1-300
