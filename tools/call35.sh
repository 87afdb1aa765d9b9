#!/bin/bash
# round-2 final evidence (session 4): suite, bench (both arms, cfg2 and cfg3), launch list, ncu --set full of the
# materialization and of formation launches, rank simulation of config 3 with 2 cores per rank
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/f_tests.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/f_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 600 python tools/phase_profile.py 2 --tag aca --flops > gpurun_out/f_phase.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python tools/phase_profile.py 2 --tag aca > gpurun_out/f_launch_ncu.log 2>&1
HX_OVERLAP=0 timeout 1200 ncu --profile-from-start off --nvtx --nvtx-include "hx::materialize/" -k regex:grouped_gemm --set full --clock-control none --import-source on -o gpurun_out/f_mat python tools/phase_profile.py 2 --tag aca > gpurun_out/f_mat_ncu.log 2>&1
HX_OVERLAP=0 timeout 1200 ncu --profile-from-start off --nvtx --nvtx-include "hx::form/" -k regex:grouped_gemm -s 20 -c 4 --set full --clock-control none --import-source on -o gpurun_out/f_form python tools/phase_profile.py 2 --tag aca > gpurun_out/f_form_ncu.log 2>&1
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/f_bench_cfg3.log 2>&1; echo "cfg3 rc=$?"
timeout 1500 python tools/rank_sim.py 3 --worlds 8 --tag aca > gpurun_out/f_rank_sim_cfg3_full.log 2>&1
OMP_NUM_THREADS=2 timeout 1500 taskset -c 0-1 python tools/rank_sim.py 3 --worlds 8 --tag aca --skip-full > gpurun_out/f_rank_sim_cfg3_2c.log 2>&1
tail -1 gpurun_out/f_bench.log | cut -c1-400; tail -3 gpurun_out/f_rank_sim_cfg3_2c.log
