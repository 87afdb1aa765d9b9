#!/bin/bash
# final profiles: launch list of one config-2 product and an ncu --set full capture of the
# dominant kernel's launches (materialization), both after the same program ran clean
cd "$(dirname "$0")/.."
timeout 900 python bench.py > gpurun_out/bench_final2.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1
timeout 600 python tools/phase_profile.py 2 --tag aca > gpurun_out/final_phase.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python tools/phase_profile.py 2 --tag aca > gpurun_out/final_launch_ncu.log 2>&1
HX_OVERLAP=0 timeout 1200 ncu --profile-from-start off --nvtx --nvtx-include "hx::materialize/" -k regex:grouped_gemm --set full --clock-control none --import-source on -o gpurun_out/final_mat python tools/phase_profile.py 2 --tag aca > gpurun_out/final_mat_ncu.log 2>&1
tail -2 gpurun_out/final_phase.log
