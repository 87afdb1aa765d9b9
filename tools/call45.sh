#!/bin/bash
cd "$(dirname "$0")/.."
HX_PP_EXTRA=0 timeout 2400 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c45_launches_cfg4.csv python tools/phase_profile.py 4 --tag dense-svd > gpurun_out/c45_cfg4.log 2>&1
HX_RECOMP_TIMING=1 HX_PP_EXTRA=1 timeout 1200 python tools/phase_profile.py 4 --tag dense-svd > gpurun_out/c45_cfg4_timing.log 2>&1
tail -2 gpurun_out/c45_cfg4.log | cut -c1-200
