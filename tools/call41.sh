#!/bin/bash
cd "$(dirname "$0")/.."
HX_IMPLICIT=256 HX_PP_EXTRA=0 HX_OVERLAP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c41_launches_impl256.csv python tools/phase_profile.py 2 --tag dense-svd > gpurun_out/c41.log 2>&1
HX_RECOMP_TIMING=1 HX_IMPLICIT=256 HX_PP_EXTRA=0 HX_OVERLAP=0 timeout 900 python tools/phase_profile.py 2 --tag dense-svd > gpurun_out/c41_timing.log 2>&1
