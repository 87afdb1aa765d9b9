#!/bin/bash
# config 5 (dense-svd): per-kernel launch list of one product
cd "$(dirname "$0")/.."
HX_PP_EXTRA=0 timeout 2400 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c38_launches_cfg5.csv python tools/phase_profile.py 5 --tag dense-svd > gpurun_out/c38_cfg5.log 2>&1
tail -2 gpurun_out/c38_cfg5.log | cut -c1-300
