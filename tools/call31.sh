#!/bin/bash
# round-2 profiles of the current state: launch list of one config-2 product, ncu --set full of the
# materialization launches and of six formation launches (after the same program ran clean)
cd "$(dirname "$0")/.."
timeout 600 python tools/phase_profile.py 2 --tag aca --flops > gpurun_out/p31_phase.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p31_launches.csv python tools/phase_profile.py 2 --tag aca > gpurun_out/p31_launch_ncu.log 2>&1
HX_OVERLAP=0 timeout 1200 ncu --profile-from-start off --nvtx --nvtx-include "hx::materialize/" -k regex:grouped_gemm --set full --clock-control none --import-source on -o gpurun_out/p31_mat python tools/phase_profile.py 2 --tag aca > gpurun_out/p31_mat_ncu.log 2>&1
HX_OVERLAP=0 timeout 1200 ncu --profile-from-start off --nvtx --nvtx-include "hx::form/" -k regex:grouped_gemm -s 20 -c 6 --set full --clock-control none --import-source on -o gpurun_out/p31_form python tools/phase_profile.py 2 --tag aca > gpurun_out/p31_form_ncu.log 2>&1
tail -3 gpurun_out/p31_phase.log
