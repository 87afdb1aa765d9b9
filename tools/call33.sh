#!/bin/bash
cd "$(dirname "$0")/.."
HX_OVERLAP=0 timeout 1200 ncu --profile-from-start off --nvtx --nvtx-include "hx::form/" -k regex:grouped_gemm -s 20 -c 4 --set full --clock-control none --import-source on -o gpurun_out/p33_form python tools/phase_profile.py 2 --tag aca > gpurun_out/p33_form_ncu.log 2>&1
tail -2 gpurun_out/p33_form_ncu.log
