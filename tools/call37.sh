#!/bin/bash
cd "$(dirname "$0")/.."
for v in head new; do
  if [ $v = head ]; then export HX_LIB=$PWD/build/libhx_head.so; else export HX_LIB=$PWD/paper_1805_08998_b200/libhx.so; fi
  HX_OVERLAP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c37_launches_$v.csv python tools/phase_profile.py 2 --tag dense-svd > gpurun_out/c37_$v.log 2>&1
done
