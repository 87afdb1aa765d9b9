#!/bin/bash
# A/B of library builds on one box: tools/ab_lib.sh TAG lib1.so lib2.so ... (interleaved, 2 rounds;
# one isolated config-2 product per line, CUDA events per phase, HX_OVERLAP=0)
cd "$(dirname "$0")/.."
tag=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (run $rep)"
    HX_LIB=$PWD/$lib HX_OVERLAP=0 timeout 600 python tools/phase_profile.py 2 --tag $tag 2>&1 | grep "^plan"
  done
done
