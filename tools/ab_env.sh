#!/bin/bash
# A/B of environment variants on one box: tools/ab_env.sh TAG "ENV1" "ENV2" ... (2 interleaved rounds, HX_OVERLAP=0)
cd "$(dirname "$0")/.."
tag=$1; shift
for rep in 1 2; do
  for env in "$@"; do
    echo "== $env (run $rep)"
    env $env HX_OVERLAP=0 timeout 600 python tools/phase_profile.py 2 --tag $tag 2>&1 | grep "^plan"
  done
done
