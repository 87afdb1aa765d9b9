#!/bin/bash
# A/B of product phases on config 2 (one isolated product after a warm-up, CUDA events per
# phase) for environment variants: tools/ab_phases.sh TAG "ENV1" "ENV2" ...
tag=$1; shift
for env in "$@"; do
  for rep in 1 2; do
    echo "== $env (run $rep)"
    env $env timeout 600 python tools/phase_profile.py 2 --tag $tag 2>&1 | grep "^plan"
  done
done
