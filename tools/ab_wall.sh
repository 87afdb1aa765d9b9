#!/bin/bash
# overlapped steady-state wall of the config-2 product for environment variants:
# tools/ab_wall.sh TAG "ENV1" "ENV2" ...  (2 interleaved rounds, 9 products each, median of the last 6)
cd "$(dirname "$0")/.."
tag=$1; shift
for rep in 1 2; do
  for env in "$@"; do
    env $env timeout 600 python tools/probe.py 2 --tag $tag --steps 9 2>&1 | grep "^wall" | tail -6 | sed 's/^wall \([0-9.]*\)s.*/\1/' | sort -n | python3 -c "
import sys
w=[1e3*float(x) for x in sys.stdin.read().split()]
print('== $env (run $rep): median wall %.1f ms  min %.1f  max %.1f' % ((w[2]+w[3])/2, w[0], w[-1]))"
  done
done
