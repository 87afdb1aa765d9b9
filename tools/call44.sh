#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for g in 0 1; do echo -n "HX_BENCH_GC=$g run $rep: "; HX_BENCH_GC=$g timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --alt-tag '' 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"; done; done
