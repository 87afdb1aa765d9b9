#!/bin/bash
# final state: suite, smoke, bench (both arms), config 5 and config 4 (aca) products
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g_tests.log
timeout 600 python __graft_entry__.py > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g_smoke.log
timeout 900 python bench.py > gpurun_out/g_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/g_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/g_bench_torchrun.log 2>&1; echo "torchrun rc=$?"
timeout 1500 python tools/probe.py 5 --tag dense-svd --steps 4 > gpurun_out/g_cfg5.log 2>&1; grep -E "^wall|^cfg5" gpurun_out/g_cfg5.log
timeout 1500 python tools/probe.py 4 --tag aca --steps 4 --estimate 16 > gpurun_out/g_cfg4_aca.log 2>&1; grep -E "^wall|^cfg4|estimated" gpurun_out/g_cfg4_aca.log
tail -1 gpurun_out/g_bench.log | cut -c1-300
