#!/bin/bash
# correctness + headline bench + prefill tcgen05 micro-bench (one GPU)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python scripts/bench_prefill.py 14336 > gpurun_out/prefill.log 2>&1
timeout 600 python scripts/bench_prefill.py 7168 >> gpurun_out/prefill.log 2>&1
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo done
