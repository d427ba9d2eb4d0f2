#!/bin/bash
# correctness + GEMV micro-bench + host CC micro-bench + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python scripts/bench_gemv.py --T 1 2 4 --hidden 1024 4096 7168 14336 --reps 8 > gpurun_out/gemv.log 2>&1
timeout 300 python scripts/bench_cc.py > gpurun_out/cc.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --trace-out gpurun_out/timeline.json > gpurun_out/bench.log 2>&1
echo done
