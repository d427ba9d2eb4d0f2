#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --trace-out gpurun_out/timeline.json > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/bench_cfg1.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo done
