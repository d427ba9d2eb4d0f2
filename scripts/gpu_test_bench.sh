#!/bin/bash
# GPU tests (bounded) then the headline bench with a timeline
mkdir -p gpurun_out
timeout 180 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
grep -q "rc=0" gpurun_out/gpu_tests.log || exit 1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --trace-out gpurun_out/timeline.json ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline.json >> gpurun_out/bench.log 2>&1
echo done
