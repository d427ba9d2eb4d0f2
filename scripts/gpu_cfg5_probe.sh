#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for i in 1 2 3 4; do
SP_TRACE_KEEP_CALLS=100000 timeout 600 python bench.py --config cfg5 --moe 8x22b --batch 4 --steps 30 --no-cpu-baseline --trace-out gpurun_out/tl_$i.json > gpurun_out/bench_8x22b_b4_$i.log 2>&1
python scripts/slowest_call.py gpurun_out/tl_$i.json 2>&1 | head -3 >> gpurun_out/bench_8x22b_b4_$i.log
done
echo done
