#!/bin/bash
# GPU tests then the headline bench, repeated (run-to-run spread of the host side)
mkdir -p gpurun_out
timeout 180 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
grep -q "rc=0" gpurun_out/gpu_tests.log || exit 1
timeout 120 python scripts/bench_cc.py --quick > gpurun_out/cc.log 2>&1
for i in 1 2 3; do
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --trace-out gpurun_out/timeline$i.json ${BENCH_ARGS} > gpurun_out/bench$i.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline$i.json >> gpurun_out/bench$i.log 2>&1
done
echo done
