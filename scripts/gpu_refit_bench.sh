#!/bin/bash
# concurrent-load decode refit, bench on the refit profile (+ timeline)
mkdir -p gpurun_out
timeout 900 python -m paper_2411_15715_b200.b200_profile --out profiles > gpurun_out/refit.log 2>&1
cp profiles/b200_decode.json profiles/b200_samples_decode.csv gpurun_out/ 2>/dev/null
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --trace-out gpurun_out/timeline.json > gpurun_out/bench.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline.json >> gpurun_out/bench.log 2>&1
echo done
