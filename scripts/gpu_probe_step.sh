#!/bin/bash
# decode step anatomy: link micro-bench + traced bench timeline
mkdir -p gpurun_out
timeout 300 python scripts/bench_link.py > gpurun_out/link.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --trace-out gpurun_out/timeline.json > gpurun_out/bench.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline.json > gpurun_out/timeline_summary.txt 2>&1
echo done
