#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg5 --moe phimoe --batch 32 --steps 20 --no-cpu-baseline --trace-out gpurun_out/timeline_phimoe32.json > gpurun_out/bench_phimoe32.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_phimoe32.json >> gpurun_out/bench_phimoe32.log 2>&1
echo done
