#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg3 --layers 8 --distinct-layers 2 --decode-steps 4 --steps 2 --warmup 1 --trace-out gpurun_out/timeline_cfg3.json > gpurun_out/bench_cfg3.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_cfg3.json >> gpurun_out/bench_cfg3.log 2>&1
echo done
