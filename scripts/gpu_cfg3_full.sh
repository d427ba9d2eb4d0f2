#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg3 --layers 8 --distinct-layers 2 --decode-steps 4 --steps 2 --warmup 1 --trace-out gpurun_out/timeline_cfg3.json > gpurun_out/bench_cfg3_probe.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_cfg3.json >> gpurun_out/bench_cfg3_probe.log 2>&1
timeout 1200 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32 > gpurun_out/bench_cfg3.log 2>&1
timeout 900 python bench.py --config model --layers 32 --distinct-layers 4 --prompt 512 --steps 16 --warmup 3 > gpurun_out/bench_model.log 2>&1
echo done
