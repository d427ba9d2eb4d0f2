#!/bin/bash
# cfg3 with the committed profiles: 8-layer probe (device + host I/O timelines), then the 32-layer run
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg3 --layers 8 --distinct-layers 2 --decode-steps 4 --steps 2 --warmup 1 --trace-out gpurun_out/timeline_cfg3.json > gpurun_out/bench_cfg3_probe.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_cfg3.json >> gpurun_out/bench_cfg3_probe.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_cfg3_hostio.json >> gpurun_out/bench_cfg3_probe.log 2>&1
timeout 1200 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32 > gpurun_out/bench_cfg3.log 2>&1
echo done
