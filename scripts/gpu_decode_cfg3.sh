#!/bin/bash
# decode in-situ refit + headline bench; cfg3 probe with device- and host-I/O timelines
mkdir -p gpurun_out
timeout 900 python -m paper_2411_15715_b200.b200_profile --out profiles > gpurun_out/refit.log 2>&1
cp profiles/b200_decode.json profiles/b200_samples_decode.csv gpurun_out/ 2>/dev/null
timeout 300 python bench.py --steps 50 --warmup 5 --trace-out gpurun_out/timeline.json > gpurun_out/bench.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline.json >> gpurun_out/bench.log 2>&1
timeout 600 python bench.py --config cfg3 --layers 8 --distinct-layers 2 --decode-steps 4 --steps 2 --warmup 1 --trace-out gpurun_out/timeline_cfg3.json > gpurun_out/bench_cfg3_probe.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_cfg3.json >> gpurun_out/bench_cfg3_probe.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_cfg3_hostio.json >> gpurun_out/bench_cfg3_probe.log 2>&1
echo done
