#!/bin/bash
# GPU tests, prompt-phase refit (in-situ), cfg3 (8-layer probe with timeline, then 32 layers)
mkdir -p gpurun_out
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
grep -q "rc=0" gpurun_out/gpu_tests.log || exit 1
timeout 900 python -m paper_2411_15715_b200.b200_profile --phase prompt --out profiles > gpurun_out/refit_prompt.log 2>&1
cp profiles/b200_prompt.json profiles/b200_samples_prompt.csv gpurun_out/ 2>/dev/null
timeout 600 python bench.py --config cfg3 --layers 8 --distinct-layers 2 --decode-steps 4 --steps 2 --warmup 1 --trace-out gpurun_out/timeline_cfg3.json > gpurun_out/bench_cfg3_probe.log 2>&1
python scripts/timeline_summary.py gpurun_out/timeline_cfg3.json >> gpurun_out/bench_cfg3_probe.log 2>&1
timeout 1200 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32 > gpurun_out/bench_cfg3.log 2>&1
echo done
