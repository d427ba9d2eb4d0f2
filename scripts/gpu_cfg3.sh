#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m paper_2411_15715_b200.b200_profile --phase prompt --out profiles > gpurun_out/refit_prompt.log 2>&1
cp profiles/b200_prompt.json profiles/b200_samples_prompt.csv gpurun_out/ 2>/dev/null
timeout 1200 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32 > gpurun_out/bench_cfg3.log 2>&1
echo done
