#!/bin/bash
# profile refit + bench + reference arm + ncu launch list (one GPU)
set -x
mkdir -p gpurun_out
timeout 600 python -m paper_2411_15715_b200.b200_profile --out profiles > gpurun_out/refit.log 2>&1
cp profiles/b200_decode.json profiles/b200_samples_decode.csv gpurun_out/ 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 3 --trace-out gpurun_out/timeline.json > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo done
