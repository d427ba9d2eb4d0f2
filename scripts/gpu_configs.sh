#!/bin/bash
# BASELINE configs 4 and 5 on one B200 (cfg4: the 1-GPU shard = the whole layer)
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg4 --steps 30 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1
for b in 1 4 16 32; do
  timeout 900 python bench.py --config cfg5 --moe 8x22b --batch $b --steps 30 --no-cpu-baseline > gpurun_out/bench_cfg5_8x22b_b$b.log 2>&1
done
for b in 1 8 32; do
  timeout 900 python bench.py --config cfg5 --moe phimoe --batch $b --steps 30 --no-cpu-baseline > gpurun_out/bench_cfg5_phimoe_b$b.log 2>&1
done
echo done
