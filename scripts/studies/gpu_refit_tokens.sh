#!/bin/bash
# batched-decode profiles (tokens per expert 2, 4, 8), then the cfg5 sweep on them
mkdir -p gpurun_out/cfg
for t in 2 4 8; do
  timeout 900 python -m paper_2411_15715_b200.b200_profile --tokens $t --out profiles > gpurun_out/refit_t$t.log 2>&1
  cp profiles/b200_decode_t$t.json profiles/b200_samples_decode_t$t.csv gpurun_out/ 2>/dev/null
done
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/cfg/$name.log 2>&1; grep '^{' gpurun_out/cfg/$name.log | tail -1 > gpurun_out/cfg/$name.json; }
for b in 4 16 32; do run bench_cfg5_8x22b_b$b --config cfg5 --moe 8x22b --batch $b --steps 30 --no-cpu-baseline; done
for b in 8 32; do run bench_cfg5_phimoe_b$b --config cfg5 --moe phimoe --batch $b --steps 30 --no-cpu-baseline; done
echo done
