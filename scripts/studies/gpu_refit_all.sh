#!/bin/bash
# decode refits (T = 1, 2, 4, 8 tokens per expert) after a host-kernel change, then cfg2 + cfg5 benches
mkdir -p gpurun_out/cfg
timeout 900 python -m paper_2411_15715_b200.b200_profile --out profiles > gpurun_out/refit.log 2>&1
cp profiles/b200_decode.json profiles/b200_samples_decode.csv gpurun_out/ 2>/dev/null
for t in 2 4 8; do
  timeout 900 python -m paper_2411_15715_b200.b200_profile --tokens $t --out profiles > gpurun_out/refit_t$t.log 2>&1
  cp profiles/b200_decode_t$t.json profiles/b200_samples_decode_t$t.csv gpurun_out/ 2>/dev/null
done
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/cfg/$name.log 2>&1; grep '^{' gpurun_out/cfg/$name.log | tail -1 > gpurun_out/cfg/$name.json; }
run bench_cfg2 --steps 100 --warmup 5 --trace-out gpurun_out/timeline.json
for b in 4 16 32; do run bench_cfg5_8x22b_b$b --config cfg5 --moe 8x22b --batch $b --steps 30 --no-cpu-baseline; done
for b in 1 8 32; do run bench_cfg5_phimoe_b$b --config cfg5 --moe phimoe --batch $b --steps 30 --no-cpu-baseline; done
run bench_cfg5_8x22b_b1 --config cfg5 --moe 8x22b --batch 1 --steps 30 --no-cpu-baseline
run bench_cfg4 --config cfg4 --steps 30 --no-cpu-baseline
run bench_cfg1 --config cfg1 --steps 100 --warmup 5
echo done
