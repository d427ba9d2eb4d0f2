#!/bin/bash
# every BASELINE config on one B200 (+ the reference arm), JSON lines into gpurun_out/cfg/
mkdir -p gpurun_out/cfg
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/cfg/$name.log 2>&1; grep '^{' gpurun_out/cfg/$name.log | tail -1 > gpurun_out/cfg/$name.json; }
run bench_cfg2 --steps 100 --warmup 5
run bench_reference --impl reference --steps 3 --warmup 1
run bench_cfg1 --config cfg1 --steps 100 --warmup 5
run bench_cfg4 --config cfg4 --steps 30 --no-cpu-baseline
for b in 1 4 16 32; do run bench_cfg5_8x22b_b$b --config cfg5 --moe 8x22b --batch $b --steps 30 --no-cpu-baseline; done
for b in 1 8 32; do run bench_cfg5_phimoe_b$b --config cfg5 --moe phimoe --batch $b --steps 30 --no-cpu-baseline; done
run bench_cfg3 --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 128
run bench_cfg3_layerplan --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 128 --token-plan layer
run bench_model_decode --config model --layers 32 --distinct-layers 4 --prompt 512 --steps 16 --warmup 3
run bench_cfg2_all_gg --budget-frac 1.0 --steps 200 --warmup 10 --no-cpu-baseline
echo done
