#!/bin/bash
mkdir -p gpurun_out/cfg
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
grep -q "rc=0" gpurun_out/gpu_tests.log || exit 1
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/cfg/$name.log 2>&1; grep '^{' gpurun_out/cfg/$name.log | tail -1 > gpurun_out/cfg/$name.json; }
for b in 4 16 32; do run bench_cfg5_8x22b_b$b --config cfg5 --moe 8x22b --batch $b --steps 30 --no-cpu-baseline --trace-out gpurun_out/tl_8x22b_b$b.json; done
for b in 8 32; do run bench_cfg5_phimoe_b$b --config cfg5 --moe phimoe --batch $b --steps 30 --no-cpu-baseline --trace-out gpurun_out/tl_phimoe_b$b.json; done
run bench_cfg2 --steps 100
echo done
