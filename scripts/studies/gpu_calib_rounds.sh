#!/bin/bash
# Fixed-point calibration (--calib-rounds 3) vs one round (--calib-rounds 1) on the
# lines whose predicted / measured step was off after one round (batched decode).
mkdir -p gpurun_out/calib
F=gpurun_out/calib
run() { local name=$1; shift; timeout 600 python bench.py "$@" > $F/$name.log 2>&1; grep '^{' $F/$name.log | tail -1 > $F/$name.json; }
run cfg1 --config cfg1 --steps 100 --warmup 5 --no-cpu-baseline
for r in 3 1; do
  run b16_r$r --config cfg5 --moe 8x22b --batch 16 --steps 30 --no-cpu-baseline --calib-rounds $r
  run phi32_r$r --config cfg5 --moe phimoe --batch 32 --steps 30 --no-cpu-baseline --calib-rounds $r
  run phi8_r$r --config cfg5 --moe phimoe --batch 8 --steps 30 --no-cpu-baseline --calib-rounds $r
  run cfg2_r$r --steps 100 --no-cpu-baseline --calib-rounds $r
done
echo done
