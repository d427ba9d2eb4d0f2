#!/bin/bash
# GEMV kernel with packed FFMA2 (new) vs scalar FFMA (old): parity with the new
# library, then the GG GEMV microbench and the default bench, alternating.
# _ab/{old,new}.so are built from the two kernels.cuh versions.
mkdir -p gpurun_out/ffma2
F=gpurun_out/ffma2/ab.txt
L=paper_2411_15715_b200/_native/libsliced.so
: > $F
cp _ab/new.so $L
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/ffma2/gputest.log 2>&1; echo "gpu tests rc=$?" >> $F
tail -2 gpurun_out/ffma2/gputest.log >> $F
for r in 1 2 3; do
  for v in old new; do
    cp _ab/$v.so $L
    echo "== round $r $v" >> $F
    timeout 300 python scripts/bench_gemv.py --T 1 2 4 --hidden 14336 --reps 20 >> $F 2>&1
    timeout 300 python scripts/bench_gemv.py --T 1 2 --model 6144 --hidden 8192 --reps 20 >> $F 2>&1
    timeout 300 python scripts/bench_gemv.py --T 1 4 --model 1024 --hidden 1792 --dtype f32 --reps 20 >> $F 2>&1
  done
done
for r in 1 2; do
  for v in old new; do
    cp _ab/$v.so $L
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); rf=d['roofline']
print('bench $v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'gg_frac', round(rf['frac'],3), 'dev', round(rf['frac_device_span'],3))" >> $F 2>&1
    timeout 300 python bench.py --config cfg5 --moe phimoe --batch 32 --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); rf=d['roofline']
print('phimoe b32 $v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'gg_frac', round(rf['frac'],3), 'dev', round(rf['frac_device_span'],3))" >> $F 2>&1
  done
done
cp _ab/new.so $L
echo done
