#!/bin/bash
# default bench (cfg2 decode), packed-FFMA2 GEMV (new) vs scalar (old), alternating
mkdir -p gpurun_out/ffma2b
F=gpurun_out/ffma2b/ab.txt
L=paper_2411_15715_b200/_native/libsliced.so
: > $F
for r in 1 2 3 4; do
  for v in new old; do
    cp _ab/$v.so $L
    timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); rf=d['roofline']
print('bench $v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'gg_frac', round(rf['frac'],3), 'dev', round(rf['frac_device_span'],3), 'cc', round(d['split']['rates']['cc'],4))" >> $F 2>&1
  done
done
cp _ab/new.so $L
echo done
