#!/bin/bash
# metadata copies on the copy stream from double-buffered device metadata (new) vs on the compute stream (old):
# headline (fixed rates), batched decode, cfg3 layer plan; alternating builds
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2 3; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    for cfg in "--steps 100" "--config cfg5 --moe phimoe --batch 32 --steps 40" "--config cfg5 --moe 8x22b --batch 4 --steps 40"; do
      timeout 600 python bench.py $cfg --no-cpu-baseline --calibrate 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $cfg', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
    done
  done
done
for r in 1 2; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    timeout 900 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 8 --token-plan layer --calibrate 0 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'decode', round(d['decode_tokens_per_s'],2))"
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
