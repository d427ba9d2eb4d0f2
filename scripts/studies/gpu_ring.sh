#!/bin/bash
# CG ring depth A/B: cfg3 prefill and cfg2 decode, alternating on one box
mkdir -p gpurun_out
for r in 1 2; do
  for v in 3 6; do
    SP_RING_SLOTS=$v timeout 600 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 8 --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 slots=$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done > gpurun_out/ring.log 2>&1
for r in 1 2; do
  for v in 3 6; do
    SP_RING_SLOTS=$v timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 slots=$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done >> gpurun_out/ring.log 2>&1
