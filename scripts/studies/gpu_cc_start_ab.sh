#!/bin/bash
# CC block start (x read-back ahead of the ring copies, CC submitted before the
# host-side x staging, parallel row gather): old vs new build, cfg3 layer plan
# (fixed plan) and cfg2 decode, alternating; [cc] phase lines from the new build
# (the phase lines: SP_CC_PROF=1 python bench.py --config cfg3 ... --calibrate 0 2>&1 | grep "^\[cc\]")
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2 3; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    timeout 900 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 8 --token-plan layer 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 $v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ng0', d['config']['layer_plan_n_g_layer0'], 'k_cpu', round(d['prompt_calibration']['k_cpu'],3))"
    true
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
