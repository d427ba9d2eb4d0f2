#!/bin/bash
# AMX CC kernel with the layer's prepacked W2 (new) vs repack per round (old): phase medians
# (bench_amx, alternating builds), the AMX parity tests, then cfg3 layer plan (calibrated) old vs new
mkdir -p gpurun_out
: > gpurun_out/amx_prepack.txt
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2 3; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    echo "== $v" | tee -a gpurun_out/amx_prepack.txt
    SP_AMX_PROF=1 TS=64,128,256 REPS=8 timeout 600 python scripts/bench_amx.py 2>&1 | grep -v thread | python scripts/amx_phases.py | tee -a gpurun_out/amx_prepack.txt
  done
done
cp _ab/new.so paper_2411_15715_b200/_native/libsliced.so
timeout 600 python -m pytest tests/test_abi.py tests/test_tc_shapes.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for r in 1 2; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    timeout 900 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 8 --token-plan layer 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 $v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ng0', d['config']['layer_plan_n_g_layer0'])" | tee -a gpurun_out/amx_prepack.txt
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
