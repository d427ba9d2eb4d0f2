#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for pf in 0 1024 2048 4096 8192; do
  echo "== SP_CC_PREFETCH=$pf" >> gpurun_out/cc_pf.log
  SP_CC_PREFETCH=$pf TH=16 HH=5018 TS=1,1,1 timeout 120 python scripts/bench_cc_tokens.py >> gpurun_out/cc_pf.log 2>&1
done
done
echo "== 15 threads" >> gpurun_out/cc_pf.log
TH=15 HH=5018 TS=1,1,1 timeout 120 python scripts/bench_cc_tokens.py >> gpurun_out/cc_pf.log 2>&1
echo done
