#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
echo "== AMX 16 threads" >> gpurun_out/amx.log
TH=16 HH=5018 TS=1,4,8,16,32,128 timeout 300 python scripts/bench_cc_tokens.py >> gpurun_out/amx.log 2>&1
done
echo "== AVX 16 threads" >> gpurun_out/amx.log
SP_AMX=0 TH=16 HH=5018 TS=4,8,16 timeout 300 python scripts/bench_cc_tokens.py >> gpurun_out/amx.log 2>&1
echo done
