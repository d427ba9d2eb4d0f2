#!/bin/bash
mkdir -p gpurun_out
echo "== 16 threads" >> gpurun_out/amx.log
TH=16 HH=4742 TS=1,4,16,32,64,128 timeout 300 python scripts/bench_cc_tokens.py >> gpurun_out/amx.log 2>&1
echo "== 1 thread, cycle split" >> gpurun_out/amx.log
SP_AMX_PROF=1 TH=1 HH=512 TS=16,64 timeout 300 python scripts/bench_cc_tokens.py 2>&1 | tail -8 >> gpurun_out/amx.log
grep MHz /proc/cpuinfo | head -2 >> gpurun_out/amx.log
echo done
