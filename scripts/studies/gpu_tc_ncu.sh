#!/bin/bash
# tcgen05 expert microbench (read flush) + ncu --set full of the up / down GEMMs at T=16 and 128
mkdir -p gpurun_out
timeout 300 python scripts/bench_prefill.py 14336 > gpurun_out/tc_micro.txt 2>&1; cat gpurun_out/tc_micro.txt
SP_PREFILL_T="16" timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -s 4 -c 2 -o gpurun_out/tc_T16 python scripts/bench_prefill.py 14336 > gpurun_out/tc_ncu16.log 2>&1; echo "ncu16 rc=$?"
SP_PREFILL_T="128" timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -s 4 -c 2 -o gpurun_out/tc_T128 python scripts/bench_prefill.py 14336 > gpurun_out/tc_ncu128.log 2>&1; echo "ncu128 rc=$?"
