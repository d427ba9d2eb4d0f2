#!/bin/bash
# tcgen05 prefill chain A/B (SP_TC_PDL on/off, alternating, read-flush microbench),
# GPU parity of every tc path, then an ncu launch list at T = 16 / 128.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_config_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/tc_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/tc_parity.log
for r in 1 0 1 0; do echo "SP_TC_PDL=$r"; SP_TC_PDL=$r timeout 300 python scripts/bench_prefill.py 14336; done > gpurun_out/tc_ab.txt 2>&1
cat gpurun_out/tc_ab.txt
SP_PREFILL_T="16 128" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm|gather|swiglu|final|reduce" --csv --log-file gpurun_out/tc_launches.csv python scripts/bench_prefill.py 14336 > /dev/null 2>&1; echo "ncu rc=$?"
