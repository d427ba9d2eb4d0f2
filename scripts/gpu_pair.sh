#!/bin/bash
# CTA-pair up GEMM: parity first (short timeouts), then A/B prefill timings
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" > gpurun_out/pair_tests.log 2>&1
echo "rc=$?" >> gpurun_out/pair_tests.log
if grep -q "rc=0" gpurun_out/pair_tests.log; then
  for H in 14336 7168; do
    for v in 0 1; do echo "SP_TC_PAIR=$v"; SP_TC_PAIR=$v timeout 120 python scripts/bench_prefill.py $H 2>&1 | tail -5; done
  done > gpurun_out/pair_bench.log 2>&1
  timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
fi
