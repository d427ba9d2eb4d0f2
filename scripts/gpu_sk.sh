#!/bin/bash
mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "prefill" > gpurun_out/sk_tests.log 2>&1
echo "prefill tests rc=$?" >> gpurun_out/sk_tests.log
grep -q "rc=0" gpurun_out/sk_tests.log || exit 1
timeout 200 python -m pytest tests -x -q -m gpu >> gpurun_out/sk_tests.log 2>&1
echo "all tests rc=$?" >> gpurun_out/sk_tests.log
for sk in 0 1 0 1; do
  echo "== SP_TC_STREAMK=$sk" >> gpurun_out/sk_bench.log
  SP_TC_STREAMK=$sk timeout 150 python scripts/bench_prefill.py 14336 >> gpurun_out/sk_bench.log 2>&1
  SP_TC_STREAMK=$sk timeout 150 python scripts/bench_prefill.py 7168 >> gpurun_out/sk_bench.log 2>&1
done
echo done
