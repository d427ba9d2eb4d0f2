#!/bin/bash
# CTA-pair up GEMM also at 16-token tiles (SP_TC_PAIR_MIN_NT=16) vs 32 (default): tc shape parity with 16 forced, then alternating
mkdir -p gpurun_out/tcp4
F=gpurun_out/tcp4/ab.txt
SP_TC_PAIR_MIN_NT=16 timeout 900 python -m pytest tests/test_tc_shapes.py tests/test_config_parity.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/tcp4/gputest.log 2>&1; echo "parity (pair from 16) rc=$?" > $F
tail -1 gpurun_out/tcp4/gputest.log >> $F
for round in 1 2 3; do
  for nt in 16 32; do
    echo "== round $round SP_TC_PAIR_MIN_NT=$nt" >> $F
    SP_TC_PAIR_MIN_NT=$nt SP_PREFILL_T="16" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
  done
done
echo done
