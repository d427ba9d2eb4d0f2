#!/bin/bash
# CTA-pair up GEMM at 32-128-token tiles (SP_TC_PAIR_MIN_NT) vs single-CTA tiles:
# parity of the tensor-core shapes with the pair path forced, then the
# one-expert prefill chain alternating, two rounds.
mkdir -p gpurun_out/tcp
F=gpurun_out/tcp/ab.txt
: > $F
SP_TC_PAIR_MIN_NT=32 timeout 600 python -m pytest tests/test_tc_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/tcp/parity.log 2>&1; echo "parity rc=$?" >> $F
tail -2 gpurun_out/tcp/parity.log >> $F
for round in 1 2; do
  for nt in 256 32; do
    echo "== round $round SP_TC_PAIR_MIN_NT=$nt" >> $F
    SP_TC_PAIR_MIN_NT=$nt SP_PREFILL_T="16 32 64 128" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
  done
done
echo done
