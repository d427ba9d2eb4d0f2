#!/bin/bash
# pair up GEMM from 32-token tiles as the default: GPU suite, then the one-expert chain (new default vs 256), alternating
mkdir -p gpurun_out/tcp3
F=gpurun_out/tcp3/ab.txt
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/tcp3/gputest.log 2>&1; echo "gpu suite rc=$?" > $F
tail -1 gpurun_out/tcp3/gputest.log >> $F
for round in 1 2 3; do
  for nt in 32 256; do
    echo "== round $round SP_TC_PAIR_MIN_NT=$nt" >> $F
    SP_TC_PAIR_MIN_NT=$nt SP_PREFILL_T="16 32 64 128" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
  done
done
echo done
