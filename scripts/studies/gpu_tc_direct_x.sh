#!/bin/bash
# up GEMM reading bf16 x through its own TMA map (no gather kernel) for calls whose
# tokens are x's rows in order: GPU suite, then the one-expert chain with the
# direct map on / off (SP_TC_DIRECT_X), alternating
mkdir -p gpurun_out/dx
F=gpurun_out/dx/out.txt
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/dx/gputest.log 2>&1; echo "gpu suite rc=$?" > $F
tail -1 gpurun_out/dx/gputest.log >> $F
for r in 1 2; do
  for v in 1 0; do
    echo "== round $r SP_TC_DIRECT_X=$v" >> $F
    SP_TC_DIRECT_X=$v SP_PREFILL_T="16 32 64 128 256 512" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
  done
done
echo done
