#!/bin/bash
# (SP_TC_DN_SUB was a local probe switch, not committed)
# down GEMM: 128-column sub-tiles per CTA (SP_TC_DN_SUB = 1 / 2 (default) / 4), parity with 1 and 4, then alternating
mkdir -p gpurun_out/dsub
F=gpurun_out/dsub/ab.txt
: > $F
for v in 1 4; do
  SP_TC_DN_SUB=$v timeout 400 python -m pytest tests/test_tc_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/dsub/p$v.log 2>&1; echo "tc shapes SP_TC_DN_SUB=$v rc=$?" >> $F
done
for round in 1 2 3; do
  for v in 2 1 4; do
    echo "== round $round SP_TC_DN_SUB=$v" >> $F
    SP_TC_DN_SUB=$v SP_PREFILL_T="16 64 128" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
  done
done
echo done
