#!/bin/bash
# CTA-pair up GEMM from 64-token tiles vs from 256 (default), with the direct x map; 4 alternating rounds
mkdir -p gpurun_out/tcp2
F=gpurun_out/tcp2/ab.txt
: > $F
for round in 1 2 3 4; do
  for nt in 256 64; do
    echo "== round $round SP_TC_PAIR_MIN_NT=$nt" >> $F
    SP_TC_PAIR_MIN_NT=$nt SP_PREFILL_T="64 128 256" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
  done
done
echo done
