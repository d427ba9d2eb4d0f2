#!/bin/bash
# tcgen05 prefill chain with and without its MMAs (SP_TC_DBG_NOMMA=1: operands streamed, no MMA; output garbage), alternating
for r in 1 2; do
  for v in 0 1; do
    echo "== SP_TC_DBG_NOMMA=$v"; SP_TC_DBG_NOMMA=$v SP_PREFILL_T="16 64 128" timeout 120 python scripts/bench_prefill.py 2>&1 | tail -3
  done
done
