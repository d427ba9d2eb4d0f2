#!/bin/bash
# Prefill chain (one resident Mixtral expert): CTA targets of the up / down GEMMs
# (SP_TC_UP_CTAS / SP_TC_DN_CTAS; default = one per SM), alternating, two rounds.
mkdir -p gpurun_out/tct
F=gpurun_out/tct/ab.txt
: > $F
for round in 1 2; do
  for cfg in "0 0" "296 0" "0 296" "296 296" "0 74"; do
    set -- $cfg
    echo "== round $round UP_CTAS=$1 DN_CTAS=$2" >> $F
    SP_TC_UP_CTAS=$1 SP_TC_DN_CTAS=$2 SP_PREFILL_T="16 64 128" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
  done
done
echo done
