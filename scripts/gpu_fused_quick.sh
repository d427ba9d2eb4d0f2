#!/bin/bash
# expert_tc_kernel quick loop: its parity tests, then the one-expert prefill
# microbench against the four-kernel chain (SP_TC_FUSED=0), alternating.
mkdir -p gpurun_out/fused
F=gpurun_out/fused
timeout 300 python -m pytest tests/test_expert_tc.py -q -s -x -p no:cacheprovider > $F/test_expert_tc.log 2>&1; echo "fused tests rc=$?" >> $F/test_expert_tc.log
grep -E "PARITY|passed|failed|rc=" $F/test_expert_tc.log
for i in 1 2; do
  SP_TC_FUSED=0 SP_PREFILL_T="${PT:-16 64 128}" timeout 120 python scripts/bench_prefill.py > $F/prefill_chain_$i.txt 2>&1
  SP_TC_FUSED=1 SP_PREFILL_T="${PT:-16 64 128}" timeout 120 python scripts/bench_prefill.py > $F/prefill_fused_$i.txt 2>&1
done
tail -n 3 $F/prefill_*.txt
SP_PREFILL_T="16 128" timeout 120 python scripts/fused_stamps.py > $F/stamps.txt 2>&1; cat $F/stamps.txt
