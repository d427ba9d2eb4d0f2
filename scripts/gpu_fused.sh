#!/bin/bash
# expert_tc_kernel: parity (new tests + the whole GPU suite) and the one-expert
# prefill microbench against the four-kernel chain (SP_TC_FUSED=0), alternating.
mkdir -p gpurun_out/fused
F=gpurun_out/fused
timeout 600 python -m pytest tests/test_expert_tc.py -q -s -p no:cacheprovider > $F/test_expert_tc.log 2>&1; echo "fused tests rc=$?" >> $F/test_expert_tc.log
tail -3 $F/test_expert_tc.log
grep PARITY $F/test_expert_tc.log
for i in 1 2; do
  SP_TC_FUSED=0 SP_PREFILL_T="16 64 128" timeout 300 python scripts/bench_prefill.py > $F/prefill_chain_$i.txt 2>&1
  SP_TC_FUSED=1 SP_PREFILL_T="16 64 128" timeout 300 python scripts/bench_prefill.py > $F/prefill_fused_$i.txt 2>&1
done
tail -n 3 $F/prefill_*.txt
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $F/gputest.log 2>&1; echo "tests rc=$?" >> $F/gputest.log
tail -5 $F/gputest.log
