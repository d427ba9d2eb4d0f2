#!/bin/bash
# L2 prefetch depth sweep of the tcgen05 GEMMs (read-flush microbench, one expert)
# (record of the sweep in profiles/r2/tc_l2_prefetch_sweep.txt: the SP_TC_PF knob was removed after it --
# every prefetch depth was slower, so this no longer changes anything)
mkdir -p gpurun_out
for rep in 1 2; do for pf in 0 4 8 16 32; do echo "SP_TC_PF=$pf"; SP_PREFILL_T="16 64 128 512" SP_TC_PF=$pf timeout 300 python scripts/bench_prefill.py 14336; done; done > gpurun_out/tc_pf.txt 2>&1
cat gpurun_out/tc_pf.txt
