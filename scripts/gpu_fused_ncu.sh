#!/bin/bash
# ncu launch lists (per-kernel device time, DRAM bytes) of the one-expert prefill microbench, chain vs fused
mkdir -p gpurun_out/fused
for f in 0 1; do
SP_TC_FUSED=$f SP_PREFILL_T="16 128" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fused/ncu_launch_f$f.csv python scripts/bench_prefill.py > /dev/null 2>&1
python scripts/ncu_launch_table.py gpurun_out/fused/ncu_launch_f$f.csv | grep -v "at::" | head -12
done
