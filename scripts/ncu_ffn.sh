#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,smsp__cycles_active.avg --clock-control none --csv \
  --log-file gpurun_out/ffn_launches.csv python scripts/bench_gemv.py --T 1 --hidden 1024 7168 14336 --reps 3 > gpurun_out/ncu_ffn_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_block -s 3 -c 1 \
  -o gpurun_out/ffn7168 -f python scripts/bench_gemv.py --T 1 --hidden 7168 --reps 3 > gpurun_out/ncu_ffn_full.log 2>&1
echo done
