#!/bin/bash
# ncu: launch list + full capture of the up (gated) and down rowdot kernels at H=7168, T=1
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/gemv_launches.csv python scripts/bench_gemv.py --T 1 --hidden 7168 --reps 3 > gpurun_out/ncu_gemv_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowdot -s 4 -c 2 \
  -o gpurun_out/gemv_prof -f python scripts/bench_gemv.py --T 1 --hidden 7168 --reps 3 > gpurun_out/ncu_gemv_full.log 2>&1
echo done
