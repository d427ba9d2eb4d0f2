#!/bin/bash
# launch list of a short bench run + full captures of the grouped GG ffn_block launch and the prefill tcgen05 GEMMs
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_list.log 2>&1
# the grouped GG launch of a decode step (2 experts x 7168 rows), third forward
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_block --launch-skip 2 -c 1 \
  -o gpurun_out/ffn_gg_bench -f python scripts/gg_group_one.py > gpurun_out/ncu_bench_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 2 \
  -o gpurun_out/gemm_tc -f python scripts/bench_prefill.py 7168 > gpurun_out/ncu_gemm_full.log 2>&1
echo done
