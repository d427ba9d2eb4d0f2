#!/bin/bash
# ncu --set full of the GEMV at 4 tokens (one Mixtral expert, 4096/14336) and 1 token
mkdir -p gpurun_out/gemv_ncu
for T in 4 1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_block_kernel -s 3 -c 1 \
    -o gpurun_out/gemv_ncu/gemv_t$T python scripts/bench_gemv.py --T $T --hidden 14336 --reps 3 > gpurun_out/gemv_ncu/t$T.log 2>&1
done
echo done
