# per-kernel durations of the tensor-core block path, data-parallel vs stream-K up GEMM
mkdir -p gpurun_out
for sk in 0 1; do
SP_TC_STREAMK=$sk timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
  --log-file gpurun_out/sk_launch_$sk.csv python scripts/bench_prefill.py 14336 > gpurun_out/sk_ncu_$sk.log 2>&1
done
