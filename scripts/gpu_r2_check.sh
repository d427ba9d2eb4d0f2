#!/bin/bash
# Round-2 check on one box: GPU tests (parity lines kept), default bench, the
# reference arm, and the 2-rank plumbing on one GPU (gloo).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider -s > gpurun_out/r2_gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_gputest.log
grep -E "PARITY|passed|failed" gpurun_out/r2_gputest.log | tail -60
timeout 600 python bench.py > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_n1.json 2> gpurun_out/r2_ref_n1.err; echo "ref rc=$?"
SP_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r2_bench_n2_onegpu.json 2> gpurun_out/r2_bench_n2_onegpu.err; echo "n2 rc=$?"
SP_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_n2.json 2> gpurun_out/r2_ref_n2.err; echo "ref n2 rc=$?"
tail -c 600 gpurun_out/r2_bench_n1.err
