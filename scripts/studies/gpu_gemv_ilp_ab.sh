#!/bin/bash
# GEMV phase 1 with the accumulator chains interleaved (e outermost, ilp) vs the
# committed packed-FFMA2 kernel (ffma2), alternating; GPU parity with ilp first.
mkdir -p gpurun_out/ilp
F=gpurun_out/ilp/ab.txt
L=paper_2411_15715_b200/_native/libsliced.so
: > $F
cp _ab/ilp.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_config_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/ilp/gputest.log 2>&1; echo "gpu parity rc=$?" >> $F
tail -1 gpurun_out/ilp/gputest.log >> $F
for r in 1 2 3; do
  for v in ffma2 ilp; do
    cp _ab/$v.so $L
    echo "== round $r $v" >> $F
    timeout 300 python scripts/bench_gemv.py --T 1 2 4 --hidden 14336 --reps 20 >> $F 2>&1
    timeout 300 python scripts/bench_gemv.py --T 1 2 --model 6144 --hidden 8192 --reps 20 >> $F 2>&1
  done
done
cp _ab/ilp.so $L
echo done
