#!/bin/bash
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
for st in 16 32 64; do for ns in 4 8; do
  SP_BULK_STAGE_KB=$st SP_BULK_STAGES=$ns timeout 300 python scripts/bench_gemv.py --T 1 --hidden 7168 14336 --reps 8 2>&1 | sed "s/^/st=$st ns=$ns /"
done; done
timeout 300 python scripts/bench_gemv.py --T 1 2 4 8 --hidden 7168 --reps 8
SP_BULK=0 timeout 300 python scripts/bench_gemv.py --T 1 --hidden 7168 --reps 8
