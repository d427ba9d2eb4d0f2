#!/bin/bash
# prefill chain: CUDA-event span and in-kernel device span (first CTA start of
# the gather / GEMMs -> last CTA end of the down GEMM) of one resident expert
mkdir -p gpurun_out/tcspan
F=gpurun_out/tcspan/out.txt
timeout 900 python -m pytest tests/test_tc_shapes.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/tcspan/gputest.log 2>&1; echo "gpu parity rc=$?" > $F
tail -1 gpurun_out/tcspan/gputest.log >> $F
for r in 1 2; do SP_PREFILL_T="16 32 64 128 256 512" timeout 300 python scripts/bench_prefill.py >> $F 2>&1; done
echo done
