#!/bin/bash
# (the kernel and the SP_TC_DOWN_PAIR switch exist only at commit 475dfe0)
# down GEMM on CTA pairs (SP_TC_DOWN_PAIR=1): parity first (bounded), then the one-expert chain, alternating
mkdir -p gpurun_out/dp
F=gpurun_out/dp/ab.txt
SP_TC_DOWN_PAIR=1 timeout 400 python -m pytest tests/test_tc_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/dp/tcshapes.log 2>&1; echo "tc shapes (down pair) rc=$?" > $F
tail -3 gpurun_out/dp/tcshapes.log >> $F
if grep -q "passed" gpurun_out/dp/tcshapes.log && ! grep -q "failed" gpurun_out/dp/tcshapes.log; then
  SP_TC_DOWN_PAIR=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_config_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/dp/parity.log 2>&1; echo "parity (down pair) rc=$?" >> $F
  tail -1 gpurun_out/dp/parity.log >> $F
  for round in 1 2 3; do
    for v in 1 0; do
      echo "== round $round SP_TC_DOWN_PAIR=$v" >> $F
      SP_TC_DOWN_PAIR=$v SP_PREFILL_T="16 64 128 256 512" timeout 300 python scripts/bench_prefill.py >> $F 2>&1
    done
  done
fi
echo done
