#!/bin/bash
# batched decode: routing on the host pool + pooled output copy-out (new) vs old, cfg5 PhiMoE b32 / 8x22B b16, alternating
timeout 600 python -m pytest tests/test_abi.py tests/test_config_parity.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2 3; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    for cfg in "--moe phimoe --batch 32" "--moe 8x22b --batch 16"; do
      timeout 600 python bench.py --config cfg5 $cfg --steps 40 --no-cpu-baseline --calibrate 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $cfg', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
    done
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
