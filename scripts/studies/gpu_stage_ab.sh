#!/bin/bash
# host-I/O x staging order (small x before the ring copies) old vs new: batched decode e2e, cfg2 decode, alternating
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2 3; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    for cfg in "--config cfg5 --moe phimoe --batch 32 --steps 40" "--config cfg5 --moe 8x22b --batch 16 --steps 40" "--steps 100"; do
      timeout 600 python bench.py $cfg --no-cpu-baseline --calibrate 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $cfg', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
    done
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
