#!/bin/bash
# cfg5 batched decode, two builds (_ab/old.so, _ab/new.so), calibrated as the evidence runs, alternating
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    for cfg in "--moe 8x22b --batch 16" "--moe phimoe --batch 32" "--moe phimoe --batch 8"; do
      timeout 600 python bench.py --config cfg5 $cfg --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $cfg', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'step', round(d['link']['step_roofline_frac'],2))"
    done
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
