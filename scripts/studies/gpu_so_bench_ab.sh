#!/bin/bash
# A/B of two builds (_ab/old.so vs _ab/new.so) on the default bench line, fixed rates, alternating on one box
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2 3 4 5; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    timeout 300 python bench.py --no-cpu-baseline --steps 100 --calibrate 0 ${ARGS:-} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); rf=d.get('roofline') or {}
print('$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'gg_frac', round(rf['frac'],3), 'dev', round(rf['frac_device_span'],3), 'launch_us', round(rf['mean_launch_us'],2), 'span_us', round(rf['device_span_us'],2))"
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
