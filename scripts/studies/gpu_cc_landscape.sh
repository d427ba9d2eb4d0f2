#!/bin/bash
# decode step vs a forced r_CC around the planner's split (r_GG fixed by the budget), two alternating passes
mkdir -p gpurun_out
for r in 1 2; do
  for cc in 0.30 0.34 0.376 0.41 0.44; do
    timeout 300 python bench.py --no-cpu-baseline --force-cc $cc 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cc=$cc', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done > gpurun_out/cc_landscape.log 2>&1
