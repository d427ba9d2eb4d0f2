#!/bin/bash
# A/B of one env switch on the default bench, alternating on the same box:
#   bash scripts/gpu_ab.sh VAR "A B" "bench args" [skip-tests]
mkdir -p gpurun_out
VAR=${1:-SP_PREREDUCE}; VALS=${2:-"0 1"}; ARGS=${3:-}
if [ -z "$4" ]; then
  timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
fi
for r in 1 2 3; do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --no-cpu-baseline $ARGS 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms', round(d['ms_per_step'],4), 'rates', d['config'].get('rates'))"
  done
done > gpurun_out/ab.log 2>&1
