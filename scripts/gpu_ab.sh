#!/bin/bash
# A/B of one env switch on the default bench, alternating on the same box:
#   bash scripts/gpu_ab.sh VAR "A B" "bench args" [rounds]
mkdir -p gpurun_out
VAR=${1:-SP_PREREDUCE}; VALS=${2:-"0 1"}; ARGS=${3:-}; ROUNDS=${4:-3}
for r in $(seq $ROUNDS); do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --no-cpu-baseline $ARGS 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); rf=d.get('roofline') or {}
print('$VAR=$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms', round(d['ms_per_step'],4),
      'gg_frac', rf.get('frac') and round(rf['frac'],3), 'dev', rf.get('frac_device_span') and round(rf['frac_device_span'],3),
      'rates', (d.get('split') or {}).get('rates'))"
  done
done 2>&1 | tee gpurun_out/ab_$VAR.log
