#!/bin/bash
# cfg3 host-I/O layer anatomy with the x staging deferred behind the first ring copies, then
# ring depth for long streams 6 vs 8 (cfg3 layer plan, calibrated), alternating
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_tc_shapes.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
bash scripts/studies/gpu_cfg3_trace.sh 2>&1 | grep -E "wall|== host|copy_start|cc_start|period" | tail -5
for r in 1 2; do
  for v in 6 8; do
    SP_RING_SLOTS_LONG=$v timeout 900 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 8 --token-plan layer 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ring $v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done
