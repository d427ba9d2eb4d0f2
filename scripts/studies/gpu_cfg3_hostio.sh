#!/bin/bash
# cfg3 host-I/O: parity of the host-I/O paths, the host-I/O layer anatomy, then cfg3 (layer plan, calibrated) twice
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_tc_shapes.py tests/test_config_parity.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
bash scripts/studies/gpu_cfg3_trace.sh 2>&1 | grep -E "wall|==|copy_start|cc_start|cc_end|copy_end|merge_end|return_end|period"
for r in 1 2; do
  timeout 900 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 8 --token-plan layer 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
