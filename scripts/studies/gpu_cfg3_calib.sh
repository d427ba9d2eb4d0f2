#!/bin/bash
# cfg3 prefill with and without the per-box prompt-profile recalibration, both token plans, alternating on one box
mkdir -p gpurun_out/cfg3cal
for r in 1 2; do
  for plan in solve_ng layer; do
    for cal in 0 1; do
      timeout 900 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32 --token-plan $plan --calibrate $cal \
        > gpurun_out/cfg3cal/${plan}_cal${cal}_$r.log 2>&1
      grep '^{' gpurun_out/cfg3cal/${plan}_cal${cal}_$r.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d.get('prompt_calibration') or {}
print('$plan cal=$cal', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'k_cpu', c.get('k_cpu') and round(c['k_cpu'],3), 'k_link', c.get('k_link') and round(c['k_link'],3), 'ng0', c.get('n_g_layer0_before'), '->', c.get('n_g_layer0_after'))"
    done
  done
done
