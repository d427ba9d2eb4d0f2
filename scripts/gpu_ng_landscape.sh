#!/bin/bash
# cfg3 (8 layers) prefill vs a forced token split, all on one box, next to solve_ng's splits
mkdir -p gpurun_out
for f in solver-rs solver-lit 0.6 0.7 0.8 0.85 0.95 1.0 solver-rs; do
  case $f in solver-rs) a="--transfer-model rate_scaled";; solver-lit) a="--transfer-model literal";; *) a="--ng-frac $f";; esac
  echo "== $f" >> gpurun_out/ng_landscape.log
  timeout 600 python bench.py --config cfg3 --layers 8 --distinct-layers 2 --decode-steps 2 --steps 3 --warmup 1 $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']/8,2), 'ms/layer', d['config']['n_g_by_expert_tokens'].get('128'))" >> gpurun_out/ng_landscape.log 2>&1
done
echo done
