#!/bin/bash
# cfg3 (8 layers): solve_ng (rate_scaled), the layer-level plan, forced splits -- one box
mkdir -p gpurun_out
for f in solver layer 1.0 layer solver; do
  case $f in solver) a="";; layer) a="--token-plan layer";; *) a="--ng-frac $f";; esac
  echo "== $f" >> gpurun_out/ng_landscape.log
  timeout 600 python bench.py --config cfg3 --layers 8 --distinct-layers 2 --decode-steps 2 --steps 3 --warmup 1 $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']/8,2), 'ms/layer', d['config']['n_g_by_expert_tokens'].get('128'), d['config'].get('layer_plan_n_g_layer0'), round(d['e2e']['value'],1))" >> gpurun_out/ng_landscape.log 2>&1
done
echo done
