#!/bin/bash
# cfg3 with prompt profiles whose host CC samples are taken at 32 vs 128 tokens (new AMX kernel)
mkdir -p gpurun_out/cfg3b _ab/p32 _ab/p128
timeout 900 python -m paper_2411_15715_b200.b200_profile --phase prompt --out _ab/p32 > gpurun_out/cfg3b/refit32.log 2>&1
timeout 900 python -m paper_2411_15715_b200.b200_profile --phase prompt --cpu-tokens 128 --tag _t128 --out _ab/p128 > gpurun_out/cfg3b/refit128.log 2>&1
cp _ab/p32/b200_prompt.json _ab/p32/b200_samples_prompt.csv _ab/p128/b200_prompt_t128.json _ab/p128/b200_samples_prompt_t128.csv gpurun_out/cfg3b/ 2>/dev/null
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/cfg3b/$name.log 2>&1; grep '^{' gpurun_out/cfg3b/$name.log | tail -1 > gpurun_out/cfg3b/$name.json; python -c "
import json; d=json.load(open('gpurun_out/cfg3b/$name.json')); c=d['config']; print('$name', 'value %.1f'%d['value'], 'e2e %.1f'%d['e2e']['value'], c.get('layer_plan_n_g_layer0'), c.get('n_g_by_expert_tokens'))" 2>&1 | cut -c1-300; }
A="--config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32"
for r in 1 2; do
run p32_solve $A --prompt-profile _ab/p32/b200_prompt.json
run p32_layer $A --prompt-profile _ab/p32/b200_prompt.json --token-plan layer
run p128_solve $A --prompt-profile _ab/p128/b200_prompt_t128.json
run p128_layer $A --prompt-profile _ab/p128/b200_prompt_t128.json --token-plan layer
done
