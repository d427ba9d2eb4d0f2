#!/bin/bash
# cfg3 prefill with the new AMX CC kernel (prompt profile refit on this box) vs
# the round-1 kernel with the committed prompt profile, same box
mkdir -p gpurun_out/cfg3 _ab/prof_new
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
timeout 900 python -m paper_2411_15715_b200.b200_profile --phase prompt --out _ab/prof_new > gpurun_out/cfg3/refit_prompt.log 2>&1
cp _ab/prof_new/b200_prompt.json _ab/prof_new/b200_samples_prompt.csv gpurun_out/cfg3/ 2>/dev/null
tail -8 gpurun_out/cfg3/refit_prompt.log
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/cfg3/$name.log 2>&1; grep '^{' gpurun_out/cfg3/$name.log | tail -1 > gpurun_out/cfg3/$name.json; python -c "
import json; d=json.load(open('gpurun_out/cfg3/$name.json')); print('$name', 'value %.1f'%d['value'], 'e2e %.1f'%d['e2e']['value'], {k: d[k] for k in ('prefill', 'decode') if k in d})" 2>&1 | cut -c1-400; }
A="--config cfg3 --layers 32 --distinct-layers 4 --decode-steps 32"
run new_solve_ng $A --prompt-profile _ab/prof_new/b200_prompt.json
run new_layer $A --prompt-profile _ab/prof_new/b200_prompt.json --token-plan layer
cp _ab/old.so paper_2411_15715_b200/_native/libsliced.so
run old_solve_ng $A
run old_layer $A --token-plan layer
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
