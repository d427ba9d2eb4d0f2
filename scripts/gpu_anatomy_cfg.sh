#!/bin/bash
# step anatomy (device-I/O and e2e regions fully traced) of one config: $1 = bench args
mkdir -p gpurun_out/anat
A=gpurun_out/anat
SP_TRACE_KEEP_CALLS=1000 SP_BENCH_TRACE_E2E=$A/trace_e2e.json timeout 600 python bench.py --no-cpu-baseline $1 --trace-out $A/trace_dev.json > $A/bench.json 2> $A/bench.err; echo "bench rc=$?"
echo "== device I/O (full-trace region)"; python scripts/step_anatomy.py $A/trace_dev.json
echo "== e2e (host I/O)"; python scripts/step_anatomy.py $A/trace_e2e.json
python -c "import json;d=json.loads(open('$A/bench.json').read().splitlines()[-1]);print('value',d['value'],'e2e',d['e2e']['value'],'ms',d['ms_per_step'],'full',d['model_vs_measured']['step_full_trace_s'])"
