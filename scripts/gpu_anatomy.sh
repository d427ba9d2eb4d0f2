#!/bin/bash
# default decode bench with the device-I/O and the e2e regions fully traced; step anatomy of both
mkdir -p gpurun_out
SP_TRACE_KEEP_CALLS=1000 SP_BENCH_TRACE_E2E=gpurun_out/trace_e2e.json timeout 600 python bench.py --no-cpu-baseline --trace-out gpurun_out/trace_dev.json > gpurun_out/anat_bench.json 2> gpurun_out/anat_bench.err; echo "bench rc=$?"
echo "== device I/O (full-trace region)"; python scripts/step_anatomy.py gpurun_out/trace_dev.json
echo "== e2e (host I/O)"; python scripts/step_anatomy.py gpurun_out/trace_e2e.json
python -c "import json;d=json.loads(open('gpurun_out/anat_bench.json').read().splitlines()[-1]);print('value',d['value'],'e2e',d['e2e']['value'],'ms',d['ms_per_step'],'full',d['model_vs_measured']['step_full_trace_s'])"
