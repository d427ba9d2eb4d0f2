#!/bin/bash
# one cfg3 layer-plan run with its prefill traced (first 4 layers, device and host I/O), anatomy of both
mkdir -p gpurun_out/cfg3tr
timeout 900 python bench.py --config cfg3 --layers 32 --distinct-layers 4 --decode-steps 8 --token-plan layer \
  --trace-out gpurun_out/cfg3tr/trace.json > gpurun_out/cfg3tr/bench.log 2>&1
grep '^{' gpurun_out/cfg3tr/bench.log | tail -1 | cut -c1-200
grep "host-I/O prefill layer wall" gpurun_out/cfg3tr/bench.log
echo "== device I/O"; python scripts/step_anatomy.py gpurun_out/cfg3tr/trace.json
echo "== host I/O"; python scripts/step_anatomy.py gpurun_out/cfg3tr/trace_hostio.json
