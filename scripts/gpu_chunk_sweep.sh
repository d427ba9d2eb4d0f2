#!/bin/bash
mkdir -p gpurun_out
for mb in 8 16 32 8 16; do
  echo "== SP_CHUNK_MB=$mb" >> gpurun_out/chunk_sweep.log
  SP_CHUNK_MB=$mb timeout 300 python bench.py --config cfg5 --moe 8x22b --batch 32 --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['link']['cg_copy_GBps_while_busy'])" >> gpurun_out/chunk_sweep.log 2>&1
  SP_CHUNK_MB=$mb timeout 300 python bench.py --config cfg5 --moe phimoe --batch 32 --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['link']['cg_copy_GBps_while_busy'])" >> gpurun_out/chunk_sweep.log 2>&1
done
echo done
