#!/bin/bash
mkdir -p gpurun_out
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag > gpurun_out/hp.log 2>&1
for rep in 1 2; do
for hp in 0 1; do
  echo "== SP_HUGEPAGES=$hp" >> gpurun_out/hp.log
  SP_HUGEPAGES=$hp TH=16 HH=5018 TS=1,1,1,16 timeout 120 python scripts/bench_cc_tokens.py >> gpurun_out/hp.log 2>&1
  grep AnonHugePages /proc/meminfo >> gpurun_out/hp.log
done
done
for hp in 0 1 0 1; do
  echo "== bench SP_HUGEPAGES=$hp" >> gpurun_out/hp.log
  SP_HUGEPAGES=$hp timeout 300 python bench.py --steps 100 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))" >> gpurun_out/hp.log 2>&1
done
echo done
