#!/bin/bash
# host CC kernel variants: software prefetch distance, THP host region, pinned threads
mkdir -p gpurun_out
(nproc; lscpu; numactl -H 2>/dev/null; cat /sys/kernel/mm/transparent_hugepage/enabled; free -g) > gpurun_out/host_info.txt 2>&1
for v in "" "SP_CC_PREFETCH=4096" "SP_CC_PREFETCH=8192" "SP_CC_PREFETCH=16384" "SP_HUGEPAGES=1" "SP_HUGEPAGES=1 SP_CC_PREFETCH=8192" "SP_PIN_THREADS=1" "SP_HUGEPAGES=1 SP_CC_PREFETCH=8192 SP_PIN_THREADS=1"; do
  echo "== $v" >> gpurun_out/cc_variants.log
  env $v timeout 120 python scripts/bench_cc.py --quick >> gpurun_out/cc_variants.log 2>&1
done
for v in "" "SP_HUGEPAGES=1 SP_CC_PREFETCH=8192"; do
  echo "== $v" >> gpurun_out/bench_variants.log
  env $v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --trace-out gpurun_out/timeline_v.json >> gpurun_out/bench_variants.log 2>&1
  python scripts/timeline_summary.py gpurun_out/timeline_v.json >> gpurun_out/bench_variants.log 2>&1
done
echo done
