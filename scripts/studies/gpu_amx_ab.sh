#!/bin/bash
# AMX CC kernel A/B (_ab/old.so vs _ab/new.so, alternating, one box): phase medians per token count
# (scripts/amx_phases.py), then the AMX parity tests with the new build
mkdir -p gpurun_out
: > gpurun_out/amx_ab.txt
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in 1 2 3 4 5 6; do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    echo "== $v" | tee -a gpurun_out/amx_ab.txt
    SP_AMX_PROF=1 TS=16,64,128,256 REPS=12 timeout 600 python scripts/bench_amx.py 2>&1 | grep -v thread | python scripts/amx_phases.py | tee -a gpurun_out/amx_ab.txt
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
timeout 600 python -m pytest tests/test_abi.py -q -m gpu -k amx -p no:cacheprovider 2>&1 | tail -3
