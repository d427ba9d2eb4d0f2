#!/bin/bash
# A/B of two builds of libsliced.so (_ab/old.so vs _ab/new.so) on one box,
# alternating: bash scripts/studies/gpu_so_ab.sh "<command>" [rounds]
CMD=${1:-"TS=16,64,128,256 python scripts/bench_amx.py"}; ROUNDS=${2:-3}
cp paper_2411_15715_b200/_native/libsliced.so _ab/keep.so
for r in $(seq $ROUNDS); do
  for v in old new; do
    cp _ab/$v.so paper_2411_15715_b200/_native/libsliced.so
    echo "== $v"; timeout 600 bash -c "$CMD" 2>&1 | tail -8
  done
done
cp _ab/keep.so paper_2411_15715_b200/_native/libsliced.so
