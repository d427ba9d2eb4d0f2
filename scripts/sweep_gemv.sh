#!/bin/bash
# sweep GEMV tunables; one process per setting (env is read at library load)
for c in 1 2 3 4; do for w in 0 1 2 4 8; do
  SP_CTAS_PER_SM=$c SP_WPR=$w timeout 300 python scripts/bench_gemv.py --T 1 --hidden 7168 14336 --reps 8 2>&1 | grep -v Warn
done; done
SP_CTAS_PER_SM=2 timeout 300 python scripts/bench_gemv.py --T 1 2 4 8 --hidden 7168 --reps 8
