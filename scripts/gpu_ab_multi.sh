#!/bin/bash
# alternating A/B of two env settings over N rounds of the default bench: "A-env" "B-env" N
mkdir -p gpurun_out
A=$1; B=$2; N=${3:-6}
for r in $(seq 1 $N); do
  for tag in A B; do
    if [ $tag = A ]; then E=$A; else E=$B; fi
    env $E timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['value'],1), round(d['e2e']['value'],1))"
  done
done > gpurun_out/abm.log 2>&1
python - <<'PY'
import statistics as st
rows=[l.split() for l in open("gpurun_out/abm.log") if l.strip()]
for tag in "AB":
    v=[float(r[1]) for r in rows if r[0]==tag]; e=[float(r[2]) for r in rows if r[0]==tag]
    print(tag, "value median", st.median(v), "mean", round(st.mean(v),1), "| e2e median", st.median(e), "mean", round(st.mean(e),1), "n", len(v))
PY
