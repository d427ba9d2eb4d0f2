#!/bin/bash
# the default bench line N times on one box (median / spread of value and e2e)
mkdir -p gpurun_out
N=${1:-10}
for r in $(seq 1 $N); do
  timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1
done > gpurun_out/repeat.jsonl
python - <<'PY'
import json, statistics as st
rows = [json.loads(l) for l in open("gpurun_out/repeat.jsonl") if l.strip()]
v = [r["value"] for r in rows]; e = [r["e2e"]["value"] for r in rows]
f = [r["roofline"]["frac"] for r in rows]; fd = [r["roofline"]["frac_device_span"] for r in rows]
for name, xs in (("value", v), ("e2e", e), ("frac", f), ("frac_device_span", fd)):
    print(f"{name:18s} n={len(xs)} median {st.median(xs):8.3f}  min {min(xs):8.3f}  max {max(xs):8.3f}")
PY
