"""First spans of a mid-run traced call (bench --trace-out / SP_BENCH_TRACE_E2E json): when the GPU starts."""
import json
import sys

recs = json.load(open(sys.argv[1]))
calls = sorted(set(r["call"] for r in recs))
c = calls[len(calls) // 2]
rs = sorted([r for r in recs if r["call"] == c], key=lambda r: r["start_s"])
t0 = min(r["start_s"] for r in rs)
for r in rs[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"  {r['kind']:8s} {(r['start_s'] - t0) * 1e6:8.1f} -> {(r['end_s'] - t0) * 1e6:8.1f} us")
