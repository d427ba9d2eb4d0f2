"""Median anatomy of traced decode steps (bench --trace-out / SP_BENCH_TRACE_E2E):
per call, when each stage starts and ends relative to the call's first span,
the copy stream's busy time and gaps, and the step period (call start to next
call start)."""
import json
import statistics as st
import sys
from collections import defaultdict

recs = json.load(open(sys.argv[1]))
by = defaultdict(list)
for r in recs:
    by[r["call"]].append(r)
calls = sorted(by)
starts = {c: min(r["start_s"] for r in by[c]) for c in calls}
rows = []
for i, c in enumerate(calls[1:-1], 1):
    rs = by[c]
    t0 = starts[c]
    row = {}
    for kind in ("route", "launch", "cc", "copy", "cg", "gg", "merge", "ycc", "return"):
        xs = [r for r in rs if r["kind"] == kind]
        if not xs:
            continue
        row[f"{kind}_start"] = (min(r["start_s"] for r in xs) - t0) * 1e6
        row[f"{kind}_end"] = (max(r["end_s"] for r in xs) - t0) * 1e6
        row[f"{kind}_busy"] = sum(r["end_s"] - r["start_s"] for r in xs) * 1e6
        row[f"{kind}_n"] = len(xs)
    cps = sorted((r["start_s"], r["end_s"]) for r in rs if r["kind"] == "copy")
    row["copy_gaps"] = sum(max(0.0, b[0] - a[1]) for a, b in zip(cps, cps[1:])) * 1e6
    row["period"] = (starts[calls[i + 1]] - t0) * 1e6
    rows.append(row)
keys = []
for r in rows:
    for k in r:
        if k not in keys:
            keys.append(k)
for k in keys:
    vals = [r[k] for r in rows if k in r]
    print(f"{k:14s} median {st.median(vals):9.1f}   (n={len(vals)})")
