"""Median per-call anatomy of a bench trace (--trace-out): where the CC block
and the CG copy stream start and end relative to the call's first host span."""
import json
import statistics as st
import sys
from collections import defaultdict

recs = json.load(open(sys.argv[1]))
by = defaultdict(list)
for r in recs:
    by[r["call"]].append(r)
rows = []
for c, rs in sorted(by.items()):
    t0 = min(r["start_s"] for r in rs)
    def first(kind):
        xs = [r["start_s"] for r in rs if r["kind"] == kind]
        return (min(xs) - t0) * 1e6 if xs else float("nan")
    def last(kind):
        xs = [r["end_s"] for r in rs if r["kind"] == kind]
        return (max(xs) - t0) * 1e6 if xs else float("nan")
    rows.append({"cc_start": first("cc"), "cc_end": last("cc"), "copy_start": first("copy"), "copy_end": last("copy"),
                 "merge_end": last("merge"), "return_end": last("return")})
for k in rows[0]:
    print(f"{k:11s} median {st.median(r[k] for r in rows[1:]):8.1f} us")
