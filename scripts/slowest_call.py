"""Find the slowest forwards in a full bench trace and print their spans."""
import json
import sys
from collections import defaultdict

recs = json.load(open(sys.argv[1]))
by = defaultdict(list)
for r in recs:
    by[r["call"]].append(r)
calls = sorted(by)
starts = {c: min(r["start_s"] for r in by[c]) for c in calls}
ends = {c: max(r["end_s"] for r in by[c]) for c in calls}
gaps = [(starts[b] - ends[a], a, b) for a, b in zip(calls, calls[1:])]
dur = sorted(((ends[c] - starts[c], c) for c in calls), reverse=True)
print("longest calls (ms):", [(round(d * 1e3, 2), c) for d, c in dur[:5]])
print("longest gaps between calls (ms):", [(round(g * 1e3, 2), a, b) for g, a, b in sorted(gaps, reverse=True)[:5]])
for d, c in dur[:2]:
    t0 = starts[c]
    print(f"-- call {c}")
    for r in sorted(by[c], key=lambda r: r["start_s"]):
        if r["kind"] != "copy" or r["end_s"] - r["start_s"] > 0.001:
            print(f'  {r["kind"]:8s} {r["stream"]:8s} {1e3 * (r["start_s"] - t0):9.3f} {1e3 * (r["end_s"] - t0):9.3f}')
