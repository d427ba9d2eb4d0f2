"""Per-call critical-path summary of a bench.py --trace-out timeline (µs from the call's first span)."""
import json
import sys
from collections import defaultdict

recs = json.load(open(sys.argv[1]))
by = defaultdict(list)
for r in recs:
    by[r["call"]].append(r)
for c in sorted(by):
    rs = by[c]
    t0 = min(r["start_s"] for r in rs)
    f = lambda kinds, key, agg: agg([r[key] for r in rs if r["kind"] in kinds] or [float("nan")])  # noqa: E731
    us = lambda v: (v - t0) * 1e6  # noqa: E731
    cps = sorted([r for r in rs if r["kind"] == "copy"], key=lambda r: r["start_s"])
    gaps = [b["start_s"] - a["end_s"] for a, b in zip(cps, cps[1:])]
    busy = sum(r["end_s"] - r["start_s"] for r in cps)
    byt = sum(r["bytes"] for r in cps)
    print(f"call {c}: launch {us(f({'launch'}, 'start_s', min)):7.1f}-{us(f({'launch'}, 'end_s', max)):7.1f} | "
          f"gg {us(f({'gg'}, 'start_s', min)):7.1f}-{us(f({'gg'}, 'end_s', max)):7.1f} | "
          f"copy {us(f({'copy'}, 'start_s', min)):7.1f}-{us(f({'copy'}, 'end_s', max)):7.1f} "
          f"({len(cps)} x, {byt / busy / 1e9 if busy else 0:5.1f} GB/s busy, gaps sum {sum(gaps) * 1e6:6.1f}) | "
          f"cg end {us(f({'cg'}, 'end_s', max)):7.1f} | cc {us(f({'cc'}, 'start_s', min)):7.1f}-{us(f({'cc'}, 'end_s', max)):7.1f} | "
          f"merge {us(f({'merge'}, 'start_s', min)):7.1f}-{us(f({'merge'}, 'end_s', max)):7.1f} | "
          f"route {us(f({'route'}, 'start_s', min)):7.1f}-{us(f({'route'}, 'end_s', max)):7.1f} | "
          f"return {us(f({'return'}, 'start_s', min)):7.1f}-{us(f({'return'}, 'end_s', max)):7.1f}")
