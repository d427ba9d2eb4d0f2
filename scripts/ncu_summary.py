"""Summarise an ncu --csv launch list: per kernel, launches, mean/total gpu time, DRAM bytes per launch."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
for r in rows[start + 1:]:
    if len(r) > vi:
        per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for (_, name), m in per.items():
    short = name.split("(")[0].replace("void ", "")[:70]
    a = agg[short]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':72s} {'n':>5s} {'mean us':>9s} {'share':>6s} {'MB/launch':>10s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:72s} {n:5d} {t / n / 1e3:9.1f} {t / tot:6.1%} {b / n / 1e6:10.2f}")
