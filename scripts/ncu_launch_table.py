"""Per-launch table from an `ncu --metrics ... --csv` log: kernel, grid, time, DRAM bytes.
`--summary`: per kernel name (this library's kernels only), launches, mean time, share of
the library's GPU time and DRAM MB per launch."""
import csv
import sys
from collections import OrderedDict

rows = OrderedDict()
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    e = rows.setdefault(key, {"name": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
    e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
if "--summary" in sys.argv:
    from collections import defaultdict

    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for e in rows.values():
        if e["name"].startswith(("at::", "void at::")):
            continue  # torch's input setup, outside the path
        name = e["name"].replace("void ", "").split("(")[0]
        a = agg[name]
        a[0] += 1
        a[1] += e.get("gpu__time_duration.sum", 0)
        a[2] += e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
    total = sum(a[1] for a in agg.values()) or 1.0
    print(f"{'kernel':60s} {'n':>5s} {'mean us':>9s} {'share':>7s} {'MB/launch':>10s}")
    for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {n:5d} {t / n / 1e3:9.1f} {t / total:7.1%} {b / n / 1e6:10.2f}")
    sys.exit(0)
for k, e in rows.items():
    t = e.get("gpu__time_duration.sum", 0)
    rd = e.get("dram__bytes_read.sum", 0)
    wr = e.get("dram__bytes_write.sum", 0)
    name = e["name"].replace("void ", "")[:48]
    gbs = (rd + wr) / t if t else 0
    print(f"{k:>4} {name:48s} {e['grid']:>14s} {t/1e3:8.2f} us  rd {rd/1e6:8.2f} MB  wr {wr/1e6:7.2f} MB  {gbs:7.0f} GB/s")
