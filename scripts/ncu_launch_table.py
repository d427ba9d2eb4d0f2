"""Per-launch table from an `ncu --metrics ... --csv` log: kernel, grid, time, DRAM bytes."""
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
for k, e in rows.items():
    t = e.get("gpu__time_duration.sum", 0)
    rd = e.get("dram__bytes_read.sum", 0)
    wr = e.get("dram__bytes_write.sum", 0)
    name = e["name"].replace("void ", "")[:48]
    gbs = (rd + wr) / t if t else 0
    print(f"{k:>4} {name:48s} {e['grid']:>14s} {t/1e3:8.2f} us  rd {rd/1e6:8.2f} MB  wr {wr/1e6:7.2f} MB  {gbs:7.0f} GB/s")
