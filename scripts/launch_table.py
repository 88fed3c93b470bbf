"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = (d["ID"], d["Kernel Name"].split("(")[0][:48])
        agg.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
print(f"{'id':>4} {'kernel':48} {'ms':>8} {'rd GB':>7} {'wr GB':>7}")
for (i, k), m in agg.items():
    t = m.get("gpu__time_duration.sum", 0)
    unit_ms = t / 1e6 if t > 1e3 else t
    print(f"{i:>4} {k:48} {t / 1e6:8.3f} {m.get('dram__bytes_read.sum', 0) / 1e9:7.2f} {m.get('dram__bytes_write.sum', 0) / 1e9:7.2f}")
