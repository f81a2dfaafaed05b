"""Per-kernel mean duration from an ncu gpu__time_duration launch list.

    python scripts/launch_table.py launches.csv [first_index]
"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0].split("::")[-1][:40], float(d["Metric Value"].replace(",", ""))))
agg = OrderedDict()
for k, v in out[first:]:
    agg.setdefault(k, []).append(v)
for k, v in agg.items():
    print(f"{k:42s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.2f} us  min={min(v)/1e3:9.2f}")
