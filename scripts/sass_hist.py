"""Per-instruction execution counts of one kernel from an ncu source-page CSV.

Usage: ncu -i REP --page source --csv --print-source sass > x.csv
       python scripts/sass_hist.py x.csv [min_count]
Prints the total warp-instruction count, the share in instructions executed at least
`min_count` times (the hot loop), and the listing of instructions above a tenth of it.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
h = rows[1]
ie = h.index("Instructions Executed")
src = h.index("Source")
smp = h.index("Warp Stall Sampling (All Samples)")
seen, d = set(), []
for r in rows[2:]:
    if len(r) != len(h) or not r[ie].isdigit():
        continue
    if r[0] in seen:
        break
    seen.add(r[0])
    d.append(r)
tot = sum(int(r[ie]) for r in d)
hot = sum(int(r[ie]) for r in d if int(r[ie]) >= thr)
s_tot = sum(int(r[smp] or 0) for r in d)
s_hot = sum(int(r[smp] or 0) for r in d if int(r[ie]) >= thr)
print(f"instructions {tot/1e6:.2f}M, >= {thr}: {hot/1e6:.2f}M; samples {s_tot}, hot {s_hot}")
for r in d:
    n = int(r[ie])
    if n >= thr // 10:
        print(f"{r[0][-5:]} {n/1e6:6.3f}M smp={int(r[smp] or 0):5d} {r[src].strip()[:90]}")
