"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, gi, bi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
mi = h.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0, ""])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    k = r[ki][:70]
    agg[k][0] += 1
    agg[k][1] += v
    agg[k][2] = f"grid {r[gi]} block {r[bi]}"
for k, (n, t, g) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:4d} {t / 1e6:10.3f} ms  {k:70s} {g}")
