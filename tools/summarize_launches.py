"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = defaultdict(lambda: [0, 0.0])
for r in data:
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(x[1] for x in agg.values())
print(f"{len(data)} launches, {tot:.1f} ms total (ncu-serialised, cold-cache)")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:6d} launches {ms:10.2f} ms {100 * ms / tot:5.1f}%  avg {ms / n:8.3f} ms  {k}")
