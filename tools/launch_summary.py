"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, total
time and share per kernel name.   python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    ms = float(r[vi].replace(",", "")) * SCALE[r[ui]]
    a = agg[r[ki][:90]]
    a[0] += 1
    a[1] += ms
tot = sum(v[1] for v in agg.values())
print(f"{sum(v[0] for v in agg.values())} launches, {tot:.1f} ms (cold, serialised under ncu)")
for name, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{c:6d} launches {ms:10.2f} ms {100 * ms / tot:5.1f}%  {name}")
