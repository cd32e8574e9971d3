"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python scripts/launch_table.py launches.csv [steps] [top]"""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(path)):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum" or "materialize" in d["Kernel Name"]:
        continue
    us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-3)
    k = d["Kernel Name"].split("(")[0][-48:]
    agg[k][0] += 1
    agg[k][1] += us
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{k:48s} {n:5d} {t / steps:9.1f} us/step {100 * t / tot:5.1f}%")
print(f"total {tot / steps:.1f} us/step over {steps} steps")
