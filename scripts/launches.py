"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
launches = [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr + 1:] if len(r) > vi]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
launches = launches[skip:]
agg, cnt = collections.defaultdict(float), collections.Counter()
for _, k, v in launches:
    name = k.split("(")[0][:70]
    agg[name] += v; cnt[name] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:30]:
    print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}% x{cnt[k]:3d} {k}")
print(f"total {tot/1e3:.1f} us over {len(launches)} launches")
