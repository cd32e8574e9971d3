"""Top SASS stall sites from `ncu -i rep --page source --csv --kernel-name regex:X`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ai, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Address"), h.index("Source")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[si]), r[ai], r[src].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
order = sorted(range(len(data)), key=lambda i: -data[i][0])
for i in order[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    v, a, s = data[i]
    ctx = " | ".join(d[2][:40] for d in data[max(0, i - 2):i])
    print(f"{100 * v / tot:5.1f}%  {s[:70]:70s}  <- {ctx}")
