"""Summarise `ncu -i rep --page source --csv --kernel-name regex:X` (SASS view):
executed warp-instructions by opcode and the top stall sites with their stall
reason breakdown.  Usage: python scripts/sass_hot.py file.csv [top_n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = 1 if rows[0][0] == "Kernel Name" else 0
h = rows[start]
col = {n: i for i, n in enumerate(h)}
data = []
for r in rows[start + 1:]:
    try:
        data.append(r)
    except Exception:
        pass


def f(r, name):
    try:
        return float(r[col[name]])
    except (ValueError, IndexError, KeyError):
        return 0.0


tot_inst = sum(f(r, "Instructions Executed") for r in data)
print(f"total warp-instructions executed: {tot_inst:.4g}")
ops = collections.Counter()
for r in data:
    op = r[col["Source"]].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    ops[o.split(".")[0]] += f(r, "Instructions Executed")
for o, n in ops.most_common(25):
    print(f"  {o:12s} {100 * n / tot_inst:5.1f}%")
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
agg = collections.Counter()
for r in data:
    for c in stall_cols:
        agg[c] += f(r, c)
print("stall reasons (all samples):", ", ".join(f"{c[6:]} {100 * v / tot:.1f}%" for c, v in agg.most_common(8)))
top = sorted(range(len(data)), key=lambda i: -f(data[i], "Warp Stall Sampling (All Samples)"))
for i in top[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    r = data[i]
    s = f(r, "Warp Stall Sampling (All Samples)")
    why = sorted(((f(r, c), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{100 * s / tot:5.1f}% {r[col['Address']]:>6s} {r[col['Source']].strip()[:60]:60s} "
          + " ".join(f"{w}:{100 * v / max(s, 1):.0f}%" for v, w in why))
