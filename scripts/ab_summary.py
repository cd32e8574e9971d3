"""Summarize gpurun_out/<tag>_ab.log (scripts/ab.sh): per env setting, the
ms/step, samples/s, SM clock and the probed kernel times of each run."""
import json
import sys

cur = None
for line in open(sys.argv[1]):
    if line.startswith("== "):
        cur = line[3:].strip()
    elif line.startswith("{"):
        d = json.loads(line)
        r = d.get("roofline") or {}
        ks = {k: round(v["ms"] * 1e3, 1) for k, v in (r.get("kernels") or {}).items()}
        print(f"{cur:28s} {d['ms_per_step']:.4f} ms  {d['value'] / 1e6:.3f} M/s  {d['clocks'].get('sm_mhz')} MHz  {ks}")
