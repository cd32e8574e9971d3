"""Copy the bench JSON line of each given log into profiles/<name>.json.

    python scripts/save_lines.py gpurun_out/r2l_cfg2_n1.log:r02_bench_cfg2_n1 ...
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for arg in sys.argv[1:]:
    src, name = arg.split(":")
    lines = [line for line in open(src) if line.startswith("{")]
    if not lines:
        print(f"{src}: no JSON line")
        continue
    d = json.loads(lines[-1])
    with open(os.path.join(ROOT, "profiles", name + ".json"), "w") as fh:
        json.dump(d, fh, indent=1)
    print(f"{name}: {d.get('value')} {d.get('unit')}  ms/step {d.get('ms_per_step')}")
