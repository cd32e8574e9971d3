"""Summarize an ncu --set full report of the hot-path kernels into profiles/.

    python scripts/ncu_summary.py <full.ncu-rep> <launches.csv> <config> <precision> <tag> <unique_images>

Writes profiles/<tag>_<config>_<precision>_ncu.md (per-kernel DRAM bytes,
throughput, tensor-pipe activity, coalescing counters, plus the launch-list
share of the step) and merges the per-launch DRAM traffic of every captured
kernel into profiles/ncu_traffic.json, which bench.py reports as
roofline.traffic.
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = {"k_fwd": "img_fwd_l0", "k_fwd2": "img_fwd_l0", "k_fwd4": "img_fwd_l0", "k_l12_fwd": "img_fwd_l12", "k_l12f": "img_fwd_l12",
         "k_l12_bwd": "img_bwd_l12", "k_l12b": "img_bwd_l12", "k_dw1": "img_bwd_dw1", "k_dw1b": "img_bwd_dw1",
         "k_dw0": "img_bwd_dw0", "k_dw0p": "img_bwd_dw0", "k_sample_fwd": "sample_fwd", "k_sample_bwd": "sample_bwd",
         "k_attn_bwd": "sample_bwd", "k_sample_scatter": "sample_bwd"}
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "tmem pipe %"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "LSU ld sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "LSU ld requests"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    """Bare function name: 'void dicm::<unnamed>::k_fwd<1>(CUtensorMap ...)' -> 'k_fwd'."""
    head = name.split("(")[0]
    head = re.sub(r"<[^<>]*>$", "", head.strip())  # trailing template arguments
    m = re.search(r"([A-Za-z_][A-Za-z0-9_]*)\s*$", head)
    return m.group(1) if m else name[:40]


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for m, _ in METRICS)],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for m, _ in METRICS:
            for i, h in enumerate(hdr):
                if h == m:
                    v = r[i].replace(",", "")
                    try:
                        d[m] = float(v) * SCALE.get(units[i], 1.0)
                    except ValueError:
                        d[m] = None
        d["name"] = short(r[hdr.index("Kernel Name")])
        res.append(d)
    return res


def launch_share(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        n = short(r[ki])
        if "materialize" in r[ki] or "Fill" in r[ki]:
            continue  # pool build / buffer init, outside the step
        agg[n] += float(r[vi].replace(",", ""))
        cnt[n] += 1
    return agg, cnt


def main():
    rep, launches, cfg, prec, tag, U = sys.argv[1:7]
    U = int(U)
    kern = read_raw(rep)
    agg, cnt = launch_share(launches)
    tot = sum(agg.values())
    steps = max(cnt.get("k_fwd4", 0) or cnt.get("k_fwd2", 0) or cnt.get("k_fwd", 1), 1)
    lines = [f"# ncu summary: {cfg} / {prec} ({tag})", "",
             f"Source: `{os.path.basename(rep)}` (`ncu --set full --clock-control none --import-source on`, "
             "one launch per kernel, cold-cache replay) and the launch list "
             f"`{os.path.basename(launches)}` (`--metrics gpu__time_duration.sum`, {steps} steps incl. warm-up; "
             f"pool materialization excluded). Unique images in the captured step: ~{U}.", "",
             "## Per-kernel counters (one captured launch each)", "",
             "| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " | DRAM GB/s |",
             "|---" * (len(METRICS) + 2) + "|"]
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    seen, fresh = set(), {}
    for d in kern:
        t = d.get("gpu__time_duration.sum") or 0
        rd, wr = d.get("dram__bytes_read.sum") or 0, d.get("dram__bytes_write.sum") or 0
        cells = []
        for m, _ in METRICS:
            v = d.get(m)
            if v is None:
                cells.append("-")
            elif m.startswith("dram__bytes"):
                cells.append(f"{v / 1e6:.1f} MB")
            elif m == "gpu__time_duration.sum":
                cells.append(f"{v * 1e6:.1f} us")
            else:
                cells.append(f"{v:.1f}" if v % 1 else f"{int(v)}")
        gbs = (rd + wr) / t / 1e9 if t else 0
        lines.append(f"| {d['name']} | " + " | ".join(cells) + f" | {gbs:.0f} |")
        if d["name"] in PROBE and d["name"] not in seen:  # one launch per kernel; probes may span kernels
            seen.add(d["name"])
            key = f"{cfg}/{prec}/{PROBE[d['name']]}"
            e = fresh.setdefault(key, {"dram_bytes": 0.0, "unique_images": U, "ncu_time_s": 0.0,
                                       "source": f"{tag}:{rep}"})
            e["dram_bytes"] += rd + wr
            e["ncu_time_s"] += t
    traffic.update(fresh)
    lines += ["", "## Launch list: share of the step (serialized, cold-cache)", "",
              "| kernel | launches | total us | us / step | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:25]:
        lines.append(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / 1e3 / steps:.1f} | {100 * v / tot:.1f}% |")
    lines.append(f"| total | {sum(cnt.values())} | {tot / 1e3:.1f} | {tot / 1e3 / steps:.1f} | 100% |")
    out = os.path.join(ROOT, "profiles", f"{tag}_{cfg}_{prec}_ncu.md")
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
    print(out)


if __name__ == "__main__":
    main()
