"""DICM training-step benchmark on B200 (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
                    [--precision auto|fp32|tf32|bf16] [--impl b200|reference]

Workload (BASELINE.json configs):
  cfg1  sum pooling, B=256, L=50, pool 10k            (the CPU-runnable case)
  cfg2  single-head attn, B=4096, L=200, pool 1M       (default at N=1)
  cfg3  multi-query attn, B=8192/GPU, L=200, pool 20M sharded
  cfg4  sum, Zipf(1.1) keys, B=8192/GPU, L=50, pool 1M
  cfg5  attn, lengths lognormal(ln 40, 1) clipped 1..500, 100M-row tables
A step = one full training iteration (dedup, image MLP fwd/bwd, pooling,
head, BCE, backward, Adam on every dense parameter and every touched ID row)
over one batch of synthetic data.  ``value`` times K steps with the inputs
already in HBM; ``e2e`` times the public API (LocalTrainer.train_batch_async on
a host Batch: H2D of the packed batch + D2H of the loss inside the region).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(kind="sum", B=256, L=50, P=10_000, vocab=100_000, zipf=None, lengths=None, tables=None),
    "cfg2": dict(kind="attn", B=4096, L=200, P=1_000_000, vocab=100_000, zipf=None, lengths=None, tables=None),
    "cfg3": dict(kind="multiquery-attn", B=8192, L=200, P=20_000_000, vocab=100_000, zipf=None, lengths=None,
                 tables=None),
    "cfg4": dict(kind="sum", B=8192, L=50, P=1_000_000, vocab=100_000, zipf=1.1, lengths=None, tables=None),
    "cfg5": dict(kind="attn", B=8192, L=500, P=20_000_000, vocab=100_000_000, zipf=None, lengths="lognormal",
                 tables=None),
}
DESC = {
    "cfg1": "DICM sum pooling, batch 256, 50 behavior images/user, 10k-image pool, 100k-row ID tables",
    "cfg2": "DICM single-head attentive pooling (ad-image query), batch 4096, 200 behavior images/user, "
            "1M-image pool, 1xB200",
    "cfg3": "DICM double-head attentive pooling, batch 8192/GPU, 200 behaviors/user, 20M-image pool",
    "cfg4": "DICM sum pooling, Zipf(1.1) image keys, batch 8192/GPU, 50 behaviors/user, 1M-image pool",
    "cfg5": "DICM attentive pooling, behavior lengths lognormal 1-500, 100M-row ID tables",
}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def build_workload(name, rank, world, precision, seed=0, device="cuda"):
    import torch

    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema
    c = CONFIGS[name]
    b_max = 500 if c["lengths"] == "lognormal" else c["L"]
    v = c["vocab"]
    schema = default_schema(v, 4, v, 8, c["P"], b_max=b_max)
    pool_dtype = "bf16" if precision == "bf16" else "fp32"
    pool = ImagePool.synthetic(c["P"], seed=seed, dtype=pool_dtype, device=device, world=world, rank=rank)
    big = max(f.vocab for f in schema.fields) > (1 << 21)
    model = DicmModel(schema, AggregatorSpec(c["kind"]), None, seed=0, device=device,
                      shard=(world, rank) if world > 1 else None, table_init="device" if big else "reference")
    torch.cuda.synchronize()
    return schema, model, pool


def make_batches(name, schema, n, seed):
    from paper_1711_06505_b200.batch import synthetic_batch
    c = CONFIGS[name]
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        if c["lengths"] == "lognormal":
            L = np.clip(np.round(rng.lognormal(np.log(40), 1.0, c["B"])), 1, 500).astype(np.int64)
        else:
            L = c["L"]
        out.append(synthetic_batch(rng, schema, c["B"], L, c["P"], zipf=c["zipf"]))
    return out


# ---------------------------------------------------------------------------
# CPU baseline (the reference's own LocalTrainer when baseline/_ref holds it,
# else the oracle port), timed on this host's cores on a bounded sample
# ---------------------------------------------------------------------------

def cpu_baseline(name, schema, pool, batch, max_seconds=25.0, sample_b=256):
    import torch
    threads = os.cpu_count() or 1
    sub = batch.slice(0, min(sample_b, batch.size))
    lay_kind = CONFIGS[name]["kind"]
    # compact monotone remap of the touched pool rows
    ids = np.unique(np.concatenate([sub.ad_image_ids, sub.beh_image_ids]).astype(np.int64))
    rows = pool.gather(ids).double().cpu().numpy()
    kind = "port"
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    t0 = time.perf_counter()
    times = []
    try:
        if os.path.isdir(os.path.join(ref_dir, "dicm")):
            sys.path.insert(0, ref_dir)
            import dicm.model as RM
            import dicm.training as RT
            kind = "reference"
            fields = [RM.FieldSpec(f.name, f.vocab, f.multi) for f in schema.fields]
            rs = RM.FeatureSchema(fields=fields, d_id=12, d_raw=schema.d_raw, d_img=12, b_max=schema.b_max)

            class Ext:
                out_dim = schema.d_raw

            class Store:
                def __len__(self):
                    return pool.global_size

                def raw_features(self, q, extractor):
                    return rows[np.searchsorted(ids, np.asarray(q, dtype=np.int64))]

            model = RM.DicmModel(rs, RM.AggregatorSpec(lay_kind), Ext(), seed=0)
            tr = RT.LocalTrainer(model, Store(), RT.TrainConfig(batch_size=sub.size))
            samples = _samples_of(sub)
            step = lambda: tr.train_batch(samples)  # noqa: E731
        else:
            raise ImportError
    except Exception:
        from oracle import dicm_oracle as O
        kind = "port"
        from paper_1711_06505_b200.schema import init_params, ModelLayout, AggregatorSpec
        lay = ModelLayout(schema, AggregatorSpec(lay_kind), (128, 64), True, True)
        params = init_params(lay, 0, include_tables=True)
        cfg = O.make_cfg([(f.name, f.vocab, f.multi) for f in schema.fields], b_max=schema.b_max, kind=lay_kind)
        # remap image ids into the compact pool
        ob = {"size": sub.size, "labels": sub.labels.astype(np.float64),
              "onehot": {k: v.astype(np.int64) for k, v in sub.onehot.items()},
              "multihot": {k: (a.astype(np.int64), o.astype(np.int64)) for k, (a, o) in sub.multihot.items()},
              "ad_image_ids": np.searchsorted(ids, sub.ad_image_ids), "beh_image_ids": np.searchsorted(ids,
                                                                                                       sub.beh_image_ids),
              "beh_off": sub.beh_off.astype(np.int64)}
        tr = O.OracleTrainer(params, cfg, rows)
        step = lambda: tr.train_batch(ob)  # noqa: E731
    # one warm-up, then as many steps as fit the budget (>= 1)
    step()
    while True:
        a = time.perf_counter()
        step()
        times.append(time.perf_counter() - a)
        if time.perf_counter() - t0 > max_seconds or len(times) >= 3:
            break
    med = statistics.median(times)
    return {"value": sub.size / med, "unit": "samples/s", "cores": threads, "kind": kind,
            "sample": f"{sub.size} samples of {name} (L={CONFIGS[name]['L']}, pool {CONFIGS[name]['P']}), "
                      f"1 warm-up + median of {len(times)} steps, f64, {threads} host threads"}


def _samples_of(b):
    out = []
    for i in range(b.size):
        s = {"label": float(b.labels[i]), "ad_image": int(b.ad_image_ids[i]), "day": 0}
        for f, v in b.onehot.items():
            s[f] = int(v[i])
        for f, (fl, of) in b.multihot.items():
            s[f] = fl[of[i]:of[i + 1]].tolist()
        s["behavior_images"] = b.beh_image_ids[b.beh_off[i]:b.beh_off[i + 1]].tolist()

        class S_:
            pass
        o = S_()
        o.__dict__.update(s)
        out.append(o)
    return out


# ---------------------------------------------------------------------------

def run_reference_arm(args):
    rank, world, local = env_rank()
    if rank != 0:
        return
    import torch
    name = args.config
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
        schema, model, pool = build_workload(name, 0, 1, "fp32")
    else:
        raise SystemExit("reference arm needs the GPU box to materialize the same pool rows")
    batch = make_batches(name, schema, 1, seed=1234)[0]
    times = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(name, schema, pool, batch, max_seconds=20.0)
        times.append(cb["value"])
    v = statistics.median(times[args.warmup:]) if args.steps else times[-1]
    line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * 256 / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": name, "description": DESC[name], "sample_batch": 256},
            "cpu_baseline": {**cb, "value": v},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "DICM train samples/sec (fwd+bwd)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="auto", choices=["auto", "fp32", "tf32", "bf16"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.config
    kind = CONFIGS[name]["kind"]
    precision = args.precision
    if precision == "auto":
        # bf16 layer-0 operands stay inside the north star's 2e-2 on logits for
        # attentive pooling; sum pooling's large logits need tf32
        precision = os.environ.get("DICM_PRECISION", "tf32" if kind == "sum" else "bf16")
    from paper_1711_06505_b200.runtime import Cluster, ClusterConfig
    B = CONFIGS[name]["B"]
    schema, model, pool = build_workload(name, rank, world, precision)
    cluster = Cluster(ClusterConfig(workers=world, servers=world, batch_per_worker=B), model, pool,
                      precision=precision)
    eng = cluster.engine
    batches = make_batches(name, schema, args.warmup + args.steps, seed=1000 + rank)
    staged = [eng.upload(b, own=True) for b in batches]
    torch.cuda.synchronize()
    union = world * B

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(db):
        eng.forward_backward(db, denominator=union)
        eng.optimizer_step(eng.lr())
        eng.iteration += 1

    for db in staged[:args.warmup]:
        step(db)
    barrier()
    eng.probe = {"imgmlp_fwd": [], "imgmlp_bwd": []}
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        start.record()
        for db in staged[args.warmup:]:
            step(db)
        end.record()
        barrier()
    ms = start.elapsed_time(end)
    eng.raise_status()
    probes = {k: [a.elapsed_time(b) for a, b in v] for k, v in eng.probe.items()}
    eng.probe = None
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / max(args.steps, 1)
    value = union * args.steps / (ms / 1000.0)

    # e2e through the public API with host batches: H2D inside the region,
    # the loss read back (async D2H into pinned memory) every step
    e2e = None
    if not args.no_e2e:
        host = batches[args.warmup:]
        pinned_loss = torch.empty(len(host), dtype=torch.float32, pin_memory=True)
        barrier()
        s2, e2_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        for i, b in enumerate(host):
            loss = cluster.train_batch_async(b, union)
            pinned_loss[i:i + 1].copy_(loss, non_blocking=True)
        e2_.record()
        barrier()
        ems = s2.elapsed_time(e2_)
        eng.raise_status()
        te = torch.tensor([ems], device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        e2e = {"value": union * len(host) / (ems / 1000.0), "unit": "samples/s",
               "h2d_bytes_per_step": int(np.mean([eng.h2d_bytes(b) for b in host])), "d2h_bytes_per_step": 4,
               "api": "Cluster.train_batch_async (host CSR batch -> pinned H2D -> step -> loss D2H)"}

    # roofline of the dominant launch pair: dicm_imgmlp_fwd (tcgen05 layer 0 +
    # fused layers 1-2) per step, algorithmic bytes
    U = int(eng.counts[2].item()) if world > 1 else int(eng.counts[0].item())
    fwd_ms = statistics.mean(probes["imgmlp_fwd"]) if probes.get("imgmlp_fwd") else None
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    elem = 2 if precision == "bf16" else 4
    roof = None
    if fwd_ms:
        # X rows once, W0 once, act0 write + re-read, h1 write, act1 + emb write
        bytes_fwd = U * schema.d_raw * elem + 256 * schema.d_raw * elem + U * (256 * 4 * 3 + 64 * 4 + 12 * 4)
        ach = bytes_fwd / (fwd_ms / 1000.0) / 1e9
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            ent = prof.get(f"{name}/{precision}")
            if ent:
                traffic = ent["dram_bytes_per_launch"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": "dicm_imgmlp_fwd (tcgen05 layer-0 GEMM + fused layers 1-2)",
                "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json (measured)" if peaks else "fallback",
                "algorithmic_bytes_per_launch": bytes_fwd, "ms_per_launch": fwd_ms,
                "bwd_ms_per_launch": statistics.mean(probes["imgmlp_bwd"]) if probes.get("imgmlp_bwd") else None,
                "unique_images_per_step": U,
                "tensor_tflops_fwd_bwd": (U * 4297216 / 1e12) / ((fwd_ms + (statistics.mean(
                    probes["imgmlp_bwd"]) if probes.get("imgmlp_bwd") else 0)) / 1000.0)}
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(name, schema, pool, batches[-1])
        except Exception as ex:  # reported, never fatal
            cb = {"value": None, "error": repr(ex)[:200]}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": precision, "data": "synthetic",
                "config": {"workload": name, "description": DESC[name], "global_batch": union,
                           "batch_per_gpu": B, "behaviors_per_user": CONFIGS[name]["L"],
                           "pool_images": CONFIGS[name]["P"], "aggregator": kind,
                           "precision": f"image-MLP layer-0 operands {precision}, fp32 accumulate; "
                                        "layers 1-2 tf32 tensor cores; pooling/head/Adam fp32",
                           "parallelism": f"AMS: pool + ID tables sharded over {world} GPU(s), dense dp{world}",
                           "l2": "inputs larger than L2 (each step gathers ~U x 8-16 KB of distinct pool rows)"},
                "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": eng.launches_per_step * args.steps,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
