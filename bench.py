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
already in HBM; ``e2e`` times the public API (Cluster.train_batch_async on
host Batches: host packing, H2D of the packed batch + D2H of the loss inside
the region; the host side of step i+1 overlaps step i).
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
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region:
    one `nvidia-smi -lms 20` stream started before the region, samples kept
    between enter() and exit()."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples = []
        self._proc = None
        self._t = None
        self._window = [None, None]
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                                           "--format=csv,noheader,nounits", "-lms", "20"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.3)  # let the stream start before the timed region
        except Exception:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            now = time.perf_counter()
            w0, w1 = self._window
            if w0 is not None and now >= w0 and (w1 is None or now <= w1):
                self.samples.append([x.strip() for x in line.split(",")])

    def __enter__(self):
        self._window[0] = time.perf_counter()
        return self

    def __exit__(self, *a):
        self._window[1] = time.perf_counter()
        if self._proc is not None:
            time.sleep(0.05)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()

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


def fields_of(name):
    """The benchmark schema's ID fields (reference experiments.py:17-32 with
    image_id_fields=True): (name, vocab, multi)."""
    c = CONFIGS[name]
    v = c["vocab"]
    return [("user", v, False), ("scenario", 4, False), ("ad", v, False), ("ad_category", 8, False),
            ("behavior_items", v, True), ("ad_image", c["P"], False), ("behavior_images", c["P"], True)]


def b_max_of(name):
    c = CONFIGS[name]
    return 500 if c["lengths"] == "lognormal" else c["L"]


def build_workload(name, rank, world, precision, seed=0, device="cuda"):
    import torch

    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.schema import AggregatorSpec, FeatureSchema, FieldSpec
    c = CONFIGS[name]
    schema = FeatureSchema([FieldSpec(n, v, m) for n, v, m in fields_of(name)], d_id=12, d_raw=4096, d_img=12,
                           b_max=b_max_of(name))
    pool_dtype = "bf16" if precision == "bf16" else "fp32"
    pool = ImagePool.synthetic(c["P"], seed=seed, dtype=pool_dtype, device=device, world=world, rank=rank)
    big = max(f.vocab for f in schema.fields) > (1 << 21)
    model = DicmModel(schema, AggregatorSpec(c["kind"]), None, seed=0, device=device,
                      shard=(world, rank) if world > 1 else None, table_init="device" if big else "reference")
    torch.cuda.synchronize()
    return schema, model, pool


# FP32 CUDA-core peak for the per-sample kernels (no measured figure exists):
# 148 SMs x 4 SMSPs x 32 lanes x 2 FMAs (paired FFMA2, one every 2 cycles,
# B300_MICROARCH.md pipe rates) x 2 FLOP at 1.965 GHz
FP32_PEAK_TFLOPS = 148 * 4 * 32 * 2 * 2 / 2 * 1.965e9 / 1e12


def attn_flops_per_ref(kind):
    """(forward, backward) FP32 FLOP per behavior reference of the attention
    channels (the 12 -> 32 key projection, PReLU and score per
    hidden unit, the softmax and weighted sum; backward: the projection again,
    the PReLU / softmax backward, dWk, dk)."""
    ch = {"attn": 1, "multiquery-attn": 2}.get(kind, 0)
    return ch * (2 * 12 * 32 + 4 * 32 + 2 * 12 + 8), ch * (3 * 2 * 12 * 32 + 8 * 32 + 4 * 12 + 16)


def kernel_work(U, B, R, W, D, e, kind="attn"):
    """Algorithmic (bytes, tensor flops, CUDA-core flops) per launch of each
    probed kernel, counting only what the math needs: U unique
    images, B samples, R behaviors, W head-input width, D = d_raw, e = layer-0
    operand bytes.  The saved activations act0/act1 (and da1/da0) are stored
    in the operand dtype in bf16 mode (e = 2) and in fp32 otherwise."""
    Rimg = B + R
    a = e  # bytes per saved activation
    af, ab = attn_flops_per_ref(kind)
    return {
        # X rows + W0 in, act0 out
        "img_fwd_l0": (U * D * e + 256 * D * e + U * 256 * a, 2 * U * D * 256, 0),
        # act0 in, act1 + emb out
        "img_fwd_l12": (U * ((256 + 64) * a + 12 * 4), 2 * U * (256 * 64 + 64 * 12), 0),
        # dE, act1, act0 in; da1, da0 out (dh2, dW2, dh1)
        "img_bwd_l12": (U * (12 * 4 + (64 + 256 + 64 + 256) * a), 2 * U * (2 * 12 * 64 + 64 * 256), 0),
        # act0 (-> h1), da1 in
        "img_bwd_dw1": (U * (256 + 64) * a, 2 * U * 64 * 256, 0),
        # X rows + da0 in, dW0 out
        "img_bwd_dw0": (U * D * e + U * 256 * e + 256 * D * 4, 2 * U * D * 256, 0),
        # image columns of the head input: inverse ids + embedding rows per reference, the attention math
        "sample_fwd": (Rimg * (4 + 48) + B * W * 4, 0, R * af),
        # attention backward + the ordered sums into dE: rows per reference in, dE out
        "sample_bwd": (Rimg * (4 + 48) + U * 48 + B * W * 4, 0, R * ab),
    }


def _zipf_keys(rng, n, pool, s=1.1, perm_seed=0):
    """rank r ~ (r+1)^-s over [0, pool), through a seeded permutation (cfg 4)."""
    p = (np.arange(pool, dtype=np.float64) + 1.0) ** (-s)
    cdf = np.cumsum(p / p.sum())
    r = np.minimum(np.searchsorted(cdf, rng.random(n), side="right"), pool - 1)
    return np.random.default_rng(perm_seed).permutation(pool)[r]


def gen_columns(name, n, seed):
    """``n`` synthetic batches of workload ``name`` as plain numpy columns
    (no package import: the reference arm encodes the same draws as reference
    ``Sample`` objects).  Labels ~ Bernoulli(0.3) (data.py:66); uniform or
    Zipf image keys; behavior_items / behavior_images share each sample's
    length (data.py:207-209)."""
    c = CONFIGS[name]
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        B = c["B"]
        if c["lengths"] == "lognormal":
            L = np.clip(np.round(rng.lognormal(np.log(40), 1.0, B)), 1, 500).astype(np.int64)
        else:
            L = np.full(B, c["L"], dtype=np.int64)
        off = np.zeros(B + 1, dtype=np.int32)
        np.cumsum(L, out=off[1:])
        R = int(off[-1])
        draw = (lambda k: _zipf_keys(rng, k, c["P"], c["zipf"])) if c["zipf"] else \
            (lambda k: rng.integers(0, c["P"], k))
        beh = draw(R).astype(np.int32)
        ad_img = draw(B).astype(np.int32)
        onehot, multi = {}, {}
        for f, v, m in fields_of(name):
            if m:
                multi[f] = (beh if f == "behavior_images" else rng.integers(0, v, R).astype(np.int32), off)
            else:
                onehot[f] = ad_img if f == "ad_image" else rng.integers(0, v, B).astype(np.int32)
        labels = (rng.random(B) < 0.3).astype(np.float32)
        out.append(dict(size=B, labels=labels, onehot=onehot, multihot=multi, ad_image_ids=ad_img,
                        beh_image_ids=beh, beh_off=off))
    return out


def make_batches(name, schema, n, seed):
    from paper_1711_06505_b200.batch import Batch
    return [Batch(**c) for c in gen_columns(name, n, seed)]


def pool_latents(name, seed=0):
    """The pool's float32 latents [P, 32], drawn exactly as ImagePool.synthetic
    draws them for an unsharded pool (torch CPU generator, seed)."""
    import torch
    gen = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randn((CONFIGS[name]["P"], 32), generator=gen, dtype=torch.float32).numpy()


def config_of(name, world):
    """The workload description: identical in both arms' JSON lines."""
    c = CONFIGS[name]
    B = c["B"]
    return {"workload": name, "description": DESC[name], "global_batch": world * B, "batch_per_gpu": B,
            "behaviors_per_user": c["L"] if c["lengths"] is None else "lognormal(ln 40, 1) clipped 1-500",
            "pool_images": c["P"], "id_table_rows": c["vocab"], "aggregator": c["kind"],
            "parallelism": f"AMS: pool + ID tables sharded over {world} GPU(s), dense dp{world}",
            "l2": "L2 flushed between timed steps (256 MB write outside each step's events)" if l2_flush(name)
            else "inputs larger than L2 (each step gathers ~U x 8-16 KB of distinct pool rows)"}


def l2_flush(name):
    """cfg1's whole pool (10k x 16 KB) is about the size of the 126 MB L2."""
    return CONFIGS[name]["P"] * 4096 * 4 < (1 << 30)


# ---------------------------------------------------------------------------
# The reference's own CPU implementation (baseline/_ref: the unmodified
# dicm package) on a bounded sample of the same workload.  Nothing of this
# repository's package or kernel library is imported on this path.
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
REF_TABLE_CAP = 1_000_000  # cfg5's 100M-row tables allocate O(V) dense grads per step on the CPU


def reference_step(name, cols, sample_b):
    """-> (step, kind, threads, n, note): ``step()`` runs the stock
    ``dicm.training.LocalTrainer.train_batch`` (training.py:66-91) on the first
    ``sample_b`` samples of ``cols``, with the stock ``ImageFeatureStore`` /
    ``FixedExtractor`` (images.py:48-101) over the benchmark pool's latents."""
    threads = os.cpu_count() or 1
    n = int(min(sample_b, cols["size"]))
    note = ""
    if not os.path.isdir(os.path.join(REF_DIR, "dicm")):
        return _oracle_port_step(name, cols, n) + (note,)
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import dicm.data as RD
    import dicm.images as RI
    import dicm.model as RM
    import dicm.training as RT
    c = CONFIGS[name]
    fields = []
    for f, v, m in fields_of(name):
        if v > REF_TABLE_CAP and f not in ("ad_image", "behavior_images"):
            v = REF_TABLE_CAP
            note = f"; ID tables capped at {REF_TABLE_CAP} rows on the CPU (ids drawn modulo the cap)"
        fields.append(RM.FieldSpec(f, v, m))
    schema = RM.FeatureSchema(fields=fields, d_id=12, d_raw=4096, d_img=12, b_max=b_max_of(name))
    store = RI.ImageFeatureStore(pool_latents(name))
    extractor = RI.FixedExtractor(0x5EED, 32, 4096)
    model = RM.DicmModel(schema, RM.AggregatorSpec(c["kind"]), extractor, seed=0)
    tr = RT.LocalTrainer(model, store, RT.TrainConfig(batch_size=n))
    vocab = {f.name: f.vocab for f in fields}
    samples = []
    off = cols["beh_off"]
    for i in range(n):
        kw = {f: int(v[i]) % vocab[f] for f, v in cols["onehot"].items()}
        for f, (fl, of) in cols["multihot"].items():
            kw[f] = [int(x) % vocab[f] for x in fl[of[i]:of[i + 1]]]
        kw["behavior_images"] = cols["beh_image_ids"][off[i]:off[i + 1]].tolist()
        samples.append(RD.Sample(label=int(cols["labels"][i]), day=0, **kw))
    return (lambda: tr.train_batch(samples)), "reference", threads, n, note


def _oracle_port_step(name, cols, n):
    """Fallback when baseline/_ref is absent: the oracle's restatement
    (oracle/dicm_oracle.py) of the same step, rows from numpy tanh(z R^T)."""
    from oracle import dicm_oracle as O
    from paper_1711_06505_b200.schema import AggregatorSpec, FeatureSchema, FieldSpec, ModelLayout, init_params
    threads = os.cpu_count() or 1
    kind = CONFIGS[name]["kind"]
    schema = FeatureSchema([FieldSpec(f, v, m) for f, v, m in fields_of(name)], d_id=12, d_raw=4096, d_img=12,
                           b_max=b_max_of(name))
    lay = ModelLayout(schema, AggregatorSpec(kind), (128, 64), True, True)
    params = init_params(lay, 0, include_tables=True)
    cfg = O.make_cfg(fields_of(name), b_max=schema.b_max, kind=kind)
    off = cols["beh_off"]
    R = int(off[n])
    ids = np.unique(np.concatenate([cols["ad_image_ids"][:n], cols["beh_image_ids"][:R]]).astype(np.int64))
    proj = np.random.default_rng(0x5EED).normal(0.0, 1.0 / np.sqrt(32), (4096, 32))
    rows = np.tanh(pool_latents(name)[ids].astype(np.float64) @ proj.T)
    ob = {"size": n, "labels": cols["labels"][:n].astype(np.float64),
          "onehot": {k: v[:n].astype(np.int64) for k, v in cols["onehot"].items()},
          "multihot": {k: (a[:R].astype(np.int64), o[:n + 1].astype(np.int64))
                       for k, (a, o) in cols["multihot"].items()},
          "ad_image_ids": np.searchsorted(ids, cols["ad_image_ids"][:n]),
          "beh_image_ids": np.searchsorted(ids, cols["beh_image_ids"][:R]), "beh_off": off[:n + 1].astype(np.int64)}
    tr = O.OracleTrainer(params, cfg, rows)
    return (lambda: tr.train_batch(ob)), "port", threads, n


def cpu_baseline(name, cols, max_seconds=25.0, sample_b=256):
    """The reference CPU step on this host's cores: 1 warm-up + up to 3 timed
    steps (median), bounded to ~``max_seconds``."""
    step, kind, threads, n, note = reference_step(name, cols, sample_b)
    t0 = time.perf_counter()
    step()
    times = []
    while True:
        a = time.perf_counter()
        step()
        times.append(time.perf_counter() - a)
        if time.perf_counter() - t0 > max_seconds or len(times) >= 3:
            break
    med = statistics.median(times)
    return {"value": n / med, "unit": "samples/s", "cores": threads, "kind": kind,
            "sample": f"first {n} samples of one {name} batch (same per-sample shape: L, pool, tables, aggregator), "
                      f"1 warm-up + median of {len(times)} steps of the stock dicm LocalTrainer.train_batch, f64, "
                      f"{threads} host threads{note}"}


def run_reference_arm(args):
    """The reference's own CPU implementation (the unmodified dicm package in
    baseline/_ref): W warm-up + K timed ``LocalTrainer.train_batch`` steps,
    each over a bounded slice of the same synthetic batch the GPU arm trains
    on.  Imports neither this repository's package nor its kernel library."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    world = max(world, args.gpus)
    name = args.config
    # torchrun sets OMP_NUM_THREADS=1 for every rank; rank 0 runs alone here,
    # so the reference's numpy/BLAS gets every host thread back
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:  # reported through the thread count in cpu_baseline
        pass
    cols = gen_columns(name, 1, seed=1000)[0]
    # ~10 ms of host work per sample at L = 200: size the slice so W + K steps take ~2.5 min
    per_sample = 0.01 * max(CONFIGS[name]["L"], 40) / 200.0
    sample_b = int(max(16, min(256, 150.0 / max(args.warmup + args.steps, 1) / per_sample)))
    step, kind, threads, n, note = reference_step(name, cols, sample_b)
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(max(args.steps, 1)):
        a = time.perf_counter()
        step()
        times.append(time.perf_counter() - a)
    med = statistics.median(times)
    v = n / med
    sample = (f"first {n} samples of the {name} batch per step (same per-sample shape as the GPU arm), "
              f"{args.warmup} warm-up + median of {len(times)} steps of the stock dicm LocalTrainer.train_batch, "
              f"f64, {threads} host threads{note}")
    line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * med, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_of(name, world), "sample_batch": n,
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "DICM train samples/sec (fwd+bwd)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="auto", choices=["auto", "fp32", "tf32", "bf16"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each step from a CUDA graph (auto: when every batch has the same layout)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus is authoritative: one process per GPU under torchrun
        import socket
        with socket.socket() as s_:
            s_.bind(("127.0.0.1", 0))
            port = s_.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))

    import torch
    import torch.distributed as dist
    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
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
    # up to 64 distinct batches, cycled (each step still gathers GBs of pool
    # rows, far beyond L2)
    distinct = make_batches(name, schema, min(args.warmup + args.steps, 64), seed=1000 + rank)
    batches = [distinct[i % len(distinct)] for i in range(args.warmup + args.steps)]
    staged_d = [eng.upload(b, own=True) for b in distinct]
    staged = [staged_d[i % len(staged_d)] for i in range(args.warmup + args.steps)]
    torch.cuda.synchronize()
    union = world * B
    same_layout = len({d.pk.signature() for d in staged_d}) == 1
    p2p_ok = world == 1 or getattr(eng, "exchange", "p2p") == "p2p"
    graphs = p2p_ok and (args.graph == "on" or (args.graph == "auto" and same_layout))
    cluster.use_graphs = graphs

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(db, eager=False):
        if graphs and not eager:
            eng.step_graphed(db, denominator=union)
            return
        eng.forward_backward(db, denominator=union)
        eng.optimizer_step(eng.lr())
        eng.iteration += 1

    for db in staged[:args.warmup]:
        step(db)
    barrier()
    from paper_1711_06505_b200 import _lib as LIB
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = l2_flush(name)
    if flush:
        # a step's inputs fit in L2: flush it (a 2 x L2 write) between timed
        # steps, outside each step's own pair of events
        junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in staged]
    with ClockSampler(local) as clk:
        barrier()
        start.record()
        if flush:
            for db, (a, b) in zip(staged[args.warmup:], evs):
                junk.fill_(1)
                a.record()
                step(db)
                b.record()
        else:
            for db in staged[args.warmup:]:
                step(db)
        end.record()
        barrier()
    ms = start.elapsed_time(end) if not flush else sum(a.elapsed_time(b) for a, b in evs[:args.steps])
    if os.environ.get("DICM_BENCH_NOCHECK") != "1":  # =1 only for timing-only measurement builds (scripts/)
        eng.raise_status()
    if os.environ.get("DICM_PHASE_TIMING") == "1" and hasattr(eng, "phase_times"):
        barrier()  # the ranks start the timed eager step together
        step(staged[-1], eager=True)
        pt = eng.phase_times()
        if rank == 0:
            print("phases(ms):", json.dumps({k: round(v, 3) for k, v in pt.items()}), flush=True)
    # per-kernel times: the library's own event probes on its stream, over a
    # few eager steps after the timed region (events are not graph nodes)
    LIB.check(LIB.lib.dicm_probe_enable(1))
    for db in staged[args.warmup:args.warmup + min(args.steps, 8)]:
        step(db, eager=True)
    barrier()
    probes = {k: LIB.probe_read(k) for k in LIB.PROBE_KERNELS}
    LIB.check(LIB.lib.dicm_probe_enable(0))
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
        t_cpu = time.perf_counter()
        # default: one call per iteration (the host packs step i+1 while the
        # device runs step i; measured 0.98 x value at cfg2); train_stream
        # (worker-thread packing) contends for the GIL and measured 0.85 (r2e)
        if os.environ.get("DICM_E2E_API", "batch") == "stream":
            for i, loss in enumerate(cluster.train_stream(host)):
                pinned_loss[i:i + 1].copy_(loss, non_blocking=True)
        else:  # one call per iteration, host side of step i+1 after step i is enqueued
            for i, b in enumerate(host):
                loss = cluster.train_batch_async(b, union)
                pinned_loss[i:i + 1].copy_(loss, non_blocking=True)
        t_cpu = time.perf_counter() - t_cpu
        e2_.record()
        barrier()
        ems = s2.elapsed_time(e2_)
        if os.environ.get("DICM_E2E_DEBUG") and rank == 0:
            print(f"e2e: cpu enqueue {1e3 * t_cpu / len(host):.3f} ms/step, device {ems / len(host):.3f} ms/step",
                  flush=True)
        eng.raise_status()
        te = torch.tensor([ems], device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        e2e = {"value": union * len(host) / (ems / 1000.0), "unit": "samples/s",
               "h2d_bytes_per_step": int(np.mean([eng.h2d_bytes(b) for b in host])), "d2h_bytes_per_step": 4,
               "api": "Cluster.train_batch_async per iteration (host CSR batch -> multithreaded pack into pinned "
                      "memory -> H2D on a copy stream, overlapping the previous step -> step -> loss D2H into "
                      "pinned memory)" if os.environ.get("DICM_E2E_API", "batch") != "stream" else
                      "Cluster.train_stream (worker-thread slice + pack, H2D on a copy stream, loss D2H)"}

    # roofline: per-kernel algorithmic bytes / flops over the
    # kernel times the library's own event probe measured on its stream
    U = int(eng.counts[2].item()) if world > 1 else int(eng.counts[0].item())
    last = batches[-1]
    R = int(last.beh_off[-1])
    width = model.layout.mlp_input_width()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    src = "MEASURED_PEAKS.json (measured)" if peaks else "B200_PROFILING.md fallback"
    hbm_peak = peaks.get("hbm_gbs", 6550.1)
    tc_peak = peaks.get("bf16_tflops_sustained", 1362.2) if precision == "bf16" else \
        peaks.get("bf16_tflops_sustained", 1362.2) / 2.0
    elem = 2 if precision == "bf16" else 4
    kern = kernel_work(U, B, R, width, schema.d_raw, elem, kind)
    table = {}
    for k, (nbytes, flops, sflops) in kern.items():
        t = probes.get(k) or []
        if not t:
            continue
        ms_k = statistics.mean(t)
        ideal = max(nbytes / (hbm_peak * 1e9), flops / (tc_peak * 1e12), sflops / (FP32_PEAK_TFLOPS * 1e12))
        table[k] = {"ms": ms_k, "launches": len(t), "alg_bytes": nbytes, "GB_s": nbytes / (ms_k / 1e3) / 1e9,
                    "flops": flops, "TFLOP_s": flops / (ms_k / 1e3) / 1e12,
                    "roofline_frac": ideal / (ms_k / 1e3)}
        if sflops:
            table[k].update({"fp32_flops": sflops, "fp32_TFLOP_s": sflops / (ms_k / 1e3) / 1e12,
                             "fp32_peak_TFLOP_s": FP32_PEAK_TFLOPS,
                             "bound": "fp32" if sflops / FP32_PEAK_TFLOPS / 1e12 > nbytes / hbm_peak / 1e9
                             else "hbm"})
    img = [k for k in table if k.startswith("img")]
    mlp_ms = sum(table[k]["ms"] for k in img)
    mlp_flops = sum(table[k]["flops"] for k in img)
    roof = None
    if "img_fwd_l0" in table:
        top = table["img_fwd_l0"]
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            ent = prof.get(f"{name}/{precision}/img_fwd_l0")
            if ent:
                # ncu's DRAM bytes for the captured launch, rescaled to this run's U
                traffic = ent["dram_bytes"] * U / ent["unique_images"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": "k_fwd4: pool-row gather + layer-0 tcgen05 GEMM on CTA pairs (dicm_imgmlp_fwd)",
                "achieved": top["GB_s"], "peak": hbm_peak, "unit": "GB/s", "frac": top["GB_s"] / hbm_peak,
                "traffic": traffic, "peak_source": src, "algorithmic_bytes_per_launch": top["alg_bytes"],
                "ms_per_launch": top["ms"], "unique_images_per_step": U,
                "tensor": {"image_mlp_TFLOP_s": mlp_flops / (mlp_ms / 1e3) / 1e12, "peak": tc_peak,
                           "frac": mlp_flops / (mlp_ms / 1e3) / 1e12 / tc_peak,
                           "peak_kind": "dense bf16 sustained" if precision == "bf16" else "tf32 = bf16/2",
                           "flops_per_unique_image": 4297216, "kernels": img},
                "kernels": table}
    if roof is not None:
        # whole-step roofline: sum over the step's components of
        # max(algorithmic bytes / HBM, tensor flops / TC), against the step time
        n_id = sum(len(v) for v in last.onehot.values()) + sum(len(f) for f, _ in last.multihot.values())
        K = int(eng.counts[3].item()) if world > 1 else int(eng.counts[1].item())
        Rimg = B + R
        comp = {k: max(kern[k][0] / (hbm_peak * 1e9), kern[k][1] / (tc_peak * 1e12)) for k in kern
                if k.startswith("img")}
        comp["dedup"] = (Rimg * 12 + U * 8 + n_id * 12 + K * 8) / (hbm_peak * 1e9)
        comp["pooling"] = sum(max(kern[k][0] / (hbm_peak * 1e9), kern[k][2] / (FP32_PEAK_TFLOPS * 1e12))
                              for k in ("sample_fwd", "sample_bwd"))
        comp["id_rows"] = (2 * n_id * (4 + 48) + K * 48 + K * (6 * 48 + 16)) / (hbm_peak * 1e9)
        comp["head"] = 2 * B * width * 4 / (hbm_peak * 1e9)
        comp["dense_adam"] = int(model.dense.numel()) * 20 / (hbm_peak * 1e9)
        t_roof = sum(comp.values())
        roof["step"] = {"roofline_ms": 1e3 * t_roof, "measured_ms": ms_step, "frac": 1e3 * t_roof / ms_step,
                        "components_ms": {k: round(1e3 * v, 4) for k, v in comp.items()},
                        "note": "per-GPU step; image MLP at max(bytes/HBM, flops/TC) per kernel, pooling at "
                                "max(bytes/HBM, attention FP32 flops/CUDA-core peak), the rest HBM-bound "
                                "(SURVEY.md 8d byte counts)",
                        "fp32_peak_TFLOP_s": FP32_PEAK_TFLOPS}
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(name, gen_columns(name, 1, seed=1000)[0])
        except Exception as ex:  # reported, never fatal
            cb = {"value": None, "error": repr(ex)[:200]}
    # kernel launches inside the timed region: the captured step graph's kernel
    # nodes (this library's only; NCCL / torch nodes excluded) x steps, or the
    # engine's per-call kernel sequence for eager steps
    kn, src = (eng.kernel_nodes(detail=True), "captured step graph") if graphs else (None, None)
    if kn is None:  # eager steps: one representative step captured (never replayed) and counted
        try:
            kn, src = eng.count_step_kernels(staged[-1], union), "one eager step captured for counting"
        except Exception as ex:  # e.g. the NCCL exchange (host syncs) cannot be captured
            src = f"uncounted: {ex!r}"[:120]
    launches = kn[0] * args.steps if kn else None
    launch_src = ({"own_kernels_per_step": kn[0], "cub_scan_kernels_per_step": kn[1],
                   "kernel_nodes_per_step": kn[2], "source": src} if kn else {"source": src})
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": precision, "data": "synthetic",
                "config": config_of(name, world),
                "precision": {"image_mlp_layer0": f"{precision} operands, fp32 accumulate (tcgen05)"
                              if precision != "fp32" else "fp32 CUDA cores",
                              "image_mlp_layers12": {"bf16": "bf16 operands (tcgen05 kind::f16), fp32 accumulate",
                                                     "tf32": "tf32 operands (tcgen05 kind::tf32), fp32 accumulate",
                                                     "fp32": "fp32 CUDA cores"}[precision],
                              "pooling_head_adam": "fp32 (BCE gradient in fp64)"},
                "cuda_graph": graphs,
                "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": launches, "gpu_launches_detail": launch_src,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dbg = os.environ.get("DICM_EXIT_DEBUG") == "1"
    if dbg:
        print(f"[rank {rank}] releasing graphs", flush=True)
    cluster.close()
    if world > 1:
        if dbg:
            print(f"[rank {rank}] destroy", flush=True)
        dist.destroy_process_group()
    if dbg:
        print(f"[rank {rank}] done", flush=True)


if __name__ == "__main__":
    main()
