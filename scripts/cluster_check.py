"""Multi-GPU parity check (run under torchrun, one rank per GPU):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29517 scripts/cluster_check.py [kind] [precision]

The AMS cluster (workers = servers = world) must match the single-process
oracle on the union batch (reference runtime.py:19-21): loss per iteration,
dense parameters (identical on every rank) and every ID-table row after Adam.
Exits non-zero on a mismatch; rank 0 prints one JSON line.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "multiquery-attn"
    precision = sys.argv[2] if len(sys.argv) > 2 else "fp32"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from oracle import dicm_oracle as O
    import gpu_helpers as H
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.model import DicmModel, PrerankModel
    from paper_1711_06505_b200.pool import FixedExtractor, ImagePool
    from paper_1711_06505_b200.runtime import Cluster, ClusterConfig
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema, init_params, ModelLayout, prerank_layout

    P, bpw, iters = 2000, 96, 3
    schema = default_schema(3001, 4, 2999, 8, P, b_max=30)
    if kind == "prerank":  # two-tower pre-rank model (reference model.py:420-531)
        full = init_params(prerank_layout(schema), 0)
        model = PrerankModel(schema, None, seed=0, shard=(world, rank))
    else:
        agg = AggregatorSpec(kind)
        full = init_params(ModelLayout(schema, agg, (128, 64), True, True), 0)
        model = DicmModel(schema, agg, None, seed=0, shard=(world, rank))
    gen = torch.Generator().manual_seed(11)
    lat = torch.randn((P, 32), generator=gen)
    ext = FixedExtractor(0x5EED, 32, 4096)
    pdt = "bf16" if precision == "bf16" else "fp32"
    pool = ImagePool.from_latents(lat, ext, dtype=pdt, world=world, rank=rank)
    full_rows = ImagePool.from_latents(lat, ext, dtype=pdt).rows.double().cpu().numpy()
    cl = Cluster(ClusterConfig(workers=world, servers=world, batch_per_worker=bpw), model, pool, precision=precision)
    graphs = len(sys.argv) > 3 and sys.argv[3] == "graphs"
    cl.use_graphs = graphs  # steps 2.. replay a captured CUDA graph
    rng = np.random.default_rng(5)
    lengths = rng.integers(0, 31, world * bpw)
    unions = [synthetic_batch(rng, schema, world * bpw, lengths, P) for _ in range(iters)]
    out = [cl.run_iteration(u, digests=True) for u in unions]
    # gather every rank's table shard
    snap = cl.snapshot()
    tables = {}
    for f in model.layout.schema.fields:
        t = torch.as_tensor(snap[f"id_emb/{f.name}"], device="cuda")
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        full_t = np.zeros((f.vocab, 12))
        for r in range(world):
            rows = parts[r].cpu().numpy()
            n = len(range(r, f.vocab, world))
            full_t[r::world] = rows[:n]
        tables[f.name] = full_t
    ok = True
    report = {}
    if rank == 0:
        cfg = H.oracle_cfg_of(model)
        tr = O.OracleTrainer(full, cfg, full_rows)
        tol = 1e-4 if precision == "fp32" else 2e-2
        for i, u in enumerate(unions):
            ref = tr.train_batch(H.oracle_batch(u))
            report[f"loss{i}"] = [out[i][0], float(ref["loss"])]
            ok &= O.rel_err(out[i][0], ref["loss"]) < tol
            ok &= out[i][1] == out[i][2] == len(ref["uniq"])   # forwards == union unique
            ok &= len(set(out[i][3])) == 1                    # bit-identical replicas
        worst = {}
        for n, a in tr.p.items():
            got = tables[n[len("id_emb/"):]] if n.startswith("id_emb/") else snap[n]
            d = np.abs(got - a) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(a)))
            noise = n.startswith("attn/") and n.endswith("/1/b")
            frac_bad = float((d > tol).mean())
            worst[n] = float(d.max())
            lim = 2.5 * 0.001 * iters
            ok &= (d.max() <= lim + 1e-6) if noise else (frac_bad <= 0.05 and d.max() <= lim + tol)
        report["worst"] = max(worst.values())
        report["worst_param"] = max(worst, key=worst.get)
        print(json.dumps({"ok": bool(ok), "world": world, "kind": kind, "precision": precision,
                          "graphs": graphs, **report}), flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    cl.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
