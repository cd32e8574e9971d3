"""Multi-GPU parity check (run under torchrun, one rank per GPU):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29517 scripts/cluster_check.py [kind] [precision] [eager|graphs]
        [--workers M] [--servers N] [--full-model] [--short-last] [--ckpt PATH]

The AMS cluster must match the single-process oracle on the union batch
(reference runtime.py:19-21, tests/test_runtime.py:46-59): loss per
iteration, forwards == union unique images, bit-identical image-net replicas
on every logical server, the assembled ``snapshot()`` (every parameter and
every ID-table row after Adam) and the assembled ``optimizer_tensors()``.

  --workers/--servers  logical topology (default: one of each per GPU);
  --full-model         pass the full (unsharded) model; ``collect_into_model``
                       must write the trained values back into it;
  --short-last         the last union batch is half a worker's batch: every
                       GPU but the first trains an empty slice (the
                       reference's final short batch, runtime.py:522-523);
  --ckpt PATH          after iteration 2 write a DCK1 checkpoint of the
                       cluster (collect_into_model + optimizer_tensors), then
                       run one more iteration and store its union batch and
                       results next to the checkpoint (PATH.npz) for the
                       single-GPU resume test.
Exits non-zero on a mismatch; rank 0 prints one JSON line.
"""
import argparse
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
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", nargs="?", default="multiquery-attn")
    ap.add_argument("precision", nargs="?", default="fp32")
    ap.add_argument("mode", nargs="?", default="eager", choices=["eager", "graphs"])
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--servers", type=int, default=0)
    ap.add_argument("--full-model", action="store_true")
    ap.add_argument("--short-last", action="store_true")
    ap.add_argument("--ckpt", default="")
    ap.add_argument("--zipf", type=float, default=0.0, help="Zipf image keys (hot keys: the chunked hot-key passes)")
    a = ap.parse_args()
    kind, precision = a.kind, a.precision
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from oracle import dicm_oracle as O
    import gpu_helpers as H
    from paper_1711_06505_b200 import checkpoint as CK
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.model import DicmModel, PrerankModel
    from paper_1711_06505_b200.pool import FixedExtractor, ImagePool
    from paper_1711_06505_b200.runtime import Cluster, ClusterConfig
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema, init_params, ModelLayout, prerank_layout

    M = a.workers or world
    N = a.servers or world
    P, bpw, iters = 2000, 96 * world // M, 3
    schema = default_schema(3001, 4, 2999, 8, P, b_max=30)
    shard = None if a.full_model else (world, rank)
    if kind == "prerank":  # two-tower pre-rank model (reference model.py:420-531)
        full = init_params(prerank_layout(schema), 0)
        model = PrerankModel(schema, None, seed=0, shard=shard)
    else:
        agg = AggregatorSpec(kind)
        full = init_params(ModelLayout(schema, agg, (128, 64), True, True), 0)
        model = DicmModel(schema, agg, None, seed=0, shard=shard)
    gen = torch.Generator().manual_seed(11)
    lat = torch.randn((P, 32), generator=gen)
    ext = FixedExtractor(0x5EED, 32, 4096)
    pdt = "bf16" if precision == "bf16" else "fp32"
    pool = ImagePool.from_latents(lat, ext, dtype=pdt, world=world, rank=rank)
    full_rows = ImagePool.from_latents(lat, ext, dtype=pdt).rows.double().cpu().numpy()
    cl = Cluster(ClusterConfig(workers=M, servers=N, batch_per_worker=bpw), model, pool, precision=precision)
    cl.use_graphs = a.mode == "graphs"  # steps 2.. replay a captured CUDA graph
    rng = np.random.default_rng(5)
    U = M * bpw
    sizes = [U] * iters
    if a.short_last:
        sizes[-1] = bpw // 2  # only worker 0 gets samples: every other GPU trains an empty slice
    unions = [synthetic_batch(rng, schema, n, rng.integers(0, 31, n), P, zipf=a.zipf or None) for n in sizes]
    out = []
    for i, u in enumerate(unions):
        out.append(cl.run_iteration(u, digests=True))
        if a.ckpt and i == 1:
            src = cl.collect_into_model() if a.full_model else None
            opt = cl.optimizer_tensors()
            snap = cl.snapshot()
            if rank == 0:
                if src is None:  # a sharded source model: build a full host-side view to save
                    src = type("Snap", (), {})()
                    src.params = {n: type("P", (), {"data": v})() for n, v in snap.items()}
                CK.save(a.ckpt, src, optimizer=opt, meta={"world": world, "iteration": cl.iteration})
    if a.ckpt and rank == 0:
        u = unions[2]
        np.savez(a.ckpt + ".npz", loss=out[2][0], size=u.size, labels=u.labels, ad=u.ad_image_ids,
                 beh=u.beh_image_ids, beh_off=u.beh_off,
                 **{f"oh/{k}": v for k, v in u.onehot.items()},
                 **{f"mh/{k}/flat": fl for k, (fl, of) in u.multihot.items()},
                 **{f"mh/{k}/off": of for k, (fl, of) in u.multihot.items()})
    snap = cl.snapshot()
    opt = cl.optimizer_tensors()
    if a.full_model:
        back = cl.collect_into_model()
        assert back is model
        if rank == 0:
            for n, v in model.snapshot().items():
                assert np.array_equal(v, snap[n].astype(np.float32).astype(np.float64)), n
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
            ok &= len(out[i][3]) == N and len(set(out[i][3])) == 1  # one bit-identical replica per server
        worst = {}
        for n, av in tr.p.items():
            got = snap[n]
            ok &= got.shape == av.shape
            d = np.abs(got - av) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(av)))
            noise = n.startswith("attn/") and n.endswith("/1/b")
            frac_bad = float((d > tol).mean())
            worst[n] = float(d.max())
            lim = 2.5 * 0.001 * iters
            ok &= (d.max() <= lim + 1e-6) if noise else (frac_bad <= 0.05 and d.max() <= lim + tol)
        # optimizer state: step counters exact, moments close (Adam state of the
        # oracle trainer: dense per name, tables per row)
        t_ok = True
        for n in tr.dense:
            t_ok &= int(opt[f"{n}#t"]) == tr.state[n]["t"] or (n.startswith("attn/") and n.endswith("/1/b"))
        for name, _v, _m in cfg["fields"]:
            st = tr.tstate[name]
            t_ok &= np.array_equal(opt[f"id_emb/{name}#t"], st["t"])
            t_ok &= O.rel_err(opt[f"id_emb/{name}#m"], st["m"]) < max(tol, 1e-3)
        ok &= t_ok
        report["opt_t_ok"] = bool(t_ok)
        if a.mode == "graphs":
            # every kernel node of the captured step: this library's, the CUB
            # sorts of dicm_ref_transpose, and the one NCCL all-reduce
            own, cub, total = cl.engine.kernel_nodes(detail=True)
            report["graph_nodes"] = {"own": own, "cub": cub, "total": total}
            ok &= total - own - cub <= 1
        report["worst"] = max(worst.values())
        report["worst_param"] = max(worst, key=worst.get)
        print(json.dumps({"ok": bool(ok), "world": world, "workers": M, "servers": N, "kind": kind,
                          "precision": precision, "mode": a.mode, "full_model": a.full_model, **report}), flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    cl.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
