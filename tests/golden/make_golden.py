"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is importable there, not on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For each case this builds a reference ``DicmModel`` (reference model.py:266),
feeds it seeded samples through ``encode_batch`` (model.py:158), records the
step-0 forward (``batch_loss_graph``, training.py:39) and its tape gradients
(``autograd.backward``, autograd.py:73), then trains two steps with
``LocalTrainer.train_batch`` (training.py:66) and records the losses and the
parameters / optimizer state afterwards.  The image store is duck-typed so the
reference consumes exactly the pool rows saved in the fixture (SURVEY.md 8c,
"input parity rule").  Large arrays are stored as fixed random projections
(see ``project``) to keep fixtures small; tests recompute the same projections.

The outputs are committed under tests/golden/*.npz.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("DICM_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from dicm import autograd as ag  # noqa: E402
from dicm.data import Sample  # noqa: E402
from dicm.images import FixedExtractor  # noqa: E402
from dicm.model import (AggregatorSpec, DicmModel, FeatureSchema, FieldSpec, PrerankModel,  # noqa: E402
                        encode_batch)
from dicm.runtime import Cluster, ClusterConfig  # noqa: E402
from dicm.training import LocalTrainer, TrainConfig, batch_loss_graph  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
BIG = 50_000
PROBE_SEED = 1234


def project(a):
    """Projections used for arrays with more than BIG elements."""
    a = np.asarray(a, dtype=np.float64)
    rng = np.random.default_rng([PROBE_SEED, a.shape[0], a.shape[1]])
    pc = rng.standard_normal((a.shape[1], 4))
    pr = rng.standard_normal((4, a.shape[0]))
    return {"pr": a @ pc, "pl": pr @ a, "row0": a[0].copy(), "sum": a.sum(axis=0)}


def put(store, key, a):
    a = np.asarray(a, dtype=np.float64)
    if a.size > BIG:
        for k, v in project(a).items():
            store[f"{key}#{k}"] = v
    else:
        store[key] = a


class PoolStore:
    """Duck-typed ImageFeatureStore returning fixed rows (images.py:99-101)."""

    def __init__(self, rows):
        self.rows = rows

    def __len__(self):
        return self.rows.shape[0]

    def raw_features(self, ids, extractor):
        ids = np.asarray(ids, dtype=np.int64)
        return self.rows[ids].astype(np.float64)


def make_samples(rng, n, vocabs, n_images, l_max, empty_every=7):
    out = []
    for i in range(n):
        L = 0 if (i % empty_every == 3) else int(rng.integers(1, l_max + 1))
        items = rng.integers(0, vocabs["behavior_items"], size=L).tolist()
        imgs = rng.integers(0, n_images, size=L).tolist()
        out.append(Sample(
            user=int(rng.integers(0, vocabs["user"])),
            scenario=int(rng.integers(0, vocabs["scenario"])),
            ad=int(rng.integers(0, vocabs["ad"])),
            ad_category=int(rng.integers(0, vocabs["ad_category"])),
            ad_image=int(rng.integers(0, n_images)),
            behavior_items=items, behavior_images=imgs,
            label=int(rng.random() < 0.3), day=0))
    return out


def samples_to_arrays(prefix, samples, store):
    keys = ["user", "scenario", "ad", "ad_category", "ad_image", "label"]
    for k in keys:
        store[f"{prefix}/{k}"] = np.array([getattr(s, k) for s in samples], dtype=np.int64)
    for k in ("behavior_items", "behavior_images"):
        lists = [getattr(s, k) for s in samples]
        off = np.zeros(len(lists) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(x) for x in lists])
        store[f"{prefix}/{k}/flat"] = np.array([i for x in lists for i in x], dtype=np.int64)
        store[f"{prefix}/{k}/off"] = off


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def build(case):
    fields = [FieldSpec(n, v, m) for n, v, m in case["fields"]]
    schema = FeatureSchema(fields=fields, d_id=case["d_id"], d_raw=case["d_raw"],
                           d_img=case["d_img"], b_max=case["b_max"],
                           query_fields=tuple(case["query_fields"]))
    ext = FixedExtractor(seed=7, latent_dim=4, out_dim=case["d_raw"])
    if case.get("towers"):  # two-tower pre-rank (reference model.py:420-531)
        tw = case["towers"]
        return PrerankModel(schema, ext, seed=case["seed"], user_fields=tuple(tw["user_fields"]),
                            ad_fields=tuple(tw["ad_fields"]), tower_hidden=tw["hidden"],
                            rep_dim=tw["rep"], use_images=case["use_ad_image"])
    agg = AggregatorSpec(case["kind"], attention_hidden=case["hidden"],
                         normalize=case["normalize"])
    return DicmModel(schema, agg, ext, seed=case["seed"], mlp_widths=tuple(case["mlp_widths"]),
                     use_ad_image=case["use_ad_image"],
                     use_behavior_images=case["use_behavior_images"])


def run_case(name, case, pool, batches, union_cluster=None):
    out = {"meta": np.array(json.dumps(case))}
    out["pool"] = pool
    store = PoolStore(pool)
    for bi, samples in enumerate(batches):
        samples_to_arrays(f"b{bi}", samples, out)

    model = build(case)
    out["init_digest"] = np.array(json.dumps({n: digest(p.data) for n, p in model.params.items()}))

    # step-0 forward + tape gradients
    batch = encode_batch(batches[0], model)
    for p in model.params.values():
        p.grad = None
    img = model.local_image_matrix(batch, store)
    loss, logits = batch_loss_graph(model, batch, img, model.local_id_rows, batch.size)
    ag.backward(loss)
    out["s0/loss"] = np.array(float(loss.data))
    out["s0/logits"] = logits.data.copy()
    out["s0/unique_images"] = batch.unique_images.copy()
    out["s0/E"] = img.data.copy()
    out["s0/dE"] = img.grad.copy() if img.grad is not None else np.zeros_like(img.data)
    for n, p in model.params.items():
        g = p.grad if p.grad is not None else np.zeros_like(p.data)
        if n.startswith("id_emb/"):
            f = n[len("id_emb/"):]
            u = batch.unique_field_ids(f)
            out[f"s0/tgrad/{f}/ids"] = u
            out[f"s0/tgrad/{f}/rows"] = g[u]
        else:
            put(out, f"s0/grad/{n}", g)

    # two LocalTrainer steps from a fresh model
    model = build(case)
    trainer = LocalTrainer(model, store, TrainConfig(batch_size=len(batches[0]), seed=0))
    losses = [trainer.train_batch(b) for b in batches]
    out["train/losses"] = np.array(losses)
    for n, p in model.params.items():
        put(out, f"train/after/{n}", p.data)
    for n, st in trainer.dense_state.items():
        out[f"train/t/{n}"] = np.array(st.t)
    for f, st in trainer.table_state.items():
        out[f"train/tt/{f}"] = st.t.copy()

    if union_cluster is not None:
        workers, servers = union_cluster
        model = build(case)
        per = len(batches[0]) // workers
        cl = Cluster(ClusterConfig(workers=workers, servers=servers, batch_per_worker=per),
                     model, store)
        closs = [cl.run_iteration(b)[0] for b in batches]
        out["cluster/losses"] = np.array(closs)
        snap = cl.snapshot()
        for n in model.params:
            put(out, f"cluster/after/{n}", snap[n])
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: losses {losses}  -> {os.path.relpath(path)} "
          f"({os.path.getsize(path) / 1e6:.2f} MB)")


def tiny_case(kind):
    # the reference's own tiny fixture dims (tests/conftest.py:9-34)
    return dict(fields=[["user", 5, False], ["ad", 7, False]], d_id=3, d_raw=8, d_img=4,
                b_max=4, query_fields=["ad"], kind=kind, normalize=True, hidden=5,
                mlp_widths=[6, 4], use_ad_image=True, use_behavior_images=True, seed=1)


def full_case(kind, normalize=True, use_ad_image=True, seed=0):
    vocabs = {"user": 50, "scenario": 4, "ad": 60, "ad_category": 8, "behavior_items": 60}
    fields = [["user", 50, False], ["scenario", 4, False], ["ad", 60, False],
              ["ad_category", 8, False], ["behavior_items", 60, True],
              ["ad_image", 40, False], ["behavior_images", 40, True]]
    return dict(fields=fields, d_id=12, d_raw=4096, d_img=12, b_max=16,
                query_fields=["ad", "ad_category"], kind=kind, normalize=normalize, hidden=32,
                mlp_widths=[128, 64], use_ad_image=use_ad_image, use_behavior_images=True,
                seed=seed), vocabs


def prerank_case(base, user_fields=("user", "behavior_items"), ad_fields=("ad", "ad_category"),
                 hidden=64, rep=16, use_images=True):
    case = dict(base)
    case.update(kind="sum", use_ad_image=use_images, use_behavior_images=use_images,
                towers=dict(user_fields=list(user_fields), ad_fields=list(ad_fields), hidden=hidden,
                            rep=rep))
    return case


def main():
    # tiny dims: pool rows straight from the reference extractor
    rng = np.random.default_rng(99)
    latents = rng.standard_normal((10, 6)).astype(np.float32)
    tiny_pool = FixedExtractor(seed=42, latent_dim=6, out_dim=8).extract(latents)
    trng = np.random.default_rng(5)
    tiny_batches = []
    for _ in range(2):
        bs = make_samples(trng, 6, {"user": 5, "scenario": 1, "ad": 7, "ad_category": 1,
                                    "behavior_items": 1}, 10, 6, empty_every=4)
        tiny_batches.append(bs)
    for kind in ("sum", "attn", "multiquery-attn", "max", "concat"):
        if os.environ.get("GOLDEN_ONLY") and f"tiny_{kind}" not in os.environ["GOLDEN_ONLY"].split(","):
            continue
        run_case(f"tiny_{kind}", tiny_case(kind), tiny_pool, tiny_batches)
    if not os.environ.get("GOLDEN_ONLY") or "tiny_prerank" in os.environ["GOLDEN_ONLY"].split(","):
        # the reference test's pre-rank schema (tests/test_model.py:236-247)
        case = prerank_case(dict(tiny_case("sum"), fields=[["user", 5, False], ["ad", 7, False],
                                                           ["ad_category", 3, False],
                                                           ["behavior_items", 9, True]]),
                            hidden=6, rep=5)
        run_case("tiny_prerank", case, tiny_pool, tiny_batches)

    # full dims (4096 -> 256 -> 64 -> 12), fp32 pool rows = tanh(z R^T)
    prng = np.random.default_rng(2024)
    z = prng.standard_normal((40, 32))
    R = prng.normal(0.0, 1.0 / np.sqrt(32), (4096, 32))
    full_pool = np.tanh(z @ R.T).astype(np.float32)
    for kind, norm, use_ad, tag in (("sum", True, True, "sum"), ("attn", True, True, "attn"),
                                    ("attn", False, True, "attn_raw"),
                                    ("multiquery-attn", True, True, "mq"),
                                    ("sum", True, False, "sum_noad"), ("max", True, True, "max"),
                                    ("concat", True, True, "concat")):
        if os.environ.get("GOLDEN_ONLY") and f"full_{tag}" not in os.environ["GOLDEN_ONLY"].split(","):
            continue
        case, vocabs = full_case(kind, norm, use_ad)
        brng = np.random.default_rng(len(tag) * 1009 + ord(tag[-1]))
        batches = [make_samples(brng, 24, vocabs, 40, 20) for _ in range(2)]
        cluster = (2, 2) if tag in ("mq", "sum") else None
        run_case(f"full_{tag}", case, full_pool, batches, union_cluster=cluster)
    for tag, kw in (("prerank", {}),
                    ("prerank_img_ids", dict(user_fields=("behavior_images", "user", "behavior_items"),
                                             ad_fields=("ad_image", "ad_category", "ad"), hidden=32, rep=8)),
                    ("prerank_noimg", dict(use_images=False))):
        if os.environ.get("GOLDEN_ONLY") and f"full_{tag}" not in os.environ["GOLDEN_ONLY"].split(","):
            continue
        base, vocabs = full_case("sum")
        case = prerank_case(base, **kw)
        brng = np.random.default_rng(len(tag) * 1013 + ord(tag[-1]))
        batches = [make_samples(brng, 24, vocabs, 40, 20) for _ in range(2)]
        run_case(f"full_{tag}", case, full_pool, batches,
                 union_cluster=(2, 2) if tag == "prerank" else None)


if __name__ == "__main__":
    main()
