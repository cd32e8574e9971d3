"""Helpers to read the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import json
import os

import numpy as np

from paper_1711_06505_b200 import schema as S

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BIG = 50_000
PROBE_SEED = 1234

TINY = ["tiny_sum", "tiny_attn", "tiny_multiquery-attn", "tiny_max", "tiny_concat", "tiny_prerank"]
FULL = ["full_sum", "full_attn", "full_attn_raw", "full_mq", "full_sum_noad", "full_max", "full_concat",
        "full_prerank",
        "full_prerank_img_ids", "full_prerank_noimg"]


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def meta(fx):
    return json.loads(str(fx["meta"]))


def full_schema(m):
    """The case's schema with every field (a pre-rank layout keeps only the
    tower fields)."""
    fields = [S.FieldSpec(n, v, mu) for n, v, mu in m["fields"]]
    return S.FeatureSchema(fields=fields, d_id=m["d_id"], d_raw=m["d_raw"], d_img=m["d_img"],
                           b_max=m["b_max"], query_fields=tuple(m["query_fields"]))


def layout_of(m):
    schema = full_schema(m)
    if m.get("towers"):
        tw = m["towers"]
        return S.prerank_layout(schema, tuple(tw["user_fields"]), tuple(tw["ad_fields"]), tw["hidden"],
                                tw["rep"], m["use_ad_image"])
    agg = S.AggregatorSpec(m["kind"], attention_hidden=m["hidden"], normalize=m["normalize"])
    return S.ModelLayout(schema, agg, tuple(m["mlp_widths"]), m["use_ad_image"],
                         m["use_behavior_images"])


def oracle_cfg(m):
    from oracle.dicm_oracle import make_cfg
    return make_cfg(m["fields"], d_id=m["d_id"], d_raw=m["d_raw"], d_img=m["d_img"],
                    b_max=m["b_max"], query_fields=m["query_fields"], kind=m["kind"],
                    normalize=m["normalize"], hidden=m["hidden"], mlp_widths=m["mlp_widths"],
                    use_ad_image=m["use_ad_image"], use_behavior_images=m["use_behavior_images"],
                    towers=m.get("towers"))


def samples(fx, bi):
    """Sample-like dicts of batch ``bi`` (the reference's Sample fields)."""
    p = f"b{bi}"
    n = len(fx[f"{p}/user"])
    out = []
    for i in range(n):
        s = {k: int(fx[f"{p}/{k}"][i]) for k in
             ("user", "scenario", "ad", "ad_category", "ad_image", "label")}
        for k in ("behavior_items", "behavior_images"):
            off = fx[f"{p}/{k}/off"]
            s[k] = fx[f"{p}/{k}/flat"][off[i]:off[i + 1]].tolist()
        s["day"] = 0
        out.append(s)
    return out


def project(a):
    a = np.asarray(a, dtype=np.float64)
    rng = np.random.default_rng([PROBE_SEED, a.shape[0], a.shape[1]])
    pc = rng.standard_normal((a.shape[1], 4))
    pr = rng.standard_normal((4, a.shape[0]))
    return {"pr": a @ pc, "pl": pr @ a, "row0": a[0].copy(), "sum": a.sum(axis=0)}


def golden_view(fx, key, a):
    """(expected, actual) pairs for ``key``: direct or through projections."""
    a = np.asarray(a, dtype=np.float64)
    if key in fx:
        return [(fx[key], a)]
    pr = project(a)
    return [(fx[f"{key}#{k}"], pr[k]) for k in ("pr", "pl", "row0", "sum")]


def pool(fx):
    return fx["pool"]
