"""Shared GPU-test helpers: build device models / pools from golden fixtures
and compare device state with the oracle or the fixtures."""

from __future__ import annotations

import numpy as np
import torch

import golden_io as G
from oracle import dicm_oracle as O


def device_model(m, pool_rows, pool_dtype="fp32", params=None):
    from paper_1711_06505_b200.model import DicmModel, PrerankModel
    from paper_1711_06505_b200.pool import ImagePool
    lay = G.layout_of(m)
    if lay.towers is not None:
        tw = lay.towers
        model = PrerankModel(G.full_schema(m), None, seed=m["seed"], user_fields=tw.user_fields,
                             ad_fields=tw.ad_fields, tower_hidden=tw.hidden, rep_dim=tw.rep,
                             use_images=lay.use_ad_image, params=params)
        return model, ImagePool.from_rows(pool_rows, dtype=pool_dtype)
    model = DicmModel(lay.schema, lay.aggregator, None, seed=m["seed"], mlp_widths=lay.mlp_widths,
                      use_ad_image=lay.use_ad_image, use_behavior_images=lay.use_behavior_images, params=params)
    pool = ImagePool.from_rows(pool_rows, dtype=pool_dtype)
    return model, pool


def dense_grads(engine):
    m = engine.model
    return {n: m.real_view(engine.grad, n).double().cpu().numpy() for n in m.dense_names}


def table_grads(engine):
    """{field: (ids, rows)} from the deduplicated row gradients."""
    keys = engine.unique_rows().astype(np.int64)
    rows = engine.d_rows[:len(keys), :engine.model.schema.d_id].double().cpu().numpy()
    out = {}
    for i, f in enumerate(engine.fields):
        lo = engine.bases[i]
        hi = lo + engine.model.tables[f.name].shape[0]
        sel = (keys >= lo) & (keys < hi)
        out[f.name] = (keys[sel] - lo, rows[sel])
    return out


def host_params(model):
    return {n: p.data for n, p in model.params.items()}


def oracle_batch(batch):
    """Product Batch -> oracle CSR dict."""
    return {
        "size": batch.size,
        "onehot": {f: v.astype(np.int64) for f, v in batch.onehot.items()},
        "multihot": {f: (fl.astype(np.int64), of.astype(np.int64)) for f, (fl, of) in batch.multihot.items()},
        "beh_image_ids": batch.beh_image_ids.astype(np.int64),
        "beh_off": batch.beh_off.astype(np.int64),
        "ad_image_ids": batch.ad_image_ids.astype(np.int64),
        "labels": batch.labels.astype(np.float64),
    }


def oracle_cfg_of(model):
    lay = model.layout
    s = lay.schema
    return O.make_cfg([(f.name, f.vocab, f.multi) for f in s.fields], d_id=s.d_id, d_raw=s.d_raw, d_img=s.d_img,
                      b_max=s.b_max, query_fields=s.query_fields, kind=lay.aggregator.kind,
                      normalize=lay.aggregator.normalize, hidden=lay.aggregator.attention_hidden,
                      mlp_widths=lay.mlp_widths, use_ad_image=lay.use_ad_image,
                      use_behavior_images=lay.use_behavior_images,
                      towers=None if lay.towers is None else dict(
                          user_fields=lay.towers.user_fields, ad_fields=lay.towers.ad_fields,
                          hidden=lay.towers.hidden, rep=lay.towers.rep))


def worst(a, b):
    return O.rel_err(a, b)


def cuda_ok():
    return torch.cuda.is_available()
