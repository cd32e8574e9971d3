"""Inference export + KV predictor on the device,
pinned like the reference's own tests (tests/test_inference.py:18-61):
the exported table equals the live embedding bit for bit, the predictor
equals the full model's forward, cold ids score through the live net, and the
logits agree with the f64 oracle at the fp32 tolerance."""
import numpy as np
import pytest
import torch

import gpu_helpers as H
from oracle import dicm_oracle as O

pytestmark = pytest.mark.gpu


def _trained(kind="multiquery-attn", P=600, steps=3):
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    schema = default_schema(900, 4, 900, 8, P + 10, b_max=16)  # image-ID vocab covers cold ids
    model = DicmModel(schema, AggregatorSpec(kind), None, seed=0)
    pool = ImagePool.synthetic(P, seed=1)
    rng = np.random.default_rng(2)
    tr = LocalTrainer(model, pool, TrainConfig(lr0=0.003))
    for _ in range(steps):
        tr.train_batch(synthetic_batch(rng, schema, 64, 16, P))
    test = synthetic_batch(rng, schema, 80, rng.integers(0, 17, 80), P)
    return schema, model, pool, test


@pytest.mark.parametrize("kind", ["sum", "multiquery-attn"])
def test_table_lookup_bit_equal_to_live_embedding(kind):
    from paper_1711_06505_b200.engine import StepEngine
    from paper_1711_06505_b200.inference import export_inference
    schema, model, pool, test = _trained(kind)
    table = export_inference(model, pool)
    assert len(table) == len(pool)
    e = StepEngine(model, pool, "fp32")
    e.forward_backward(e.upload(test))
    U = int(e.counts[0].item())
    ids = e.uniq_img[:U].long()
    assert torch.equal(table.device()[ids], e.emb[:U])


def test_kv_predictor_matches_full_model_and_oracle():
    from paper_1711_06505_b200.inference import KvPredictor, export_inference, predict_logits
    schema, model, pool, test = _trained()
    probs, logits = KvPredictor(model, export_inference(model, pool), pool).predict(test)
    full = predict_logits(model, test, pool)
    assert np.array_equal(logits, full)  # same kernels, same embeddings
    assert np.all((probs > 0) & (probs < 1))
    params = H.host_params(model)
    ref = O.forward_backward(params, H.oracle_cfg_of(model), H.oracle_batch(test), pool.rows.double().cpu().numpy())
    assert O.rel_err(logits, ref["logits"]) < 1e-4


def test_cold_image_id_scores_via_live_path():
    from paper_1711_06505_b200.inference import KvPredictor, export_inference, predict_logits
    from paper_1711_06505_b200.pool import ImagePool
    schema, model, pool, test = _trained()
    table = export_inference(model, pool)
    # the pool grows after export: three fresh rows beyond the table
    extra = ImagePool.synthetic(3, seed=9).rows
    grown = ImagePool.from_rows(torch.cat([pool.rows, extra]).cpu().numpy())
    cold = test.slice(0, 4)
    cold.ad_image_ids[:] = len(pool)  # beyond the exported table
    probs, logits = KvPredictor(model, table, grown).predict(cold)
    assert np.all(np.isfinite(logits)) and np.all((probs > 0) & (probs < 1))
    assert np.array_equal(logits, predict_logits(model, cold, grown))
