"""Two-tower pre-rank model on the B200 (reference
PrerankModel, model.py:420-531): the device step against the oracle at
benchmark-like shapes, forward scoring against the reference's golden
vectors, and the reference's own pre-rank properties
(tests/test_model.py:236-273).  The golden step-0 / two-step training parity
of the pre-rank cases runs with the other golden cases in test_gpu_step.py.
fp32 tolerance 1e-4 (metric |a-b| / max(1,|a|,|b|))."""

import numpy as np
import pytest
import torch

import golden_io as G
import gpu_helpers as H
from oracle import dicm_oracle as O

pytestmark = pytest.mark.gpu
FP32_TOL = 1e-4


def _prerank(B=256, L=50, P=3000, vocab=20_000, seed=0, **kw):
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.model import PrerankModel
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.schema import default_schema
    schema = default_schema(vocab, 4, vocab, 8, P, b_max=max(L, 1))
    model = PrerankModel(schema, None, seed=seed, **kw)
    pool = ImagePool.synthetic(P, seed=seed)
    batch = synthetic_batch(np.random.default_rng(seed), schema, B, L, P)
    return model, pool, batch


CASES = {
    "default": {},
    "no_images": dict(use_images=False),
    "image_id_fields_max_width": dict(user_fields=("behavior_images", "user", "behavior_items", "scenario"),
                                      ad_fields=("ad_image", "ad", "ad_category", "user"), tower_hidden=128,
                                      rep_dim=64),
    "narrow": dict(user_fields=("user",), ad_fields=("ad",), tower_hidden=6, rep_dim=5),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_prerank_step_matches_oracle(case):
    from paper_1711_06505_b200.engine import StepEngine
    model, pool, batch = _prerank(**CASES[case])
    params = H.host_params(model)
    e = StepEngine(model, pool, "fp32")
    loss = e.forward_backward(e.upload(batch))
    torch.cuda.synchronize()
    e.raise_status()
    out = O.forward_backward(params, H.oracle_cfg_of(model), H.oracle_batch(batch), pool.rows.double().cpu().numpy())
    if model.use_images:
        assert np.array_equal(e.unique_images(), out["uniq"])
    assert O.rel_err(loss.item(), out["loss"]) < FP32_TOL
    assert O.rel_err(e.logits[:batch.size].cpu().numpy(), out["logits"]) < FP32_TOL
    for n, g in H.dense_grads(e).items():
        assert O.rel_err(g, out["grads"][n]) < FP32_TOL, n
    for f, (ids, rows) in H.table_grads(e).items():
        u, r = out["tgrads"][f]
        assert np.array_equal(ids, u), f
        assert O.rel_err(rows, r) < FP32_TOL, f


@pytest.mark.parametrize("name", ["full_prerank", "full_prerank_img_ids", "full_prerank_noimg"])
def test_forward_prerank_matches_reference(name):
    from paper_1711_06505_b200.inference import forward_prerank
    fx = G.load(name)
    model, pool = H.device_model(G.meta(fx), G.pool(fx))
    probs, z = forward_prerank(model, G.samples(fx, 0), pool)
    assert O.rel_err(z, fx["s0/logits"]) < FP32_TOL
    np.testing.assert_allclose(probs, 1.0 / (1.0 + np.exp(-fx["s0/logits"])), rtol=1e-4, atol=1e-6)


def test_swapping_ads_reorders_scores():
    """reference tests/test_model.py:261-273: scores follow their samples."""
    from paper_1711_06505_b200.inference import forward_prerank
    fx = G.load("full_prerank")
    model, pool = H.device_model(G.meta(fx), G.pool(fx))
    s = G.samples(fx, 0)
    _, z = forward_prerank(model, s, pool)
    _, z_rev = forward_prerank(model, s[::-1], pool)
    np.testing.assert_allclose(z, z_rev[::-1], rtol=1e-6, atol=1e-7)


def test_prerank_training_loss_decreases():
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    model, pool, batch = _prerank(B=128, L=20, P=800)
    tr = LocalTrainer(model, pool, TrainConfig(lr0=0.003))
    losses = [tr.train_batch(batch) for _ in range(30)]
    assert np.mean(losses[-5:]) < np.mean(losses[:5]) - 0.05


def test_prerank_graphed_steps_match_eager():
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    runs = []
    for graphs in (False, True):
        model, pool, batch = _prerank(B=96, L=12, P=500)
        tr = LocalTrainer(model, pool, TrainConfig(lr0=1e-4))
        tr.engine.use_graphs = graphs
        runs.append(([tr.train_batch(batch) for _ in range(4)], model.snapshot()))
    (l0, s0), (l1, s1) = runs
    np.testing.assert_allclose(l1, l0, rtol=1e-4, atol=1e-6)
    for n in s0:
        d = np.abs(s1[n] - s0[n])
        assert (d > 1e-5 * np.abs(s0[n]) + 1e-6).mean() <= 1e-3 and d.max() <= 8e-4, n


def test_prerank_checkpoint_round_trip(tmp_path):
    from paper_1711_06505_b200 import checkpoint as ck
    from paper_1711_06505_b200.training import LocalTrainer
    model, pool, batch = _prerank(B=64, L=10, P=400)
    tr = LocalTrainer(model, pool)
    tr.train_batch(batch)
    path = tmp_path / "p.ckpt"
    ck.save(path, model, tr, meta={"model_type": "prerank"})
    fresh, _, _ = _prerank(B=64, L=10, P=400, seed=3)
    ck.load_warmup(path, fresh, ck.WarmupMask.full(), fresh_seed=0)
    a, b = model.snapshot(), fresh.snapshot()
    assert sorted(a) == sorted(b)
    for n in a:
        assert np.array_equal(a[n], b[n]), n
    assert {g for g in ck.load(path).groups} == {"id-embeddings", "image-embedding-model", "mlp"}
