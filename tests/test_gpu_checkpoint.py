"""DCK1 checkpoints of the device state, pinned like
the reference's tests/test_checkpoint.py:19-119 plus byte compatibility with
files the reference itself writes (tests/golden/ckpt_hashes.json, made by
tests/golden/make_ckpt_golden.py)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ckpt_hashes.json")))


def _model(kind, seed, users=300, scen=4, ads=200, cats=8, images=96, b_max=12):
    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema
    return DicmModel(default_schema(users, scen, ads, cats, images, b_max=b_max), AggregatorSpec(kind), None,
                     seed=seed)


def _trained(tmp_path, kind="multiquery-attn", seed=1, steps=4):
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    model = _model(kind, seed)
    pool = ImagePool.synthetic(96, seed=2)
    tr = LocalTrainer(model, pool, TrainConfig(lr0=0.003))
    rng = np.random.default_rng(3)
    batches = [synthetic_batch(rng, model.schema, 32, 8, 96) for _ in range(steps + 1)]
    for b in batches[:steps]:
        tr.train_batch(b)
    return model, pool, tr, batches[steps]


def _sha(p):
    return hashlib.sha256(open(p, "rb").read()).hexdigest()


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c[0]}-seed{c[7]}")
def test_writer_reproduces_reference_bytes(tmp_path, case):
    from paper_1711_06505_b200.checkpoint import load, save
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    kind, users, scen, ads, cats, images, b_max, seed, meta = case
    model = _model(kind, seed, users, scen, ads, cats, images, b_max)
    p = tmp_path / "x.ckpt"
    save(p, model, meta=meta)
    assert _sha(p) == GOLD[f"{kind}/seed{seed}/params"]
    tr = LocalTrainer(model, ImagePool.synthetic(images, seed=0), TrainConfig())
    save(p, model, tr, meta=meta)
    assert _sha(p) == GOLD[f"{kind}/seed{seed}/params+adam"]
    assert load(p).meta == {k: str(v) for k, v in meta.items()}


def test_save_load_round_trip_bit_exact(tmp_path):
    from paper_1711_06505_b200.checkpoint import WarmupMask, load, load_warmup, save
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    model, pool, tr, _ = _trained(tmp_path)
    p1 = tmp_path / "a.ckpt"
    save(p1, model, tr, meta={"aggregator": "multiquery-attn"})
    ckpt = load(p1)
    for n, prm in model.params.items():
        assert np.array_equal(ckpt.tensors()[n], prm.data)
    model2 = _model("multiquery-attn", 9)
    tr2 = LocalTrainer(model2, pool, TrainConfig())
    load_warmup(ckpt, model2, WarmupMask.full(), fresh_seed=0, trainer=tr2)
    p2 = tmp_path / "b.ckpt"
    save(p2, model2, tr2, meta={"aggregator": "multiquery-attn"})
    assert p1.read_bytes() == p2.read_bytes()


def test_partial_and_non_warmup(tmp_path):
    from paper_1711_06505_b200.checkpoint import WarmupMask, load_warmup, save
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    model, pool, tr, _ = _trained(tmp_path)
    path = tmp_path / "f.ckpt"
    save(path, model, tr)
    fresh = _model("multiquery-attn", 77)
    new_tr = LocalTrainer(fresh, pool, TrainConfig())
    for f in new_tr.engine.tt:
        new_tr.engine.tt[f].fill_(9)  # seeded optimizer state the reinit must reset
    load_warmup(path, fresh, WarmupMask.partial(), fresh_seed=123, trainer=new_tr)
    ref = _model("multiquery-attn", 123)
    for n in model.params:
        if n.startswith("id_emb/"):
            assert np.array_equal(fresh.params[n].data, ref.params[n].data), n
        else:
            assert np.array_equal(fresh.params[n].data, model.params[n].data), n
    for st in new_tr.table_state.values():
        assert not st.t.any()
    load_warmup(path, fresh, WarmupMask.non(), fresh_seed=321)
    ref = _model("multiquery-attn", 321)
    for n in model.params:
        assert np.array_equal(fresh.params[n].data, ref.params[n].data), n


def test_schema_mismatch_raises(tmp_path):
    from paper_1711_06505_b200.checkpoint import CheckpointError, WarmupMask, load_warmup, save
    model, pool, tr, _ = _trained(tmp_path)
    path = tmp_path / "d.ckpt"
    save(path, model)
    other = _model("multiquery-attn", 0, users=301)
    with pytest.raises(CheckpointError, match="shape mismatch"):
        load_warmup(path, other, WarmupMask.full(), fresh_seed=0)
    summ = _model("sum", 0)
    with pytest.raises(CheckpointError, match="group"):
        load_warmup(path, summ, WarmupMask.full(), fresh_seed=0)


def test_restored_optimizer_state_resumes(tmp_path):
    """The reference pins exact equality (checkpoint.py resume); here the
    continuing steps agree up to the run-to-run noise of the fp32 scatter
    reductions (see test_gpu_step.test_graphed_steps_match_eager)."""
    from paper_1711_06505_b200.checkpoint import WarmupMask, load_warmup, save
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    a, pool, ta, nxt = _trained(tmp_path)
    path = tmp_path / "h.ckpt"
    save(path, a, ta)
    b = _model("multiquery-attn", 50)
    tb = LocalTrainer(b, pool, TrainConfig(lr0=0.003))
    load_warmup(path, b, WarmupMask.full(), fresh_seed=0, trainer=tb)
    tb.engine.iteration = ta.engine.iteration
    la, lb = ta.train_batch(nxt), tb.train_batch(nxt)
    assert abs(la - lb) <= 1e-6 * max(1.0, abs(la))
    for n in a.params:
        d = np.abs(a.params[n].data - b.params[n].data)
        assert d.max() <= 2 * 0.003 + 1e-6, n
