"""Training from a JSONL file through the native reader and the prefetching
input pipeline follows the reference path
``run(read_samples(path))`` batch for batch."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
KEYS = ("user", "scenario", "ad", "ad_category", "ad_image", "behavior_items", "behavior_images", "label", "day")


def test_run_file_matches_run_on_samples(tmp_path):
    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    P = 400
    schema = default_schema(500, 4, 300, 8, P, b_max=10)
    rng = np.random.default_rng(0)
    samples = []
    for _ in range(300):
        L = int(rng.integers(0, 14))
        samples.append({"user": int(rng.integers(0, 500)), "scenario": int(rng.integers(0, 4)),
                        "ad": int(rng.integers(0, 300)), "ad_category": int(rng.integers(0, 8)),
                        "ad_image": int(rng.integers(0, P)), "behavior_items": rng.integers(0, 300, L).tolist(),
                        "behavior_images": rng.integers(0, P, L).tolist(), "label": int(rng.random() < 0.3),
                        "day": 0})
    path = tmp_path / "train.jsonl"
    with open(path, "w") as fh:
        for s in samples:
            fh.write(json.dumps({k: s[k] for k in KEYS}, separators=(",", ":")) + "\n")
    pool = ImagePool.synthetic(P, seed=1)
    cfg = TrainConfig(epochs=2, batch_size=64, seed=5, lr0=1e-4)
    logs = []
    for use_file in (False, True):
        model = DicmModel(schema, AggregatorSpec("attn"), None, seed=0)
        tr = LocalTrainer(model, pool, cfg)
        logs.append(tr.run_file(path) if use_file else tr.run(samples))
    a, b = logs
    assert len(a.losses) == len(b.losses) == 10
    np.testing.assert_allclose(b.losses, a.losses, rtol=1e-4, atol=1e-6)
    assert a.lrs == b.lrs
