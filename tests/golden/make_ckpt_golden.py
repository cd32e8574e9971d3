"""Golden hashes of DCK1 checkpoints written by the REFERENCE (run in the build
container, where /root/reference is importable):

    python tests/golden/make_ckpt_golden.py

For each case a reference DicmModel at its seeded init (reference
model.py:266-335) is saved with ``dicm.checkpoint.save`` (checkpoint.py:142),
once without and once with a fresh LocalTrainer's optimizer state; the sha256
of each file goes to tests/golden/ckpt_hashes.json.  The device keeps
parameters in fp32, so the reference's f64 init is rounded to fp32 first (the
values a device model holds); the GPU test builds the same model on the
device, saves it with paper_1711_06505_b200.checkpoint and must reproduce the
bytes exactly (byte-compatible writer), then loads the file back."""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF = os.environ.get("DICM_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from dicm.checkpoint import save  # noqa: E402
from dicm.model import AggregatorSpec, DicmModel, FeatureSchema, FieldSpec  # noqa: E402
from dicm.training import LocalTrainer, TrainConfig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
# (kind, user vocab, scenarios, ad vocab, categories, images, b_max, seed, meta)
CASES = [("sum", 300, 4, 200, 8, 96, 12, 0, {}), ("multiquery-attn", 300, 4, 200, 8, 96, 12, 3,
                                                    {"aggregator": "multiquery-attn", "note": "golden"})]


class _Ext:
    out_dim = 4096


class _Store:
    def __len__(self):
        return 96


def schema_of(users, scen, ads, cats, images, b_max):
    fields = [FieldSpec("user", users), FieldSpec("scenario", scen), FieldSpec("ad", ads),
              FieldSpec("ad_category", cats), FieldSpec("behavior_items", ads, multi=True),
              FieldSpec("ad_image", images), FieldSpec("behavior_images", images, multi=True)]
    return FeatureSchema(fields=fields, d_id=12, d_raw=4096, d_img=12, b_max=b_max)


def digest(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def main():
    out = {}
    for kind, users, scen, ads, cats, images, b_max, seed, meta in CASES:
        model = DicmModel(schema_of(users, scen, ads, cats, images, b_max), AggregatorSpec(kind), _Ext(), seed=seed)
        for prm in model.params.values():
            prm.data[...] = prm.data.astype(np.float32).astype(np.float64)
        key = f"{kind}/seed{seed}"
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "a.ckpt")
            save(p, model, meta=meta)
            out[key + "/params"] = digest(p)
            tr = LocalTrainer(model, _Store(), TrainConfig())
            save(p, model, tr, meta=meta)
            out[key + "/params+adam"] = digest(p)
    out["cases"] = [list(c[:8]) + [c[8]] for c in CASES]
    json.dump(out, open(os.path.join(HERE, "ckpt_hashes.json"), "w"), indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
