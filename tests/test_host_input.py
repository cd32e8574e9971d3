"""Native JSONL reader and columnar minibatching:
equal to the reference path read_samples (data.py:293-311) + encode_batch
(model.py:158-198) + minibatches (data.py:284-290), at any thread count.
CPU only (the reader is host code in libdicm_b200.so)."""
import json

import numpy as np
import pytest

from paper_1711_06505_b200.batch import encode_batch, iter_minibatches, read_jsonl
from paper_1711_06505_b200.schema import default_schema

KEYS = ("user", "scenario", "ad", "ad_category", "ad_image", "behavior_items", "behavior_images", "label", "day")


class _M:
    def __init__(self, schema):
        self.schema = schema


def _samples(rng, n, b_max):
    out = []
    for _ in range(n):
        L = int(rng.integers(0, 2 * b_max))
        out.append({"user": int(rng.integers(0, 500)), "scenario": int(rng.integers(0, 4)),
                    "ad": int(rng.integers(0, 300)), "ad_category": int(rng.integers(0, 8)),
                    "ad_image": int(rng.integers(0, 900)),
                    "behavior_items": [int(x) for x in rng.integers(0, 300, L)],
                    "behavior_images": [int(x) for x in rng.integers(0, 900, L)],
                    "label": int(rng.random() < 0.3), "day": int(rng.integers(0, 3))})
    return out


def _write(path, samples):  # the reference writer (data.py:293-297)
    with open(path, "w", encoding="utf-8") as fh:
        for s in samples:
            fh.write(json.dumps({k: s[k] for k in KEYS}, separators=(",", ":")) + "\n")


def _same(a, b):
    assert a.size == b.size
    assert np.array_equal(a.labels, b.labels)
    for f in a.onehot:
        assert np.array_equal(a.onehot[f], b.onehot[f]), f
    for f in a.multihot:
        assert np.array_equal(a.multihot[f][0], b.multihot[f][0]), f
        assert np.array_equal(a.multihot[f][1], b.multihot[f][1]), f
    assert np.array_equal(a.ad_image_ids, b.ad_image_ids)
    assert np.array_equal(a.beh_image_ids, b.beh_image_ids)
    assert np.array_equal(a.beh_off, b.beh_off)


@pytest.mark.parametrize("nthreads", [1, 3, 0])
def test_jsonl_reader_equals_encode_batch(tmp_path, nthreads):
    schema = default_schema(500, 4, 300, 8, 900, b_max=6)
    samples = _samples(np.random.default_rng(0), 3000, 6)
    path = tmp_path / "s.jsonl"
    _write(path, samples)
    with open(path, "a") as fh:
        fh.write("\n   \n")  # blank lines are skipped
    _same(read_jsonl(path, schema, nthreads), encode_batch(samples, _M(schema)))


def test_minibatches_follow_the_reference_order(tmp_path):
    schema = default_schema(500, 4, 300, 8, 900, b_max=6)
    samples = _samples(np.random.default_rng(1), 203, 6)
    path = tmp_path / "s.jsonl"
    _write(path, samples)
    full = read_jsonl(path, schema)
    order = np.random.default_rng([7, 2]).permutation(len(samples))  # data.py:287
    got = list(iter_minibatches(full, 64, seed=7, epoch=2))
    assert [g.size for g in got] == [64, 64, 64, 11]
    for i, g in enumerate(got):
        _same(g, encode_batch([samples[j] for j in order[64 * i:64 * (i + 1)]], _M(schema)))


def test_malformed_records_name_their_line(tmp_path):
    schema = default_schema(500, 4, 300, 8, 900, b_max=6)
    samples = _samples(np.random.default_rng(2), 5, 6)
    path = tmp_path / "bad.jsonl"
    _write(path, samples)
    lines = path.read_text().splitlines()
    lines[3] = lines[3].replace('"ad":', '"ad_missing":')
    path.write_text("\n".join(lines) + "\n")
    with pytest.raises(ValueError, match=r":4: .*missing key 'ad'"):
        read_jsonl(path, schema)
    lines[3] = "{not json"
    path.write_text("\n".join(lines) + "\n")
    with pytest.raises(ValueError, match=r":4: "):
        read_jsonl(path, schema)
