"""The DCK1 codec on the host (no GPU): the streaming writer reproduces the
bytes the reference's writer produced (tests/golden/ckpt_hashes.json, made by
tests/golden/make_ckpt_golden.py), the memory-mapped reader returns the
values, and the reference's error cases raise CheckpointError."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1711_06505_b200 import checkpoint as CK
from paper_1711_06505_b200 import schema as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ckpt_hashes.json")))


class _P:
    def __init__(self, a):
        self.data = a
        self.shape = a.shape


class _HostModel:
    """params -> host arrays (the writer's numpy source path)."""

    def __init__(self, params):
        self.params = {n: _P(a) for n, a in params.items()}


def _case_params(kind, users, scen, ads, cats, images, b_max, seed):
    schema = S.default_schema(users, scen, ads, cats, images, b_max=b_max)
    lay = S.ModelLayout(schema, S.AggregatorSpec(kind), (128, 64), True, True)
    p = S.init_params(lay, seed, include_tables=True)
    return {n: np.asarray(a, np.float64).astype(np.float32).astype(np.float64) for n, a in p.items()}


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c[0]}-seed{c[7]}")
def test_streaming_writer_reproduces_reference_bytes(tmp_path, case, monkeypatch):
    kind, users, scen, ads, cats, images, b_max, seed, meta = case
    params = _case_params(kind, users, scen, ads, cats, images, b_max, seed)
    monkeypatch.setattr(CK, "_CHUNK_BYTES", 4096)  # many chunks per tensor
    p = tmp_path / "x.ckpt"
    CK.save(p, _HostModel(params), meta=meta)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == GOLD[f"{kind}/seed{seed}/params"]
    opt = {}
    for n, a in params.items():
        opt[f"{n}#m"], opt[f"{n}#v"] = np.zeros_like(a), np.zeros_like(a)
        opt[f"{n}#t"] = np.zeros(a.shape[0], np.int64) if n.startswith("id_emb/") else np.array(0, np.int64)
    CK.save(p, _HostModel(params), optimizer=opt, meta=meta)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == GOLD[f"{kind}/seed{seed}/params+adam"]
    ck = CK.load(p)
    assert ck.meta == {k: str(v) for k, v in meta.items()}
    t = ck.tensors()
    for n, a in params.items():
        assert np.array_equal(t[n], a) and t[n].dtype == np.float64, n
        assert t[f"{n}#t"].dtype == np.int64
    assert sorted(ck.groups) == sorted({S.group_of(n) for n in params})


def test_reader_rejects_damaged_files(tmp_path):
    params = {"mlp/0/w": np.arange(6.0).reshape(2, 3), "img/0/b": np.ones(4)}
    p = tmp_path / "a.ckpt"
    CK.save(p, _HostModel(params))
    raw = bytearray(p.read_bytes())
    bad = tmp_path / "b.ckpt"
    bad.write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(CK.CheckpointError, match="not a checkpoint"):
        CK.load(bad)
    raw2 = bytearray(raw)
    raw2[-1] ^= 0xFF
    bad.write_bytes(bytes(raw2))
    with pytest.raises(CK.CheckpointError, match="checksum"):
        CK.load(bad)
    raw3 = bytearray(raw)
    raw3[4] = 2
    bad.write_bytes(bytes(raw3))
    with pytest.raises(CK.CheckpointError, match="version"):
        CK.load(bad)
    with pytest.raises(CK.CheckpointError, match="cannot read"):
        CK.load(tmp_path / "missing.ckpt")


def test_warmup_masks():
    assert CK.WarmupMask.full().restored_groups() == list(CK.GROUPS)
    assert CK.WarmupMask.non().restored_groups() == []
    assert S.GROUP_ID not in CK.WarmupMask.partial().restored_groups()
    assert CK.WarmupMask.named("partial") == CK.WarmupMask.partial()
    with pytest.raises(CK.CheckpointError, match="strategy"):
        CK.WarmupMask.named("half")
    with pytest.raises(CK.CheckpointError, match="unknown parameter group"):
        CK.WarmupMask({"nope": CK.RESTORE})
    with pytest.raises(CK.CheckpointError, match="bad warm-up flag"):
        CK.WarmupMask({S.GROUP_MLP: "maybe"})
