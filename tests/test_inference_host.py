"""Inference table host logic (reference inference.py:19-45, images.py:18-45):
FMX1 round trip, header layout, bounds errors.  CPU only."""
import struct

import numpy as np
import pytest

from paper_1711_06505_b200.inference import InferenceTable, read_matrix_f32, write_matrix_f32


def test_table_file_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    emb = rng.normal(size=(37, 12))
    table = InferenceTable(emb)
    path = tmp_path / "table.bin"
    table.save(path)
    again = InferenceTable.load(path)
    assert len(again) == len(table)
    assert np.allclose(again.embeddings, table.embeddings, atol=1e-6)  # disk format is float32


def test_fmx1_header_is_the_reference_layout(tmp_path):
    a = np.arange(6, dtype=np.float32).reshape(2, 3)
    p = tmp_path / "m.bin"
    write_matrix_f32(p, a)
    raw = p.read_bytes()
    assert raw[:4] == b"FMX1"
    assert struct.unpack("<III", raw[4:16]) == (1, 2, 3)
    assert np.array_equal(np.frombuffer(raw[16:], dtype="<f4").reshape(2, 3), a)
    assert np.array_equal(read_matrix_f32(p), a)


def test_bad_files_raise(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"XXXX" + struct.pack("<III", 1, 1, 1) + b"\0" * 4)
    with pytest.raises(ValueError, match="bad magic"):
        read_matrix_f32(p)
    p.write_bytes(b"FMX1" + struct.pack("<III", 1, 2, 2) + b"\0" * 4)
    with pytest.raises(ValueError, match="truncated"):
        read_matrix_f32(p)


def test_lookup_beyond_table_raises():
    table = InferenceTable(np.zeros((5, 12)))
    with pytest.raises(KeyError, match="exported table"):
        table.lookup([5])
    with pytest.raises(KeyError, match="exported table"):
        table.lookup([-1])
    assert table.lookup([0, 4]).shape == (2, 12)


def test_checkpoint_host_format(tmp_path):
    """DCK1 writer/reader on host arrays (duck-typed model), checksum and
    mask validation (reference tests/test_checkpoint.py:36-44, 122-129)."""
    from paper_1711_06505_b200.checkpoint import CheckpointError, WarmupMask, load, save

    class P:
        def __init__(self, a):
            self.data = a

    class M:
        params = {"img/0/w": P(np.arange(6.0).reshape(2, 3)), "id_emb/user": P(np.ones((3, 12))),
                  "mlp/2/b": P(np.zeros(1))}

    path = tmp_path / "c.ckpt"
    save(path, M(), optimizer={"mlp/2/b#t": np.array(4, dtype=np.int64)}, meta={"k": 1})
    ck = load(path)
    assert ck.meta == {"k": "1"}
    assert set(ck.groups) == {"image-embedding-model", "id-embeddings", "mlp"}
    assert np.array_equal(ck.tensors()["img/0/w"], M.params["img/0/w"].data)
    assert ck.tensors()["mlp/2/b#t"] == 4
    raw = bytearray(path.read_bytes())
    raw[-1] ^= 0xFF
    path.write_bytes(bytes(raw))
    with pytest.raises(CheckpointError, match="checksum"):
        load(path)
    with pytest.raises(CheckpointError, match="unknown parameter group"):
        WarmupMask({"bogus": "restore"})
    with pytest.raises(CheckpointError, match="bad warm-up flag"):
        WarmupMask({"mlp": "maybe"})
    with pytest.raises(CheckpointError, match="unknown warm-up strategy"):
        WarmupMask.named("half")
    assert WarmupMask.named("partial").flags["id-embeddings"] == "reinitialize"
