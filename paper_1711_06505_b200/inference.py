"""Inference export and the key-value predictor: the
drop-in for the reference ``dicm.inference`` (inference.py:1-81) and
``training.predict_logits`` (training.py:109-118).

After training, every pool image goes through the image net once
(``export_inference``: the training forward kernels over M = P rows); scoring
(``KvPredictor.predict``) then looks image embeddings up in the exported table
(one row gather on the device) instead of running the image net, except for
cold ids beyond the table, which are embedded on the fly from the pool.
Everything after the embeddings -- ID rows, pooling, head -- is the training
forward (``StepEngine.forward_logits``).

Tables are stored on disk in the reference's FMX1 float32 matrix format
(images.py:18-45), so files interchange with ``dicm.inference.InferenceTable``.
"""

from __future__ import annotations

import struct

import numpy as np

from .batch import Batch, encode_batch

MATRIX_MAGIC = b"FMX1"
MATRIX_VERSION = 1


def write_matrix_f32(path, array):
    """16-byte header (magic, version, rows, cols) + little-endian float32
    values row-major (reference images.py:22-31)."""
    a = np.ascontiguousarray(array, dtype="<f4")
    if a.ndim != 2:
        raise ValueError(f"matrix file requires a 2-D array, got shape {a.shape}")
    with open(path, "wb") as fh:
        fh.write(MATRIX_MAGIC)
        fh.write(struct.pack("<III", MATRIX_VERSION, a.shape[0], a.shape[1]))
        fh.write(a.tobytes())


def read_matrix_f32(path):
    """Reference images.py:34-45 (same errors for bad magic / version / size)."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != MATRIX_MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}, expected {MATRIX_MAGIC!r}")
        version, rows, cols = struct.unpack("<III", fh.read(12))
        if version != MATRIX_VERSION:
            raise ValueError(f"{path}: unsupported matrix version {version}")
        payload = fh.read(rows * cols * 4)
        if len(payload) != rows * cols * 4:
            raise ValueError(f"{path}: truncated payload")
    return np.frombuffer(payload, dtype="<f4").reshape(rows, cols).copy()


class InferenceTable:
    """Dense id -> embedding map, row index = image id (reference
    inference.py:19-45).  Holds the float32 rows the device computed; the
    device copy (``device()``) is what the predictor gathers from."""

    def __init__(self, embeddings):
        import torch
        if isinstance(embeddings, torch.Tensor):
            self._dev = embeddings.detach().float().contiguous()
            self.embeddings = None
        else:
            self._dev = None
            self.embeddings = np.asarray(embeddings, dtype=np.float64)

    def _host(self):
        if self.embeddings is None:
            self.embeddings = self._dev.double().cpu().numpy()
        return self.embeddings

    def device(self, dev="cuda", width=None):
        """The rows on the device, zero-padded to ``width`` columns (the
        kernels' 12-wide embedding rows) when given."""
        import torch
        if self._dev is None:
            self._dev = torch.as_tensor(self._host(), dtype=torch.float32, device=dev).contiguous()
        if width is not None and self._dev.shape[1] < width:
            out = torch.zeros((self._dev.shape[0], width), dtype=torch.float32, device=self._dev.device)
            out[:, :self._dev.shape[1]] = self._dev
            return out
        return self._dev

    def __len__(self):
        return int(self._dev.shape[0]) if self._dev is not None else self.embeddings.shape[0]

    def lookup(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        if ids.size and (ids.min() < 0 or ids.max() >= len(self)):
            raise KeyError("image id outside the exported table")
        return self._host()[ids]

    def save(self, path):
        write_matrix_f32(path, self._host())

    @classmethod
    def load(cls, path):
        return cls(read_matrix_f32(path).astype(np.float64))


def _engine_for(model, store, precision="fp32"):
    from .engine import StepEngine
    eng = getattr(model, "_infer_engine", None)
    if eng is None or eng.store is not store or eng.precision != precision:
        eng = StepEngine(model, store, precision)
        model._infer_engine = eng
    return eng


def export_inference(model, store, precision="fp32", chunk=1 << 19):
    """Embed every image id of the store with the trained net (reference
    inference.py:42-46): the forward image-MLP kernels over all P rows."""
    import torch
    eng = _engine_for(model, store, precision)
    n = len(store)
    rows = torch.arange(n, dtype=torch.int32, device=eng.dev)
    out = torch.empty((max(n, 1), 12), dtype=torch.float32, device=eng.dev)
    eng.embed_rows(rows, n, out, chunk=chunk)
    eng.raise_status()
    return InferenceTable(out[:n, :model.schema.d_img])


def _as_batch(samples, model):
    return samples if isinstance(samples, Batch) else encode_batch(samples, model)


def predict_logits(model, samples, store, chunk=1024, precision="fp32"):
    """Forward-only scores with the live image net (reference
    training.py:109-118)."""
    eng = _engine_for(model, store, precision)
    b = _as_batch(samples, model)
    out = np.empty(b.size)
    for start in range(0, b.size, chunk):
        part = b.slice(start, min(b.size, start + chunk))
        out[start:start + part.size] = eng.forward_logits(eng.upload(part)).double().cpu().numpy()
    eng.raise_status()
    return out


def forward_ctr(model, samples, store, precision="fp32"):
    """Score samples with the live model -> (probabilities, logits)
    (reference forward_ctr, model.py:411-417)."""
    z = predict_logits(model, samples, store, precision=precision)
    return 1.0 / (1.0 + np.exp(-z)), z


def forward_prerank(model, samples, store, precision="fp32"):
    """Two-tower scores (inner products) -> (probabilities, scores)
    (reference forward_prerank, model.py:529-535)."""
    return forward_ctr(model, samples, store, precision)


class KvPredictor:
    """Scores samples from frozen parameters plus the exported table
    (reference inference.py:49-81); ids beyond the table take the cold path
    through the live image net on the store's rows."""

    def __init__(self, model, table, store, precision="fp32"):
        self.model = model
        self.table = table
        self.store = store
        self.precision = precision

    def predict(self, samples, chunk=1024):
        """(probabilities, logits) for the samples via table lookups."""
        eng = _engine_for(self.model, self.store, self.precision)
        tab = self.table.device(eng.dev, width=12)
        b = _as_batch(samples, self.model)
        logits = np.empty(b.size)
        for start in range(0, b.size, chunk):
            part = b.slice(start, min(b.size, start + chunk))
            logits[start:start + part.size] = eng.forward_logits(eng.upload(part), table=tab).double().cpu().numpy()
        eng.raise_status()
        return 1.0 / (1.0 + np.exp(-logits)), logits
