"""Host-side batch encoding: samples -> CSR index arrays.

Mirror of the reference's ``Batch`` / ``encode_batch`` (model.py:138-198):
behavior lists keep their most recent ``b_max`` entries (model.py:168, 176),
multi-hot fields become (flat ids, CSR offsets) instead of (flat, segment),
and ids are int32 (every vocabulary in this build is < 2^31).  The
deduplication the reference does here with ``np.unique`` (model.py:187) is
NOT done on the host: the device step deduplicates (``dicm_dedup``).  The
``unique_images`` / ``unique_field_ids`` helpers exist for inspection only.

``synthetic_batch`` draws pre-encoded batches of the benchmark shapes
 without building Python sample objects.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Batch:
    size: int
    labels: np.ndarray                 # [B] float32
    onehot: dict                       # field -> ids [B] int32
    multihot: dict                     # field -> (flat ids [R_f] int32, offsets [B+1] int32)
    ad_image_ids: np.ndarray           # [B] int32
    beh_image_ids: np.ndarray          # [R] int32
    beh_off: np.ndarray                # [B+1] int32
    meta: dict = field(default_factory=dict)

    @property
    def refs(self):
        return int(self.beh_off[-1]) if len(self.beh_off) else 0

    @property
    def beh_seg(self):
        return np.repeat(np.arange(self.size), np.diff(self.beh_off))

    def unique_field_ids(self, fname):
        """Host-side inspection helper (reference model.py:152-155)."""
        if fname in self.onehot:
            return np.unique(self.onehot[fname])
        return np.unique(self.multihot[fname][0])

    def unique_images(self, use_ad_image=True, use_behavior_images=True):
        """Host-side inspection helper (reference model.py:182-187)."""
        parts = []
        if use_ad_image:
            parts.append(self.ad_image_ids)
        if use_behavior_images:
            parts.append(self.beh_image_ids)
        return np.unique(np.concatenate(parts).astype(np.int64)) if parts else np.zeros(0, np.int64)

    def take(self, idx):
        """Samples ``idx`` (any order) as a new batch: the vectorised CSR
        gather behind shuffled minibatches (reference data.py:284-290)."""
        idx = np.asarray(idx, dtype=np.int64)

        def gather(flat, off):
            lens = (off[1:] - off[:-1])[idx]
            o = np.zeros(len(idx) + 1, dtype=np.int32)
            np.cumsum(lens, out=o[1:])
            starts = np.repeat(off[:-1][idx].astype(np.int64) - o[:-1], lens)
            return flat[starts + np.arange(int(o[-1]))], o

        mh = {f: gather(fl, of) for f, (fl, of) in self.multihot.items()}
        beh, boff = gather(self.beh_image_ids, self.beh_off)
        return Batch(len(idx), self.labels[idx], {f: v[idx] for f, v in self.onehot.items()}, mh,
                     self.ad_image_ids[idx], beh, boff, dict(self.meta))

    def slice(self, start, stop):
        """Samples [start, stop) as a new batch (the contiguous per-worker split
        of reference runtime.py:379-382)."""
        def cut(flat, off):
            lo, hi = int(off[start]), int(off[stop])
            return flat[lo:hi].copy(), (off[start:stop + 1] - lo).astype(np.int32)

        mh = {f: cut(fl, of) for f, (fl, of) in self.multihot.items()}
        beh, boff = cut(self.beh_image_ids, self.beh_off)
        return Batch(stop - start, self.labels[start:stop].copy(),
                     {f: v[start:stop].copy() for f, v in self.onehot.items()}, mh,
                     self.ad_image_ids[start:stop].copy(), beh, boff, dict(self.meta))


def _get(s, k):
    return s[k] if isinstance(s, dict) else getattr(s, k)


def _csr(lists, b_max):
    tails = [list(x)[-b_max:] if len(x) > b_max else list(x) for x in lists]
    off = np.zeros(len(tails) + 1, dtype=np.int32)
    np.cumsum([len(x) for x in tails], out=off[1:])
    flat = np.fromiter((i for x in tails for i in x), dtype=np.int64, count=int(off[-1]))
    return _i32(flat), off


def _i32(a):
    a = np.asarray(a, dtype=np.int64)
    if a.size and (a.min() < -2**31 or a.max() >= 2**31):
        bad = a[(a < -2**31) | (a >= 2**31)][0]
        raise KeyError(f"id {bad} outside the int32 id range of this build")
    return a.astype(np.int32)


def encode_batch(samples, model):
    """Index arrays for one minibatch (reference model.py:158-198)."""
    schema = model.schema
    b_max = schema.b_max
    onehot, multihot = {}, {}
    for f in schema.fields:
        if f.multi:
            multihot[f.name] = _csr([_get(s, f.name) for s in samples], b_max)
        else:
            onehot[f.name] = _i32([_get(s, f.name) for s in samples])
    beh, beh_off = _csr([_get(s, "behavior_images") for s in samples], b_max)
    return Batch(
        size=len(samples),
        labels=np.array([_get(s, "label") for s in samples], dtype=np.float32),
        onehot=onehot,
        multihot=multihot,
        ad_image_ids=_i32([_get(s, "ad_image") for s in samples]),
        beh_image_ids=beh,
        beh_off=beh_off,
    )


def read_jsonl(path, schema, nthreads=0):
    """All samples of a JSONL file (reference data.py:293-311) as one Batch,
    parsed by the native reader (csrc/host_io.cpp) straight into CSR columns
    -- no per-sample Python objects.  Same result as
    ``encode_batch(read_samples(path), model)``; a malformed record raises
    ``ValueError`` naming its line, like the reference."""
    import ctypes as C
    from . import _lib as L
    keys, is_list = [], []
    for f in schema.fields:
        keys.append(f.name)
        is_list.append(bool(f.multi))
    for k, lst in (("ad_image", False), ("behavior_images", True), ("label", False)):
        if k not in keys:
            keys.append(k)
            is_list.append(lst)
    spec = L.JsonlSpec()
    spec.n_keys = len(keys)
    enc = [k.encode() for k in keys]
    for i, k in enumerate(enc):
        spec.keys[i] = k
        spec.key_is_list[i] = int(is_list[i])
    spec.b_max = int(schema.b_max)
    with open(path, "rb") as fh:
        raw = fh.read()
    n, bad = C.c_int64(0), C.c_int64(-1)
    h = L.lib.dicm_jsonl_parse(raw, len(raw), C.byref(spec), int(nthreads), C.byref(n), C.byref(bad))
    if not h:
        raise ValueError(f"{path}:{bad.value}: {L.lib.dicm_last_error().decode()}")
    try:
        n = n.value
        cols = {}
        for i, k in enumerate(keys):
            if k == "label":
                lab = np.empty(n, dtype=np.float32)
                L.check(L.lib.dicm_jsonl_export(h, i, None, None, lab.ctypes.data))
                cols[k] = lab
            elif is_list[i]:
                vals = np.empty(L.lib.dicm_jsonl_list_total(h, i), dtype=np.int32)
                off = np.empty(n + 1, dtype=np.int32)
                L.check(L.lib.dicm_jsonl_export(h, i, vals.ctypes.data, off.ctypes.data, None))
                cols[k] = (vals, off)
            else:
                vals = np.empty(n, dtype=np.int32)
                L.check(L.lib.dicm_jsonl_export(h, i, vals.ctypes.data, None, None))
                cols[k] = vals
    finally:
        L.lib.dicm_jsonl_free(h)
    onehot = {f.name: cols[f.name] for f in schema.fields if not f.multi}
    multihot = {f.name: cols[f.name] for f in schema.fields if f.multi}
    beh, beh_off = cols["behavior_images"]
    return Batch(n, cols["label"], onehot, multihot, cols["ad_image"], beh, beh_off)


def minibatch_order(n, seed, epoch=0):
    """The reference's deterministic shuffle (data.py:284-290)."""
    return np.random.default_rng([int(seed) & 0xFFFFFFFF, epoch]).permutation(n)


def iter_minibatches(batch, batch_size, seed, epoch=0):
    """Shuffled minibatches of a columnar Batch in the reference's order
    (data.py:284-290: the final short batch is emitted)."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    order = minibatch_order(batch.size, seed, epoch)
    for start in range(0, batch.size, batch_size):
        yield batch.take(order[start:start + batch_size])


def zipf_keys(rng, n, pool, s=1.1, perm_seed=0):
    """Zipf-skewed keys: rank r ~ (r+1)^-s over [0, pool), mapped through a
    seeded permutation (cfg 4)."""
    ranks = np.arange(pool, dtype=np.float64)
    p = (ranks + 1.0) ** (-s)
    p /= p.sum()
    cdf = np.cumsum(p)
    r = np.searchsorted(cdf, rng.random(n), side="right")
    r = np.minimum(r, pool - 1)
    perm = np.random.default_rng(perm_seed).permutation(pool)
    return perm[r]


def synthetic_batch(rng, schema, batch, lengths, n_images, base_ctr=0.3, zipf=None):
    """A pre-encoded batch of the benchmark shapes.

    ``lengths``: int (fixed behaviors per sample) or an array [B];
    ``zipf``: None for uniform image keys, else the exponent s.
    behavior_items / behavior_images share the per-sample length (the
    reference generator maps items onto images one to one, data.py:207-209).
    """
    B = int(batch)
    L = np.full(B, int(lengths), dtype=np.int64) if np.isscalar(lengths) else np.asarray(lengths, np.int64)
    L = np.minimum(L, schema.b_max)
    off = np.zeros(B + 1, dtype=np.int32)
    np.cumsum(L, out=off[1:])
    R = int(off[-1])
    draw_img = (lambda n: zipf_keys(rng, n, n_images, zipf)) if zipf else (lambda n: rng.integers(0, n_images, n))
    onehot, multihot = {}, {}
    beh = _i32(draw_img(R))
    for f in schema.fields:
        if f.multi:
            ids = beh if f.name == "behavior_images" else _i32(rng.integers(0, f.vocab, R))
            multihot[f.name] = (ids, off)
        else:
            onehot[f.name] = None
    ad_img = _i32(draw_img(B))
    for f in schema.fields:
        if not f.multi:
            onehot[f.name] = ad_img if f.name == "ad_image" else _i32(rng.integers(0, f.vocab, B))
    labels = (rng.random(B) < base_ctr).astype(np.float32)
    return Batch(B, labels, onehot, multihot, ad_img, beh, off)
