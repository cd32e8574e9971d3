"""CPU-only tests: the C ABI library loads and exports every declared entry
point; host-side encoding / layout logic matches the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest

import golden_io as G
from oracle import dicm_oracle as O
from paper_1711_06505_b200 import schema as S
from paper_1711_06505_b200.batch import Batch, encode_batch, synthetic_batch, zipf_keys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dicm_b200.h")
LIB = os.path.join(ROOT, "paper_1711_06505_b200", "libdicm_b200.so")


def _ensure_lib():
    if not os.path.exists(LIB):
        import subprocess
        subprocess.run(["make", "-j8"], cwd=ROOT, check=True, capture_output=True)
    return LIB


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dicm_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_ensure_lib())
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.dicm_version() == 1


def test_python_binding_covers_header():
    _ensure_lib()
    from paper_1711_06505_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_library_reports_no_device_here_without_crashing():
    lib = ctypes.CDLL(_ensure_lib())
    arch = lib.dicm_device_arch()
    assert isinstance(arch, int)


def test_workspace_queries_are_pure_host():
    _ensure_lib()
    from paper_1711_06505_b200 import _lib as L
    assert L.lib.dicm_dedup_workspace(1_000_000) >= 1_000_000 // 8
    assert L.lib.dicm_head_partial_size(120) == 128 + 128 + 128 * 120 + 64 + 64 + 64 * 128 + 1 + 64
    lay = L.Layout()
    lay.kind, lay.use_behavior_images, lay.n_query = 2, 1, 2
    assert L.lib.dicm_attn_partial_size(ctypes.byref(lay)) == (97 + 32 * 24) + (97 + 32 * 36)


@pytest.mark.parametrize("name", G.FULL + G.TINY)
def test_encode_batch_matches_oracle_encode(name):
    fx = G.load(name)
    m = G.meta(fx)
    lay = G.layout_of(m)

    class M:
        schema = lay.schema

    samples = G.samples(fx, 0)
    b = encode_batch(samples, M)
    ob = O.encode(samples, G.oracle_cfg(m))
    for f, v in b.onehot.items():
        assert np.array_equal(v, ob["onehot"][f])
    for f, (fl, of) in b.multihot.items():
        assert np.array_equal(fl, ob["multihot"][f][0]) and np.array_equal(of, ob["multihot"][f][1])
    assert np.array_equal(b.beh_image_ids, ob["beh_image_ids"])
    assert np.array_equal(b.beh_off, ob["beh_off"])
    assert np.array_equal(b.labels, ob["labels"])
    assert np.array_equal(b.unique_images(lay.use_ad_image, lay.use_behavior_images),
                          np.unique(O.needed_image_keys(G.oracle_cfg(m), ob)))


def test_head_offsets_follow_reference_hstack_order():
    lay = S.ModelLayout(S.default_schema(10, 4, 10, 8, 10), S.AggregatorSpec("multiquery-attn"), (128, 64),
                        True, True)
    ho = lay.head_offsets()
    names = [f.name for f in lay.schema.fields]
    assert [ho["field/" + n] for n in names] == [12 * i for i in range(7)]
    assert ho["ad_image_emb"] == 84 and ho["pool"] == 96 and ho["width"] == 120 == lay.mlp_input_width()


def test_dense_groups_are_contiguous_in_sorted_order():
    for kind in ("sum", "attn", "multiquery-attn"):
        lay = S.ModelLayout(S.default_schema(10, 4, 10, 8, 10), S.AggregatorSpec(kind), (128, 64), True, True)
        names = S.dense_param_names(lay)
        groups = [n.split("/")[0] for n in names]
        # attn/*, mlp/*, img/* each contiguous
        seen = []
        for g in groups:
            if not seen or seen[-1] != g:
                assert g not in seen
                seen.append(g)


def test_batch_slice_is_contiguous_worker_split():
    schema = S.default_schema(100, 4, 100, 8, 50, b_max=16)
    b = synthetic_batch(np.random.default_rng(0), schema, 40, 10, 50)
    parts = [b.slice(i * 10, (i + 1) * 10) for i in range(4)]
    assert np.array_equal(np.concatenate([p.beh_image_ids for p in parts]), b.beh_image_ids)
    assert all(p.size == 10 and p.beh_off[0] == 0 for p in parts)


def test_synthetic_batch_shapes_and_zipf():
    schema = S.default_schema(1000, 4, 1000, 8, 5000, b_max=50)
    rng = np.random.default_rng(1)
    b = synthetic_batch(rng, schema, 256, 50, 5000)
    assert b.refs == 256 * 50 and b.beh_off[-1] == b.refs
    assert np.array_equal(b.multihot["behavior_images"][0], b.beh_image_ids)
    assert np.array_equal(b.onehot["ad_image"], b.ad_image_ids)
    z = zipf_keys(rng, 100_000, 1_000_000, 1.1)
    top = np.bincount(z).max() / len(z)
    assert 0.05 < top < 0.2  # the hottest key takes ~11% of the references


def test_lr_schedule_paper_values():
    from paper_1711_06505_b200.engine import lr_schedule
    assert lr_schedule(0) == 0.001
    assert abs(lr_schedule(24000) - 0.0009) < 1e-15
    assert abs(lr_schedule(48000) - 0.00081) < 1e-15
    with pytest.raises(ValueError):
        lr_schedule(-1)


def test_model_validation_errors_mirror_reference():
    lay = S.ModelLayout(S.default_schema(10, 4, 10, 8, 10), S.AggregatorSpec("attn"), (128, 64), False, True)
    with pytest.raises(ValueError, match="needs the ad image"):
        S.validate_layout(lay)
    with pytest.raises(ValueError, match="unknown aggregator"):
        S.AggregatorSpec("bogus")


def test_host_pack_matches_numpy_layout():
    """dicm_host_pack (the multithreaded batch packing behind Packed.fill):
    every segment lands at its offset, any thread count, ragged sizes."""
    _ensure_lib()
    from paper_1711_06505_b200 import _lib as L
    rng = np.random.default_rng(4)
    sizes = [0, 1, 7, 100_003, 3, 65_536, 250_001]
    arrs = [rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32) for n in sizes]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]) + 5  # a gap in front
    total = int(offs[-1] + sizes[-1])
    ref = np.zeros(total, np.int32)
    for a, o in zip(arrs, offs):
        ref[o:o + len(a)] = a
    n = len(arrs)
    for nt in (1, 3, 0, 8, 2, 0, 5):  # the persistent pool grows and is reused
        out = np.zeros(total, np.int32)
        L.check(L.lib.dicm_host_pack(out.ctypes.data, (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrs]),
                                     (ctypes.c_int64 * n)(*[a.nbytes for a in arrs]),
                                     (ctypes.c_int64 * n)(*[4 * int(o) for o in offs]), n, nt))
        assert np.array_equal(out, ref), nt


def test_packed_fill_matches_column_copies():
    """Packed.fill (one dicm_host_pack call) == the per-column layout."""
    _ensure_lib()
    from paper_1711_06505_b200.engine import Packed
    schema = S.default_schema(500, 4, 600, 8, 900, b_max=20)

    class M:
        pass

    m = M()
    m.schema = schema
    m.layout = S.ModelLayout(schema, S.AggregatorSpec("attn"), (128, 64), True, True)
    b = synthetic_batch(np.random.default_rng(1), schema, 64, np.arange(64) % 21, 900)
    pk = Packed(m, b)
    host = np.full(pk.total, -7, np.int32)
    pk.fill(m, b, host)
    ref = np.full(pk.total, -7, np.int32)
    for f in schema.fields:
        if f.multi:
            a, n, o = pk.multi[f.name]
            fl, of = b.multihot[f.name]
            ref[a:a + n], ref[o:o + pk.B + 1] = fl, of
        else:
            ref[pk.onehot[f.name]:pk.onehot[f.name] + pk.B] = b.onehot[f.name]
    ref[pk.ad:pk.ad + pk.B] = b.ad_image_ids
    ref[pk.beh:pk.beh + pk.R] = b.beh_image_ids
    ref[pk.beh_off:pk.beh_off + pk.B + 1] = b.beh_off
    ref[pk.labels:pk.labels + pk.B] = np.asarray(b.labels, np.float32).view(np.int32)
    assert np.array_equal(host, ref)


def test_narrow_models_embed_into_the_kernel_widths():
    """schema.KernelGeometry: the reference's own narrow test model (d_id 3,
    d_img 4, d_raw 8, attention 5, head (6, 4); reference tests/conftest.py:9-34)
    is stored zero-padded in the compiled widths; the real entries are the
    reference init, every padded entry is 0, and copy_/data round-trip."""
    import torch
    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200 import schema as S
    sch = S.FeatureSchema(fields=[S.FieldSpec("user", 5), S.FieldSpec("ad", 7)], d_id=3, d_raw=8, d_img=4,
                          b_max=4, query_fields=("ad",))
    for kind in ("sum", "attn", "multiquery-attn", "max", "concat"):
        m = DicmModel(sch, S.AggregatorSpec(kind, attention_hidden=5), None, seed=1, mlp_widths=(6, 4),
                      device="cpu")
        lay = m.layout
        ref = S.init_params(lay, 1)
        assert m.geometry.d_raw == 256 and not m.geometry.identity
        for n, a in ref.items():
            p = m.params[n]
            assert p.shape == a.shape, n
            assert np.array_equal(p.data, a.astype(np.float32).astype(np.float64)), n
        # everything outside the real entries is zero
        mask = m.real_mask()
        assert not m.dense[~mask].any(), kind
        assert int(mask.sum()) == sum(a.size for n, a in ref.items() if not n.startswith("id_emb/"))
        for f in sch.fields:
            assert m.tables[f.name].shape == (f.vocab, 12) and not m.tables[f.name][:, 3:].any()
        # copy_ writes the real entries only; real_view reads the fused span
        w = m.params["mlp/0/w"]
        v = np.arange(np.prod(w.shape), dtype=np.float64).reshape(w.shape)
        w.copy_(v)
        assert np.array_equal(w.data, v)
        assert np.array_equal(m.real_view(m.dense, "mlp/0/w").double().numpy(), v)
        assert int((m.dense_view(m.dense, "mlp/0/w") != 0).sum()) == np.count_nonzero(v)
    with pytest.raises(NotImplementedError, match="compiled"):
        DicmModel(S.FeatureSchema(fields=[S.FieldSpec("user", 5)], d_id=16), S.AggregatorSpec("sum"), None,
                  device="cpu")
