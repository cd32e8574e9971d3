"""Parity at the benchmarked shapes (BASELINE.json configs[0] and configs[1]).

The headline number comes from cfg2 (B = 4096, L = 200, 1M-image pool, bf16):
~561k unique images per step, so every persistent CTA of the tensor-core
image-MLP kernels loops over many row tiles (TMEM double buffers and
mbarrier phases wrap) and the pair dW0 kernel runs ~62k-row chunks.  These
tests run exactly those shapes through the C-ABI and compare with the f64
oracle (oracle/dicm_oracle.py, the chunked image MLP of SURVEY.md 8c's
compact remap: rows are read back from the device pool, every op is
row-local).

Tolerances:
  * integer work (unique images, owner counts): bit-exact;
  * fp32 CUDA-core path: 1e-4 in the reference metric |a-b|/max(1,|a|,|b|);
  * tensor-core layer 0: logits and loss within the north star's 2e-2 (same
    metric); tensors (E, act0, gradients) within 2e-2 (bf16) / 3e-3 (tf32)
    of the f64 result relative to the result's largest magnitude -- bf16
    rounds operands to 8 mantissa bits (2^-9 relative), tf32 to 11.
"""

import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import gpu_helpers as H
from oracle import dicm_oracle as O

pytestmark = pytest.mark.gpu

P_BENCH = 1_000_000
CAP_CFG2 = 4096 + 4096 * 200  # the bench's image capacity (B + R): rows_max of every launch
TOL = {"tf32": 3e-3, "bf16": 2e-2}


def relmax(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


_POOLS = {}


def bench_pool(dtype):
    """The cfg2 pool (1M rows, materialized tanh(z R^T)) -- one per dtype per session."""
    from paper_1711_06505_b200.pool import ImagePool
    if dtype not in _POOLS:
        _POOLS.clear()
        torch.cuda.empty_cache()
        _POOLS[dtype] = ImagePool.synthetic(P_BENCH, seed=0, dtype=dtype)
    return _POOLS[dtype]


def rows_reader(pool, chunk=1 << 15):
    """ids -> f64 host rows of the device pool (the exact values the kernels read)."""
    def rows_of(ids):
        ids = np.asarray(ids)
        out = np.empty((len(ids), pool.d_raw))
        for s in range(0, len(ids), chunk):
            out[s:s + chunk] = pool.gather(ids[s:s + chunk]).double().cpu().numpy()
        return out
    return rows_of


def _mlp_params(seed):
    rng = np.random.default_rng(seed)
    return {"img/0/w": rng.normal(0, np.sqrt(2 / 4096), (256, 4096)), "img/0/b": rng.normal(0, 0.1, 256),
            "img/0/a": np.full(256, 0.25), "img/1/w": rng.normal(0, np.sqrt(2 / 256), (64, 256)),
            "img/1/b": rng.normal(0, 0.05, 64), "img/1/a": np.full(64, 0.25),
            "img/2/w": rng.normal(0, np.sqrt(2 / 64), (12, 64)), "img/2/b": rng.normal(0, 0.05, 12)}


@pytest.mark.parametrize("U", [20_000, 100_000, 561_018])
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_image_mlp_at_bench_sizes_matches_oracle(U, prec):
    """dicm_imgmlp_fwd / dicm_imgmlp_bwd over U sorted unique rows of the 1M
    pool with the bench's capacity (rows_max = B + R of cfg2), against the
    chunked f64 image_mlp_fwd/_bwd (oracle/dicm_oracle.py:177-201).  At
    U = 561k each k_fwd4 pair runs ~15 tiles, each k_l12f/k_l12b CTA ~30,
    and k_dw0p's 9 row chunks are ~62k rows long."""
    from paper_1711_06505_b200 import _lib as L
    pool = bench_pool("bf16" if prec == "bf16" else "fp32")
    pc = L.PRECISIONS[prec]
    rng = np.random.default_rng(U)
    rows = np.sort(rng.choice(P_BENCH, size=U, replace=False)).astype(np.int32)
    p = _mlp_params(U)
    dev = "cuda"
    cap = CAP_CFG2
    pt = {k: torch.as_tensor(v, dtype=torch.float32, device=dev).contiguous() for k, v in p.items()}
    keys = ("w0", "b0", "a0", "w1", "b1", "a1", "w2", "b2")
    names = ("img/0/w", "img/0/b", "img/0/a", "img/1/w", "img/1/b", "img/1/a", "img/2/w", "img/2/b")
    prm = L.ImgMlpParams(**{k: pt[n].data_ptr() for k, n in zip(keys, names)})
    rt = torch.zeros(cap, dtype=torch.int32, device=dev)
    rt[:U] = torch.as_tensor(rows, device=dev)
    cnt = torch.tensor([U], dtype=torch.int32, device=dev)
    act0 = torch.zeros((cap, 256), device=dev)
    act1 = torch.zeros((cap, 64), device=dev)
    emb = torch.zeros((cap, 12), device=dev)
    ws = torch.zeros(L.lib.dicm_imgmlp_workspace(cap, 4096, pc), dtype=torch.uint8, device=dev)
    s = L.stream_handle()
    L.check(L.lib.dicm_imgmlp_fwd(pool.rows.data_ptr(), pool.dtype_code, 4096, rt.data_ptr(), cnt.data_ptr(), cap,
                                  C.byref(prm), act0.data_ptr(), act1.data_ptr(), emb.data_ptr(), pc, ws.data_ptr(),
                                  ws.numel(), s))
    dE = rng.normal(0, 1e-2, (U, 12))
    demb = torch.full((cap, 12), float("nan"), device=dev)  # rows past the count must never be read
    demb[:U] = torch.as_tensor(dE, dtype=torch.float32, device=dev)
    g = {n: torch.zeros_like(pt[n]) for n in names}
    gs = L.ImgMlpGrads(**{k: g[n].data_ptr() for k, n in zip(keys, names)})
    L.check(L.lib.dicm_imgmlp_bwd(pool.rows.data_ptr(), pool.dtype_code, 4096, rt.data_ptr(), cnt.data_ptr(), cap,
                                  C.byref(prm), act0.data_ptr(), act1.data_ptr(), demb.data_ptr(), C.byref(gs), pc,
                                  ws.data_ptr(), ws.numel(), s))
    torch.cuda.synchronize()
    # forward: the oracle on the same rows
    rows_of = rows_reader(pool)
    uniq = rows.astype(np.int64)
    E, cache = O.image_mlp_fwd_rows(p, rows_of, uniq)
    tol = TOL[prec]
    got_e = emb[:U].double().cpu().numpy()
    assert not torch.isnan(emb[:U]).any()
    assert relmax(got_e, E) < tol, ("E", relmax(got_e, E))
    a0 = saved(act0, cap, 256, prec)
    a1 = saved(act1, cap, 64, prec)
    assert relmax(a0[:U].double().cpu().numpy(), cache[1]) < tol, "act0"
    assert relmax(a1[:U].double().cpu().numpy(), cache[3]) < tol, "act1"
    assert torch.count_nonzero(a0[U:].float()) == 0, "rows past the count were written"
    # backward: the oracle's backward from the activations the device saved
    # (dE rounded to fp32 like the device input).  Starting it from its own
    # f64 forward instead would compare different PReLU branches wherever
    # |a| is below the forward's operand rounding: each such entry moves a
    # gradient by (1 - alpha) dh, a 1-4 % floor (printed for the record).
    dE32 = dE.astype(np.float32).astype(np.float64)
    og, _ = O.image_mlp_bwd_from(p, a0[:U].double().cpu().numpy(), a1[:U].double().cpu().numpy(), dE32, rows_of,
                                 uniq)
    errs = {n: relmax(g[n].double().cpu().numpy(), og[n]) for n in names}
    ref_f64, _ = O.image_mlp_bwd_rows(p, cache, dE32, rows_of, uniq)
    print(f"U={U} {prec}: backward vs oracle from device activations",
          {n: f"{e:.1e}" for n, e in errs.items()}, "| from the oracle's own forward (branch flips included)",
          {n: f"{relmax(g[n].double().cpu().numpy(), ref_f64[n]):.1e}" for n in names})
    bad = {n: e for n, e in errs.items() if not e < tol}
    assert not bad, errs


def saved(buf, cap, width, prec):
    """Decode a saved-activation buffer: bf16 mode stores bf16 rows packed at
    the start of the (fp32-sized) buffer."""
    if prec != "bf16":
        return buf
    return buf.view(torch.bfloat16).reshape(-1)[:cap * width].reshape(cap, width).float()


def test_persistent_loops_wrap_at_small_sizes():
    """DICM_GRID_CAP=4 (read once per process) caps every persistent
    image-MLP grid at 4 CTAs (2 pairs), so the small tensor-core parity cases
    of test_gpu_tensorcore.py run 6-24 tiles per CTA and one dW0 row chunk."""
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, DICM_GRID_CAP="4")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(here, "test_gpu_tensorcore.py"), "-k",
                        "test_layer0_tensorcore_matches_fp32 or test_step_logits"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("epi", ["0", "1"])
def test_layer0_epilogue_variants_match_oracle(epi):
    """The non-default act0 epilogues of k_fwd4 (DICM_FWD4_EPI, read once per
    process: 1 = shared-memory transposes, also taken for an unaligned bias;
    0 = per-lane row stores) at U = 20k, bf16 and tf32, against the oracle."""
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, DICM_FWD4_EPI=epi)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(here, "test_gpu_bench_shapes.py"), "-k",
                        "test_image_mlp_at_bench_sizes_matches_oracle and 20000"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def _cfg_model(kind, P, vocab, b_max, pool_dtype):
    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema
    schema = default_schema(vocab, 4, vocab, 8, P, b_max=b_max)
    model = DicmModel(schema, AggregatorSpec(kind), None, seed=0)
    return schema, model


@pytest.mark.slow
def test_cfg2_full_step_matches_oracle():
    """One full cfg2 step (attn, B = 4096, L = 200, 1M pool, bf16 tensor
    cores -- the bench's configuration; ~561k unique images) in four checks:
      1. integer work bit-exact (unique images), logits and loss within the
         north star's 2e-2 of the pure f64 oracle (compact remap, chunked
         image MLP over the device pool's rows);
      2. everything downstream of the image embeddings (pooling, attention,
         head, BCE, their backward, dE, ID-row gradients) against the oracle
         run from the device's own E: fp32 vs f64, 1e-4;
      3. the image-MLP gradients against the oracle's backward from the
         device's saved activations and dE: within 2e-2 of their magnitude;
      4. the same batch through the fp32 CUDA-core engine against the pure
         oracle at 1e-4 on loss, logits and every gradient."""
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.engine import StepEngine
    from paper_1711_06505_b200.pool import ImagePool
    pool = bench_pool("bf16")
    schema, model = _cfg_model("attn", P_BENCH, 100_000, 200, "bf16")
    params = H.host_params(model)
    batch = synthetic_batch(np.random.default_rng(1000), schema, 4096, 200, P_BENCH)
    e = StepEngine(model, pool, "bf16")
    e.forward_backward(e.upload(batch))
    torch.cuda.synchronize()
    e.raise_status()
    cfg = H.oracle_cfg_of(model)
    ob = H.oracle_batch(batch)
    rows_of = rows_reader(pool)
    # 1. the pure oracle
    out = O.forward_backward(params, cfg, ob, rows_of, want_grads=False)
    U = len(out["uniq"])
    assert U > 500_000  # the multi-tile regime
    assert np.array_equal(e.unique_images(), out["uniq"])
    r1 = {"loss": O.rel_err(e.loss.item(), out["loss"]),
          "logits": O.rel_err(e.logits[:batch.size].cpu().numpy(), out["logits"]),
          "E": relmax(e.emb[:U].double().cpu().numpy(), out["E"])}
    print("cfg2 bf16 vs pure oracle:", r1)
    assert r1["loss"] < 2e-2 and r1["logits"] < 2e-2 and r1["E"] < 2e-2, r1
    # 2. downstream of E from the device's E
    E_dev = e.emb[:U].double().cpu().numpy()
    ds = O.forward_backward(params, cfg, ob, None, emb=E_dev)
    r2 = {"loss": O.rel_err(e.loss.item(), ds["loss"]),
          "logits": O.rel_err(e.logits[:batch.size].cpu().numpy(), ds["logits"]),
          "dE": O.rel_err(e.d_emb[:U].double().cpu().numpy(), ds["dE"]),
          "dE_of_max": relmax(e.d_emb[:U].double().cpu().numpy(), ds["dE"])}
    for n, g in H.dense_grads(e).items():
        if not n.startswith("img/") and not (n.startswith("attn/") and n.endswith("/1/b")):
            r2[n] = O.rel_err(g, ds["grads"][n])
    for f, (ids, rows_) in H.table_grads(e).items():
        u, r = ds["tgrads"][f]
        assert np.array_equal(ids, u), f
        r2["id_emb/" + f] = O.rel_err(rows_, r)
    print("cfg2 bf16 downstream of E:", {k: f"{v:.1e}" for k, v in r2.items()})
    bad = {k: v for k, v in r2.items() if k != "dE_of_max" and not v < 1e-4}
    assert not bad and r2["dE_of_max"] < 1e-3, bad or r2["dE_of_max"]
    # 3. the image-MLP backward from the device's activations and dE
    cap = e.net.cap
    og, _ = O.image_mlp_bwd_from(params, saved(e.net.act0, cap, 256, "bf16")[:U].double().cpu().numpy(),
                                 saved(e.net.act1, cap, 64, "bf16")[:U].double().cpu().numpy(),
                                 e.d_emb[:U].double().cpu().numpy(), rows_of, out["uniq"])
    r3 = {n: relmax(model.real_view(e.grad, n).double().cpu().numpy(), og[n]) for n in og}
    print("cfg2 bf16 image-MLP backward:", {k: f"{v:.1e}" for k, v in r3.items()})
    assert all(v < 2e-2 for v in r3.values()), r3
    # 4. the fp32 engine on the same (bf16-valued) rows vs the pure oracle
    del e
    torch.cuda.empty_cache()
    pool32 = ImagePool(pool.rows.float(), 1, 0, P_BENCH)
    e32 = StepEngine(model, pool32, "fp32")
    e32.forward_backward(e32.upload(batch))
    torch.cuda.synchronize()
    e32.raise_status()
    full = O.forward_backward(params, cfg, ob, rows_of)
    r4 = {"loss": O.rel_err(e32.loss.item(), full["loss"]),
          "logits": O.rel_err(e32.logits[:batch.size].cpu().numpy(), full["logits"]),
          "dE": O.rel_err(e32.d_emb[:U].double().cpu().numpy(), full["dE"])}
    for n, g in H.dense_grads(e32).items():
        if not (n.startswith("attn/") and n.endswith("/1/b")):
            r4[n] = O.rel_err(g, full["grads"][n])
    for f, (ids, rows_) in H.table_grads(e32).items():
        r4["id_emb/" + f] = O.rel_err(rows_, full["tgrads"][f][1])
    print("cfg2 fp32 engine vs pure oracle:", {k: f"{v:.1e}" for k, v in r4.items()})
    bad = {k: v for k, v in r4.items() if not v < 1e-4}
    assert not bad, bad


def _reference_dicm():
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "dicm")):
        pytest.skip("the reference install (baseline/_ref) is absent")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import dicm.data as RD
    import dicm.model as RM
    import dicm.training as RT
    return RD, RM, RT


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_cfg1_full_size_steps_match_oracle(prec):
    """BASELINE.json configs[0] at its stated size: sum pooling, B = 256,
    L = 50, 10k-image pool, 100k-row user/ad/behavior_items tables; two full
    training steps (Adam included) against the oracle trainer."""
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    schema, model = _cfg_model("sum", 10_000, 100_000, 50, "fp32")
    pool = ImagePool.synthetic(10_000, seed=0)
    params = H.host_params(model)
    rng = np.random.default_rng(1000)
    batches = [synthetic_batch(rng, schema, 256, 50, 10_000) for _ in range(2)]
    tr = LocalTrainer(model, pool, TrainConfig(batch_size=256), precision=prec)
    ot = O.OracleTrainer(params, H.oracle_cfg_of(model), pool.rows.double().cpu().numpy())
    tol = 1e-4 if prec == "fp32" else 2e-2
    for b in batches:
        loss = tr.train_batch(b)
        out = ot.train_batch(H.oracle_batch(b))
        assert O.rel_err(loss, out["loss"]) < tol
        assert O.rel_err(tr.engine.logits[:b.size].cpu().numpy(), out["logits"]) < tol
    snap = model.snapshot()
    for n, a in snap.items():
        exp = ot.p[n]
        if n.startswith("id_emb/"):
            # only touched rows moved; compare them all (100k-row tables)
            assert O.rel_err(a, exp) < (1e-4 if prec == "fp32" else 5e-3), n
        else:
            d = np.abs(a - exp) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(exp)))
            # Adam's normalised step: entries whose gradient is below fp32
            # rounding may move +-lr the other way (2 steps)
            assert np.all(d <= 2 * 2 * 0.001 + 1e-6) and (d > 1e-4).mean() <= 0.05, n


def test_cfg1_full_size_matches_reference_itself():
    """cfg1 against the unmodified reference (baseline/_ref, stock
    LocalTrainer.train_batch, training.py:66-91) on the same samples and the
    exact fp32 pool rows: two training steps, losses and parameters."""
    RD, RM, RT = _reference_dicm()
    from paper_1711_06505_b200.batch import synthetic_batch
    from paper_1711_06505_b200.pool import ImagePool
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    schema, model = _cfg_model("sum", 10_000, 100_000, 50, "fp32")
    pool = ImagePool.synthetic(10_000, seed=0)
    rows = pool.rows.double().cpu().numpy()
    rng = np.random.default_rng(1000)
    batches = [synthetic_batch(rng, schema, 256, 50, 10_000) for _ in range(2)]
    rs = RM.FeatureSchema(fields=[RM.FieldSpec(f.name, f.vocab, f.multi) for f in schema.fields], d_id=12,
                          d_raw=4096, d_img=12, b_max=50)

    class Ext:
        out_dim = 4096

    class Store:
        def __len__(self):
            return len(rows)

        def raw_features(self, ids, extractor):
            return rows[np.asarray(ids, dtype=np.int64)]

    rmodel = RM.DicmModel(rs, RM.AggregatorSpec("sum"), Ext(), seed=0)
    rtr = RT.LocalTrainer(rmodel, Store(), RT.TrainConfig(batch_size=256))
    tr = LocalTrainer(model, pool, TrainConfig(batch_size=256), precision="fp32")
    for b in batches:
        samples = []
        for i in range(b.size):
            kw = {f: int(v[i]) for f, v in b.onehot.items()}
            for f, (fl, of) in b.multihot.items():
                kw[f] = fl[of[i]:of[i + 1]].tolist()
            samples.append(RD.Sample(label=int(b.labels[i]), day=0, **kw))
        ref_loss = rtr.train_batch(samples)
        loss = tr.train_batch(b)
        assert O.rel_err(loss, ref_loss) < 1e-4
    snap, rsnap = model.snapshot(), rtr.snapshot()
    for n in rsnap:
        a, exp = snap[n], rsnap[n]
        d = np.abs(a - exp) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(exp)))
        assert np.all(d <= 2 * 2 * 0.001 + 1e-6) and (d > 1e-4).mean() <= 0.05, n
    for f, st in tr.table_state.items():
        assert np.array_equal(st.t, rtr.table_state[f].t), f
