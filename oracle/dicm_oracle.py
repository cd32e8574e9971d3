"""CPU oracle for the DICM / AMS training hot path -- TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference algorithm (reference package
``dicm``, /root/reference/pkg/src/dicm) for the path named by BASELINE.json's
north star: batch encoding, image-key dedup, the image MLP, sum / attentive /
multi-query pooling, sparse ID embeddings, the MLP head with BCE, the explicit
backward pass and both Adam variants.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
reference leg may import this module, and only as the checker.  The product
path (``paper_1711_06505_b200``) never calls it.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``); parity is therefore pinned, not assumed.

Where the reference builds a tape (``autograd.py``), this module writes the
backward pass out by hand; every formula cites the reference line it restates.
"""

from __future__ import annotations

import numpy as np

BETA1, BETA2, EPS = 0.9, 0.999, 1e-8  # reference optim.py:16-19


# ---------------------------------------------------------------------------
# configuration
# ---------------------------------------------------------------------------

def make_cfg(fields, d_id=12, d_raw=4096, d_img=12, b_max=32, query_fields=("ad", "ad_category"),
             kind="sum", normalize=True, hidden=32, mlp_widths=(128, 64), use_ad_image=True,
             use_behavior_images=True, towers=None):
    """Plain-dict model description. ``fields`` = [(name, vocab, multi)].

    ``towers`` = dict(user_fields, ad_fields, hidden, rep) describes the
    two-tower pre-rank model (reference PrerankModel, model.py:420-531)
    instead of the MLP head; ``fields`` are then the tower fields only (the
    reference builds tables for those alone, model.py:470-475), the
    aggregator is "sum" and both image flags equal ``use_images``."""
    h1, h2 = max(d_raw // 16, d_img), max(d_raw // 64, d_img)  # reference model.py:88-91
    names = [f[0] for f in fields]
    qf = [q for q in query_fields if q in names]
    if towers is not None:
        towers = dict(user_fields=tuple(towers["user_fields"]), ad_fields=tuple(towers["ad_fields"]),
                      hidden=int(towers["hidden"]), rep=int(towers["rep"]))
        keep = set(towers["user_fields"]) | set(towers["ad_fields"])
        fields = [f for f in fields if f[0] in keep]
        kind = "sum"
    return dict(fields=[tuple(f) for f in fields], d_id=d_id, d_raw=d_raw, d_img=d_img,
                b_max=b_max, query_fields=qf, kind=kind, normalize=normalize, hidden=hidden,
                mlp_widths=tuple(mlp_widths), use_ad_image=use_ad_image,
                use_behavior_images=use_behavior_images, h1=h1, h2=h2, towers=towers)


# ---------------------------------------------------------------------------
# elementwise pieces (reference autograd.py)
# ---------------------------------------------------------------------------

def prelu(x, a):
    """autograd.py:219-220: x > 0 ? x : a*x (x == 0 takes the alpha branch)."""
    return np.where(x > 0, x, a * x)


def prelu_bwd(x, a, g):
    """autograd.py:222-225 -> (dx, dalpha summed over rows)."""
    pos = x > 0
    dx = np.where(pos, g, a * g)
    da = np.where(pos, 0.0, x * g)
    return dx, (da if x.ndim == 1 else da.sum(axis=0))


def seg_of(off):
    """CSR offsets [B+1] -> segment id per row (the reference's ``seg``)."""
    counts = np.diff(off)
    return np.repeat(np.arange(len(counts)), counts)


def segment_sum(x, seg, n):
    """autograd.py:275-287 (np.add.at in row order)."""
    out = np.zeros((n,) + x.shape[1:])
    np.add.at(out, seg, x)
    return out


def segment_max(x, seg, n):
    """Per-segment elementwise max, empty segments -> 0, first argmax per
    column (reference autograd.py:289-319)."""
    x = np.asarray(x, dtype=np.float64)
    R, d = x.shape
    out = np.zeros((n, d))
    arg = np.full((n, d), -1, dtype=np.int64)
    filled = np.zeros(n, dtype=bool)
    for r in range(R):
        s_ = seg[r]
        if not filled[s_]:
            out[s_] = x[r]
            arg[s_] = r
            filled[s_] = True
        else:
            better = x[r] > out[s_]
            out[s_] = np.where(better, x[r], out[s_])
            arg[s_] = np.where(better, r, arg[s_])
    return out, arg


def segment_softmax(s, seg, n):
    """autograd.py:322-332."""
    hi = np.full(n, -np.inf)
    np.maximum.at(hi, seg, s)
    e = np.exp(s - hi[seg])
    denom = np.zeros(n)
    np.add.at(denom, seg, e)
    return e / denom[seg]


def bce(z, y):
    """autograd.py:240-241 -> (per-sample loss, sigmoid)."""
    out = np.maximum(z, 0.0) - z * y + np.log1p(np.exp(-np.abs(z)))
    return out, 1.0 / (1.0 + np.exp(-z))


def dedup(keys):
    """Sorted distinct keys and the inverse index: ``np.unique`` (model.py:187)
    followed by ``np.searchsorted(unique, ids)`` (model.py:374, 378)."""
    keys = np.asarray(keys, dtype=np.int64)
    uniq = np.unique(keys)
    return uniq, np.searchsorted(uniq, keys)


# ---------------------------------------------------------------------------
# encode (reference model.py:158-198)
# ---------------------------------------------------------------------------

def encode(samples, cfg):
    """list of sample dicts/objects -> CSR batch dict.  Behavior lists keep
    their last b_max entries (model.py:168, 176)."""
    b_max = cfg["b_max"]
    get = (lambda s, k: s[k]) if samples and isinstance(samples[0], dict) else getattr
    out = {"size": len(samples), "onehot": {}, "multihot": {}}
    for name, _vocab, multi in cfg["fields"]:
        if multi:
            lists = [list(get(s, name))[-b_max:] if b_max else [] for s in samples]
            out["multihot"][name] = _csr(lists)
        else:
            out["onehot"][name] = np.array([get(s, name) for s in samples], dtype=np.int64)
    beh = [list(get(s, "behavior_images"))[-b_max:] for s in samples]
    out["beh_image_ids"], out["beh_off"] = _csr(beh)
    out["ad_image_ids"] = np.array([get(s, "ad_image") for s in samples], dtype=np.int64)
    out["labels"] = np.array([get(s, "label") for s in samples], dtype=np.float64)
    return out


def _csr(lists):
    off = np.zeros(len(lists) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(x) for x in lists])
    flat = np.array([i for x in lists for i in x], dtype=np.int64)
    return flat, off


def needed_image_keys(cfg, batch):
    """model.py:182-187: ad images iff use_ad_image, behaviors iff
    use_behavior_images."""
    parts = []
    if cfg["use_ad_image"]:
        parts.append(np.asarray(batch["ad_image_ids"], dtype=np.int64))
    if cfg["use_behavior_images"]:
        parts.append(np.asarray(batch["beh_image_ids"], dtype=np.int64))
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


# ---------------------------------------------------------------------------
# image MLP (reference model.py:108-120, autograd.py:194-227)
# ---------------------------------------------------------------------------

def image_mlp_fwd(p, X):
    a0 = X @ p["img/0/w"].T + p["img/0/b"]
    h1 = prelu(a0, p["img/0/a"])
    a1 = h1 @ p["img/1/w"].T + p["img/1/b"]
    h2 = prelu(a1, p["img/1/a"])
    E = h2 @ p["img/2/w"].T + p["img/2/b"]
    return E, (X, a0, h1, a1, h2)


def image_mlp_bwd(p, cache, dE):
    """linear bwd autograd.py:201-204 (w: g.T @ x, b: g.sum(0)); the input
    gradient of layer 0 is not formed -- the features are frozen leaves."""
    X, a0, h1, a1, h2 = cache
    g = {}
    g["img/2/w"] = dE.T @ h2
    g["img/2/b"] = dE.sum(axis=0)
    dh2 = dE @ p["img/2/w"]
    da1, g["img/1/a"] = prelu_bwd(a1, p["img/1/a"], dh2)
    g["img/1/w"] = da1.T @ h1
    g["img/1/b"] = da1.sum(axis=0)
    dh1 = da1 @ p["img/1/w"]
    da0, g["img/0/a"] = prelu_bwd(a0, p["img/0/a"], dh1)
    g["img/0/w"] = da0.T @ X
    g["img/0/b"] = da0.sum(axis=0)
    return g, da0


def image_mlp_fwd_rows(p, rows_of, uniq, chunk=1 << 15):
    """image_mlp_fwd over ``rows_of(ids) -> [n, d_raw] f64`` in row chunks,
    for row counts whose [U, d_raw] f64 feature matrix does not fit host
    memory (the compact monotone remap of SURVEY.md 8c: every op is row-local,
    so chunking changes nothing but the order of the f64 sums).  The cache
    keeps the activations, not X: the backward re-reads the rows."""
    U = len(uniq)
    E = np.zeros((U, p["img/2/w"].shape[0]))
    a0s, h1s, a1s, h2s = [], [], [], []
    for s0 in range(0, U, chunk):
        e, (_, a0, h1, a1, h2) = image_mlp_fwd(p, rows_of(uniq[s0:s0 + chunk]))
        E[s0:s0 + len(e)] = e
        a0s.append(a0), h1s.append(h1), a1s.append(a1), h2s.append(h2)
    cat = (lambda xs, w: np.concatenate(xs) if xs else np.zeros((0, w)))
    return E, (None, cat(a0s, p["img/0/w"].shape[0]), cat(h1s, p["img/0/w"].shape[0]),
               cat(a1s, p["img/1/w"].shape[0]), cat(h2s, p["img/1/w"].shape[0]))


def image_mlp_bwd_rows(p, cache, dE, rows_of, uniq, chunk=1 << 15):
    """image_mlp_bwd with dW0 = da0^T X accumulated over row chunks of X."""
    _, a0, h1, a1, h2 = cache
    g, da0 = image_mlp_bwd(p, (np.zeros((len(uniq), 0)), a0, h1, a1, h2), dE)
    gw0 = np.zeros((a0.shape[1], p["img/0/w"].shape[1]))
    for s0 in range(0, len(uniq), chunk):
        gw0 += da0[s0:s0 + chunk].T @ rows_of(uniq[s0:s0 + chunk])
    g["img/0/w"] = gw0
    return g, da0


def image_mlp_bwd_from(p, a0, a1, dE, rows_of, uniq, chunk=1 << 15):
    """image_mlp_bwd from given pre-activations a0 [U, h1], a1 [U, h2] (a
    device's saved activations): the PReLU branches are those the device took,
    so the comparison isolates the backward kernels' own rounding -- a flipped
    branch (|a| below the forward's operand rounding) would otherwise move a
    gradient entry by a full (1 - alpha) dh."""
    h1 = prelu(a0, p["img/0/a"])
    h2 = prelu(a1, p["img/1/a"])
    return image_mlp_bwd_rows(p, (None, a0, h1, a1, h2), dE, rows_of, uniq, chunk)


# ---------------------------------------------------------------------------
# attentive pooling (reference model.py:206-215, autograd.py:322-352)
# ---------------------------------------------------------------------------

def attention_fwd(p, prefix, Q, K, seg, n, normalize):
    q = Q[seg]
    inp = np.hstack([q, K])
    pre = inp @ p[prefix + "0/w"].T + p[prefix + "0/b"]
    h = prelu(pre, p[prefix + "0/a"])
    s = (h @ p[prefix + "1/w"].T + p[prefix + "1/b"])[:, 0]
    w = segment_softmax(s, seg, n) if normalize else s
    out = segment_sum(K * w[:, None], seg, n)
    return out, (inp, pre, h, w)


def attention_bwd(p, prefix, K, seg, n, normalize, cache, dout, grads):
    """-> (dQ [n, dq], dK [R, d]); parameter grads accumulate into ``grads``."""
    inp, pre, h, w = cache
    g = dout[seg]                                   # segment_sum bwd  (autograd.py:284-285)
    dK = g * w[:, None]                             # col_scale bwd    (autograd.py:348-350)
    dw = (g * K).sum(axis=1)
    if normalize:                                   # segment_softmax bwd (autograd.py:334-337)
        dot = np.zeros(n)
        np.add.at(dot, seg, dw * w)
        ds = w * (dw - dot[seg])
    else:
        ds = dw
    w1 = p[prefix + "1/w"]
    grads[prefix + "1/w"] = ds[None, :] @ h
    grads[prefix + "1/b"] = np.array([ds.sum()])
    dh = ds[:, None] @ w1
    dpre, grads[prefix + "0/a"] = prelu_bwd(pre, p[prefix + "0/a"], dh)
    grads[prefix + "0/w"] = dpre.T @ inp
    grads[prefix + "0/b"] = dpre.sum(axis=0)
    dinp = dpre @ p[prefix + "0/w"]
    dq_rows = dinp[:, : inp.shape[1] - K.shape[1]]
    dK = dK + dinp[:, inp.shape[1] - K.shape[1]:]
    dQ = segment_sum(dq_rows, seg, n)               # rows bwd (autograd.py:267-271)
    return dQ, dK


# ---------------------------------------------------------------------------
# full forward / backward (reference model.py:358-401, training.py:39-42)
# ---------------------------------------------------------------------------

def forward_backward(p, cfg, batch, pool, denominator=None, want_grads=True, emb=None):
    """Loss, logits and every parameter gradient of one batch.

    ``p``: name -> float64 array (tables included).  ``pool``: [P, d_raw]
    rows the image ids index (the exact rows the device pool holds).
    Table gradients come back compact: ``tgrads[field] = (uniq_ids, rows)``,
    the dense reference gradient restricted to the rows touched.

    ``emb``: image embeddings [U, d_img] aligned with the batch's sorted unique
    images, used instead of the image MLP (whose gradients are then not
    formed): checks everything downstream of E against a device's own E.
    """
    B = batch["size"]
    denom = B if denominator is None else denominator
    d_id = cfg["d_id"]
    keys = needed_image_keys(cfg, batch)
    uniq, _ = dedup(keys)
    if emb is not None:
        E, img_cache = np.asarray(emb, dtype=np.float64), None
    elif callable(pool):  # rows on demand (chunked image MLP)
        E, img_cache = image_mlp_fwd_rows(p, pool, uniq)
    else:
        X = np.asarray(pool, dtype=np.float64)[uniq] if len(uniq) else np.zeros((0, cfg["d_raw"]))
        E, img_cache = image_mlp_fwd(p, X)

    parts, field_vecs, field_info = [], {}, {}
    for name, _vocab, multi in cfg["fields"]:
        T = p[f"id_emb/{name}"]
        if multi:
            flat, off = batch["multihot"][name]
            seg = seg_of(off)
            vec = segment_sum(T[flat], seg, B)
            field_info[name] = (np.asarray(flat), seg)
        else:
            ids = np.asarray(batch["onehot"][name])
            vec = T[ids]
            field_info[name] = (ids, None)
        field_vecs[name] = vec
        parts.append(vec)
    ad_local = beh_local = None
    if cfg["use_ad_image"]:
        ad_local = np.searchsorted(uniq, batch["ad_image_ids"])
        ad_vec = E[ad_local]
        parts.append(ad_vec)
    agg_cache = None
    if cfg["use_behavior_images"]:
        beh_local = np.searchsorted(uniq, batch["beh_image_ids"])
        beh_seg = seg_of(batch["beh_off"])
        K = E[beh_local]
        kind = cfg["kind"]
        if kind == "sum":
            pooled = segment_sum(K, beh_seg, B)
        elif kind == "max":
            pooled, argmax = segment_max(K, beh_seg, B)
            agg_cache = (argmax,)
        elif kind == "concat":                       # scatter_concat (autograd.py:370-385)
            pos = np.arange(len(beh_seg)) - np.asarray(batch["beh_off"])[beh_seg]
            d = cfg["d_img"]
            pooled = np.zeros((B, cfg["b_max"] * d))
            cols = pos[:, None] * d + np.arange(d)[None, :]
            np.add.at(pooled, (beh_seg[:, None], cols), K)
            agg_cache = (cols,)
        elif kind == "attn":
            pooled, c1 = attention_fwd(p, "attn/img/", ad_vec, K, beh_seg, B, cfg["normalize"])
            agg_cache = (c1,)
        elif kind == "multiquery-attn":
            qid = np.hstack([field_vecs[q] for q in cfg["query_fields"]])
            o1, c1 = attention_fwd(p, "attn/img/", ad_vec, K, beh_seg, B, cfg["normalize"])
            o2, c2 = attention_fwd(p, "attn/id/", qid, K, beh_seg, B, cfg["normalize"])
            pooled = np.hstack([o1, o2])
            agg_cache = (c1, c2)
        else:
            raise ValueError(f"aggregator {kind!r} is outside the hot path")
        parts.append(pooled)
    x = np.hstack(parts)
    y = np.asarray(batch["labels"], dtype=np.float64)
    if cfg.get("towers"):
        z, tower_cache = towers_fwd(p, cfg, field_vecs, ad_vec if cfg["use_ad_image"] else None,
                                    pooled if cfg["use_behavior_images"] else None)
    else:
        acts = [x]
        nh = len(cfg["mlp_widths"])
        pre_acts = []
        for i in range(nh):
            a = acts[-1] @ p[f"mlp/{i}/w"].T + p[f"mlp/{i}/b"]
            pre_acts.append(a)
            acts.append(prelu(a, p[f"mlp/{i}/a"]))
        z = (acts[-1] @ p[f"mlp/{nh}/w"].T + p[f"mlp/{nh}/b"])[:, 0]
    per, sig = bce(z, y)
    loss = per.sum() / denom
    out = {"loss": loss, "logits": z, "uniq": uniq, "E": E, "ad_local": ad_local,
           "beh_local": beh_local}
    if not want_grads:
        return out

    grads = {}
    dz = (sig - y) / denom                           # autograd.py:243-244 * scale(1/denominator)
    if cfg.get("towers"):
        dx = towers_bwd(p, cfg, tower_cache, dz, x.shape[1], grads)
    else:
        grads[f"mlp/{nh}/w"] = dz[None, :] @ acts[-1]
        grads[f"mlp/{nh}/b"] = np.array([dz.sum()])
        dh = dz[:, None] @ p[f"mlp/{nh}/w"]
        for i in reversed(range(nh)):
            da, grads[f"mlp/{i}/a"] = prelu_bwd(pre_acts[i], p[f"mlp/{i}/a"], dh)
            grads[f"mlp/{i}/w"] = da.T @ acts[i]
            grads[f"mlp/{i}/b"] = da.sum(axis=0)
            dh = da @ p[f"mlp/{i}/w"]
        dx = dh

    dE = np.zeros_like(E)
    dfield = {}
    off = 0
    for name, _vocab, _multi in cfg["fields"]:
        dfield[name] = dx[:, off: off + d_id].copy()
        off += d_id
    if cfg["use_ad_image"]:
        d_ad = dx[:, off: off + cfg["d_img"]].copy()
        off += cfg["d_img"]
    if cfg["use_behavior_images"]:
        dpool = dx[:, off:]
        kind = cfg["kind"]
        if kind == "sum":
            dK = dpool[beh_seg]
        elif kind == "concat":
            dK = dpool[beh_seg[:, None], agg_cache[0]]
        elif kind == "max":                          # segment_max bwd (autograd.py:307-315)
            dK = np.zeros_like(K)
            argmax = agg_cache[0]
            for s_ in range(B):
                for c in range(K.shape[1]):
                    if argmax[s_, c] >= 0:
                        dK[argmax[s_, c], c] += dpool[s_, c]
        elif kind == "attn":
            dQ, dK = attention_bwd(p, "attn/img/", K, beh_seg, B, cfg["normalize"], agg_cache[0],
                                   dpool, grads)
            d_ad += dQ
        else:
            d = cfg["d_img"]
            dQ1, dK1 = attention_bwd(p, "attn/img/", K, beh_seg, B, cfg["normalize"],
                                     agg_cache[0], dpool[:, :d], grads)
            dQ2, dK2 = attention_bwd(p, "attn/id/", K, beh_seg, B, cfg["normalize"],
                                     agg_cache[1], dpool[:, d:], grads)
            d_ad += dQ1
            dK = dK1 + dK2
            qo = 0
            for q in cfg["query_fields"]:
                dfield[q] += dQ2[:, qo: qo + d_id]
                qo += d_id
        np.add.at(dE, beh_local, dK)                 # rows bwd (autograd.py:267-271)
    if cfg["use_ad_image"]:
        np.add.at(dE, ad_local, d_ad)

    tgrads = {}
    for name, _vocab, multi in cfg["fields"]:
        ids, seg = field_info[name]
        g = dfield[name][seg] if multi else dfield[name]
        u, inv = dedup(ids)
        rows = np.zeros((len(u), d_id))
        np.add.at(rows, inv, g)
        tgrads[name] = (u, rows)

    if img_cache is None:
        ig, da0 = {}, None
    elif callable(pool):
        ig, da0 = image_mlp_bwd_rows(p, img_cache, dE, pool, uniq)
    else:
        ig, da0 = image_mlp_bwd(p, img_cache, dE)
    grads.update(ig)
    out.update(grads=grads, tgrads=tgrads, dE=dE, da0=da0)
    return out


# ---------------------------------------------------------------------------
# two-tower pre-rank (reference PrerankModel, model.py:420-531)
# ---------------------------------------------------------------------------

def _tower_parts(cfg, tower):
    """Column blocks of one tower's input in hstack order (model.py:510-520):
    its fields in the tower's order, then the pooled behavior images (user
    tower) or the ad image (ad tower) when images are used.  Each entry is
    the block's (column offset, width) in the head-input layout of ``forward_backward``
    (fields in schema order, ad image, pooled)."""
    d = cfg["d_id"]
    names = [f[0] for f in cfg["fields"]]
    tw = cfg["towers"]
    cols = [(names.index(f) * d, d) for f in tw[tower + "_fields"]]
    img_col, di = len(names) * d, cfg["d_img"]
    if tower == "user" and cfg["use_behavior_images"]:
        cols.append((img_col + (di if cfg["use_ad_image"] else 0), di))
    if tower == "ad" and cfg["use_ad_image"]:
        cols.append((img_col, di))
    return cols


def towers_fwd(p, cfg, field_vecs, ad_vec, pooled):
    """Both towers (``_tower``, model.py:503-506: PReLU layer, then a linear
    layer) and the row-wise inner product (autograd.py:388-392)."""
    tw = cfg["towers"]
    cache = {}
    reps = {}
    for tower, extra in (("user", pooled), ("ad", ad_vec)):
        parts = [field_vecs[f] for f in tw[tower + "_fields"]]
        if extra is not None:
            parts.append(extra)
        xin = np.hstack(parts) if len(parts) > 1 else parts[0]
        pre = xin @ p[f"{tower}_tower/0/w"].T + p[f"{tower}_tower/0/b"]
        h = prelu(pre, p[f"{tower}_tower/0/a"])
        reps[tower] = h @ p[f"{tower}_tower/1/w"].T + p[f"{tower}_tower/1/b"]
        cache[tower] = (xin, pre, h)
    cache["reps"] = reps
    return np.einsum("ij,ij->i", reps["user"], reps["ad"]), cache


def towers_bwd(p, cfg, cache, dz, width, grads):
    """rowwise_dot bwd (autograd.py:394-396), then each tower's linear / PReLU
    backward; returns d(head input) in the ``forward_backward`` column layout."""
    reps = cache["reps"]
    dx = np.zeros((len(dz), width))
    for tower, other in (("user", "ad"), ("ad", "user")):
        xin, pre, h = cache[tower]
        pre_ = f"{tower}_tower/"
        dr = dz[:, None] * reps[other]
        grads[pre_ + "1/w"] = dr.T @ h
        grads[pre_ + "1/b"] = dr.sum(axis=0)
        dh = dr @ p[pre_ + "1/w"]
        dpre, grads[pre_ + "0/a"] = prelu_bwd(pre, p[pre_ + "0/a"], dh)
        grads[pre_ + "0/w"] = dpre.T @ xin
        grads[pre_ + "0/b"] = dpre.sum(axis=0)
        dxin = dpre @ p[pre_ + "0/w"]
        k = 0
        for c, w in _tower_parts(cfg, tower):
            dx[:, c:c + w] += dxin[:, k:k + w]
            k += w
    return dx


# ---------------------------------------------------------------------------
# optimizer (reference optim.py)
# ---------------------------------------------------------------------------

def lr_schedule(iteration, lr0=0.001, decay=0.9, interval=24000):
    """optim.py:24-28."""
    return lr0 * decay ** (iteration // interval)


def adam_step(value, grad, state, lr):
    """optim.py:44-63: skip an all-zero gradient, raise on non-finite."""
    if not np.all(np.isfinite(grad)):
        raise FloatingPointError("adam: non-finite gradient, parameter untouched")
    if not grad.any():
        return
    state["t"] += 1
    t = state["t"]
    state["m"] = BETA1 * state["m"] + (1.0 - BETA1) * grad
    state["v"] = BETA2 * state["v"] + (1.0 - BETA2) * grad * grad
    m_hat = state["m"] / (1.0 - BETA1 ** t)
    v_hat = state["v"] / (1.0 - BETA2 ** t)
    value -= lr * m_hat / (np.sqrt(v_hat) + EPS)


def adam_rows(table, ids, grads, st, lr):
    """optim.py:83-104: per-row step counter, zero rows skipped."""
    for rid, g in zip(ids, grads):
        if not g.any():
            continue
        st["t"][rid] += 1
        t = int(st["t"][rid])
        st["m"][rid] = BETA1 * st["m"][rid] + (1.0 - BETA1) * g
        st["v"][rid] = BETA2 * st["v"][rid] + (1.0 - BETA2) * g * g
        m_hat = st["m"][rid] / (1.0 - BETA1 ** t)
        v_hat = st["v"][rid] / (1.0 - BETA2 ** t)
        table[rid] -= lr * m_hat / (np.sqrt(v_hat) + EPS)


class OracleTrainer:
    """training.py:45-91 restated: dense Adam on worker + image params, row
    Adam on the unique ids of each table, lr by the iteration counter."""

    def __init__(self, params, cfg, pool, lr0=0.001, decay=0.9, interval=24000):
        self.p = {k: np.array(v, dtype=np.float64, copy=True) for k, v in params.items()}
        self.cfg = cfg
        self.pool = pool
        self.lr0, self.decay, self.interval = lr0, decay, interval
        self.iteration = 0
        self.dense = sorted(n for n in self.p if not n.startswith("id_emb/"))
        self.state = {n: {"m": np.zeros_like(self.p[n]), "v": np.zeros_like(self.p[n]), "t": 0}
                      for n in self.dense}
        self.tstate = {}
        for name, vocab, _ in cfg["fields"]:
            T = self.p[f"id_emb/{name}"]
            self.tstate[name] = {"m": np.zeros_like(T), "v": np.zeros_like(T),
                                 "t": np.zeros(T.shape[0], dtype=np.int64)}

    def train_batch(self, batch, denominator=None):
        out = forward_backward(self.p, self.cfg, batch, self.pool, denominator)
        if not np.isfinite(out["loss"]):
            raise FloatingPointError(f"non-finite loss at iteration {self.iteration}")
        lr = lr_schedule(self.iteration, self.lr0, self.decay, self.interval)
        for n in self.dense:
            adam_step(self.p[n], out["grads"][n], self.state[n], lr)
        for name, _v, _m in self.cfg["fields"]:
            u, rows = out["tgrads"][name]
            adam_rows(self.p[f"id_emb/{name}"], u, rows, self.tstate[name], lr)
        self.iteration += 1
        return out


def rel_err(a, b):
    """The reference's comparison metric (tests/test_autograd.py:10-11),
    elementwise max: |a-b| / max(1, |a|, |b|)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))
