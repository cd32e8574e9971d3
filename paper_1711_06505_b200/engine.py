"""The device training step (single GPU): the kernel sequence behind
``LocalTrainer.train_batch`` (reference training.py:66-91).

One step, all on one CUDA stream, no host round trip until the loss is read:

  H2D   one packed copy of the CSR batch (ids, offsets, labels)
  a2    dicm_dedup over the image keys  -> unique rows + inverse
  a2    dicm_dedup over every ID field  -> unique (field,row) keys + inverse
  a3-a4 dicm_imgmlp_fwd on the unique rows -> E [U,12]
  a6-10 dicm_sample_fwd -> head input x [B, W]
  a11-12 dicm_head_fwd_bwd -> logits, dLoss/dx, head-grad partials
  a6-10 dicm_sample_bwd -> dE [U,12], dRows [K,12], attention-grad partials
  a5    dicm_imgmlp_bwd -> img/* gradients
  a14   dicm_adam_dense (all dense params) + dicm_adam_rows (unique ID rows)

Buffers are sized by capacity and reused; the dedup counts never leave the
device.  Status words latch out-of-vocabulary ids and non-finite values; the
update kernels refuse to run on a flagged step and the host raises the
reference's exception when it reads the status.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from .model import KIND_CODE

BETA1, BETA2, EPS = 0.9, 0.999, 1e-8  # reference optim.py:16-19


def lr_schedule(iteration, lr0=0.001, decay=0.9, interval=24000):
    """reference optim.py:24-28."""
    if iteration < 0:
        raise ValueError(f"iteration must be >= 0, got {iteration}")
    return lr0 * decay ** (iteration // interval)


def _u8(n, dev):
    return torch.empty(max(int(n), 1), dtype=torch.uint8, device=dev)


class Packed:
    """Offsets of one batch inside the packed int32 upload buffer."""

    def __init__(self, model, batch):
        self.B = batch.size
        self.R = batch.refs
        off = 0
        self.onehot, self.multi = {}, {}
        for f in model.schema.fields:
            if f.multi:
                flat, o = batch.multihot[f.name]
                self.multi[f.name] = (off, len(flat), off + len(flat))
                off += len(flat) + self.B + 1
            else:
                self.onehot[f.name] = off
                off += self.B
        self.ad = off
        self.beh = off + self.B
        off += self.B + self.R
        self.beh_off = off
        off += self.B + 1
        self.labels = off
        off += self.B
        self.total = off

    def fill(self, model, batch, host):
        for f in model.schema.fields:
            if f.multi:
                a, n, o = self.multi[f.name]
                flat, offs = batch.multihot[f.name]
                host[a:a + n] = flat
                host[o:o + self.B + 1] = offs
            else:
                host[self.onehot[f.name]:self.onehot[f.name] + self.B] = batch.onehot[f.name]
        host[self.ad:self.ad + self.B] = batch.ad_image_ids
        host[self.beh:self.beh + self.R] = batch.beh_image_ids
        host[self.beh_off:self.beh_off + self.B + 1] = batch.beh_off
        host[self.labels:self.labels + self.B] = np.asarray(batch.labels, dtype=np.float32).view(np.int32)


class DeviceBatch:
    __slots__ = ("pk", "packed")

    def __init__(self, pk, packed):
        self.pk, self.packed = pk, packed


class StepEngine:
    """Owns the optimizer state and the step buffers of one model replica."""

    def __init__(self, model, pool, precision="fp32", lr0=0.001, lr_decay=0.9, lr_interval=24000):
        if precision not in L.PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(L.PRECISIONS)}")
        if precision == "bf16" and pool.dtype_name != "bf16":
            raise ValueError("bf16 tensor-core mode needs a bf16 pool")
        if pool.d_raw != model.schema.d_raw:
            raise ValueError(f"pool rows are {pool.d_raw}-D, schema expects {model.schema.d_raw}")
        self.model, self.pool = model, pool
        self.precision = precision
        self.prec_code = L.PRECISIONS[precision]
        self.lr0, self.lr_decay, self.lr_interval = lr0, lr_decay, lr_interval
        self.iteration = 0
        dev = self.dev = model.device
        lay = model.layout
        self.fields = list(model.schema.fields)
        # ID key space: tables back to back
        self.bases, base = [], 0
        for f in self.fields:
            self.bases.append(base)
            base += model.tables[f.name].shape[0]
        self.id_key_space = base
        self.status = torch.zeros(L.STATUS_WORDS, dtype=torch.int32, device=dev)
        # optimizer state (reference training.py:53-60)
        self.grad = torch.zeros_like(model.dense)
        self.m = torch.zeros_like(model.dense)
        self.v = torch.zeros_like(model.dense)
        self.spans = (L.Span * len(model.dense_spans))()
        self.span_index = {}
        for i, (o, size, n) in enumerate(model.dense_spans):
            self.spans[i].offset, self.spans[i].size = o, size
            if n is not None:
                self.span_index[n] = i
        self.t = torch.zeros(len(model.dense_spans), dtype=torch.int32, device=dev)
        self.adam_ws = _u8(L.lib.dicm_adam_dense_workspace(len(model.dense_spans)), dev)
        self.tm = {f.name: torch.zeros_like(model.tables[f.name]) for f in self.fields}
        self.tv = {f.name: torch.zeros_like(model.tables[f.name]) for f in self.fields}
        self.tt = {f.name: torch.zeros(model.tables[f.name].shape[0], dtype=torch.int32, device=dev)
                   for f in self.fields}
        self.tabstate = (L.TableState * len(self.fields))()
        for i, f in enumerate(self.fields):
            ts = self.tabstate[i]
            ts.table, ts.m, ts.v, ts.t = (model.tables[f.name].data_ptr(), self.tm[f.name].data_ptr(),
                                         self.tv[f.name].data_ptr(), self.tt[f.name].data_ptr())
            ts.base, ts.vocab = self.bases[i], model.tables[f.name].shape[0]
        self.ws_id = _u8(L.lib.dicm_dedup_workspace(max(self.id_key_space, 1)), dev)
        self.ws_img = _u8(L.lib.dicm_dedup_workspace(max(pool.local_rows, 1)), dev)
        # static kernel descriptors
        self.layout = self._layout_struct()
        self.attn = (L.AttnParams * 2)()
        if lay.attentive:
            for ch, pre in ((0, "attn/img/"), (1, "attn/id/")):
                if ch == 1 and not lay.multiquery:
                    continue
                a = self.attn[ch]
                a.w0 = model.params[pre + "0/w"].tensor.data_ptr()
                a.b0 = model.params[pre + "0/b"].tensor.data_ptr()
                a.a0 = model.params[pre + "0/a"].tensor.data_ptr()
                a.w1 = model.params[pre + "1/w"].tensor.data_ptr()
                a.b1 = model.params[pre + "1/b"].tensor.data_ptr()
        p = lambda n: model.params[n].tensor.data_ptr()  # noqa: E731
        g = lambda n: model.dense_view(self.grad, n).data_ptr()  # noqa: E731
        names = ("w0", "b0", "a0", "w1", "b1", "a1", "w2", "b2")
        pnames = ("img/0/w", "img/0/b", "img/0/a", "img/1/w", "img/1/b", "img/1/a", "img/2/w", "img/2/b")
        self.img_p = L.ImgMlpParams(**{k: p(n) for k, n in zip(names, pnames)})
        self.img_g = L.ImgMlpGrads(**{k: g(n) for k, n in zip(names, pnames)})
        hn = ("mlp/0/w", "mlp/0/b", "mlp/0/a", "mlp/1/w", "mlp/1/b", "mlp/1/a", "mlp/2/w", "mlp/2/b")
        self.head_p = L.HeadParams(**{k: p(n) for k, n in zip(names, hn)})
        self.width = lay.mlp_input_width()
        self.head_range = model.group_range("mlp/")
        assert self.head_range[1] - self.head_range[0] == L.lib.dicm_head_partial_size(self.width)
        self.attn_range = model.group_range("attn/")
        self.attn_part = int(L.lib.dicm_attn_partial_size(C.byref(self.layout)))
        if self.attn_range is not None:
            assert self.attn_range[1] - self.attn_range[0] == self.attn_part
        self.cap = None
        self.probe = None  # name -> [(start, end)] CUDA events around the image-MLP launches
        self._pinned = [None, None]
        self._pin_ev = [None, None]
        self._pin_i = 0

    # ------------------------------------------------------------------
    def _layout_struct(self):
        m = self.model
        lay = m.layout
        ho = m.head_offsets
        st = L.Layout()
        st.kind = KIND_CODE[lay.aggregator.kind]
        st.normalize = int(bool(lay.aggregator.normalize))
        st.use_ad_image = int(lay.use_ad_image)
        st.use_behavior_images = int(lay.use_behavior_images)
        st.n_fields = len(self.fields)
        for i, f in enumerate(self.fields):
            st.field_multi[i] = int(f.multi)
            st.field_col[i] = ho["field/" + f.name]
        st.ad_col = ho.get("ad_image_emb", -1)
        st.pool_col = ho.get("pool", -1)
        st.width = ho["width"]
        qf = lay.query_fields_present() if lay.multiquery else []
        st.n_query = len(qf)
        names = [f.name for f in self.fields]
        for i, q in enumerate(qf):
            st.query_field[i] = names.index(q)
            st.query_col[i] = ho["field/" + q]
        return st

    def _ensure(self, pk):
        B, R = pk.B, pk.R
        n_id = sum(B if not f.multi else pk.multi[f.name][1] for f in self.fields)
        need = (pk.total, B, R, n_id)
        if self.cap is not None and all(a <= b for a, b in zip(need, self.cap)):
            return
        if self.cap is not None:  # grow with headroom
            need = tuple(max(int(a * 1.25), b) for a, b in zip(need, self.cap))
        total, B, R, n_id = need
        dev = self.dev
        lay = self.model.layout
        n_img = (B if lay.use_ad_image else 0) + (R if lay.use_behavior_images else 0)
        self.cap_u = min(n_img, self.pool.local_rows)
        self.cap_k = min(n_id, self.id_key_space)
        i32 = dict(dtype=torch.int32, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.packed = torch.empty(max(total, 1), **i32)
        self.uniq_img = torch.empty(max(self.cap_u, 1), **i32)
        self.inv_img = torch.empty(max(n_img, 1), **i32)
        self.uniq_id = torch.empty(max(self.cap_k, 1), **i32)
        self.inv_id = torch.empty(max(n_id, 1), **i32)
        self.counts = torch.zeros(4, **i32)  # [U_img, K_id, ...]
        cu = max(self.cap_u, 1)
        self.act0 = torch.empty((cu, 256), **f32)
        self.act1 = torch.empty((cu, 64), **f32)
        self.emb = torch.empty((cu, 12), **f32)
        self.d_emb = torch.empty((cu, 12), **f32)
        self.d_rows = torch.empty((max(self.cap_k, 1), 12), **f32)
        self.head_in = torch.empty((max(B, 1), self.width), **f32)
        self.d_head_in = torch.empty((max(B, 1), self.width), **f32)
        self.logits = torch.empty(max(B, 1), **f32)
        self.scores = torch.empty((2, max(R, 1)), **f32)
        self.stats = torch.empty((2, max(B, 1), 2), **f32)
        self.head_part = torch.empty((L.lib.dicm_head_blocks(max(B, 1)), self.head_range[1] - self.head_range[0]),
                                     **f32)
        self.loss_part = torch.empty(L.lib.dicm_head_blocks(max(B, 1)), **f32)
        self.attn_partial = torch.empty((L.lib.dicm_sample_blocks(max(B, 1)), max(self.attn_part, 1)), **f32)
        self.loss = torch.zeros(1, **f32)
        # zeroed once: rows past the live count are read (and multiplied by
        # zero-filled gathers) by the tensor-core backward, so they must be finite
        self.mlp_ws = torch.zeros(max(int(L.lib.dicm_imgmlp_workspace(self.cap_u, self.pool.d_raw, self.prec_code)),
                                      1), dtype=torch.uint8, device=dev)
        self.cap = need

    def _pinned_buf(self, n):
        i = self._pin_i
        self._pin_i ^= 1
        if self._pin_ev[i] is not None:
            self._pin_ev[i].synchronize()
        buf = self._pinned[i]
        if buf is None or buf.numel() < n:
            buf = torch.empty(max(n, 1), dtype=torch.int32, pin_memory=True)
            self._pinned[i] = buf
        return i, buf

    # ------------------------------------------------------------------
    def upload(self, batch, own=False):
        """H2D of one batch (async).  ``own=True`` gives the batch its own
        device buffer (pre-staged inputs); otherwise the engine's buffer is
        reused."""
        pk = Packed(self.model, batch)
        self._ensure(pk)
        dst = torch.empty(max(pk.total, 1), dtype=torch.int32, device=self.dev) if own else self.packed
        i, buf = self._pinned_buf(pk.total)
        pk.fill(self.model, batch, buf.numpy())
        dst[:pk.total].copy_(buf[:pk.total], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._pin_ev[i] = ev
        return DeviceBatch(pk, dst)

    def h2d_bytes(self, batch):
        return Packed(self.model, batch).total * 4

    def forward_backward(self, db, denominator=None):
        """Everything up to (and including) the dense gradients."""
        m, lay = self.model, self.model.layout
        pk = db.pk
        base_ptr = db.packed.data_ptr()
        self._dptr = lambda off: base_ptr + 4 * off
        s = L.stream_handle()
        B, R = pk.B, pk.R
        denom = float(B if denominator is None else denominator)
        st = self.status.data_ptr()
        cnt = self.counts
        # a2: image-key dedup (model.py:182-187)
        img_segs, inv_off = [], 0
        if lay.use_ad_image:
            img_segs.append(L.KeySeg(self._dptr(pk.ad), B, 0, self.pool.local_rows, inv_off))
            inv_off += B
        if lay.use_behavior_images:
            img_segs.append(L.KeySeg(self._dptr(pk.beh), R, 0, self.pool.local_rows, inv_off))
        n_img = len(img_segs)
        if n_img:
            arr = (L.KeySeg * n_img)(*img_segs)
            L.check(L.lib.dicm_dedup(arr, n_img, self.pool.local_rows, self.ws_img.data_ptr(), self.ws_img.numel(),
                                     self.uniq_img.data_ptr(), self.inv_img.data_ptr(), cnt[0:].data_ptr(), 0, st, s))
        # a2: ID dedup over all tables (Batch.unique_field_ids, model.py:152-155)
        id_segs, inv_id_off, off = [], {}, 0
        for i, f in enumerate(self.fields):
            if f.multi:
                a, n, _ = pk.multi[f.name]
                id_segs.append(L.KeySeg(self._dptr(a), n, self.bases[i], m.tables[f.name].shape[0], off))
            else:
                n = B
                id_segs.append(L.KeySeg(self._dptr(pk.onehot[f.name]), n, self.bases[i],
                                        m.tables[f.name].shape[0], off))
            inv_id_off[f.name] = off
            off += n
        arr = (L.KeySeg * len(id_segs))(*id_segs)
        L.check(L.lib.dicm_dedup(arr, len(id_segs), self.id_key_space, self.ws_id.data_ptr(), self.ws_id.numel(),
                                 self.uniq_id.data_ptr(), self.inv_id.data_ptr(), cnt[1:].data_ptr(), 1, st, s))
        # a3-a4: image MLP forward on the unique rows
        cu = self.cap_u
        ev = self._ev("imgmlp_fwd")
        if n_img:
            L.check(L.lib.dicm_imgmlp_fwd(self.pool.rows.data_ptr(), self.pool.dtype_code, self.pool.d_raw,
                                          self.uniq_img.data_ptr(), cnt[0:].data_ptr(), cu, C.byref(self.img_p),
                                          self.act0.data_ptr(), self.act1.data_ptr(), self.emb.data_ptr(),
                                          self.prec_code, self.mlp_ws.data_ptr(), self.mlp_ws.numel(), s))
        self._ev_end(ev)
        # a6-a10 forward
        bv = L.BatchView()
        bv.batch, bv.refs = B, R
        for i, f in enumerate(self.fields):
            if f.multi:
                a, n, o = pk.multi[f.name]
                bv.field_ids[i] = self._dptr(a)
                bv.field_off[i] = self._dptr(o)
            else:
                bv.field_ids[i] = self._dptr(pk.onehot[f.name])
            bv.tables[i] = m.tables[f.name].data_ptr()
            bv.field_inv[i] = self.inv_id.data_ptr() + 4 * inv_id_off[f.name]
        bv.ad_local = self.inv_img.data_ptr() if lay.use_ad_image else None
        bv.beh_local = self.inv_img.data_ptr() + 4 * (B if lay.use_ad_image else 0)
        bv.beh_off = self._dptr(pk.beh_off)
        bv.emb = self.emb.data_ptr()
        self._bv = bv
        L.check(L.lib.dicm_sample_fwd(C.byref(self.layout), C.byref(bv), self.attn, self.head_in.data_ptr(),
                                      self.scores.data_ptr(), self.stats.data_ptr(), s))
        # a11-a12 head forward + backward
        L.check(L.lib.dicm_head_fwd_bwd(self.head_in.data_ptr(), B, self.width, self._dptr(pk.labels),
                                        1.0 / denom, C.byref(self.head_p), self.logits.data_ptr(),
                                        self.d_head_in.data_ptr(), self.head_part.data_ptr(),
                                        self.loss_part.data_ptr(), s))
        nhb = L.lib.dicm_head_blocks(B)
        L.check(L.lib.dicm_loss_finalize(self.loss_part.data_ptr(), nhb, 1.0 / denom, self.loss.data_ptr(), st, s))
        # a6-a10 backward
        self.d_emb.zero_()
        self.d_rows.zero_()
        L.check(L.lib.dicm_sample_bwd(C.byref(self.layout), C.byref(bv), self.attn, self.head_in.data_ptr(),
                                      self.d_head_in.data_ptr(), self.scores.data_ptr(), self.stats.data_ptr(),
                                      self.d_emb.data_ptr(), self.d_rows.data_ptr(), self.attn_partial.data_ptr(),
                                      s))
        h0, h1 = self.head_range
        L.check(L.lib.dicm_reduce_partials(self.head_part.data_ptr(), nhb, h1 - h0,
                                           self.grad.data_ptr() + 4 * h0, 0, s))
        if self.attn_range is not None:
            a0, a1 = self.attn_range
            L.check(L.lib.dicm_reduce_partials(self.attn_partial.data_ptr(), L.lib.dicm_sample_blocks(B), a1 - a0,
                                               self.grad.data_ptr() + 4 * a0, 0, s))
        # a5: image MLP backward
        ev = self._ev("imgmlp_bwd")
        L.check(L.lib.dicm_imgmlp_bwd(self.pool.rows.data_ptr(), self.pool.dtype_code, self.pool.d_raw,
                                      self.uniq_img.data_ptr(), cnt[0:].data_ptr(), cu if n_img else 0,
                                      C.byref(self.img_p), self.act0.data_ptr(), self.act1.data_ptr(),
                                      self.d_emb.data_ptr(), C.byref(self.img_g), self.prec_code,
                                      self.mlp_ws.data_ptr(), self.mlp_ws.numel(), s))
        self._ev_end(ev)
        return self.loss

    def _ev(self, name):
        if self.probe is None:
            return None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        self.probe.setdefault(name, []).append((a, b))
        return b

    @staticmethod
    def _ev_end(ev):
        if ev is not None:
            ev.record()

    @property
    def launches_per_step(self):
        """Kernels this engine launches per step (memsets included), counted
        from the kernel sequence of each C-ABI call."""
        lay = self.model.layout
        n = 6 + 6  # two dedups: memset + mark + tile sums + scan + emit + inverse
        n += 3 if self.prec_code == L.PREC_FP32 else 3  # image MLP fwd: layer0, layer1, layer2
        n += 1 + 1 + 1  # sample fwd, head, loss
        n += 2 + 1 + 1 + (1 if lay.attentive else 0)  # zero dE/dRows, sample bwd, reduces
        n += 12  # image MLP bwd (layer-2 bwd + 4 reduces, dh1 GEMM + 2 reduces, dW1 + reduce, dW0 + reduce)
        n += 1 + 4 + 1  # check_finite, adam dense (memset + 3), adam rows
        return n

    def optimizer_step(self, lr):
        s = L.stream_handle()
        st = self.status.data_ptr()
        L.check(L.lib.dicm_check_finite(self.d_rows.data_ptr(), self.d_rows.numel(), self.counts[1:].data_ptr(), 12,
                                        4, st, s))
        L.check(L.lib.dicm_adam_dense(self.model.dense.data_ptr(), self.grad.data_ptr(), self.m.data_ptr(),
                                      self.v.data_ptr(), self.t.data_ptr(), self.spans, len(self.spans), lr, BETA1,
                                      BETA2, EPS, self.adam_ws.data_ptr(), self.adam_ws.numel(), st, s))
        L.check(L.lib.dicm_adam_rows(self.tabstate, len(self.fields), self.uniq_id.data_ptr(),
                                     self.counts[1:].data_ptr(), self.cap_k, self.d_rows.data_ptr(), lr, BETA1, BETA2,
                                     EPS, st, s))

    def lr(self):
        return lr_schedule(self.iteration, self.lr0, self.lr_decay, self.lr_interval)

    def step(self, batch, denominator=None):
        """Upload + full step; returns the device loss (no sync)."""
        db = self.upload(batch)
        loss = self.forward_backward(db, denominator)
        self.optimizer_step(self.lr())
        self.iteration += 1
        return loss

    def raise_status(self):
        """Sync point: raise the reference's exception for a flagged step."""
        st = self.status.cpu().numpy()
        if st[L.ST_KEY_FLAG]:
            self.status.zero_()
            tag, seg = divmod(int(st[L.ST_KEY_SEG]), 16)
            if tag == 0:
                raise KeyError(f"unknown image id {int(st[L.ST_KEY_VALUE])} (store holds 0.."
                               f"{self.pool.local_rows - 1})")
            f = self.fields[seg]
            raise KeyError(f"id {int(st[L.ST_KEY_VALUE])} outside vocabulary of size {f.vocab} "
                           f"(field {f.name})")
        if st[L.ST_NONFINITE]:
            self.status.zero_()
            bits = int(st[L.ST_NONFINITE])
            if bits & 1:
                raise FloatingPointError(f"non-finite loss at iteration {self.iteration - 1}")
            raise FloatingPointError("adam: non-finite gradient, parameter untouched")

    # -- inspection ---------------------------------------------------
    def unique_images(self):
        n = int(self.counts[0].item())
        return self.uniq_img[:n].cpu().numpy()

    def unique_rows(self):
        n = int(self.counts[1].item())
        return self.uniq_id[:n].cpu().numpy()
