"""The device training step: the kernel sequence behind ``LocalTrainer.train_batch``
(reference training.py:66-91) and, in ``runtime.ClusterEngine``, behind one
rank of ``Cluster.run_iteration`` (runtime.py:370-470).

One step, no host round trip until the loss is read (the ID chain and the
partial reduces run on a forked stream, see forward_backward):

  H2D    one packed copy of the CSR batch (ids, offsets, labels)
  a2     dicm_dedup over the image keys    -> unique pool rows + inverse
  a2     dicm_dedup over every ID field    -> unique (field,row) keys + inverse
  a3-a4  dicm_imgmlp_fwd on the unique rows -> E [U,12]
  a10    dicm_gather_rows_by_key           -> compact ID rows [K,12]
  a6-10  dicm_sample_fwd                   -> head input x [B, W]
  a11-12 dicm_head_fwd_bwd                 -> logits, dLoss/dx, head-grad partials
         (pre-rank model: dicm_towers_fwd_bwd, the two towers + inner product)
  a6-10  dicm_sample_bwd                   -> dE [U,12], dRows [K,12], attention partials
  a5     dicm_imgmlp_bwd                   -> img/* gradients
  a14    dicm_adam_dense + dicm_adam_rows

Buffers are sized by capacity and reused; data-dependent counts never leave
the device.  Status words latch out-of-vocabulary ids and non-finite values;
the update kernels refuse to run on a flagged step and the host raises the
reference's exception when it reads the status.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib as L
from .model import HEAD_SMEM_WIDTH, KIND_CODE

BETA1, BETA2, EPS = 0.9, 0.999, 1e-8  # reference optim.py:16-19


def lr_schedule(iteration, lr0=0.001, decay=0.9, interval=24000):
    """reference optim.py:24-28."""
    if iteration < 0:
        raise ValueError(f"iteration must be >= 0, got {iteration}")
    return lr0 * decay ** (iteration // interval)


def _u8(n, dev, zero=False):
    f = torch.zeros if zero else torch.empty
    return f(max(int(n), 1), dtype=torch.uint8, device=dev)


class Packed:
    """Offsets of one batch inside the packed int32 upload buffer."""

    def __init__(self, model, batch):
        self.B = batch.size
        self.R = batch.refs
        off = 0
        self.onehot, self.multi = {}, {}
        for f in model.layout.schema.fields:
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
        """Pack the batch's columns into ``host`` (int32) with the library's
        multithreaded copy (dicm_host_pack)."""
        segs = []  # (array, int32 offset in host)
        for f in model.layout.schema.fields:
            if f.multi:
                a, n, o = self.multi[f.name]
                flat, offs = batch.multihot[f.name]
                segs += [(flat, a), (offs, o)]
            else:
                segs.append((batch.onehot[f.name], self.onehot[f.name]))
        segs += [(batch.ad_image_ids, self.ad), (batch.beh_image_ids, self.beh), (batch.beh_off, self.beh_off),
                 (np.asarray(batch.labels, dtype=np.float32).view(np.int32), self.labels)]
        keep = [np.ascontiguousarray(a, dtype=np.int32) for a, _ in segs]
        n = len(keep)
        srcs = (C.c_void_p * n)(*[a.ctypes.data for a in keep])
        nbytes = (C.c_int64 * n)(*[a.nbytes for a in keep])
        offs = (C.c_int64 * n)(*[4 * o for _, o in segs])
        assert host.dtype == np.int32 and host.flags.c_contiguous and host.size >= self.total
        L.check(L.lib.dicm_host_pack(host.ctypes.data, srcs, nbytes, offs, n, 0))

    def n_id(self, fields):
        return sum(self.B if not f.multi else self.multi[f.name][1] for f in fields)

    def signature(self):
        """Everything a captured step depends on: batches with equal signatures
        share one CUDA graph."""
        return (self.B, self.R, self.total, tuple(sorted(self.multi.items())), tuple(sorted(self.onehot.items())))


class DeviceBatch:
    __slots__ = ("pk", "packed")

    def __init__(self, pk, packed):
        self.pk, self.packed = pk, packed


class Prefetcher:
    """Host input pipeline: while step i runs, a worker
    thread assembles batch i+1 on the host (``transform`` -- e.g. a Cluster
    rank's slice of the union batch -- the columnar take and the packing into
    pinned memory) and its H2D copy runs on a side stream; the compute stream
    waits for that copy only when it reaches the batch.

    Pinned host slots and device slots rotate through rings and are reused,
    never reallocated per batch: a pinned slot returns to the worker once its
    copy has been issued (the worker waits on the copy's event before
    refilling it); a device slot is rewritten only after the step that read it
    has passed (an event on the compute stream).  Yields (item, DeviceBatch)
    with ``item = transform(batch)``."""

    def __init__(self, engine, batches, depth=2, transform=None):
        import queue
        import threading
        self.e, self.depth = engine, max(1, int(depth))
        self.copy_stream = torch.cuda.Stream(device=engine.dev)
        n = self.depth + 2
        self.q = queue.Queue(maxsize=self.depth)
        self.free = queue.Queue()
        for k in range(n):
            self.free.put((k, None))
        self.pinned = [None] * n
        self.ring = [None] * n
        self.freed = [None] * n
        self._err = None
        self._stop = False

        def work():
            try:
                for b in batches:
                    if self._stop:
                        break
                    item = transform(b) if transform is not None else b
                    local = item[0] if transform is not None else item
                    engine._check_capacity(local)
                    pk = Packed(engine.model, local)
                    k, ev = self.free.get()
                    if ev is not None:
                        ev.synchronize()  # the previous copy out of this slot has finished
                    host = self.pinned[k]
                    if host is None or host.numel() < pk.total:
                        host = self.pinned[k] = torch.empty(max(pk.total, 1), dtype=torch.int32, pin_memory=True)
                    pk.fill(engine.model, local, host.numpy())
                    self.q.put((item, pk, k))
            except BaseException as ex:  # surfaced in the consumer
                self._err = ex
            self.q.put(None)

        self.t = threading.Thread(target=work, daemon=True)
        self.t.start()

    def close(self):
        self._stop = True

    def __iter__(self):
        i = 0
        while True:
            got = self.q.get()
            if got is None:
                if self._err is not None:
                    raise self._err
                return
            item, pk, k = got
            self.e._ensure(pk)
            slot = i % len(self.ring)
            buf = self.ring[slot]
            if buf is None or buf.numel() < pk.total:
                buf = self.ring[slot] = torch.empty(max(pk.total, 1), dtype=torch.int32, device=self.e.dev)
            with torch.cuda.stream(self.copy_stream):
                if self.freed[slot] is not None:
                    self.copy_stream.wait_event(self.freed[slot])  # the step that read this slot is done
                buf[:pk.total].copy_(self.pinned[k][:pk.total], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(self.copy_stream)
            self.free.put((k, ready))
            torch.cuda.current_stream().wait_event(ready)
            yield item, DeviceBatch(pk, buf)
            done = torch.cuda.Event()
            done.record(torch.cuda.current_stream())
            self.freed[slot] = done
            i += 1


class ImageNetBuffers:
    """Activations + workspace of one image-MLP pass over up to ``cap`` rows."""

    def __init__(self, cap, d_raw, prec_code, dev):
        cu = max(int(cap), 1)
        f32 = dict(dtype=torch.float32, device=dev)
        self.cap = int(cap)
        self.act0 = torch.empty((cu, 256), **f32)
        self.act1 = torch.empty((cu, 64), **f32)
        self.emb = torch.empty((cu, 12), **f32)
        self.d_emb = torch.empty((cu, 12), **f32)
        # zeroed once: rows past the live count are read (and multiplied by
        # zero-filled gathers) by the tensor-core backward, so they must be finite
        self.ws = _u8(L.lib.dicm_imgmlp_workspace(self.cap, d_raw, prec_code), dev, zero=True)


class _Joined:
    """A forked stream whose backward work is already queued (forward_backward)."""

    def __init__(self, stream):
        self.stream = stream


class StepEngine:
    """Owns the optimizer state and the step buffers of one model replica.

    ``world``/``id_align``: the ID key space puts table f at base_f, aligned to
    ``id_align`` so that a key's owner in a sharded run is simply key % world
    (see runtime.ClusterEngine); a single GPU uses id_align = 1.
    """

    def __init__(self, model, pool, precision="fp32", lr0=0.001, lr_decay=0.9, lr_interval=24000, id_align=1):
        if precision not in L.PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(L.PRECISIONS)}")
        if precision == "bf16" and pool.dtype_name != "bf16":
            raise ValueError("bf16 tensor-core mode needs a bf16 pool")
        self.store = pool  # the caller's pool (the engine may hold a padded copy)
        if pool.d_raw != model.schema.d_raw and pool.d_raw != model.geometry.d_raw:
            raise ValueError(f"pool rows are {pool.d_raw}-D, schema expects {model.schema.d_raw}")
        if pool.d_raw != model.geometry.d_raw:
            # rows narrower than the kernels' multiple of 256: one zero-padded
            # device copy (the padded columns meet zero columns of img/0/w)
            pool = pool.padded(model.geometry.d_raw)
        self.model, self.pool = model, pool
        self.precision = precision
        self.prec_code = L.PRECISIONS[precision]
        self.lr0, self.lr_decay, self.lr_interval = lr0, lr_decay, lr_interval
        self.iteration = 0
        self.hot_acc_on = True  # chunked hot-key passes (False: one block per hot key; same bits)
        dev = self.dev = model.device
        lay = model.layout
        self.fields = list(lay.schema.fields)  # the fields with tables (pre-rank: tower fields)
        # global ID key space: field f at bases[f] (aligned), vocab = schema vocab
        self.bases, base = [], 0
        for f in self.fields:
            self.bases.append(base)
            base += -(-f.vocab // id_align) * id_align
        self.id_key_space = base
        self.status = torch.zeros(L.STATUS_WORDS, dtype=torch.int32, device=dev)
        # optimizer state (reference training.py:53-60); the gradient buffer
        # carries one more slot, the loss, so that a multi-GPU step sums both
        # with a single all-reduce (Adam's spans never cover that slot)
        self.grad_ext = torch.zeros(model.dense.numel() + 1, dtype=torch.float32, device=dev)
        self.grad = self.grad_ext[:-1]
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
        self.tabstate = self._table_states(self.bases, 1)
        self.ws_id = _u8(L.lib.dicm_dedup_workspace(max(self.id_key_space, 1)), dev)
        self.ws_img = _u8(L.lib.dicm_dedup_workspace(max(self.image_key_space, 1)), dev)
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
        self.width = model.geometry.width  # the kernel head input (12-wide blocks)
        if lay.towers is None:
            hn = ("mlp/0/w", "mlp/0/b", "mlp/0/a", "mlp/1/w", "mlp/1/b", "mlp/1/a", "mlp/2/w", "mlp/2/b")
            self.head_p = L.HeadParams(**{k: p(n) for k, n in zip(names, hn)})
            self.head_range = model.group_range("mlp/")
            assert self.head_range[1] - self.head_range[0] == L.lib.dicm_head_partial_size(self.width)
        else:
            self._setup_towers(model)
        self.attn_range = model.group_range("attn/")
        self.attn_part = int(L.lib.dicm_attn_partial_size(C.byref(self.layout)))
        if self.attn_range is not None:
            assert self.attn_range[1] - self.attn_range[0] == self.attn_part
        self.cap = None
        self.probe = None  # name -> [(start, end)] CUDA events around the image-MLP launches
        self._pinned = [None, None]
        self._pin_ev = [None, None]
        self._pin_i = 0
        self._copy_stream, self._up_ring, self._up_mark, self._up_n = None, [None, None], None, 0

    def _setup_towers(self, model):
        """Pre-rank head (csrc/towers.cu): tower descriptors whose gradient
        offsets index one partial row laid out like the fused buffer's
        ad_tower/* + user_tower/* range (contiguous in sorted order)."""
        lay = model.layout
        names = [n for n in model.dense_names if n.split("/")[0] in ("user_tower", "ad_tower")]
        start = min(model.dense_offsets[n][0] for n in names)
        end = max(model.dense_offsets[n][0] + model.dense_offsets[n][1] for n in names)
        assert end - start == sum(model.dense_offsets[n][1] for n in names), "tower params not contiguous"
        self.head_range = (start, end)
        self.towers = (L.Tower * 2)()
        for i, t in enumerate(("user", "ad")):
            tw = self.towers[i]
            pre = f"{t}_tower/"
            for k, n in (("w0", "0/w"), ("b0", "0/b"), ("a0", "0/a"), ("w1", "1/w"), ("b1", "1/b")):
                setattr(tw, k, model.params[pre + n].tensor.data_ptr())
                setattr(tw, "g_" + k, model.dense_offsets[pre + n][0] - start)
            parts = model.geometry.tower_parts(t)
            tw.n_parts = len(parts)
            for j, (col, _w) in enumerate(parts):
                tw.part_col[j] = col

    def _head_blocks(self, B):
        return L.lib.dicm_towers_blocks(B) if self.model.layout.towers else L.lib.dicm_head_blocks(B)

    @property
    def wide_head(self):
        """Head input too wide for the shared-memory W0 (concat aggregator):
        layer 0 runs as GEMMs and the mlp/ gradients land directly in
        ``self.grad`` (dicm_head_wide_fwd_bwd)."""
        return self.model.layout.towers is None and self.width > HEAD_SMEM_WIDTH

    def _head_fwd_bwd(self, B, denom):
        """a11-a12: MLP head (or the two towers) + BCE -> logits, d_head_in,
        gradient partials, loss partials."""
        pk, s = self.pk, self.s
        tw = self.model.layout.towers
        if self.wide_head:
            h0, _ = self.head_range
            L.check(L.lib.dicm_head_wide_fwd_bwd(self.head_in.data_ptr(), B, self.width, self._dptr(pk.labels),
                                                 1.0 / denom, C.byref(self.head_p), self.logits.data_ptr(),
                                                 self.d_head_in.data_ptr(), self.grad.data_ptr() + 4 * h0,
                                                 self.loss_part.data_ptr(), self.head_ws.data_ptr(),
                                                 self.head_ws.numel(), s))
        elif tw is None:
            L.check(L.lib.dicm_head_fwd_bwd(self.head_in.data_ptr(), B, self.width, self._dptr(pk.labels),
                                            1.0 / denom, C.byref(self.head_p), self.logits.data_ptr(),
                                            self.d_head_in.data_ptr(), self.head_part.data_ptr(),
                                            self.loss_part.data_ptr(), s))
        else:
            L.check(L.lib.dicm_towers_fwd_bwd(self.head_in.data_ptr(), B, self.width, self.towers, tw.hidden, tw.rep,
                                              self._dptr(pk.labels), 1.0 / denom, self.logits.data_ptr(),
                                              self.d_head_in.data_ptr(), self.head_part.data_ptr(),
                                              self.head_part.shape[1], self.loss_part.data_ptr(), s))

    def _head_fwd(self, B):
        tw = self.model.layout.towers
        if self.wide_head:
            L.check(L.lib.dicm_head_wide_fwd(self.head_in.data_ptr(), B, self.width, C.byref(self.head_p),
                                             self.logits.data_ptr(), self.head_ws.data_ptr(), self.head_ws.numel(),
                                             self.s))
        elif tw is None:
            L.check(L.lib.dicm_head_fwd(self.head_in.data_ptr(), B, self.width, C.byref(self.head_p),
                                        self.logits.data_ptr(), self.s))
        else:
            L.check(L.lib.dicm_towers_fwd(self.head_in.data_ptr(), B, self.width, self.towers, tw.hidden, tw.rep,
                                          self.logits.data_ptr(), self.s))

    # ------------------------------------------------------------------
    @property
    def image_key_space(self):
        """Image ids are pool rows of THIS engine's pool."""
        return self.pool.local_rows

    def _table_states(self, bases, divisor):
        """Row-Adam / row-gather descriptors over the local tables, keyed by
        global combined keys divided by ``divisor`` (owner-local keys)."""
        ts_arr = (L.TableState * len(self.fields))()
        for i, f in enumerate(self.fields):
            ts = ts_arr[i]
            ts.table, ts.m, ts.v, ts.t = (self.model.tables[f.name].data_ptr(), self.tm[f.name].data_ptr(),
                                         self.tv[f.name].data_ptr(), self.tt[f.name].data_ptr())
            ts.base, ts.vocab = bases[i] // divisor, self.model.tables[f.name].shape[0]
        return ts_arr

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

    def _n_img(self, B, R):
        lay = self.model.layout
        return (B if lay.use_ad_image else 0) + (R if lay.use_behavior_images else 0)

    def _need(self, pk):
        return (pk.total, pk.B, pk.R, pk.n_id(self.fields))

    def _ensure(self, pk):
        need = self._need(pk)
        if self.cap is not None and all(a <= b for a, b in zip(need, self.cap)):
            return
        if self.cap is not None:  # grow with headroom
            need = tuple(max(int(a * 1.25), b) for a, b in zip(need, self.cap))
        self._alloc_caps(need)

    def _alloc_caps(self, need):
        """Every per-batch buffer at capacity ``need`` = (packed int32 words,
        samples, behaviors, ID references)."""
        total, B, R, n_id = need
        dev = self.dev
        n_img = self._n_img(B, R)
        self.cap_u = min(n_img, self.image_key_space)
        self.cap_k = min(n_id, self.id_key_space)
        i32 = dict(dtype=torch.int32, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.packed = torch.empty(max(total, 1), **i32)
        self.uniq_img = torch.empty(max(self.cap_u, 1), **i32)
        self.inv_img = torch.empty(max(n_img, 1), **i32)
        self.uniq_id = torch.empty(max(self.cap_k, 1), **i32)
        self.inv_id = torch.empty(max(n_id, 1), **i32)
        self.counts = torch.zeros(8, **i32)  # [U_img, K_id, U_owner, K_owner, ...]
        self.id_rows = torch.empty((max(self.cap_k, 1), 12), **f32)
        self.d_rows = torch.empty((max(self.cap_k, 1), 12), **f32)
        self.head_in = torch.empty((max(B, 1), self.width), **f32)
        self.d_head_in = torch.empty((max(B, 1), self.width), **f32)
        self.logits = torch.empty(max(B, 1), **f32)
        self.scores = torch.empty((2, max(R, 1)), **f32)
        self.stats = torch.empty((2, max(B, 1), 2), **f32)
        if self.wide_head:  # no per-block partial rows: the GEMMs write the gradients
            self.head_part = torch.empty((1, 1), **f32)
            self.head_ws = _u8(L.lib.dicm_head_wide_workspace(max(B, 1), self.width), dev)
        else:
            self.head_part = torch.empty((self._head_blocks(max(B, 1)), self.head_range[1] - self.head_range[0]),
                                         **f32)
        self.loss_part = torch.empty(self._head_blocks(max(B, 1)), **f32)
        self.attn_partial = torch.empty((L.lib.dicm_sample_blocks(max(B, 1)), max(self.attn_part, 1)), **f32)
        self.loss = self.grad_ext[-1:]
        lay = self.model.layout
        # deterministic backward (dicm_ref_transpose / dicm_sample_bwd): the
        # dedup inverses transposed, the sample of every CSR reference, and
        # per-reference / per-sample gradient scratch
        self.img_order = torch.empty(max(n_img, 1), **i32)
        self.img_start = torch.empty(max(self.cap_u, 1) + 1, **i32)
        self.id_order = torch.empty(max(n_id, 1), **i32)
        self.id_start = torch.empty(max(self.cap_k, 1) + 1, **i32)
        self.beh_seg = torch.empty(max(R, 1), **i32)
        self.id_seg = torch.empty(max(n_id, 1), **i32)  # multi-hot field f's refs at their ID-list positions
        own_rows = lay.use_behavior_images and lay.aggregator.kind != "sum"
        self.ref_grad = torch.empty((max(R, 1) if own_rows else 1, 12), **f32)
        self.q_grad = torch.empty((max(B, 1), 36), **f32)
        self.hot = torch.empty(4 + 2 * (max(self.cap_u, 1) + max(self.cap_k, 1)), **i32)
        self.hot_acc = torch.zeros(L.lib.dicm_hot_acc_bytes(), dtype=torch.uint8, device=dev)  # kept re-armed
        self.ws_tr_img = _u8(L.lib.dicm_ref_transpose_workspace(n_img, max(self.cap_u, 1)), dev)
        self.ws_tr_id = _u8(L.lib.dicm_ref_transpose_workspace(n_id, max(self.cap_k, 1)), dev)
        self._alloc_image_net(self.cap_u)
        self.cap = need
        self._graphs, self._graph_warm = None, False  # captured steps point at the old buffers
        self._last_graph = None

    def _alloc_image_net(self, cap):
        self.net = ImageNetBuffers(cap, self.pool.d_raw, self.prec_code, self.dev)

    # views kept for callers / tests
    @property
    def emb(self):
        return self.net.emb

    @property
    def d_emb(self):
        return self.net.d_emb

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
    def _check_capacity(self, batch):
        """concat: every kept behavior needs a slot (reference scatter_concat
        raises ShapeError for pos >= capacity, autograd.py:375-376)."""
        lay = self.model.layout
        if lay.aggregator.kind == "concat" and lay.use_behavior_images and batch.size:
            longest = int(np.max(np.diff(np.asarray(batch.beh_off))))
            if longest > lay.schema.b_max:
                raise ValueError(f"scatter_concat: slot out of range for capacity {lay.schema.b_max} "
                                 f"(a sample has {longest} behaviors)")

    def upload(self, batch, own=False):
        """H2D of one batch (async).  ``own=True`` gives the batch its own
        device buffer (pre-staged inputs) and copies on the current stream.
        Otherwise the copy runs on a side stream into one of two staging
        buffers, so it overlaps the step still running on the compute stream;
        the compute stream waits for the copy only where it reaches this
        batch.  A staging slot is rewritten only after the step that read it
        (two uploads back) has finished."""
        self._check_capacity(batch)
        pk = Packed(self.model, batch)
        self._ensure(pk)
        i, buf = self._pinned_buf(pk.total)
        pk.fill(self.model, batch, buf.numpy())
        cur = torch.cuda.current_stream()
        if own:
            dst = torch.empty(max(pk.total, 1), dtype=torch.int32, device=self.dev)
            dst[:pk.total].copy_(buf[:pk.total], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cur)
            self._pin_ev[i] = ev
            return DeviceBatch(pk, dst)
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(device=self.dev)
        k = self._up_n % 2
        self._up_n += 1
        mark = torch.cuda.Event()
        mark.record(cur)  # the work enqueued so far: every step before this batch's
        prev, self._up_mark = self._up_mark, mark
        dst = self._up_ring[k]
        if dst is None or dst.numel() < pk.total:
            torch.cuda.synchronize()  # the old slot may still be read or written
            dst = self._up_ring[k] = torch.empty(max(pk.total, 1), dtype=torch.int32, device=self.dev)
        cs = self._copy_stream
        with torch.cuda.stream(cs):
            if prev is not None:
                cs.wait_event(prev)  # slot k's last reader (two uploads back) has run
            dst[:pk.total].copy_(buf[:pk.total], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(cs)
        cur.wait_event(ready)
        self._pin_ev[i] = ready
        return DeviceBatch(pk, dst)

    def h2d_bytes(self, batch):
        return Packed(self.model, batch).total * 4

    # ---- phases --------------------------------------------------------
    def _begin(self, db):
        self.pk = db.pk
        base_ptr = db.packed.data_ptr()
        self._dptr = lambda off: base_ptr + 4 * off
        self.s = L.stream_handle()

    def _dedup_images(self, inverse=True):
        """a2 over the image keys (model.py:182-187) -> uniq_img, inv_img, counts[0]
        (``inverse=False``: inv_img is left to ``_inverse_images``)."""
        lay, pk = self.model.layout, self.pk
        segs, inv_off = [], 0
        space = self.pool.global_size if getattr(self, "world", 1) > 1 else self.image_key_space
        if lay.use_ad_image:
            segs.append(L.KeySeg(self._dptr(pk.ad), pk.B, 0, space, inv_off))
            inv_off += pk.B
        if lay.use_behavior_images:
            segs.append(L.KeySeg(self._dptr(pk.beh), pk.R, 0, space, inv_off))
        self.n_img_segs = len(segs)
        if segs:
            arr = self._img_segs = ((L.KeySeg * len(segs))(*segs), len(segs), space)
            L.check(L.lib.dicm_dedup(arr[0], len(segs), space, self.ws_img.data_ptr(), self.ws_img.numel(),
                                     self.uniq_img.data_ptr(), self.inv_img.data_ptr() if inverse else None,
                                     self.counts.data_ptr(), 0, self.status.data_ptr(), self.s))

    def _inverse_images(self):
        """The image inverse of the last ``_dedup_images(inverse=False)``."""
        if self.n_img_segs:
            arr, n, space = self._img_segs
            L.check(L.lib.dicm_dedup_inverse(arr, n, space, self.ws_img.data_ptr(), self.ws_img.numel(),
                                             self.inv_img.data_ptr(), self.s))

    def _dedup_ids(self):
        """a2 over every ID field (Batch.unique_field_ids, model.py:152-155)."""
        pk = self.pk
        segs, self.inv_id_off, off = [], {}, 0
        for i, f in enumerate(self.fields):
            if f.multi:
                a, n, _ = pk.multi[f.name]
                segs.append(L.KeySeg(self._dptr(a), n, self.bases[i], f.vocab, off))
            else:
                n = pk.B
                segs.append(L.KeySeg(self._dptr(pk.onehot[f.name]), n, self.bases[i], f.vocab, off))
            self.inv_id_off[f.name] = off
            off += n
        arr = (L.KeySeg * len(segs))(*segs)
        L.check(L.lib.dicm_dedup(arr, len(segs), self.id_key_space, self.ws_id.data_ptr(), self.ws_id.numel(),
                                 self.uniq_id.data_ptr(), self.inv_id.data_ptr(), self.counts[1:].data_ptr(), 1,
                                 self.status.data_ptr(), self.s))

    def _image_forward(self, net, rows, count_ptr):
        """a3-a4: image MLP on pool rows rows[0..*count) -> net.emb."""
        ev = self._ev("imgmlp_fwd")
        L.check(L.lib.dicm_imgmlp_fwd(self.pool.rows.data_ptr(), self.pool.dtype_code, self.pool.d_raw,
                                      rows.data_ptr(), count_ptr, net.cap, C.byref(self.img_p), net.act0.data_ptr(),
                                      net.act1.data_ptr(), net.emb.data_ptr(), self.prec_code, net.ws.data_ptr(),
                                      net.ws.numel(), self.s))
        self._ev_end(ev)

    def _image_backward(self, net, rows, count_ptr, cap):
        """a5: reverse path into the shared image MLP (img/* gradients)."""
        ev = self._ev("imgmlp_bwd")
        L.check(L.lib.dicm_imgmlp_bwd(self.pool.rows.data_ptr(), self.pool.dtype_code, self.pool.d_raw,
                                      rows.data_ptr(), count_ptr, cap, C.byref(self.img_p), net.act0.data_ptr(),
                                      net.act1.data_ptr(), net.d_emb.data_ptr(), C.byref(self.img_g), self.prec_code,
                                      net.ws.data_ptr(), net.ws.numel(), self.s))
        self._ev_end(ev)

    def _gather_id_rows(self):
        """Compact ID rows of the batch's unique keys (rows(table, ids) with
        the dedup applied, model.py:407-408)."""
        L.check(L.lib.dicm_gather_rows_by_key(self.tabstate, len(self.fields), self.uniq_id.data_ptr(),
                                              self.counts[1:].data_ptr(), self.cap_k, self.id_rows.data_ptr(),
                                              self.s))

    def _batch_view(self, emb):
        """Device pointers of the current batch for the per-sample kernels."""
        lay, pk = self.model.layout, self.pk
        B, R = pk.B, pk.R
        bv = L.BatchView()
        bv.batch, bv.refs = B, R
        for i, f in enumerate(self.fields):
            if f.multi:
                a, n, o = pk.multi[f.name]
                bv.field_ids[i] = self._dptr(a)
                bv.field_off[i] = self._dptr(o)
            else:
                bv.field_ids[i] = self._dptr(pk.onehot[f.name])
            bv.tables[i] = self.id_rows.data_ptr()
            bv.field_inv[i] = self.inv_id.data_ptr() + 4 * self.inv_id_off[f.name]
        bv.ad_local = self.inv_img.data_ptr() if lay.use_ad_image else None
        bv.beh_local = self.inv_img.data_ptr() + 4 * (B if lay.use_ad_image else 0)
        bv.beh_off = self._dptr(pk.beh_off)
        bv.emb = emb.data_ptr()
        bv.img_order, bv.img_start = self.img_order.data_ptr(), self.img_start.data_ptr()
        bv.id_order, bv.id_start = self.id_order.data_ptr(), self.id_start.data_ptr()
        for i, f in enumerate(self.fields):
            bv.field_ref_begin[i] = self.inv_id_off[f.name]
            if f.multi:
                bv.field_seg[i] = self.id_seg.data_ptr() + 4 * self.inv_id_off[f.name]
        bv.beh_seg = self.beh_seg.data_ptr()
        bv.n_img_keys, bv.n_id_keys = self.counts.data_ptr(), self.counts[1:].data_ptr()
        bv.img_cap, bv.id_cap = max(self.cap_u, 1), max(self.cap_k, 1)
        bv.ref_grad, bv.q_grad, bv.hot = self.ref_grad.data_ptr(), self.q_grad.data_ptr(), self.hot.data_ptr()
        bv.hot_acc = self.hot_acc.data_ptr() if self.hot_acc_on else 0  # 0: one block per hot key
        return bv

    def _transpose_images(self):
        """The image-key dedup inverse transposed (stable by reference) and the
        sample of every behavior reference: the fixed summation order of the
        deterministic backward.  Depends only on the batch."""
        pk = self.pk
        n = self._n_img(pk.B, pk.R)
        if n:
            L.check(L.lib.dicm_ref_transpose(self.inv_img.data_ptr(), n, max(self.cap_u, 1), self.ws_tr_img.data_ptr(),
                                             self.ws_tr_img.numel(), self.img_order.data_ptr(),
                                             self.img_start.data_ptr(), self.s))
        if self.model.layout.use_behavior_images and self.model.layout.aggregator.kind == "sum":
            L.check(L.lib.dicm_csr_segments(self._dptr(pk.beh_off), pk.B, self.beh_seg.data_ptr(), self.s))

    def _transpose_ids(self):
        """The same for the ID keys (every field's references in schema order)."""
        pk = self.pk
        n = pk.n_id(self.fields)
        if n:
            L.check(L.lib.dicm_ref_transpose(self.inv_id.data_ptr(), n, max(self.cap_k, 1), self.ws_tr_id.data_ptr(),
                                             self.ws_tr_id.numel(), self.id_order.data_ptr(), self.id_start.data_ptr(),
                                             self.s))
        for f in self.fields:
            if f.multi:
                _, _, o = pk.multi[f.name]
                L.check(L.lib.dicm_csr_segments(self._dptr(o), pk.B, self.id_seg.data_ptr() + 4 * self.inv_id_off[f.name],
                                                self.s))

    def _local_step(self, emb, d_emb, denom, reduce=True, id_rows=True, fwd=True, after_head=None):
        """a6-a12 forward and backward on the local batch: pooling, head, BCE.
        Reads image embeddings ``emb`` and compact ID rows ``self.id_rows``;
        writes ``d_emb`` / ``self.d_rows`` (``id_rows=False``: left to
        ``_id_row_grads``) and the head/attention gradients.  ``fwd=False``:
        the head input was already built (``self._bv``, split forward)."""
        pk, s = self.pk, self.s
        B = pk.B
        st = self.status.data_ptr()
        if fwd:
            bv = self._bv = self._batch_view(emb)
            L.check(L.lib.dicm_sample_fwd(C.byref(self.layout), C.byref(bv), self.attn, self.head_in.data_ptr(),
                                          self.scores.data_ptr(), self.stats.data_ptr(), s))
        bv = self._bv
        self._head_fwd_bwd(B, denom)
        nhb = self._head_blocks(B)
        L.check(L.lib.dicm_loss_finalize(self.loss_part.data_ptr(), nhb, 1.0 / denom, self.loss.data_ptr(), st, s))
        if after_head is not None:  # work that needs only the head's gradients (forked by the caller)
            after_head()
        L.check(L.lib.dicm_sample_bwd(C.byref(self.layout), C.byref(bv), self.attn, self.head_in.data_ptr(),
                                      self.d_head_in.data_ptr(), self.scores.data_ptr(), self.stats.data_ptr(),
                                      d_emb.data_ptr(), self.d_rows.data_ptr() if id_rows else None,
                                      self.attn_partial.data_ptr(), s))
        if reduce:
            self._reduce_partials(s)

    def _id_row_grads(self, s):
        L.check(L.lib.dicm_id_row_grads(C.byref(self.layout), C.byref(self._bv), self.d_head_in.data_ptr(),
                                        self.d_rows.data_ptr(), s))

    def _reduce_partials(self, s):
        """Head and attention parameter gradients from their block partials
        (fixed-order reduces)."""
        self._reduce_head_partials(s)
        self._reduce_attn_partials(s)

    def _reduce_head_partials(self, s):
        B = self.pk.B
        h0, h1 = self.head_range
        if not self.wide_head:
            L.check(L.lib.dicm_reduce_partials(self.head_part.data_ptr(), self._head_blocks(B), h1 - h0,
                                               self.grad.data_ptr() + 4 * h0, 0, s))

    def _reduce_attn_partials(self, s):
        B = self.pk.B
        if self.attn_range is not None:
            a0, a1 = self.attn_range
            L.check(L.lib.dicm_reduce_partials(self.attn_partial.data_ptr(), L.lib.dicm_sample_blocks(B), a1 - a0,
                                               self.grad.data_ptr() + 4 * a0, 0, s))

    _rows_checked = False  # dRows already checked on the forked stream this step

    def _side_stream(self):
        """Stream for the forked ID chain (None: everything on one stream;
        DICM_FORK=0 turns the fork off)."""
        if os.environ.get("DICM_FORK", "1") == "0":
            return None
        side = getattr(self, "_side", None)
        if side is None:
            side = self._side = torch.cuda.Stream(device=self.dev)
        return side

    def forward_backward(self, db, denominator=None):
        """Everything up to (and including) the dense gradients."""
        self._begin(db)
        denom = float(db.pk.B if denominator is None else denominator)
        side = self._side_stream()
        if side is not None:
            # the ID chain (dedup over every field -> compact rows -> the ID
            # columns of the head input -> its transpose) shares no buffer
            # with the image chain; it runs on a forked stream (a graph branch
            # once captured) and joins before the head
            main = self.s
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                self.s = side.cuda_stream
                self._dedup_ids()
                self._gather_id_rows()
                ids_ready = torch.cuda.Event()
                ids_ready.record(side)
                self._bv = self._batch_view(self.net.emb)
                L.check(L.lib.dicm_fields_fwd(C.byref(self.layout), C.byref(self._bv), self.head_in.data_ptr(),
                                              self.s))
                self._transpose_ids()
            self.s = main
            self._dedup_images(inverse=False)
            # the image inverse and its transpose run on the branch, beside the
            # image-MLP forward (which needs only the unique keys)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                self.s = side.cuda_stream
                self._inverse_images()
                inv_ready = torch.cuda.Event()
                inv_ready.record(side)
                self._transpose_images()
            self.s = main
            if self.n_img_segs:
                self._image_forward(self.net, self.uniq_img, self.counts.data_ptr())
            torch.cuda.current_stream().wait_event(inv_ready)  # the per-sample kernels read inv_img
            if self.model.layout.multiquery:  # the ID query rows of the second channel
                torch.cuda.current_stream().wait_event(ids_ready)
            L.check(L.lib.dicm_images_fwd(C.byref(self.layout), C.byref(self._bv), self.attn, self.head_in.data_ptr(),
                                          self.scores.data_ptr(), self.stats.data_ptr(), self.s))
            torch.cuda.current_stream().wait_stream(side)
            def id_grads_after_head():
                # the ID-row ordered sums, the head partial reduce and the
                # row-gradient finite check need only the head's gradients:
                # forked here, they run beside the attention backward
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    self._id_row_grads(side.cuda_stream)
                    self._reduce_head_partials(side.cuda_stream)
                    L.check(L.lib.dicm_check_finite(self.d_rows.data_ptr(), self.cap_k * 12,
                                                    self.counts[1:].data_ptr(), 12, 4, self.status.data_ptr(),
                                                    side.cuda_stream))

            # (multi-query attention: the ID query fields' rows also collect
            # the attention backward's query gradients, so they wait for it)
            # DICM_ID_FORK=head: measured neutral (r2 idfork A/B: k_dw1b -43 us,
            # the attention backward + image sums +46 us), so off by default
            early = os.environ.get("DICM_ID_FORK", "bwd") == "head" and not self.model.layout.multiquery
            self._local_step(self.net.emb, self.net.d_emb, denom, reduce=False, id_rows=False, fwd=False,
                             after_head=id_grads_after_head if early else None)
            if early:  # the attention partial reduce waits for the attention backward
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    self._reduce_attn_partials(side.cuda_stream)
                self._rows_checked = True
                side = _Joined(side)
        else:
            self._dedup_images()
            self._dedup_ids()
            self._transpose_images()
            self._transpose_ids()
            if self.n_img_segs:
                self._image_forward(self.net, self.uniq_img, self.counts.data_ptr())
            self._gather_id_rows()
            self._local_step(self.net.emb, self.net.d_emb, denom)
        if side is not None and not isinstance(side, _Joined):  # the ID-row gradients and the partial reduces
            side.wait_stream(torch.cuda.current_stream())       # overlap the image-MLP backward
            with torch.cuda.stream(side):
                self._id_row_grads(side.cuda_stream)
                self._reduce_partials(side.cuda_stream)
                # the row-gradient finite check (optimizer_step) needs only dRows
                L.check(L.lib.dicm_check_finite(self.d_rows.data_ptr(), self.cap_k * 12, self.counts[1:].data_ptr(),
                                                12, 4, self.status.data_ptr(), side.cuda_stream))
            self._rows_checked = True
        self._image_backward(self.net, self.uniq_img, self.counts.data_ptr(), self.cap_u if self.n_img_segs else 0)
        if side is not None:
            torch.cuda.current_stream().wait_stream(side.stream if isinstance(side, _Joined) else side)
        return self.loss

    def optimizer_step(self, lr, row_keys=None, row_count=None, row_grads=None, row_cap=None, tabstate=None):
        s = L.stream_handle()
        st = self.status.data_ptr()
        row_keys = self.uniq_id if row_keys is None else row_keys
        row_count = self.counts[1:] if row_count is None else row_count
        row_grads = self.d_rows if row_grads is None else row_grads
        row_cap = self.cap_k if row_cap is None else row_cap
        tabstate = self.tabstate if tabstate is None else tabstate
        if not self._rows_checked:  # the step checked these rows on its forked branch already
            L.check(L.lib.dicm_check_finite(row_grads.data_ptr(), row_cap * 12, row_count.data_ptr(), 12, 4, st, s))
        self._rows_checked = False
        L.check(L.lib.dicm_adam_dense(self.model.dense.data_ptr(), self.grad.data_ptr(), self.m.data_ptr(),
                                      self.v.data_ptr(), self.t.data_ptr(), self.spans, len(self.spans), lr, BETA1,
                                      BETA2, EPS, self.adam_ws.data_ptr(), self.adam_ws.numel(), st, s))
        L.check(L.lib.dicm_adam_rows(tabstate, len(self.fields), row_keys.data_ptr(), row_count.data_ptr(), row_cap,
                                     row_grads.data_ptr(), lr, BETA1, BETA2, EPS, st, s))

    def lr(self):
        return lr_schedule(self.iteration, self.lr0, self.lr_decay, self.lr_interval)

    # -- forward only (inference: reference KvPredictor, predict_logits) ---
    def _infer_net(self, cap):
        net = getattr(self, "_inet", None)
        if net is None or net.cap < cap:
            net = self._inet = ImageNetBuffers(cap, self.pool.d_raw, self.prec_code, self.dev)
        return net

    def embed_rows(self, rows, n, out, chunk=1 << 19):
        """out[i] = image-net embedding of pool row rows[i] for i < n (rows:
        device int32; out: device [>= n, 12] fp32), in chunks through the
        training forward kernels (reference model.embed_images,
        model.py:355-356)."""
        if n <= 0:
            return
        net = self._infer_net(min(chunk, n))
        cnt = torch.empty(1, dtype=torch.int32, device=self.dev)
        s = L.stream_handle()
        for s0 in range(0, n, net.cap):
            m = min(net.cap, n - s0)
            cnt.fill_(m)
            L.check(L.lib.dicm_imgmlp_fwd(self.pool.rows.data_ptr(), self.pool.dtype_code, self.pool.d_raw,
                                          rows.data_ptr() + 4 * s0, cnt.data_ptr(), net.cap, C.byref(self.img_p),
                                          net.act0.data_ptr(), net.act1.data_ptr(), out.data_ptr() + 48 * s0,
                                          self.prec_code, net.ws.data_ptr(), net.ws.numel(), s))

    def forward_logits(self, db, table=None):
        """Logits of one uploaded batch (no loss, no gradients).  Image
        embeddings come from the live image net, or -- with ``table`` (a device
        [T, 12] fp32 tensor of exported embeddings, row = image id) -- from the
        table for ids < T and the live net for the cold ids >= T (reference
        KvPredictor._embedding_matrix, inference.py:61-70)."""
        self._begin(db)
        self._dedup_images()
        self._dedup_ids()
        U = int(self.counts[0].item()) if self.n_img_segs else 0
        if U:
            if table is None:
                self.embed_rows(self.uniq_img, U, self.net.emb)
            else:
                T = int(table.shape[0])
                k = int(torch.searchsorted(self.uniq_img[:U], torch.tensor([T], dtype=torch.int32,
                                                                             device=self.dev)).item())
                if k:
                    ts = (L.TableState * 1)()
                    ts[0].table, ts[0].base, ts[0].vocab = table.data_ptr(), 0, T
                    cnt = torch.tensor([k], dtype=torch.int32, device=self.dev)
                    L.check(L.lib.dicm_gather_rows_by_key(ts, 1, self.uniq_img.data_ptr(), cnt.data_ptr(), k,
                                                          self.net.emb.data_ptr(), self.s))
                if k < U:  # cold path: ids beyond the table
                    self.embed_rows(self.uniq_img[k:U], U - k, self.net.emb[k:U])
        self._gather_id_rows()
        bv = self._batch_view(self.net.emb)
        L.check(L.lib.dicm_sample_fwd(C.byref(self.layout), C.byref(bv), self.attn, self.head_in.data_ptr(),
                                      self.scores.data_ptr(), self.stats.data_ptr(), self.s))
        self._head_fwd(self.pk.B)
        return self.logits[:self.pk.B]

    def step_device(self, db, denominator=None):
        """Full step on an already-uploaded batch; returns the device loss."""
        if self.use_graphs:
            return self.step_graphed(db, denominator)
        loss = self.forward_backward(db, denominator)
        self.optimizer_step(self.lr())
        self.iteration += 1
        return loss

    def step(self, batch, denominator=None):
        """Upload + full step; returns the device loss (no sync)."""
        db = self.upload(batch)
        if self.use_graphs:
            return self.step_graphed(db, denominator)
        loss = self.forward_backward(db, denominator)
        self.optimizer_step(self.lr())
        self.iteration += 1
        return loss

    # -- CUDA graphs ---------------------------------------------------
    use_graphs = False
    _graphs = None
    _graph_warm = False

    def step_graphed(self, db, denominator=None):
        """One full step (forward_backward + optimizer_step) replayed from a
        CUDA graph captured once per (batch layout, denominator, lr): the ~50
        library launches of a step become one graph launch.  The batch is
        copied into the engine's own upload buffer first when it lives
        elsewhere.  The first call for an engine runs eagerly (it sets kernel
        attributes and builds communicators, which must not happen inside a
        capture)."""
        lr = self.lr()
        if db.packed.data_ptr() != self.packed.data_ptr():
            self.packed[:db.pk.total].copy_(db.packed[:db.pk.total], non_blocking=True)
            db = DeviceBatch(db.pk, self.packed)
        if not self._graph_warm:
            self._graph_warm = True
            loss = self.forward_backward(db, denominator)
            self.optimizer_step(lr)
            self.iteration += 1
            return loss
        if self._graphs is None:
            self._graphs = {}
        key = (db.pk.signature(), None if denominator is None else float(denominator), lr)
        g = self._graphs.get(key)
        if g is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph(keep_graph=True)  # the node list stays inspectable (kernel_nodes)
            with torch.cuda.graph(g):
                self.forward_backward(db, denominator)
                self.optimizer_step(lr)
            g.instantiate()
            self._graphs[key] = g
        self._last_graph = g
        g.replay()
        self.iteration += 1
        return self.loss

    _OWN_SOURCES = ("capi", "dedup", "exchange", "head", "imgmlp", "imgmlp_bf16_sm100", "imgmlp_sm100",
                    "imgmlp_small_sm100", "optim", "p2p", "pool", "sample", "towers", "transpose")

    def kernel_nodes(self, detail=False):
        """(own, total) kernel nodes of the last captured step graph: every
        kernel the step launches, and those written in this library
        (csrc/*.cu).  The CUB scan kernels instantiated inside the
        library by dicm_ref_transpose (CUDA toolkit templates) are counted
        apart (``detail=True`` -> (own, cub, total)); NCCL or torch kernels
        in the graph are counted in total only."""
        g = getattr(self, "_last_graph", None)
        if g is None:
            return None
        from cuda.bindings import driver as cu
        err, _, n = cu.cuGraphGetNodes(g.raw_cuda_graph(), 0)
        err, nodes, n = cu.cuGraphGetNodes(g.raw_cuda_graph(), n)
        own = cub = total = 0
        for nd in nodes[:n]:
            err, ty = cu.cuGraphNodeGetType(nd)
            if ty != cu.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
                continue
            total += 1
            err, prm = cu.cuGraphKernelNodeGetParams(nd)
            err, name = cu.cuFuncGetName(prm.func)
            name = name.decode() if isinstance(name, bytes) else str(name)
            if "4dicm" in name or any(f"_{s}_cu_" in name for s in self._OWN_SOURCES):
                own += 1
            elif name.startswith("_ZN3cub"):
                cub += 1
        return (own, cub, total) if detail else (own, total)

    def raise_status(self):
        """Sync point: raise the reference's exception for a flagged step."""
        st = self.status.cpu().numpy()
        if st[L.ST_P2P_TIMEOUT]:
            self.status.zero_()
            raise RuntimeError("p2p barrier timeout: a peer missed a barrier (the step's updates were skipped)")
        if st[L.ST_KEY_FLAG]:
            self.status.zero_()
            tag, seg = divmod(int(st[L.ST_KEY_SEG]), 16)
            if tag == 0:
                raise KeyError(f"unknown image id {int(st[L.ST_KEY_VALUE])} (store holds 0.."
                               f"{self.pool.global_size - 1})")
            f = self.fields[seg] if tag == 1 else None
            if f is None:
                raise KeyError(f"key {int(st[L.ST_KEY_VALUE])} outside this shard")
            raise KeyError(f"id {int(st[L.ST_KEY_VALUE])} outside vocabulary of size {f.vocab} "
                           f"(field {f.name})")
        if st[L.ST_NONFINITE]:
            self.status.zero_()
            bits = int(st[L.ST_NONFINITE])
            if bits & 1:
                raise FloatingPointError(f"non-finite loss at iteration {self.iteration - 1}")
            raise FloatingPointError("adam: non-finite gradient, parameter untouched")

    # -- instrumentation ---------------------------------------------
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

    def count_step_kernels(self, db, denominator=None):
        """(own, cub, total) kernel nodes of one step (forward_backward +
        optimizer_step) captured into a throwaway graph that is never
        replayed: the launch count of an eager step, read from the same graph
        API as ``kernel_nodes``.  Needs a warmed-up engine (kernel attributes
        set) and no other thread issuing CUDA work during the capture."""
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g):
            self.forward_backward(db, denominator)
            self.optimizer_step(self.lr())
        saved, self._last_graph = getattr(self, "_last_graph", None), g
        try:
            return self.kernel_nodes(detail=True)
        finally:
            self._last_graph = saved

    # -- inspection ---------------------------------------------------
    def unique_images(self):
        n = int(self.counts[0].item())
        return self.uniq_img[:n].cpu().numpy()

    def unique_rows(self):
        n = int(self.counts[1].item())
        return self.uniq_id[:n].cpu().numpy()
