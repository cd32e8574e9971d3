"""Multi-GPU AMS training: the drop-in for the reference ``Cluster``
(runtime.py:313-516) and ``run_training`` (runtime.py:519-554).

One process per GPU; every GPU hosts one worker (a contiguous slice of the
union batch, runtime.py:379-382) and one server (the image-pool rows and
ID-table rows it owns, runtime.py:98-124).  A key is owned by rank
key % world and stored there at row key // world (any balanced placement is
valid).  One iteration (reference phases, runtime.py:378-463):

  1. local dedup of image keys and ID keys              (a2, on device)
  2. bucket unique keys by owner; all-to-all of counts (the one host sync),
     then all-to-all-v of the keys                       (C1, C3 of SURVEY 2.2)
  3. owner: dedup across sources, image MLP forward once per distinct image,
     gather ID rows; all-to-all-v the rows back          (C2, C3)
  4. local pooling + head forward/backward               (a6-a12)
  5. all-to-all-v the embedding and ID-row gradients to the owners; owners
     reduce per key in ascending source order (no float atomics) (C4, C5)
  6. owner: image MLP backward; ONE all-reduce(sum) over the fused buffer of
     every dense gradient (head, attention, image net)   (C6 + C7)
  7. Adam on the (bit-identical) dense replicas, row Adam on owned ID rows.

Collectives are NCCL calls through torch.distributed on the compute stream.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .batch import Batch, encode_batch
from .engine import ImageNetBuffers, StepEngine, _u8, lr_schedule

MODES = ("ams", "ps-store-in-server", "store-in-worker")


@dataclass
class ClusterConfig:
    workers: int = 4
    servers: int = 2
    mode: str = "ams"
    batch_per_worker: int = 64
    deterministic: bool = True

    def __post_init__(self):
        if self.workers < 1 or self.servers < 1:
            raise ValueError("cluster needs at least one worker and one server")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}; use one of {MODES}")


def shard_of(key, n):
    """Stable hash placement (reference runtime.py:60-68), kept for API parity;
    the device path places key k on rank k % n."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if not isinstance(key, (str, bytes)):
        key = repr(key)
    if isinstance(key, str):
        key = key.encode()
    return zlib.crc32(key) % n


def params_digest(params):
    """Order-independent fingerprint of a named parameter set (runtime.py:79-86)."""
    h = hashlib.sha256()
    for name in sorted(params):
        arr = params[name]
        arr = arr.data if hasattr(arr, "data") and not isinstance(arr, np.ndarray) else arr
        h.update(name.encode())
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


@dataclass
class RunLog:
    losses: list = field(default_factory=list)
    lrs: list = field(default_factory=list)
    embed_forwards: list = field(default_factory=list)
    unique_images: list = field(default_factory=list)
    replica_digests: list = field(default_factory=list)


def _a2a(out, inp, out_splits, in_splits, group=None):
    """all-to-all-v along dim 0 (NCCL on GPU tensors, gloo on CPU tensors)."""
    dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)


def exchange_counts(send_counts, group=None):
    """[world, k] int32 per-destination counts -> ([world, k] send, [world, k]
    recv) on the host; the single host synchronisation of an iteration."""
    recv = torch.empty_like(send_counts)
    dist.all_to_all_single(recv, send_counts.contiguous(), group=group)
    both = torch.cat([send_counts, recv]).cpu()
    w = send_counts.shape[0]
    return both[:w], both[w:]


def p2p_plan(cmat, rank):
    """Host restatement of the device placement plan (csrc/p2p.cu k_plan) for
    one kind of key: cmat[s][d] = rows source s sends to owner d.  Returns
    (send_off[d], pos_at_dest[d], recv_off[s], back_pos[s]):
      send_off     where this rank's segment for owner d starts in its send buffer
      pos_at_dest  where that segment lands in owner d's receive buffer
      recv_off     where source s's segment starts in this rank's receive buffer
      back_pos     where this rank's answers for requester s land in s's buffer
    (= s's send offset for this rank, so answers come back in send order)."""
    c = np.asarray(cmat, dtype=np.int64)
    w = c.shape[0]
    send_off = np.concatenate([[0], np.cumsum(c[rank])])
    pos_at_dest = np.array([c[:rank, d].sum() for d in range(w)], dtype=np.int64)
    recv_off = np.concatenate([[0], np.cumsum(c[:, rank])])
    back_pos = np.array([c[s, :rank].sum() for s in range(w)], dtype=np.int64)
    return send_off, pos_at_dest, recv_off, back_pos


class _ExtMem:
    """A device allocation the library owns, seen by torch through
    __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerExchange:
    """The AMS exchanges over NVLink peer memory (include/dicm_b200.h, a16 over
    NVLink): one exchange region per rank, identical layout on every rank,
    mapped into every peer with CUDA IPC.  Layout (byte offsets):

        flags      [64] uint32            barrier epochs, slot = source rank
        cmat       [world][world][2] i32  per-pair counts (row = source)
        recv_img   [cap_ri] i32           keys this owner receives
        recv_id    [cap_rk] i32
        push_img   [cap_ri, 12] f32       embedding gradients this owner receives
        push_id    [cap_rk, 12] f32       ID-row gradients this owner receives
        back_img   [cap_u, 12] f32        embeddings this requester receives
        back_id    [cap_k, 12] f32        ID rows this requester receives

    Capacities are agreed once (max over ranks) when the region is built."""

    def __init__(self, world, rank, cap_u, cap_k, local_rows, local_id_space, group=None, dense_n=0):
        dev = torch.device("cuda", torch.cuda.current_device())
        # every capacity the layout depends on is agreed (max over ranks):
        # a peer writes into our region at ITS offsets, so the layout must be
        # identical everywhere (pool shards differ by one row when P % world)
        caps = torch.tensor([cap_u, cap_k, local_rows, local_id_space], dtype=torch.int64, device=dev)
        dist.all_reduce(caps, op=dist.ReduceOp.MAX, group=group)
        cap_u, cap_k, local_rows, local_id_space = (int(x) for x in caps.cpu().tolist())
        self.world, self.rank = world, rank
        self.cap_u, self.cap_k = cap_u, cap_k
        self.cap_ri = min(world * cap_u, world * max(local_rows, 1))
        self.cap_rk = min(world * cap_k, world * max(local_id_space, 1))
        off, layout = 0, {}

        def take(name, nbytes):
            nonlocal off
            layout[name] = off
            off += (int(nbytes) + 255) // 256 * 256

        take("flags", 64 * 4)
        take("flags_side", 64 * 4)  # the barriers of the forked stream (their own epoch counter)
        take("cmat", world * world * 2 * 4)
        take("recv_img", self.cap_ri * 4)
        take("recv_id", self.cap_rk * 4)
        take("push_img", self.cap_ri * 48)
        take("push_id", self.cap_rk * 48)
        take("back_img", cap_u * 48)
        take("back_id", cap_k * 48)
        # the dense all-reduce (dicm_p2p_allreduce): staged gradients and sums
        self.dense_n = int(dense_n)
        take("grad_stage", (self.dense_n + 3) // 4 * 16)
        take("grad_sum", (self.dense_n + 3) // 4 * 16)
        self.off, self.bytes = layout, off
        lay = torch.tensor([off] + [layout[k] for k in sorted(layout)], dtype=torch.int64, device=dev)
        lo, hi = lay.clone(), lay.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
        if not torch.equal(lo, hi):
            raise RuntimeError("peer exchange regions differ between ranks")
        base = C.c_void_p()
        L.check(L.lib.dicm_p2p_alloc(off, C.byref(base)))
        self.base = base.value
        h = (C.c_char * 64)()
        L.check(L.lib.dicm_ipc_handle(self.base, h))
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h), group=group)
        self.peers = L.Peers()
        self.peers.world, self.peers.rank = world, rank
        self._opened = []
        for r in range(world):
            if r == rank:
                self.peers.region[r] = self.base
            else:
                p = C.c_void_p()
                L.check(L.lib.dicm_ipc_open((C.c_char * 64).from_buffer_copy(handles[r]), C.byref(p)))
                self.peers.region[r] = p.value
                self._opened.append(p.value)
        self.epoch = 0
        self.plan = torch.zeros(2 * 4 * (L.MAX_PEERS + 1), dtype=torch.int64, device=dev)
        i32, f32 = "<i4", "<f4"
        self.recv_img = self._view("recv_img", (self.cap_ri,), i32)
        self.recv_id = self._view("recv_id", (self.cap_rk,), i32)
        self.push_img = self._view("push_img", (self.cap_ri, 12), f32)
        self.push_id = self._view("push_id", (self.cap_rk, 12), f32)
        self.back_img = self._view("back_img", (cap_u, 12), f32)
        self.back_id = self._view("back_id", (cap_k, 12), f32)
        dist.barrier(group=group)

    def _view(self, name, shape, typestr):
        return torch.as_tensor(_ExtMem(self.base + self.off[name], shape, typestr), device="cuda")

    def allreduce(self, buf, status, s):
        """buf (the fused gradient buffer + loss, float32, dense_n elements) <-
        its sum over every rank, in rank order (bit-identical replicas)."""
        L.check(L.lib.dicm_p2p_allreduce(C.byref(self.peers), buf.data_ptr(), self.dense_n, self.off["grad_stage"],
                                         self.off["grad_sum"], self.off["flags"], status, buf.data_ptr(), s))

    def barrier_side(self, status, s):
        """A barrier on the forked stream: its own flag slots and epoch
        counter, so it may run concurrently with the main stream's barriers."""
        L.check(L.lib.dicm_p2p_barrier(C.byref(self.peers), self.off["flags_side"], 0, status, s))

    def barrier(self, status, s):
        # epoch 0: the kernel advances a device-side counter (CUDA-graph safe)
        L.check(L.lib.dicm_p2p_barrier(C.byref(self.peers), self.off["flags"], 0, status, s))

    def counts(self, send_counts, s):
        L.check(L.lib.dicm_p2p_counts(C.byref(self.peers), send_counts, self.off["cmat"], s))

    def plan_from_counts(self, seg_img, seg_id, cnt_dev, s):
        L.check(L.lib.dicm_p2p_plan(C.byref(self.peers), self.off["cmat"], seg_img, seg_id, cnt_dev,
                                    self.plan.data_ptr(), s))

    def scatter(self, kind, direction, src, row_bytes, dst, s):
        L.check(L.lib.dicm_p2p_scatter(C.byref(self.peers), self.plan.data_ptr(), kind, direction, src, row_bytes,
                                       self.off[dst], s))

    def gather_scatter12(self, kind, direction, rows, idx, dst, s):
        """scatter() of rows[idx[i]] (12-float rows) without a staged copy."""
        L.check(L.lib.dicm_p2p_gather_scatter12(C.byref(self.peers), self.plan.data_ptr(), kind, direction, rows,
                                                idx, self.off[dst], s))

    def close(self):
        for p in self._opened:
            L.lib.dicm_ipc_close(p)
        self._opened = []


class ClusterEngine(StepEngine):
    """One rank of the sharded AMS step."""

    def __init__(self, model, pool, precision="fp32", lr0=0.001, lr_decay=0.9, lr_interval=24000, world=1, rank=0,
                 group=None):
        if pool.world != world or pool.rank != rank:
            raise ValueError(f"pool shard ({pool.world}, {pool.rank}) != rank ({world}, {rank})")
        self.world, self.rank, self.group = world, rank, group
        import os
        # sparse exchanges: NVLink peer-memory copies (default) or NCCL all-to-all-v
        self.exchange = os.environ.get("DICM_EXCHANGE", "p2p")
        if self.exchange not in ("p2p", "nccl"):
            raise ValueError(f"DICM_EXCHANGE must be p2p or nccl, got {self.exchange!r}")
        self.px = None
        super().__init__(model, pool, precision, lr0, lr_decay, lr_interval, id_align=world)
        dev = self.dev
        # owner-side descriptors: owner-local key = global key // world
        self.owner_tabstate = self._table_states(self.bases, world)
        self.local_id_space = self.id_key_space // world
        self.ws_id_owner = _u8(L.lib.dicm_dedup_workspace(max(self.local_id_space, 1)), dev)
        self.ws_img_owner = _u8(L.lib.dicm_dedup_workspace(max(pool.local_rows, 1)), dev)
        self.segs_img = torch.zeros(world + 1, dtype=torch.int64, device=dev)
        self.segs_id = torch.zeros(world + 1, dtype=torch.int64, device=dev)
        self._seg_host = torch.zeros(2 * (world + 1), dtype=torch.int64, pin_memory=True)
        self._timing = os.environ.get("DICM_PHASE_TIMING") == "1"
        self._allreduce = os.environ.get("DICM_ALLREDUCE", "p2p")
        if self._allreduce not in ("p2p", "nccl"):
            raise ValueError(f"DICM_ALLREDUCE must be p2p or nccl, got {self._allreduce!r}")
        self._marks = None

    @property
    def image_key_space(self):
        return self.pool.global_size  # requests are in global image ids

    declared = None  # (packed words, samples, behaviors, ID refs): Cluster's per-rank maximum

    def declare_capacity(self, batch_per_worker):
        """Size every buffer once for the largest local batch any rank can see
        (``batch_per_worker`` samples of at most ``b_max`` behaviors, and
        multi-hot fields tail-truncated to ``b_max`` like the reference,
        model.py:168,176).  All ranks compute the same numbers, so the peer
        exchange built from them never has to grow -- a one-sided regrowth
        would desynchronise the collective layout."""
        B, bm = int(batch_per_worker), int(self.model.schema.b_max)
        fields = self.model.layout.schema.fields
        n_multi = sum(1 for f in self.fields if f.multi)
        n_one = len(self.fields) - n_multi
        R = B * bm
        n_id = B * n_one + R * n_multi
        total = sum((R + B + 1) if f.multi else B for f in fields) + 2 * B + R + B + 1
        self.declared = (total, B, R, n_id)

    def _ensure(self, pk):
        need = self._need(pk)
        if self.declared is None:
            return super()._ensure(pk)
        if self.cap is None:
            self._alloc_caps(tuple(max(a, b) for a, b in zip(need, self.declared)))
        elif not all(a <= b for a, b in zip(need, self.cap)):
            raise ValueError(f"local batch needs {need}, beyond the declared per-rank capacity {self.cap} "
                             "(batch_per_worker samples of at most b_max behaviors)")

    def _alloc_image_net(self, cap):
        dev, G = self.dev, self.world
        i32 = dict(dtype=torch.int32, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        cu, ck = max(self.cap_u, 1), max(self.cap_k, 1)
        # requester side
        self.emb_l = torch.empty((cu, 12), **f32)
        self.d_emb_l = torch.empty((cu, 12), **f32)
        self.send_img = torch.empty(cu, **i32)
        self.perm_img = torch.empty(cu, **i32)
        self.perm_inv_img = torch.empty(cu, **i32)  # gather form of perm_img (the gradient push)
        self.send_id = torch.empty(ck, **i32)
        self.perm_id = torch.empty(ck, **i32)
        self.perm_inv_id = torch.empty(ck, **i32)
        self.ws_bucket = _u8(L.lib.dicm_bucket_workspace(max(cu, ck), G), dev)
        self.ws_bucket_id = _u8(L.lib.dicm_bucket_workspace(max(cu, ck), G), dev)
        self.rows_buf = torch.empty((max(cu, ck), 12), **f32)  # responses in / pushes out
        # owner side (worst case: every rank asks for all its keys here)
        self._alloc_owner(G * cu, G * ck)
        self.cnt_dev = torch.zeros(4, dtype=torch.int32, device=dev)  # n_recv_img, n_recv_id, n_send_img, n_send_id

    def _alloc_owner(self, cap_ri, cap_rk):
        dev, G = self.dev, self.world
        i32 = dict(dtype=torch.int32, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.cap_ri, self.cap_rk = cap_ri, cap_rk
        if self.exchange == "nccl":
            self.recv_img = torch.empty(self.cap_ri, **i32)
            self.recv_id = torch.empty(self.cap_rk, **i32)
        self.cap_o = min(self.cap_ri, self.pool.local_rows)
        self.cap_ko = min(self.cap_rk, self.local_id_space)
        self.uniq_o = torch.empty(max(self.cap_o, 1), **i32)
        self.inv_o = torch.empty(self.cap_ri, **i32)
        self.uniq_id_o = torch.empty(max(self.cap_ko, 1), **i32)
        self.inv_id_o = torch.empty(self.cap_rk, **i32)
        self.resp = torch.empty((max(self.cap_ri, self.cap_rk), 12), **f32)
        self.d_rows_o = torch.empty((max(self.cap_ko, 1), 12), **f32)
        self.idx_ws = torch.empty(G * max(self.cap_o, self.cap_ko, 1), **i32)
        self.idx_ws_img = torch.empty(G * max(self.cap_o, 1), **i32)  # the image reduce runs beside the ID one
        self.net = ImageNetBuffers(self.cap_o, self.pool.d_raw, self.prec_code, dev)

    @property
    def emb(self):
        return self.emb_l

    @property
    def d_emb(self):
        return self.d_emb_l

    def _dedup_owner(self, keys, n, space, ws, uniq, inv, count_slot):
        seg = (L.KeySeg * 1)(L.KeySeg(keys.data_ptr(), n, 0, space, 0))
        L.check(L.lib.dicm_dedup(seg, 1, space, ws.data_ptr(), ws.numel(), uniq.data_ptr(), inv.data_ptr(),
                                 self.counts[count_slot:].data_ptr(), 2, self.status.data_ptr(), self.s))

    def _mark(self, name):
        """Phase timing (DICM_PHASE_TIMING=1): an event on the compute stream."""
        if self._marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._marks.append((name, ev))

    def phase_times(self):
        """{phase: ms} of the last iteration (needs DICM_PHASE_TIMING=1)."""
        if not self._marks:
            return {}
        torch.cuda.synchronize()
        out, prev = {}, None
        for name, ev in self._marks:
            if prev is not None:
                out[name] = out.get(name, 0.0) + prev.elapsed_time(ev)
            prev = ev
        return out

    def forward_backward(self, db, denominator=None):
        if self.exchange == "p2p":
            return self._forward_backward_p2p(db, denominator)
        G, s = self.world, None
        self._marks = [] if self._timing else None
        self._mark("start")
        self._begin(db)
        s = self.s
        denom = float(db.pk.B * G if denominator is None else denominator)
        self._dedup_images()
        self._dedup_ids()
        self._transpose_images()
        self._transpose_ids()
        cnt = self.counts
        # (2) requests: bucket by owner, exchange counts, then keys
        L.check(L.lib.dicm_bucket_by_owner(self.uniq_img.data_ptr(), cnt.data_ptr(), self.cap_u, G,
                                           self.send_img.data_ptr(), self._col(0), self.perm_img.data_ptr(), None,
                                           self.ws_bucket.data_ptr(), self.ws_bucket.numel(), s))
        L.check(L.lib.dicm_bucket_by_owner(self.uniq_id.data_ptr(), cnt[1:].data_ptr(), self.cap_k, G,
                                           self.send_id.data_ptr(), self._col(1), self.perm_id.data_ptr(), None,
                                           self.ws_bucket.data_ptr(), self.ws_bucket.numel(), s))
        self._mark("dedup+bucket")
        pair = self._cnt_both.t().contiguous()
        sent, recv = exchange_counts(pair, self.group)
        self._mark("count exchange (host sync)")
        si, sk = sent[:, 0].tolist(), sent[:, 1].tolist()
        ri, rk = recv[:, 0].tolist(), recv[:, 1].tolist()
        nsi, nsk, nri, nrk = sum(si), sum(sk), sum(ri), sum(rk)
        self._splits = (si, sk, ri, rk)
        h = self._seg_host
        h[0] = 0
        h[1:G + 1] = torch.tensor(np.cumsum(ri), dtype=torch.int64)
        h[G + 1] = 0
        h[G + 2:] = torch.tensor(np.cumsum(rk), dtype=torch.int64)
        self.segs_img.copy_(h[:G + 1], non_blocking=True)
        self.segs_id.copy_(h[G + 1:], non_blocking=True)
        self.cnt_dev.copy_(torch.tensor([nri, nrk, nsi, nsk], dtype=torch.int32), non_blocking=True)
        _a2a(self.recv_img[:nri], self.send_img[:nsi], ri, si, self.group)
        _a2a(self.recv_id[:nrk], self.send_id[:nsk], rk, sk, self.group)
        self._mark("a2a keys")
        # (3) owner: one image-MLP forward per distinct image, ID rows
        self._dedup_owner(self.recv_img, nri, self.pool.local_rows, self.ws_img_owner, self.uniq_o, self.inv_o, 2)
        self._mark("owner dedup")
        if self.n_img_segs:
            self._image_forward(self.net, self.uniq_o, cnt[2:].data_ptr())
        self._mark("image MLP fwd")
        L.check(L.lib.dicm_permute_rows12(self.net.emb.data_ptr(), self.inv_o.data_ptr(), self.cnt_dev.data_ptr(),
                                          max(nri, 0), 0, self.resp.data_ptr(), s))
        _a2a(self.rows_buf[:nsi], self.resp[:nri], si, ri, self.group)
        self._mark("a2a E rows")
        L.check(L.lib.dicm_permute_rows12(self.rows_buf.data_ptr(), self.perm_img.data_ptr(), cnt.data_ptr(),
                                          self.cap_u, 0, self.emb_l.data_ptr(), s))
        L.check(L.lib.dicm_gather_rows_by_key(self.owner_tabstate, len(self.fields), self.recv_id.data_ptr(),
                                              self.cnt_dev[1:].data_ptr(), max(nrk, 0), self.resp.data_ptr(), s))
        _a2a(self.rows_buf[:nsk], self.resp[:nrk], sk, rk, self.group)
        L.check(L.lib.dicm_permute_rows12(self.rows_buf.data_ptr(), self.perm_id.data_ptr(), cnt[1:].data_ptr(),
                                          self.cap_k, 0, self.id_rows.data_ptr(), s))
        self._mark("ID rows + a2a")
        # (4) local pooling + head
        self._local_step(self.emb_l, self.d_emb_l, denom)
        self._mark("pooling+head")
        # (5) push gradients to the owners; owners reduce in ascending source order
        L.check(L.lib.dicm_permute_rows12(self.d_emb_l.data_ptr(), self.perm_img.data_ptr(), cnt.data_ptr(),
                                          self.cap_u, 1, self.rows_buf.data_ptr(), s))
        _a2a(self.resp[:nri], self.rows_buf[:nsi], ri, si, self.group)
        L.check(L.lib.dicm_owner_reduce_rows12(self.resp.data_ptr(), self.inv_o.data_ptr(), self.segs_img.data_ptr(),
                                               G, max(nri, 0), cnt[2:].data_ptr(), self.cap_o, self.idx_ws.data_ptr(),
                                               self.net.d_emb.data_ptr(), s))
        self._mark("a2a dE + owner reduce")
        # (6) owner image-MLP backward
        self._image_backward(self.net, self.uniq_o, cnt[2:].data_ptr(), self.cap_o if self.n_img_segs else 0)
        self._mark("image MLP bwd")
        L.check(L.lib.dicm_permute_rows12(self.d_rows.data_ptr(), self.perm_id.data_ptr(), cnt[1:].data_ptr(),
                                          self.cap_k, 1, self.rows_buf.data_ptr(), s))
        _a2a(self.resp[:nrk], self.rows_buf[:nsk], rk, sk, self.group)
        self._dedup_owner(self.recv_id, nrk, self.local_id_space, self.ws_id_owner, self.uniq_id_o, self.inv_id_o, 3)
        L.check(L.lib.dicm_owner_reduce_rows12(self.resp.data_ptr(), self.inv_id_o.data_ptr(), self.segs_id.data_ptr(),
                                               G, max(nrk, 0), cnt[3:].data_ptr(), self.cap_ko,
                                               self.idx_ws.data_ptr(), self.d_rows_o.data_ptr(), s))
        # (6) every dense gradient in one all-reduce (sum: the loss is already
        # divided by the union batch, runtime.py:374, training.py:42)
        self._mark("ID grads a2a + reduce")
        dist.all_reduce(self.grad_ext, group=self.group)  # dense gradients and the loss
        self._mark("allreduce")
        return self.loss

    def _forward_backward_p2p(self, db, denominator=None):
        """The same iteration with every sparse exchange done by peer-memory
        copy kernels and device-side counts: no host synchronisation.  The ID
        chains run on a forked stream beside the image chain -- the owner's ID
        rows go out while the image-MLP forward runs, the owner's ID-gradient
        reduction and the head/attention partial reduces run beside the
        image-MLP backward -- and one all-reduce sums the dense gradients and
        the loss (a graph with parallel branches once captured)."""
        G = self.world
        self._marks = [] if self._timing else None
        self._mark("start")
        self._begin(db)
        s, st = self.s, self.status.data_ptr()
        denom = float(db.pk.B * G if denominator is None else denominator)
        if self.px is None or self.px.cap_u < self.cap_u or self.px.cap_k < self.cap_k:
            if self.px is not None:
                raise RuntimeError("batch outgrew the peer exchange region built at the first iteration")
            self.px = PeerExchange(G, self.rank, self.cap_u, self.cap_k, self.pool.local_rows,
                                   self.local_id_space, self.group, dense_n=self.grad_ext.numel())
            self._alloc_owner(self.px.cap_ri, self.px.cap_rk)  # every owner buffer at the agreed capacity
            self.resp_id = torch.empty((max(self.px.cap_rk, 1), 12), dtype=torch.float32, device=self.dev)
        px = self.px
        side = self._side_stream()
        main_stream = torch.cuda.current_stream()

        def on_side(fn):
            """Run ``fn`` on the forked stream (ordered after everything queued
            so far on the main stream), or inline without a fork."""
            if side is None:
                fn(s)
                return
            side.wait_stream(main_stream)
            with torch.cuda.stream(side):
                fn(side.cuda_stream)

        def join():
            if side is not None:
                main_stream.wait_stream(side)

        cnt = self.counts

        def swap(fn):  # run an engine phase (which launches on self.s) on stream ss
            def run(ss):
                saved, self.s = self.s, ss
                try:
                    fn(ss)
                finally:
                    self.s = saved
            return run

        def id_chain(ss):  # ID keys: dedup, bucket by owner, the backward's transpose
            self._dedup_ids()
            L.check(L.lib.dicm_bucket_by_owner(self.uniq_id.data_ptr(), cnt[1:].data_ptr(), self.cap_k, G,
                                               self.send_id.data_ptr(), self._col(1), self.perm_id.data_ptr(),
                                               self.perm_inv_id.data_ptr(), self.ws_bucket_id.data_ptr(),
                                               self.ws_bucket_id.numel(), ss))

        # the ID chain beside the image chain; the counts wait for both buckets
        on_side(swap(id_chain))
        id_bucketed = None
        if side is not None:
            id_bucketed = torch.cuda.Event()
            id_bucketed.record(side)
        self._dedup_images()
        L.check(L.lib.dicm_bucket_by_owner(self.uniq_img.data_ptr(), cnt.data_ptr(), self.cap_u, G,
                                           self.send_img.data_ptr(), self._col(0), self.perm_img.data_ptr(),
                                           self.perm_inv_img.data_ptr(), self.ws_bucket.data_ptr(),
                                           self.ws_bucket.numel(), s))
        # the backward's summation order, needed only at the local step (joined before it)
        on_side(swap(lambda ss: (self._transpose_ids(), self._transpose_images())))
        if id_bucketed is not None:
            main_stream.wait_event(id_bucketed)
        self._mark("dedup+bucket")
        # (2) counts -> every peer, then the request keys (C1, C3)
        px.counts(self._col(0), s)
        px.barrier(st, s)
        px.plan_from_counts(self.segs_img.data_ptr(), self.segs_id.data_ptr(), self.cnt_dev.data_ptr(), s)
        px.scatter(0, 0, self.send_img.data_ptr(), 4, "recv_img", s)
        px.scatter(1, 0, self.send_id.data_ptr(), 4, "recv_id", s)
        px.barrier(st, s)
        self._mark("counts + keys")

        # (3) owner: ID rows back to the requesters (C3) on the branch, beside
        # the image chain: dedup across sources, one image-MLP forward per
        # distinct image, embeddings back (C2)
        def id_rows_out(ss):
            L.check(L.lib.dicm_gather_rows_by_key(self.owner_tabstate, len(self.fields), px.recv_id.data_ptr(),
                                                  self.cnt_dev[1:].data_ptr(), px.cap_rk, self.resp_id.data_ptr(), ss))
            px.scatter(1, 1, self.resp_id.data_ptr(), 48, "back_id", ss)

        on_side(id_rows_out)
        L.check(L.lib.dicm_dedup_devn(px.recv_img.data_ptr(), self.cnt_dev.data_ptr(), px.cap_ri,
                                      self.pool.local_rows, self.ws_img_owner.data_ptr(), self.ws_img_owner.numel(),
                                      self.uniq_o.data_ptr(), self.inv_o.data_ptr(), cnt[2:].data_ptr(), 2, st, s))
        self._mark("owner dedup")
        if self.n_img_segs:
            self._image_forward(self.net, self.uniq_o, cnt[2:].data_ptr())
        self._mark("image MLP fwd")
        # the owner's embeddings gathered by key and stored into the requesters' buffers in one pass
        px.gather_scatter12(0, 1, self.net.emb.data_ptr(), self.inv_o.data_ptr(), "back_img", s)
        join()
        px.barrier(st, s)
        L.check(L.lib.dicm_permute_rows12(px.back_img.data_ptr(), self.perm_img.data_ptr(), cnt.data_ptr(),
                                          self.cap_u, 0, self.emb_l.data_ptr(), s))
        L.check(L.lib.dicm_permute_rows12(px.back_id.data_ptr(), self.perm_id.data_ptr(), cnt[1:].data_ptr(),
                                          self.cap_k, 0, self.id_rows.data_ptr(), s))
        self._mark("rows back")
        # (4) local pooling + head (the partial reduces and the ID-row sums wait)
        self._local_step(self.emb_l, self.d_emb_l, denom, reduce=False, id_rows=False)
        self._mark("pooling+head")

        # (5b, 6b) on the branch: this rank's ID-row sums, their push to the
        # owners (C5) and a barrier on the branch's own flags, then the owner's
        # ID-row reduction in ascending source order (runtime.py:208-219), the
        # finite check and the head / attention partial reduces
        def id_chain_bwd(ss):
            self._id_row_grads(ss)
            px.gather_scatter12(1, 0, self.d_rows.data_ptr(), self.perm_inv_id.data_ptr(), "push_id", ss)
            px.barrier_side(st, ss)
            L.check(L.lib.dicm_dedup_devn(px.recv_id.data_ptr(), self.cnt_dev[1:].data_ptr(), px.cap_rk,
                                          self.local_id_space, self.ws_id_owner.data_ptr(), self.ws_id_owner.numel(),
                                          self.uniq_id_o.data_ptr(), self.inv_id_o.data_ptr(), cnt[3:].data_ptr(), 3,
                                          st, ss))
            L.check(L.lib.dicm_owner_reduce_rows12(px.push_id.data_ptr(), self.inv_id_o.data_ptr(),
                                                   self.segs_id.data_ptr(), G, px.cap_rk, cnt[3:].data_ptr(),
                                                   self.cap_ko, self.idx_ws.data_ptr(), self.d_rows_o.data_ptr(), ss))
            L.check(L.lib.dicm_check_finite(self.d_rows_o.data_ptr(), self.cap_ko * 12, cnt[3:].data_ptr(), 12, 4,
                                            st, ss))
            self._reduce_partials(ss)

        on_side(id_chain_bwd)
        # (5a, 6a) main stream: image gradients to the owners (C4), barrier, the
        # owner's reduction in ascending source order, the image-MLP backward
        # this rank's image gradients, in owner order, straight into the owners' buffers
        px.gather_scatter12(0, 0, self.d_emb_l.data_ptr(), self.perm_inv_img.data_ptr(), "push_img", s)
        px.barrier(st, s)
        self._mark("grads to owners")
        L.check(L.lib.dicm_owner_reduce_rows12(px.push_img.data_ptr(), self.inv_o.data_ptr(),
                                               self.segs_img.data_ptr(), G, px.cap_ri, cnt[2:].data_ptr(),
                                               self.cap_o, self.idx_ws_img.data_ptr(), self.net.d_emb.data_ptr(), s))
        self._image_backward(self.net, self.uniq_o, cnt[2:].data_ptr(), self.cap_o if self.n_img_segs else 0)
        join()
        self._rows_checked = True
        self._mark("image MLP bwd || ID grads")
        # (7) every dense gradient and the loss in one all-reduce over peer
        # memory (rank-order sums: bit-identical replicas); DICM_ALLREDUCE=nccl
        # uses NCCL instead
        if self._allreduce == "nccl":
            dist.all_reduce(self.grad_ext, group=self.group)
        else:
            px.allreduce(self.grad_ext, st, s)
        self._mark("allreduce")
        return self.loss
    def _col(self, j):
        """Per-owner send counts: row j of one [2][world] buffer (image keys,
        ID keys) that dicm_p2p_counts reads as a whole."""
        if not hasattr(self, "_cnt_both") or self._cnt_both.shape[1] != self.world:
            self._cnt_both = torch.zeros((2, self.world), dtype=torch.int32, device=self.dev)
            self._cnt_cols = [self._cnt_both[0], self._cnt_both[1]]
        return self._cnt_both[j].data_ptr()

    def optimizer_step(self, lr):
        super().optimizer_step(lr, row_keys=self.uniq_id_o, row_count=self.counts[3:], row_grads=self.d_rows_o,
                               row_cap=self.cap_ko, tabstate=self.owner_tabstate)

    def forwards(self):
        """Image-MLP forwards this rank ran in the last iteration."""
        return int(self.counts[2].item())


class Cluster:
    """Multi-GPU AMS cluster (reference runtime.py:313-516), one rank per
    process; every rank calls ``run_iteration`` with the same union batch.

    ``ClusterConfig(workers=M, servers=N)`` is the reference's LOGICAL actor
    topology; the physical one is the G GPUs of the process group.  Worker w
    runs on GPU w * G // M ... each GPU trains the contiguous union slice of
    the workers it hosts (reference runtime.py:379-382: workers take
    consecutive ``batch_per_worker`` slices, so a GPU's slice is contiguous
    too).  Keys are sharded over the G GPUs (owner key % G); logical server s
    is hosted by GPU s % G.  Placement never changes results (every
    reduction is per key or a fixed-order sum), so any (M, N) trains exactly
    like ``LocalTrainer`` on the union batch (runtime.py:19-21).

    ``model`` may be the full model (its values are copied into this rank's
    shard and ``collect_into_model`` writes the trained values back, like the
    reference's node replicas, runtime.py:108-111,490-495) or an already
    sharded one (``DicmModel(..., shard=(G, rank))``, trained in place: the
    scalable form for tables that do not fit one host)."""

    def __init__(self, cfg, model, store, lr0=0.001, lr_decay=0.9, lr_interval=24000, precision="fp32",
                 group=None):
        if cfg.mode != "ams":
            raise ValueError(
                f"training runs under mode 'ams' only; {cfg.mode!r} is an "
                "accounting-only storage strategy (see dicm.accounting)")
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.cfg, self.source_model, self.store = cfg, model, store
        self.world, self.rank = world, rank
        self.lr0, self.lr_decay, self.lr_interval = lr0, lr_decay, lr_interval
        self.group = group
        # the contiguous block of logical workers this GPU hosts
        self.w_lo, self.w_hi = rank * cfg.workers // world, (rank + 1) * cfg.workers // world
        if world > 1 and getattr(model, "shard", None) is None:
            model = model.sharded(world, rank)  # this rank's working copy
        self.model = model
        if world > 1:
            self.engine = ClusterEngine(model, store, precision, lr0, lr_decay, lr_interval, world, rank, group)
            self.engine.declare_capacity(max(self.w_hi - self.w_lo, 1) * cfg.batch_per_worker)
        else:
            self.engine = StepEngine(model, store, precision, lr0, lr_decay, lr_interval)

    @property
    def iteration(self):
        return self.engine.iteration

    def local_slice(self, union):
        b = union if isinstance(union, Batch) else encode_batch(union, self.model)
        bpw = self.cfg.batch_per_worker
        lo = min(self.w_lo * bpw, b.size)
        return b.slice(lo, min(b.size, self.w_hi * bpw)), b

    def run_iteration(self, union_batch, digests=True):
        """-> (loss, union_unique, forwards, digests) like runtime.py:465-470:
        the union loss, the union's distinct images, the image-net forwards
        summed over the servers (== union_unique: each distinct image is
        embedded once per iteration), and one image-net replica digest per
        logical server."""
        local, union = self.local_slice(union_batch)
        e = self.engine
        loss = self.train_batch_async(local, union.size)
        value = float(loss.item())
        e.raise_status()
        if self.world > 1:
            fw = torch.tensor([e.forwards()], dtype=torch.int64, device=e.dev)
            dist.all_reduce(fw, group=self.group)
            forwards = int(fw.item())
        else:
            forwards = len(e.unique_images()) if e.n_img_segs else 0
        lay = self.model.layout
        union_unique = len(union.unique_images(lay.use_ad_image, lay.use_behavior_images))
        dig = self.server_digests() if digests else []
        return value, union_unique, forwards, dig

    def server_digests(self):
        """params_digest of the image-net replica (reference ServerNode.digest,
        runtime.py:221-222) for each logical server, computed on the GPU that
        hosts it."""
        d = params_digest({n: p.data for n, p in self.model.params.items() if n.startswith("img/")})
        per_gpu = [d]
        if self.world > 1:
            per_gpu = [None] * self.world
            dist.all_gather_object(per_gpu, d, group=self.group)
        return [per_gpu[s % self.world] for s in range(self.cfg.servers)]

    def train_batch_async(self, local_batch, union_size):
        """This rank's part of an iteration on its already-sliced local batch
        (no host sync): upload, step, optimizer; returns the device loss.
        With ``use_graphs`` the step replays a captured CUDA graph."""
        e = self.engine
        db = e.upload(local_batch)
        if self.use_graphs:
            return e.step_graphed(db, denominator=union_size)
        loss = e.forward_backward(db, denominator=union_size)
        e.optimizer_step(e.lr())
        e.iteration += 1
        return loss

    def train_stream(self, unions, prefetch=2):
        """Train on an iterable of union batches (``Batch`` or sample lists),
        yielding each iteration's device loss without a host sync.  A worker
        thread slices, packs and copies iteration i+1's input while iteration
        i runs (engine.Prefetcher): the host pipeline of run_iteration hidden
        behind the device step."""
        from .engine import Prefetcher
        e = self.engine

        def prep(u):
            local, union = self.local_slice(u)
            return local, union.size

        for (local, union_size), db in Prefetcher(e, unions, prefetch, transform=prep):
            if self.use_graphs:
                yield e.step_graphed(db, denominator=union_size)
                continue
            loss = e.forward_backward(db, denominator=union_size)
            e.optimizer_step(e.lr())
            e.iteration += 1
            yield loss

    def close(self):
        """Release captured CUDA graphs and the peer-memory mappings (call
        before destroy_process_group; graphs that captured collectives and
        live IPC mappings must not outlive the communicator)."""
        e = self.engine
        e.use_graphs = False
        e._graphs = None
        e._last_graph = None  # kept graphs hold NCCL nodes: release them before the communicator
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        px = getattr(e, "px", None)
        if px is not None:
            if self.world > 1 and dist.is_initialized():
                dist.barrier(group=self.group)  # no peer may still be writing into our region
            px.close()

    @property
    def use_graphs(self):
        return self.engine.use_graphs

    @use_graphs.setter
    def use_graphs(self, on):
        """CUDA-graph replay of whole steps: single GPU, or the peer-memory
        exchange (the NCCL exchange path has a host sync per iteration)."""
        if on and self.world > 1 and getattr(self.engine, "exchange", "p2p") != "p2p":
            raise ValueError("CUDA graphs need the peer-memory exchange (DICM_EXCHANGE=p2p)")
        self.engine.use_graphs = bool(on)

    # -- checkpoint restore into this rank's state (checkpoint.load_warmup)

    def set_adam_state(self, name, m=None, v=None, t=None):
        """Adam state of one parameter; tables take this rank's rows."""
        from .training import set_adam_state
        set_adam_state(self.engine, self.model, name, m, v, t)

    def reset_adam_state(self, name):
        from .training import reset_adam_state
        reset_adam_state(self.engine, self.model, name)

    # -- state assembled from the owning shards (reference runtime.py:474-516)

    def _assemble(self, local, vocab):
        """Full [vocab, ...] host array from every rank's shard (row r lives
        on rank r % G at local row r // G); collective: every rank calls it."""
        if self.world == 1:
            return local.cpu().numpy()[:vocab]
        local = local.contiguous()
        parts = [torch.empty_like(local) for _ in range(self.world)]
        dist.all_gather(parts, local, group=self.group)
        out = np.zeros((vocab,) + tuple(local.shape[1:]), dtype=local.cpu().numpy().dtype)
        for r in range(self.world):
            n = len(range(r, vocab, self.world))
            out[r::self.world] = parts[r][:n].cpu().numpy()
        return out

    def snapshot(self):
        """Every parameter with the ID tables assembled from their shards
        (reference Cluster.snapshot, runtime.py:474-488); f64 host arrays.
        Collective when G > 1."""
        out = {n: p.data for n, p in self.model.params.items() if not n.startswith("id_emb/")}
        for f in self.model.layout.schema.fields:
            out[f"id_emb/{f.name}"] = self._assemble(self.model.real_table(self.model.tables[f.name]),
                                                     f.vocab).astype(np.float64)
        return out

    def collect_into_model(self):
        """Write the trained parameters back into the source model
        (runtime.py:490-495).  A sharded source model already holds its
        trained shard and is returned as is."""
        src = self.source_model
        if src is self.model:
            return src
        for n, v in self.snapshot().items():
            src.params[n].copy_(v)
        return src

    def optimizer_tensors(self):
        """Checkpoint-ready Adam state (runtime.py:497-516): ``<name>#m``,
        ``#v``, ``#t`` for every dense parameter (one replica: they are
        identical on every rank) and the row-Adam state of every table
        assembled from the shards.  Collective when G > 1."""
        e, m = self.engine, self.model
        t = e.t.cpu().numpy()
        out = {}
        for n in m.dense_names:
            out[f"{n}#m"] = m.real_view(e.m, n).double().cpu().numpy()
            out[f"{n}#v"] = m.real_view(e.v, n).double().cpu().numpy()
            out[f"{n}#t"] = np.array(int(t[e.span_index[n]]), dtype=np.int64)
        for f in m.layout.schema.fields:
            base = f"id_emb/{f.name}"
            out[f"{base}#m"] = self._assemble(m.real_table(e.tm[f.name]), f.vocab).astype(np.float64)
            out[f"{base}#v"] = self._assemble(m.real_table(e.tv[f.name]), f.vocab).astype(np.float64)
            out[f"{base}#t"] = self._assemble(e.tt[f.name], f.vocab).astype(np.int64)
        return out


def run_training(cluster_cfg, model, store, train_samples, train_cfg, log=None, precision="fp32"):
    """Synchronous distributed training (reference runtime.py:519-554)."""
    from .training import minibatches
    cluster = Cluster(cluster_cfg, model, store, train_cfg.lr0, train_cfg.lr_decay, train_cfg.lr_interval,
                      precision)
    log = log or RunLog()
    union_size = cluster_cfg.workers * cluster_cfg.batch_per_worker
    stop = train_cfg.max_iterations or None
    for epoch in range(train_cfg.epochs):
        for union in minibatches(train_samples, union_size, train_cfg.seed, epoch):
            log.lrs.append(lr_schedule(cluster.iteration, train_cfg.lr0, train_cfg.lr_decay, train_cfg.lr_interval))
            loss, unique, forwards, digests = cluster.run_iteration(union, digests=True)
            if not np.isfinite(loss):
                raise FloatingPointError(f"non-finite loss at iteration {cluster.iteration}")
            log.losses.append(loss)
            log.unique_images.append(unique)
            log.embed_forwards.append(forwards)
            log.replica_digests.append(digests)
            if stop and cluster.iteration >= stop:
                cluster.collect_into_model()
                return cluster, log
    cluster.collect_into_model()
    return cluster, log
