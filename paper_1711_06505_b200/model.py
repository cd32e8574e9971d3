"""The DICM model with its parameters resident on the GPU.

API mirror of the reference ``DicmModel`` (model.py:266-408): same
constructor arguments and validation errors, same parameter names and --
through ``schema.init_params`` -- bit-identical initial values (cast to fp32
on the device).  Storage is laid out for the kernels:

* every dense parameter (attn/*, mlp/*, img/*) lives in ONE fused fp32 buffer
  in ``dense_param_names`` order (sorted worker names, then sorted image
  names, reference training.py:53), with matching gradient / Adam-moment
  buffers -- one Adam launch and one NCCL all-reduce cover all of them;
* each ID table ``id_emb/<field>`` is a [V, 12] fp32 tensor with per-row Adam
  moments and step counts (reference optim.py:66-80).
"""

from __future__ import annotations

import zlib

import numpy as np
import torch

from . import schema as S
from .schema import AggregatorSpec, FeatureSchema, FieldSpec, ModelLayout  # noqa: F401

KIND_CODE = {"sum": 0, "attn": 1, "multiquery-attn": 2, "max": 3, "concat": 4}
HEAD_SMEM_WIDTH = 128   # widest head input whose W0 stays in shared memory (csrc/head.cu)
HEAD_MAX_WIDE = 16384   # DICM_HEAD_MAX_WIDE


class Parameter:
    """A named device tensor; ``.data`` returns a float64 host copy like the
    reference's ``Parameter.data`` (autograd.py:49-53).

    ``tensor`` is the kernel-shaped storage; a model narrower than the
    compiled widths (schema.KernelGeometry) holds its real entries at
    ``tensor[rows][:, cols]`` and zeros elsewhere -- ``shape``, ``data``,
    ``real()`` and ``copy_`` see the real tensor only."""

    __slots__ = ("name", "tensor", "rows", "cols")

    def __init__(self, name, tensor, rows=None, cols=None):
        self.name = name
        self.tensor = tensor
        self.rows = None if rows is None else torch.as_tensor(rows, device=tensor.device)
        self.cols = None if cols is None else torch.as_tensor(cols, device=tensor.device)

    @property
    def shape(self):
        shp = list(self.tensor.shape)
        if self.rows is not None:
            shp[0] = len(self.rows)
        if self.cols is not None:
            shp[-1] = len(self.cols)
        return tuple(shp)

    def real(self):
        """The real entries as a device tensor (a copy when padded)."""
        return real_of(self.tensor, self.rows, self.cols)

    @property
    def data(self):
        return self.real().detach().double().cpu().numpy()

    def copy_(self, value):
        write_real(self.tensor, self.rows, self.cols, value)

    def __repr__(self):
        return f"Parameter({self.name!r}, shape={self.shape})"


def real_of(t, rows, cols):
    """kernel-shaped t -> its real entries t[rows][:, cols]."""
    if rows is not None:
        t = t.index_select(0, rows)
    if cols is not None:
        t = t.index_select(t.dim() - 1, cols)
    return t


def write_real(t, rows, cols, value):
    """t[rows][:, cols] = value (the padded entries are left as they are)."""
    v = torch.as_tensor(np.asarray(value), dtype=t.dtype if t.dtype == torch.bool else torch.float32).to(t.device)
    if rows is None and cols is None:
        t.copy_(v)
    elif t.dim() == 1:
        t[rows] = v
    elif cols is None:
        t[rows] = v
    elif rows is None:
        t[:, cols] = v
    else:
        t[rows[:, None], cols[None, :]] = v


def check_hot_path(layout):
    """The kernels are compiled for the paper's configuration; narrower
    widths embed into it (schema.KernelGeometry), wider ones raise."""
    s = layout.schema
    if layout.towers is not None:
        return _check_towers(layout)
    if layout.aggregator.kind not in S.HOT_PATH_AGGREGATORS:
        raise NotImplementedError(
            f"aggregator {layout.aggregator.kind!r} is outside this build's hot path "
            f"(supported: {S.HOT_PATH_AGGREGATORS})")
    geom = S.KernelGeometry(layout)
    if len(s.fields) > 8:
        raise NotImplementedError("at most 8 ID fields")
    if layout.multiquery:
        for q in layout.query_fields_present():
            if s.field(q).multi:
                raise NotImplementedError("multiquery-attn query fields must be one-hot")
        if len(layout.query_fields_present()) > 2:
            raise NotImplementedError("multiquery-attn takes at most 2 ID query fields")
    return geom


def _check_image_net(layout):
    s = layout.schema
    if len(s.fields) > 8:
        raise NotImplementedError("at most 8 ID fields")
    return S.KernelGeometry(layout)


def _check_towers(layout):
    from . import _lib as L
    geom = _check_image_net(layout)
    tw = layout.towers
    if not 1 <= tw.hidden <= 128 or not 1 <= tw.rep <= 64:
        raise NotImplementedError("tower kernels take hidden <= 128 and rep_dim <= 64")
    for t in ("user", "ad"):
        if not 1 <= len(layout.tower_parts(t)) <= L.TOWER_MAX_PARTS:
            raise NotImplementedError(f"{t} tower needs 1..{L.TOWER_MAX_PARTS} input blocks")
    if geom.width > 128:
        raise NotImplementedError(f"tower input layout width {geom.width} > 128")
    return geom


class DicmModel:
    """Embedding&MLP CTR net with ad-image and behavior-image paths."""

    def __init__(self, schema, aggregator, extractor=None, seed=0, mlp_widths=(128, 64),
                 use_ad_image=True, use_behavior_images=True, device="cuda", params=None,
                 table_rows=None, shard=None, table_init="reference"):
        """``shard=(world, rank)``: hold only the ID-table rows this rank owns
        (row % world == rank, at local row row // world), with exactly the
        values the full reference init gives them.  ``table_init="device"``
        draws 0.05 N(0,1) rows on the device instead (same distribution as
        model.py:316-319, not the same values; counter-based, so identical at
        every world size) -- for 100M-row tables whose reference init would
        not fit host memory."""
        layout = ModelLayout(schema, aggregator, tuple(mlp_widths), use_ad_image, use_behavior_images)
        S.validate_layout(layout, None if extractor is None else extractor.out_dim)
        self.geometry = check_hot_path(layout)
        self.schema = schema
        self.aggregator = aggregator
        self.extractor = extractor
        self.seed = seed
        self.mlp_widths = tuple(mlp_widths)
        self.use_ad_image = use_ad_image
        self.use_behavior_images = use_behavior_images
        self._build(layout, seed, device, params, table_rows, shard, table_init)

    def _build(self, layout, seed, device, params, table_rows, shard, table_init):
        """Device storage of every parameter of ``layout`` (tables of
        ``layout.schema``'s fields)."""
        schema = layout.schema
        host = params if params is not None else {}
        if table_init == "device" and table_rows is None:
            world, rank = shard if shard is not None else (1, 0)

            def table_rows(f, name):
                # counter-based: a row's values depend on (seed, name, row) only,
                # so the model is the same at every world size (dicm_table_init)
                from . import _lib as L
                n_local = -(-f.vocab // world)
                out = torch.empty((n_local, schema.d_id), dtype=torch.float32, device=device)
                key = ((int(seed) & 0xFFFFFFFF) << 32) | zlib.crc32(name.encode())
                L.check(L.lib.dicm_table_init(out.data_ptr(), n_local, schema.d_id, world, rank, f.vocab, key, 0.05,
                                              L.stream_handle()))
                return out
        elif shard is not None and table_rows is None:
            world, rank = shard

            def table_rows(f, name):
                full = host[name] if name in host else S.init_param(seed, name, (f.vocab, schema.d_id), "table")
                local = np.asarray(full)[rank::world]
                n_local = -(-f.vocab // world)
                out = np.zeros((n_local, schema.d_id))
                out[:len(local)] = local
                return torch.as_tensor(out, dtype=torch.float32).to(device)
        self.shard = shard
        self.layout = layout
        self.device = torch.device(device)
        self.specs = S.param_specs(layout)
        self.dense_names = S.dense_param_names(layout)
        geom = self.geometry
        # kernel shapes; the real tensor of each is kernel[rows][:, cols] (KernelGeometry)
        shapes = {n: geom.specs[n][0] for n, _, _ in self.specs}
        self.index_maps = {n: (None if geom.specs[n][1] is None else torch.as_tensor(geom.specs[n][1],
                                                                                      device=self.device),
                               None if geom.specs[n][2] is None else torch.as_tensor(geom.specs[n][2],
                                                                                      device=self.device))
                           for n, _, _ in self.specs}
        real_shapes = {n: shp for n, shp, _ in self.specs}
        # fused dense buffer
        # the image and head groups start on 256-B boundaries so the kernels
        # can use 16-B vector loads on their weights (mlp/0/w, mlp/1/w sit a
        # multiple of 4 floats into the group); a gap is its own (always-zero) span
        self.dense_offsets, off = {}, 0
        self.dense_spans = []  # (offset, size, name or None) tiling the buffer
        first_mlp = next((n for n in self.dense_names if n.startswith("mlp/")), None)
        for n in self.dense_names:
            if (n.startswith("img/") or n == first_mlp) and off % 64:
                pad = 64 - off % 64
                self.dense_spans.append((off, pad, None))
                off += pad
            size = int(np.prod(shapes[n]))
            self.dense_offsets[n] = (off, size, shapes[n])
            self.dense_spans.append((off, size, n))
            off += size
        self.dense_size = off
        self.dense = torch.zeros(off, dtype=torch.float32, device=self.device)
        self.params = {}
        kinds = {nm: k for nm, _, k in self.specs}
        for n in self.dense_names:
            o, size, shp = self.dense_offsets[n]
            view = self.dense[o:o + size].view(shp)
            val = host[n] if n in host else S.init_param(seed, n, real_shapes[n], kinds[n])
            rows, cols = self.index_maps[n]
            write_real(view, rows, cols, np.asarray(val, dtype=np.float64))
            self.params[n] = Parameter(n, view, rows, cols)
        # ID tables (``table_rows`` lets a sharded model hold only its rows),
        # kernel width 12 (a narrower d_id is zero-padded)
        self.tables = {}
        for f in schema.fields:
            n = f"id_emb/{f.name}"
            if table_rows is not None:
                t = table_rows(f, n)
            elif n in host:
                t = torch.as_tensor(np.asarray(host[n], dtype=np.float64), dtype=torch.float32).to(self.device)
            else:
                t = torch.as_tensor(S.init_param(seed, n, (f.vocab, schema.d_id), "table"),
                                    dtype=torch.float32).to(self.device)
            if t.shape[1] != S.KD:
                padded = torch.zeros((t.shape[0], S.KD), dtype=torch.float32, device=self.device)
                padded[:, :t.shape[1]] = t
                t = padded
            self.tables[f.name] = t.contiguous()
            self.params[n] = Parameter(n, self.tables[f.name], None, self.index_maps[n][1])
        self.head_offsets = geom.head_offsets

    # -- reference bookkeeping (model.py:339-347)
    def worker_param_names(self):
        return S.worker_param_names(self.layout)

    def image_param_names(self):
        return S.image_param_names(self.layout)

    def table_fields(self):
        return [f.name for f in self.layout.schema.fields]

    def mlp_input_width(self):
        return self.layout.mlp_input_width()

    def dense_view(self, buf, name):
        """The kernel-shaped view of one parameter's span of a fused buffer."""
        o, size, shp = self.dense_offsets[name]
        return buf[o:o + size].view(shp)

    def real_view(self, buf, name):
        """The real entries of one parameter's span (a copy when padded)."""
        rows, cols = self.index_maps[name]
        return real_of(self.dense_view(buf, name), rows, cols)

    def write_real_view(self, buf, name, value):
        rows, cols = self.index_maps[name]
        write_real(self.dense_view(buf, name), rows, cols, value)

    def real_mask(self):
        """bool mask over the fused dense buffer: True on real entries (the
        padded ones of a narrow model -- and the alignment gaps -- are False)."""
        mask = torch.zeros(self.dense.shape, dtype=torch.bool, device=self.dense.device)
        for n in self.dense_names:
            write_real(self.dense_view(mask, n), *self.index_maps[n],
                       np.ones(self.params[n].shape, dtype=bool))
        return mask

    def real_table(self, t):
        """A kernel-width [V, 12] table (or table-shaped state) -> [V, d_id]."""
        return t[:, :self.schema.d_id] if t.dim() == 2 and self.schema.d_id != t.shape[1] else t

    def group_range(self, prefix):
        """[start, end) of the contiguous fused-buffer range of a name group."""
        names = [n for n in self.dense_names if n.startswith(prefix)]
        if not names:
            return None
        start = self.dense_offsets[names[0]][0]
        o, size, _ = self.dense_offsets[names[-1]]
        return start, o + size

    def snapshot(self):
        return {n: p.data for n, p in self.params.items()}

    def sharded(self, world, rank):
        """A copy that holds only the ID-table rows rank ``rank`` of ``world``
        owns, with this model's current values (a Cluster rank's working copy
        of a full model)."""
        return DicmModel(self.schema, self.aggregator, self.extractor, self.seed, self.mlp_widths,
                         self.use_ad_image, self.use_behavior_images, device=self.device,
                         params=self.snapshot(), shard=(world, rank))


class PrerankModel(DicmModel):
    """Two-tower pre-rank variant (reference PrerankModel, model.py:420-531):
    user and ad representations scored by their inner product.  Behavior
    images enter the user tower through sum pooling, the ad image enters the
    ad tower; only the tower fields get tables.  Same constructor arguments
    and validation errors as the reference; the image net, the ID tables and
    the per-sample kernels are the DICM ones, the head is the tower kernel
    (csrc/towers.cu)."""

    def __init__(self, schema, extractor=None, seed=0, user_fields=("user", "behavior_items"),
                 ad_fields=("ad", "ad_category"), tower_hidden=64, rep_dim=16, use_images=True, device="cuda",
                 params=None, table_rows=None, shard=None, table_init="reference"):
        layout = S.prerank_layout(schema, tuple(user_fields), tuple(ad_fields), tower_hidden, rep_dim, use_images,
                                  None if extractor is None else extractor.out_dim)
        self.geometry = check_hot_path(layout)
        self.schema = schema
        self.extractor = extractor
        self.seed = seed
        self.user_fields = tuple(user_fields)
        self.ad_fields = tuple(ad_fields)
        self.tower_hidden = tower_hidden
        self.rep_dim = rep_dim
        self.use_images = use_images
        self.use_ad_image = use_images
        self.use_behavior_images = use_images
        self.aggregator = layout.aggregator
        self.mlp_widths = ()
        self._build(layout, seed, device, params, table_rows, shard, table_init)

    def sharded(self, world, rank):
        return PrerankModel(self.schema, self.extractor, self.seed, self.user_fields, self.ad_fields,
                            self.tower_hidden, self.rep_dim, self.use_images, device=self.device,
                            params=self.snapshot(), shard=(world, rank))
