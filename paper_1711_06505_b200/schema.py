"""Feature schema, aggregator spec and reference-compatible parameter init.

Host-side mirror of the reference's model description so that a user of
``dicm.model`` finds the same names, defaults, validation errors and -- bit
for bit -- the same initial parameter values:

* ``FieldSpec`` / ``FeatureSchema``      -- reference ``model.py:38-67``
* ``AggregatorSpec``                     -- reference ``model.py:70-85``
* ``image_net_widths``                   -- reference ``model.py:88-91``
* ``param_specs`` / ``init_params``      -- reference ``model.py:94-105`` and
  ``DicmModel._build_params`` ``model.py:314-335``
* ``default_schema``                     -- reference ``experiments.py:17-32``

Nothing here touches the GPU; the device model lives in ``model.py``.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass

import numpy as np

AGGREGATOR_KINDS = ("concat", "max", "sum", "attn", "multiquery-attn")
# aggregators built on the B200 hot path
HOT_PATH_AGGREGATORS = ("sum", "attn", "multiquery-attn", "max", "concat")

GROUP_ID = "id-embeddings"
GROUP_IMAGE = "image-embedding-model"
GROUP_MLP = "mlp"
GROUP_ATTN = "aggregator-attention"


def group_of(name):
    """Checkpoint group / owner side of a parameter (reference model.py:28-35)."""
    if name.startswith("id_emb/"):
        return GROUP_ID
    if name.startswith("img/"):
        return GROUP_IMAGE
    if name.startswith("attn/"):
        return GROUP_ATTN
    return GROUP_MLP


@dataclass(frozen=True)
class FieldSpec:
    name: str
    vocab: int
    multi: bool = False


@dataclass
class FeatureSchema:
    """ID fields plus dimension settings (reference model.py:45-67)."""

    fields: list
    d_id: int = 12
    d_raw: int = 64
    d_img: int = 12
    b_max: int = 32
    query_fields: tuple = ("ad", "ad_category")

    def __post_init__(self):
        if min(self.d_id, self.d_raw, self.d_img, self.b_max) < 1:
            raise ValueError("schema dimensions must be >= 1")
        for f in self.fields:
            if f.vocab < 1:
                raise ValueError(f"field {f.name}: vocabulary must be >= 1")

    def field(self, name):
        for f in self.fields:
            if f.name == name:
                return f
        raise KeyError(f"schema has no field {name!r}")


@dataclass
class AggregatorSpec:
    kind: str = "sum"
    attention_hidden: int = 32
    normalize: bool = True

    def __post_init__(self):
        if self.kind not in AGGREGATOR_KINDS:
            raise ValueError(f"unknown aggregator {self.kind!r}; use one of {AGGREGATOR_KINDS}")

    def output_width(self, d_img, b_max):
        if self.kind == "concat":
            return d_img * b_max
        if self.kind == "multiquery-attn":
            return 2 * d_img
        return d_img


def image_net_widths(d_raw, d_img):
    """Hidden widths of the image net (reference model.py:88-91)."""
    return max(d_raw // 16, d_img), max(d_raw // 64, d_img)


def default_schema(users, scenarios, ad_vocab, categories, image_count, d_id=12,
                   d_raw=4096, d_img=12, b_max=32, image_id_fields=True):
    """The benchmark field layout of reference experiments.py:17-32, with the
    vocabularies given directly instead of through a SyntheticConfig."""
    fields = [
        FieldSpec("user", users),
        FieldSpec("scenario", scenarios),
        FieldSpec("ad", ad_vocab),
        FieldSpec("ad_category", categories),
        FieldSpec("behavior_items", ad_vocab, multi=True),
    ]
    if image_id_fields:
        fields.append(FieldSpec("ad_image", image_count))
        fields.append(FieldSpec("behavior_images", image_count, multi=True))
    return FeatureSchema(fields=fields, d_id=d_id, d_raw=d_raw, d_img=d_img, b_max=b_max)


def rng_for(seed, name):
    """Per-parameter generator (reference model.py:94-95)."""
    return np.random.default_rng([int(seed) & 0xFFFFFFFF, zlib.crc32(name.encode())])


@dataclass(frozen=True)
class TowerSpec:
    """The two towers of the pre-rank model (reference PrerankModel,
    model.py:420-531): field lists in hstack order, hidden and output width."""

    user_fields: tuple
    ad_fields: tuple
    hidden: int = 64
    rep: int = 16


@dataclass(frozen=True)
class ModelLayout:
    """Everything the kernels need to know about one DICM configuration.

    ``towers`` set: the two-tower pre-rank model -- ``schema`` then holds the
    tower fields only (the reference builds tables for those alone,
    model.py:470-475), pooling is "sum", and the head input feeds the towers
    instead of the MLP head."""

    schema: FeatureSchema
    aggregator: AggregatorSpec
    mlp_widths: tuple
    use_ad_image: bool
    use_behavior_images: bool
    towers: TowerSpec = None

    def tower_parts(self, tower):
        """(head-input column, width) blocks of one tower's input in the
        reference's hstack order (model.py:510-520): the tower's fields, then
        the pooled behavior images (user) or the ad image (ad)."""
        s, off = self.schema, self.head_offsets()
        tw = self.towers
        out = [(off["field/" + f], s.d_id) for f in (tw.user_fields if tower == "user" else tw.ad_fields)]
        if tower == "user" and self.use_behavior_images:
            out.append((off["pool"], s.d_img))
        if tower == "ad" and self.use_ad_image:
            out.append((off["ad_image_emb"], s.d_img))
        return out

    def tower_input_width(self, tower):
        return sum(w for _, w in self.tower_parts(tower))

    @property
    def h1(self):
        return image_net_widths(self.schema.d_raw, self.schema.d_img)[0]

    @property
    def h2(self):
        return image_net_widths(self.schema.d_raw, self.schema.d_img)[1]

    @property
    def attentive(self):
        return self.use_behavior_images and self.aggregator.kind in ("attn", "multiquery-attn")

    @property
    def multiquery(self):
        return self.use_behavior_images and self.aggregator.kind == "multiquery-attn"

    def query_fields_present(self):
        names = [f.name for f in self.schema.fields]
        return [q for q in self.schema.query_fields if q in names]

    def id_query_width(self):
        return self.schema.d_id * len(self.query_fields_present())

    def mlp_input_width(self):
        s = self.schema
        w = len(s.fields) * s.d_id
        if self.use_ad_image:
            w += s.d_img
        if self.use_behavior_images:
            w += self.aggregator.output_width(s.d_img, s.b_max)
        return w

    def head_offsets(self):
        """Column offsets of every part of the head input (the hstack order of
        reference model.py:364-397): fields in schema order, then the ad-image
        embedding, then the aggregator output."""
        s = self.schema
        off, out = 0, {}
        for f in s.fields:
            out["field/" + f.name] = off
            off += s.d_id
        if self.use_ad_image:
            out["ad_image_emb"] = off
            off += s.d_img
        if self.use_behavior_images:
            out["pool"] = off
            off += self.aggregator.output_width(s.d_img, s.b_max)
        out["width"] = off
        return out


def prerank_layout(schema, user_fields=("user", "behavior_items"), ad_fields=("ad", "ad_category"),
                   tower_hidden=64, rep_dim=16, use_images=True, extractor_out_dim=None):
    """Layout of the reference ``PrerankModel`` (model.py:427-458), with its
    constructor checks: the extractor width and every tower field present."""
    if extractor_out_dim is not None and extractor_out_dim != schema.d_raw:
        raise ValueError(f"extractor emits {extractor_out_dim}-D features, schema expects {schema.d_raw}")
    names = [f.name for f in schema.fields]
    for fn in (*user_fields, *ad_fields):
        if fn not in names:
            raise ValueError(f"tower field {fn!r} missing from schema")
    keep = set(user_fields) | set(ad_fields)
    sub = FeatureSchema(fields=[f for f in schema.fields if f.name in keep], d_id=schema.d_id,
                        d_raw=schema.d_raw, d_img=schema.d_img, b_max=schema.b_max,
                        query_fields=tuple(schema.query_fields))
    return ModelLayout(sub, AggregatorSpec("sum"), (), bool(use_images), bool(use_images),
                       TowerSpec(tuple(user_fields), tuple(ad_fields), int(tower_hidden), int(rep_dim)))


def validate_layout(layout, extractor_out_dim=None):
    """The constructor checks of reference model.py:279-288."""
    agg = layout.aggregator
    if layout.use_behavior_images and agg.kind in ("attn", "multiquery-attn") and not layout.use_ad_image:
        raise ValueError(f"aggregator {agg.kind!r} needs the ad image as query")
    if agg.kind == "multiquery-attn" and not layout.query_fields_present():
        raise ValueError("multiquery-attn needs at least one ad-side query field")
    if extractor_out_dim is not None and extractor_out_dim != layout.schema.d_raw:
        raise ValueError(
            f"extractor emits {extractor_out_dim}-D features, schema expects {layout.schema.d_raw}"
        )


def param_specs(layout):
    """Ordered (name, shape, kind) of every parameter, in the reference's
    construction order (model.py:314-335). kind: table|w|b|a."""
    s = layout.schema
    out = []

    def lin(prefix, n_in, n_out, alpha=True):
        out.append((prefix + "w", (n_out, n_in), "w"))
        out.append((prefix + "b", (n_out,), "b"))
        if alpha:
            out.append((prefix + "a", (n_out,), "a"))

    for f in s.fields:
        out.append((f"id_emb/{f.name}", (f.vocab, s.d_id), "table"))
    h1, h2 = layout.h1, layout.h2
    lin("img/0/", s.d_raw, h1)
    lin("img/1/", h1, h2)
    lin("img/2/", h2, s.d_img, alpha=False)
    if layout.towers is not None:  # reference model.py:477-481
        tw = layout.towers
        for t in ("user", "ad"):
            lin(f"{t}_tower/0/", layout.tower_input_width(t), tw.hidden)
            lin(f"{t}_tower/1/", tw.hidden, tw.rep, alpha=False)
        return out
    if layout.attentive:
        hidden = layout.aggregator.attention_hidden
        lin("attn/img/0/", 2 * s.d_img, hidden)
        lin("attn/img/1/", hidden, 1, alpha=False)
        if layout.multiquery:
            lin("attn/id/0/", layout.id_query_width() + s.d_img, hidden)
            lin("attn/id/1/", hidden, 1, alpha=False)
    widths = [layout.mlp_input_width(), *layout.mlp_widths]
    for i in range(len(widths) - 1):
        lin(f"mlp/{i}/", widths[i], widths[i + 1])
    lin(f"mlp/{len(widths) - 1}/", widths[-1], 1, alpha=False)
    return out


def init_param(seed, name, shape, kind):
    """Initial value of one parameter, float64, identical to the reference
    (model.py:98-105 for linear layers, model.py:316-319 for tables)."""
    if kind == "table":
        return 0.05 * rng_for(seed, name).standard_normal(shape)
    if kind == "w":
        n_out, n_in = shape
        return rng_for(seed, name).normal(0.0, np.sqrt(2.0 / n_in), (n_out, n_in))
    if kind == "b":
        return np.zeros(shape)
    if kind == "a":
        return np.full(shape, 0.25)
    raise ValueError(kind)


def init_params(layout, seed, include_tables=True):
    return {
        name: init_param(seed, name, shape, kind)
        for name, shape, kind in param_specs(layout)
        if include_tables or kind != "table"
    }


def worker_param_names(layout):
    """Dense replicated parameters (reference model.py:339-341)."""
    return sorted(n for n, _, _ in param_specs(layout) if group_of(n) in (GROUP_MLP, GROUP_ATTN))


def image_param_names(layout):
    return sorted(n for n, _, _ in param_specs(layout) if group_of(n) == GROUP_IMAGE)


def dense_param_names(layout):
    """Dense parameters in the order LocalTrainer steps them (training.py:53)."""
    return worker_param_names(layout) + image_param_names(layout)


# ---------------------------------------------------------------------------
# kernel geometry: the reference's widths embedded into the compiled ones
# ---------------------------------------------------------------------------

KD = 12                 # embedding block width of the kernels (d_id and d_img)
KH1, KH2 = 256, 64      # image-net hidden widths
KATT = 32               # attention hidden width
KHEAD = (128, 64)       # head hidden widths
KRAW = 256              # the pool row width is a multiple of this
KMAX_WIDE = 16384       # widest head input (the GEMM head path)


class KernelGeometry:
    """How a layout's parameters embed into the kernels' compiled widths.

    The kernels are compiled for the paper's widths (12-d embeddings, a
    256/64 image net, 32 attention units, a 128/64 head).  A narrower model
    (e.g. the reference's own test fixtures: d_id 3, d_img 4, d_raw 8,
    attention 5, head (6, 4)) is trained by zero-padding every parameter into
    those widths: padded weights, biases and PReLU slopes are 0, so padded
    units output exactly 0 (PReLU(0) = 0), padded input columns meet zero
    weights, every padded gradient is exactly 0 and Adam leaves padded entries
    at 0 -- the real entries follow the reference bit for bit in f64 and to
    fp32 rounding on the device.  The pool is padded with zero columns to a
    multiple of 256.  ``specs`` maps every parameter name to (kernel shape,
    row index, column index): the real tensor is
    kernel[rows][:, cols]; None means the whole axis.
    Wider models than the compiled widths raise NotImplementedError."""

    def __init__(self, layout):
        s = layout.schema
        agg = layout.aggregator
        self.layout = layout
        problems = []
        if s.d_id > KD or s.d_img > KD:
            problems.append(f"d_id / d_img <= {KD} (got {s.d_id}, {s.d_img})")
        if layout.h1 > KH1 or layout.h2 > KH2:
            problems.append(f"image-net widths <= ({KH1}, {KH2}) (got {layout.h1}, {layout.h2})")
        if layout.attentive and agg.attention_hidden > KATT:
            problems.append(f"attention_hidden <= {KATT} (got {agg.attention_hidden})")
        if layout.towers is None:
            mw = tuple(layout.mlp_widths)
            if len(mw) != 2 or mw[0] > KHEAD[0] or mw[1] > KHEAD[1]:
                problems.append(f"two head layers of at most {KHEAD} units (got {mw})")
        if problems:
            raise NotImplementedError("kernels are compiled for " + "; ".join(problems))
        self.d_raw = -(-s.d_raw // KRAW) * KRAW
        self.identity = (s.d_id == KD and s.d_img == KD and s.d_raw == self.d_raw and layout.h1 == KH1
                         and layout.h2 == KH2 and (not layout.attentive or agg.attention_hidden == KATT)
                         and (layout.towers is not None or tuple(layout.mlp_widths) == KHEAD))
        # head input: every block 12 wide
        real, off, cols = layout.head_offsets(), 0, []
        kern = {}
        for f in s.fields:
            kern["field/" + f.name] = off
            cols += range(off, off + s.d_id)
            off += KD
        if layout.use_ad_image:
            kern["ad_image_emb"] = off
            cols += range(off, off + s.d_img)
            off += KD
        if layout.use_behavior_images:
            kern["pool"] = off
            nblk = {"multiquery-attn": 2, "concat": s.b_max}.get(agg.kind, 1)
            for j in range(nblk):
                cols += range(off + KD * j, off + KD * j + s.d_img)
            off += KD * nblk
        kern["width"] = off
        assert len(cols) == real["width"]
        self.head_offsets, self.width = kern, off
        self.head_cols = np.asarray(cols, dtype=np.int64)
        if self.width > KMAX_WIDE:
            raise NotImplementedError(f"head input width {self.width} > {KMAX_WIDE}")
        self.specs = self._specs()

    def tower_parts(self, tower):
        """(kernel head-input column, 12) blocks of one tower's input, in the
        reference's hstack order (model.py:510-520)."""
        kern, real = self.head_offsets, self.layout.head_offsets()
        inv = {v: k for k, v in real.items() if k != "width"}
        return [(kern[inv[col]], KD) for col, _w in self.layout.tower_parts(tower)]

    def _specs(self):
        lay, s, agg = self.layout, self.layout.schema, self.layout.aggregator
        ar = lambda n: np.arange(n, dtype=np.int64)  # noqa: E731
        out = {}

        def lin(prefix, n_in, n_out, k_in, k_out, cols=None, alpha=True):
            out[prefix + "w"] = ((k_out, k_in), ar(n_out) if n_out != k_out else None,
                                 cols if cols is not None else (ar(n_in) if n_in != k_in else None))
            out[prefix + "b"] = ((k_out,), ar(n_out) if n_out != k_out else None, None)
            if alpha:
                out[prefix + "a"] = ((k_out,), ar(n_out) if n_out != k_out else None, None)

        for f in s.fields:
            out[f"id_emb/{f.name}"] = ((f.vocab, KD), None, ar(s.d_id) if s.d_id != KD else None)
        lin("img/0/", s.d_raw, lay.h1, self.d_raw, KH1)
        lin("img/1/", lay.h1, lay.h2, KH1, KH2)
        lin("img/2/", lay.h2, s.d_img, KH2, KD, alpha=False)
        if lay.towers is not None:
            tw = lay.towers
            for t in ("user", "ad"):
                parts = lay.tower_parts(t)
                cols = np.concatenate([ar(w) + KD * j for j, (_c, w) in enumerate(parts)])
                k_in = KD * len(parts)
                lin(f"{t}_tower/0/", len(cols), tw.hidden, k_in, tw.hidden,
                    cols=cols if len(cols) != k_in else None)
                lin(f"{t}_tower/1/", tw.hidden, tw.rep, tw.hidden, tw.rep, alpha=False)
            return out
        if lay.attentive:
            h = agg.attention_hidden
            cols = np.concatenate([ar(s.d_img), KD + ar(s.d_img)])
            lin("attn/img/0/", 2 * s.d_img, h, 2 * KD, KATT, cols=cols if len(cols) != 2 * KD else None)
            lin("attn/img/1/", h, 1, KATT, 1, alpha=False)
            if lay.multiquery:
                nq = len(lay.query_fields_present())
                cols = np.concatenate([KD * q + ar(s.d_id) for q in range(nq)] + [KD * nq + ar(s.d_img)])
                lin("attn/id/0/", nq * s.d_id + s.d_img, h, KD * nq + KD, KATT,
                    cols=cols if len(cols) != KD * (nq + 1) else None)
                lin("attn/id/1/", h, 1, KATT, 1, alpha=False)
        m0, m1 = lay.mlp_widths
        lin("mlp/0/", lay.mlp_input_width(), m0, self.width, KHEAD[0],
            cols=self.head_cols if len(self.head_cols) != self.width else None)
        lin("mlp/1/", m0, m1, KHEAD[0], KHEAD[1])
        lin("mlp/2/", m1, 1, KHEAD[1], 1, alpha=False)
        return out
