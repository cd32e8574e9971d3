"""ctypes binding of the sm_100a kernel library (include/dicm_b200.h).

The library is required: there is no CPU fallback.  Importing this module
without ``libdicm_b200.so`` next to it raises ImportError; calling a kernel
without a CUDA device raises RuntimeError from the library.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DICM_LIB_PATH: an alternate build of the same library (scripts/ab_lib.sh A/B runs)
LIB_PATH = os.environ.get("DICM_LIB_PATH") or os.path.join(_HERE, "libdicm_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a kernels first "
        "(`make` in the repo root or `python -c 'import __graft_entry__ as g; g.build()'`)"
    )
lib = C.CDLL(LIB_PATH)

DICM_OK, DICM_ERR_CUDA, DICM_ERR_SHAPE, DICM_ERR_KEY, DICM_ERR_VALUE, DICM_ERR_FLOAT, DICM_ERR_UNSUPPORTED = range(7)
STATUS_WORDS = 8
ST_KEY_FLAG, ST_KEY_VALUE, ST_KEY_SEG, ST_NONFINITE, ST_P2P_TIMEOUT = 0, 1, 2, 3, 4
MAX_PEERS = 8
POOL_F32, POOL_BF16 = 0, 1
PREC_FP32, PREC_TF32, PREC_BF16 = 0, 1, 2
PRECISIONS = {"fp32": PREC_FP32, "tf32": PREC_TF32, "bf16": PREC_BF16}


class ShapeError(ValueError):
    """Operand shapes do not conform (reference autograd.py:18-19)."""


class ProtocolError(RuntimeError):
    """Distributed-step protocol violation (reference protocol.py:41-42)."""


_EXC = {
    DICM_ERR_CUDA: RuntimeError,
    DICM_ERR_SHAPE: ShapeError,
    DICM_ERR_KEY: KeyError,
    DICM_ERR_VALUE: ValueError,
    DICM_ERR_FLOAT: FloatingPointError,
    DICM_ERR_UNSUPPORTED: NotImplementedError,
}


def check(rc):
    if rc != DICM_OK:
        msg = lib.dicm_last_error().decode()
        raise _EXC.get(rc, RuntimeError)(msg)


# ---------------------------------------------------------------------------
# structs (must match include/dicm_b200.h)
# ---------------------------------------------------------------------------

P = C.c_void_p
I32, I64 = C.c_int32, C.c_int64


class KeySeg(C.Structure):
    _fields_ = [("ids", P), ("n", I64), ("base", I64), ("vocab", I64), ("inv_off", I64)]


class ImgMlpParams(C.Structure):
    _fields_ = [(n, P) for n in ("w0", "b0", "a0", "w1", "b1", "a1", "w2", "b2")]


ImgMlpGrads = ImgMlpParams


class Layout(C.Structure):
    _fields_ = [("kind", I32), ("normalize", I32), ("use_ad_image", I32), ("use_behavior_images", I32),
                ("n_fields", I32), ("field_multi", I32 * 8), ("field_col", I32 * 8), ("ad_col", I32),
                ("pool_col", I32), ("width", I32), ("n_query", I32), ("query_col", I32 * 2),
                ("query_field", I32 * 2)]


class BatchView(C.Structure):
    _fields_ = [("batch", I32), ("refs", I64), ("field_ids", P * 8), ("field_off", P * 8), ("tables", P * 8),
                ("field_inv", P * 8), ("ad_local", P), ("beh_local", P), ("beh_off", P), ("emb", P),
                ("img_order", P), ("img_start", P), ("id_order", P), ("id_start", P), ("field_ref_begin", I64 * 8),
                ("beh_seg", P), ("field_seg", P * 8), ("n_img_keys", P), ("n_id_keys", P), ("img_cap", I64),
                ("id_cap", I64), ("ref_grad", P), ("q_grad", P), ("hot", P),
                ("hot_acc", P)]


class AttnParams(C.Structure):
    _fields_ = [(n, P) for n in ("w0", "b0", "a0", "w1", "b1")]


class HeadParams(C.Structure):
    _fields_ = [(n, P) for n in ("w0", "b0", "a0", "w1", "b1", "a1", "w2", "b2")]


TOWER_MAX_PARTS = 10


class Tower(C.Structure):
    _fields_ = ([(n, P) for n in ("w0", "b0", "a0", "w1", "b1")] + [("n_parts", I32),
                                                                    ("part_col", I32 * TOWER_MAX_PARTS)]
                + [(n, I64) for n in ("g_w0", "g_b0", "g_a0", "g_w1", "g_b1")])


class Span(C.Structure):
    _fields_ = [("offset", I64), ("size", I64)]


class TableState(C.Structure):
    _fields_ = [("table", P), ("m", P), ("v", P), ("t", P), ("base", I64), ("vocab", I64)]


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


S = C.c_size_t
F = C.c_float
ST = P  # stream


class JsonlSpec(C.Structure):
    _fields_ = [("n_keys", I32), ("keys", C.c_char_p * 16), ("key_is_list", I32 * 16), ("b_max", I32)]


class Peers(C.Structure):
    _fields_ = [("world", I32), ("rank", I32), ("region", P * MAX_PEERS)]


_sig("dicm_last_error", C.c_char_p)
_sig("dicm_version", C.c_int)
_sig("dicm_device_arch", C.c_int)
_sig("dicm_dedup_workspace", S, I64)
_sig("dicm_dedup", C.c_int, C.POINTER(KeySeg), C.c_int, I64, P, S, P, P, P, C.c_int, P, ST)
_sig("dicm_dedup_inverse", C.c_int, C.POINTER(KeySeg), C.c_int, I64, P, S, P, ST)
_sig("dicm_pool_materialize", C.c_int, P, P, I64, C.c_int, C.c_int, P, C.c_int, ST)
_sig("dicm_pool_gather", C.c_int, P, C.c_int, C.c_int, P, P, I64, P, ST)
_sig("dicm_imgmlp_workspace", S, I64, C.c_int, C.c_int)
_sig("dicm_imgmlp_fwd", C.c_int, P, C.c_int, C.c_int, P, P, I64, C.POINTER(ImgMlpParams), P, P, P, C.c_int,
     P, S, ST)
_sig("dicm_imgmlp_bwd", C.c_int, P, C.c_int, C.c_int, P, P, I64, C.POINTER(ImgMlpParams), P, P, P,
     C.POINTER(ImgMlpGrads), C.c_int, P, S, ST)
_sig("dicm_attn_partial_size", I64, C.POINTER(Layout))
_sig("dicm_ref_transpose_workspace", S, I64, I64)
_sig("dicm_hot_acc_bytes", S)
_sig("dicm_ref_transpose", C.c_int, P, I64, I64, P, S, P, P, ST)
_sig("dicm_csr_segments", C.c_int, P, C.c_int, P, ST)
_sig("dicm_id_row_grads", C.c_int, C.POINTER(Layout), C.POINTER(BatchView), P, P, ST)
_sig("dicm_fields_fwd", C.c_int, C.POINTER(Layout), C.POINTER(BatchView), P, ST)
_sig("dicm_images_fwd", C.c_int, C.POINTER(Layout), C.POINTER(BatchView), C.POINTER(AttnParams), P, P, P, ST)
_sig("dicm_p2p_allreduce", C.c_int, C.POINTER(Peers), P, I64, I64, I64, I64, P, P, ST)
_sig("dicm_table_init", C.c_int, P, I64, C.c_int, C.c_int, C.c_int, I64, C.c_uint64, C.c_float, ST)
_sig("dicm_sample_blocks", C.c_int, C.c_int)
_sig("dicm_sample_fwd", C.c_int, C.POINTER(Layout), C.POINTER(BatchView), C.POINTER(AttnParams), P, P, P, ST)
_sig("dicm_sample_bwd", C.c_int, C.POINTER(Layout), C.POINTER(BatchView), C.POINTER(AttnParams), P, P, P, P,
     P, P, P, ST)
_sig("dicm_head_partial_size", I64, C.c_int)
_sig("dicm_head_blocks", C.c_int, C.c_int)
_sig("dicm_head_fwd_bwd", C.c_int, P, C.c_int, C.c_int, P, F, C.POINTER(HeadParams), P, P, P, P, ST)
_sig("dicm_head_fwd", C.c_int, P, C.c_int, C.c_int, C.POINTER(HeadParams), P, ST)
_sig("dicm_reduce_partials", C.c_int, P, C.c_int, I64, P, C.c_int, ST)
_sig("dicm_loss_finalize", C.c_int, P, C.c_int, F, P, P, ST)
_sig("dicm_check_finite", C.c_int, P, I64, P, C.c_int, C.c_int, P, ST)
_sig("dicm_adam_dense_workspace", S, C.c_int)
_sig("dicm_adam_dense", C.c_int, P, P, P, P, P, C.POINTER(Span), C.c_int, F, F, F, F, P, S, P, ST)
_sig("dicm_adam_rows", C.c_int, C.POINTER(TableState), C.c_int, P, P, I64, P, F, F, F, F, P, ST)
_sig("dicm_bucket_workspace", S, I64, C.c_int)
_sig("dicm_bucket_by_owner", C.c_int, P, P, I64, C.c_int, P, P, P, P, P, S, ST)
_sig("dicm_permute_rows12", C.c_int, P, P, P, I64, C.c_int, P, ST)
_sig("dicm_gather_rows_by_key", C.c_int, C.POINTER(TableState), C.c_int, P, P, I64, P, ST)
_sig("dicm_owner_reduce_rows12", C.c_int, P, P, P, C.c_int, I64, P, I64, P, P, ST)
_sig("dicm_p2p_alloc", C.c_int, S, C.POINTER(P))
_sig("dicm_p2p_free", C.c_int, P)
_sig("dicm_ipc_handle", C.c_int, P, P)
_sig("dicm_ipc_open", C.c_int, P, C.POINTER(P))
_sig("dicm_ipc_close", C.c_int, P)
_sig("dicm_p2p_barrier", C.c_int, C.POINTER(Peers), I64, C.c_uint32, P, ST)
_sig("dicm_p2p_counts", C.c_int, C.POINTER(Peers), P, I64, ST)
_sig("dicm_p2p_plan", C.c_int, C.POINTER(Peers), I64, P, P, P, P, ST)
_sig("dicm_p2p_scatter", C.c_int, C.POINTER(Peers), P, C.c_int, C.c_int, P, C.c_int, I64, ST)
_sig("dicm_p2p_gather_scatter12", C.c_int, C.POINTER(Peers), P, C.c_int, C.c_int, P, P, I64, ST)
_sig("dicm_dedup_devn", C.c_int, P, P, I64, I64, P, S, P, P, P, C.c_int, P, ST)
_sig("dicm_jsonl_parse", P, C.c_char_p, I64, C.POINTER(JsonlSpec), C.c_int, C.POINTER(I64), C.POINTER(I64))
_sig("dicm_jsonl_list_total", I64, P, C.c_int)
_sig("dicm_jsonl_export", C.c_int, P, C.c_int, P, P, P)
_sig("dicm_jsonl_free", None, P)
_sig("dicm_zero_async", C.c_int, P, S, ST)
_sig("dicm_host_pack", C.c_int, P, C.POINTER(P), C.POINTER(I64), C.POINTER(I64), C.c_int, C.c_int)
_sig("dicm_head_wide_workspace", S, C.c_int, C.c_int)
_sig("dicm_head_wide_fwd_bwd", C.c_int, P, C.c_int, C.c_int, P, F, C.POINTER(HeadParams), P, P, P, P, P, S, ST)
_sig("dicm_head_wide_fwd", C.c_int, P, C.c_int, C.c_int, C.POINTER(HeadParams), P, P, S, ST)
_sig("dicm_towers_blocks", C.c_int, C.c_int)
_sig("dicm_towers_fwd_bwd", C.c_int, P, C.c_int, C.c_int, C.POINTER(Tower), C.c_int, C.c_int, P, F, P, P, P, I64, P,
     ST)
_sig("dicm_towers_fwd", C.c_int, P, C.c_int, C.c_int, C.POINTER(Tower), C.c_int, C.c_int, P, ST)
_sig("dicm_probe_enable", C.c_int, C.c_int)
_sig("dicm_probe_read", C.c_int, C.c_int, C.POINTER(F), C.c_int, C.POINTER(C.c_int))

PROBE_KERNELS = {"img_fwd_l0": 0, "img_fwd_l12": 1, "img_bwd_l12": 2, "img_bwd_dw1": 3, "img_bwd_dw0": 4,
                 "sample_fwd": 5, "sample_bwd": 6}


def probe_read(kernel, max_n=4096):
    """Elapsed ms of every recorded launch of one probed kernel."""
    buf = (F * max_n)()
    n = C.c_int(0)
    check(lib.dicm_probe_read(PROBE_KERNELS[kernel], buf, max_n, C.byref(n)))
    return list(buf[:n.value])

EXPORTED = [
    "dicm_last_error", "dicm_version", "dicm_device_arch", "dicm_dedup_workspace", "dicm_dedup",
    "dicm_pool_materialize", "dicm_pool_gather", "dicm_imgmlp_workspace", "dicm_imgmlp_fwd", "dicm_imgmlp_bwd",
    "dicm_attn_partial_size", "dicm_sample_blocks", "dicm_sample_fwd", "dicm_sample_bwd",
    "dicm_head_partial_size", "dicm_head_blocks", "dicm_head_fwd_bwd", "dicm_reduce_partials",
    "dicm_loss_finalize", "dicm_check_finite", "dicm_adam_dense_workspace", "dicm_adam_dense", "dicm_adam_rows",
    "dicm_bucket_workspace", "dicm_bucket_by_owner", "dicm_permute_rows12", "dicm_gather_rows_by_key",
    "dicm_owner_reduce_rows12", "dicm_probe_enable", "dicm_probe_read",
    "dicm_p2p_alloc", "dicm_p2p_free", "dicm_ipc_handle", "dicm_ipc_open", "dicm_ipc_close", "dicm_p2p_barrier",
    "dicm_p2p_counts", "dicm_p2p_plan", "dicm_p2p_scatter", "dicm_p2p_gather_scatter12", "dicm_dedup_devn", "dicm_head_fwd",
    "dicm_ref_transpose_workspace", "dicm_hot_acc_bytes", "dicm_dedup_inverse", "dicm_ref_transpose", "dicm_csr_segments", "dicm_table_init", "dicm_id_row_grads", "dicm_p2p_allreduce", "dicm_fields_fwd", "dicm_images_fwd", "dicm_jsonl_parse", "dicm_jsonl_list_total", "dicm_jsonl_export", "dicm_jsonl_free",
    "dicm_towers_blocks", "dicm_towers_fwd_bwd", "dicm_towers_fwd", "dicm_head_wide_workspace",
    "dicm_head_wide_fwd_bwd", "dicm_head_wide_fwd", "dicm_host_pack", "dicm_zero_async",
]


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
