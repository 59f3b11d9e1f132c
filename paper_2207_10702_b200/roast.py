"""Thin ctypes binding of libroast.so (include/roast.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of libroast.so.  Functions keep the C names; `Roast` is a small convenience
wrapper that takes torch tensors (device memory and streams come from torch —
plumbing, not the product).  If the library is missing the import of this
module raises: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ROAST_LIB", os.path.join(_PKG, "libroast.so"))   # override: A/B experiments

OK, ERR_CONFIG, ERR_GEOMETRY, ERR_SHAPE, ERR_BOUNDS, ERR_CAPACITY, ERR_STATE, ERR_CUDA, ERR_NCCL, \
    ERR_UNSUPPORTED = range(10)
FP32, BF16 = 0, 1
ROW_MAJOR, SW128 = 0, 1
MAP_HASH, MAP_IDENTITY = 0, 1

EXPORTS = [
    "roast_config_default", "roast_create", "roast_create_ex", "roast_destroy", "roast_bind",
    "roast_register_linear", "roast_register_embedding", "roast_register_linear_seg",
    "roast_register_embedding_seg", "roast_linear_fwd", "roast_linear_bwd", "roast_linear_bwd_fused",
    "roast_linear_bwd_dx", "roast_linear_bwd_dm", "roast_embedding_fwd", "roast_embedding_bwd",
    "roast_embedding_fwd_multi", "roast_embedding_bwd_multi", "roast_set_autotune", "roast_get_tuned", "roast_set_tuned",
    "roast_linear_fwd_bias", "roast_bias_fwd", "roast_bias_bwd", "roast_bias_bwd_ld", "roast_colsum", "roast_colsum_ex", "roast_register_linear_concat", "roast_linear_fwd_chain",
    "roast_linear_bwd_dx_chain", "roast_linear_bwd_chain", "roast_comm_unique_id", "roast_comm_init",
    "roast_grad_allreduce", "roast_set_exchange", "roast_touched_size", "roast_touched_intervals",
    "roast_debug_exchange", "roast_zero_grad", "roast_sync_shadow", "roast_sgd_step", "roast_optimizer_step", "roast_grad_exchange_step",
    "roast_p2p_window", "roast_p2p_ipc_handle", "roast_p2p_open", "roast_p2p_attach", "roast_p2p_post",
    "roast_p2p_finish", "roast_grad_exchange_p2p", "roast_p2p_reduce", "roast_p2p_gather",
    "roast_grad_exchange_p2p2", "roast_nvls_supported", "roast_nvls_create", "roast_nvls_import",
    "roast_nvls_add_device", "roast_nvls_bind", "roast_nvls_bound", "roast_nvls_reset", "roast_layernorm_fwd",
    "roast_linear_fwd_act", "roast_linear_bwd_dx_act", "roast_linear_fwd_chain_act", "roast_linear_bwd_chain_act",
    "roast_layernorm_bwd", "roast_get_error",
    "roast_status_str", "roast_last_error", "roast_debug_tile_map", "roast_debug_chunk_map",
    "roast_debug_materialize", "roast_debug_hash_host", "roast_launch_count", "roast_lms_segments",
    "roast_debug_opt_state",
]


class roast_tile_t(ctypes.Structure):
    _fields_ = [("z1", ctypes.c_int32), ("z2", ctypes.c_int32)]


class roast_config_t(ctypes.Structure):
    _fields_ = [("C", ctypes.c_double), ("align_elems", ctypes.c_int32), ("tile_layout", ctypes.c_int32),
                ("mapping", ctypes.c_int32), ("use_sign", ctypes.c_int32), ("deterministic", ctypes.c_int32),
                ("simt_bf16", ctypes.c_int32)]


class roast_opt_config_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("lr", ctypes.c_float), ("beta1", ctypes.c_float),
                ("beta2", ctypes.c_float), ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("zero_grad", ctypes.c_int32), ("touched_only", ctypes.c_int32)]


OPT_SGD, OPT_ADAGRAD, OPT_ADAM = 0, 1, 2


class RoastError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        super().__init__(f"{where}: {_lib.roast_status_str(status).decode()} ({status}): "
                         f"{_lib.roast_last_error().decode()}")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2207_10702_b200.build` "
                          "(no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    H, I32, I64, U64, P, S = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                              ctypes.c_void_p, ctypes.c_void_p)
    st = ctypes.c_int
    sig = {
        "roast_config_default": (None, [ctypes.POINTER(roast_config_t)]),
        "roast_create": (st, [ctypes.POINTER(H), I64, U64, roast_tile_t]),
        "roast_create_ex": (st, [ctypes.POINTER(H), I64, U64, roast_tile_t, ctypes.POINTER(roast_config_t)]),
        "roast_destroy": (st, [H]),
        "roast_bind": (st, [H, P, P, S]),
        "roast_register_linear": (st, [H, I64, I64, ctypes.POINTER(I32)]),
        "roast_register_embedding": (st, [H, I64, I32, I32, ctypes.c_double, ctypes.POINTER(I32)]),
        "roast_set_autotune": (st, [H, ctypes.c_int]),
        "roast_linear_fwd_bias": (st, [H, I32, P, P, I64, ctypes.c_int, P, S]),
        "roast_linear_fwd_act": (st, [H, I32, P, P, P, I64, ctypes.c_int, P, I32, S]),
        "roast_linear_bwd_dx_act": (st, [H, I32, P, P, P, I64, ctypes.c_int, I32, S]),
        "roast_linear_fwd_chain_act": (st, [H, I32, I32, P, P, P, P, I64, ctypes.c_int, P, P, I32, S]),
        "roast_linear_bwd_chain_act": (st, [H, I32, I32, P, P, P, P, P, P, I64, ctypes.c_int, I32, S]),
        "roast_bias_fwd": (st, [H, I32, P, S]),
        "roast_linear_fwd_chain": (st, [H, I32, I32, P, P, P, I64, ctypes.c_int, P, P, S]),
        "roast_linear_bwd_dx_chain": (st, [H, I32, I32, P, P, P, I64, ctypes.c_int, S]),
        "roast_linear_bwd_chain": (st, [H, I32, I32, P, P, P, P, P, I64, ctypes.c_int, S]),
        "roast_bias_bwd": (st, [H, I32, P, I64, ctypes.c_int, S]),
        "roast_bias_bwd_ld": (st, [H, I32, P, I64, I64, ctypes.c_int, S]),
        "roast_colsum": (st, [P, I64, I32, I64, ctypes.c_int, P, S]),
        "roast_colsum_ex": (st, [P, I64, I32, I64, ctypes.c_int, P, I32, S]),
        "roast_register_linear_concat": (st, [H, P, I32, ctypes.POINTER(I32)]),
        "roast_get_tuned": (st, [H, I32, I32, I64, ctypes.POINTER(I32), ctypes.POINTER(I32)]),
        "roast_set_tuned": (st, [H, I32, I32, I64, I32, I32]),
        "roast_register_linear_seg": (st, [H, I64, I64, I64, I64, ctypes.POINTER(I32)]),
        "roast_register_embedding_seg": (st, [H, I64, I32, I32, ctypes.c_double, I64, I64, ctypes.POINTER(I32)]),
        "roast_linear_fwd": (st, [H, I32, P, P, I64, ctypes.c_int, S]),
        "roast_linear_bwd": (st, [H, I32, P, P, P, I64, ctypes.c_int, S]),
        "roast_linear_bwd_fused": (st, [H, I32, P, P, P, I64, ctypes.c_int, S]),
        "roast_linear_bwd_dx": (st, [H, I32, P, P, I64, ctypes.c_int, S]),
        "roast_linear_bwd_dm": (st, [H, I32, P, P, I64, ctypes.c_int, S]),
        "roast_embedding_fwd": (st, [H, I32, P, I64, P, S]),
        "roast_embedding_bwd": (st, [H, I32, P, I64, P, S]),
        "roast_embedding_fwd_multi": (st, [H, ctypes.POINTER(I32), I32, P, I64, P, S]),
        "roast_embedding_bwd_multi": (st, [H, ctypes.POINTER(I32), I32, P, I64, P, S]),
        "roast_comm_unique_id": (st, [ctypes.c_char_p]),
        "roast_comm_init": (st, [H, I32, I32, ctypes.c_char_p]),
        "roast_grad_allreduce": (st, [H, S]),
        "roast_set_exchange": (st, [H, I32]),
        "roast_touched_size": (st, [H, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "roast_touched_intervals": (st, [P, I64, I64, P, P, I64, ctypes.POINTER(I64)]),
        "roast_debug_exchange": (st, [H, ctypes.c_float, S]),
        "roast_zero_grad": (st, [H, S]),
        "roast_sync_shadow": (st, [H, S]),
        "roast_sgd_step": (st, [H, ctypes.c_float, S]),
        "roast_optimizer_step": (st, [H, ctypes.POINTER(roast_opt_config_t), I64, S]),
        "roast_grad_exchange_step": (st, [H, ctypes.POINTER(roast_opt_config_t), I64, S]),
        "roast_p2p_window": (st, [H, ctypes.POINTER(P), ctypes.POINTER(I64)]),
        "roast_p2p_ipc_handle": (st, [H, ctypes.c_char_p]),
        "roast_p2p_open": (st, [H, I32, I32, ctypes.c_char_p]),
        "roast_p2p_attach": (st, [H, I32, I32, ctypes.POINTER(P)]),
        "roast_p2p_post": (st, [H, S]),
        "roast_p2p_finish": (st, [H, ctypes.POINTER(roast_opt_config_t), I64, S]),
        "roast_grad_exchange_p2p": (st, [H, ctypes.POINTER(roast_opt_config_t), I64, S]),
        "roast_p2p_reduce": (st, [H, ctypes.POINTER(roast_opt_config_t), I64, S]),
        "roast_p2p_gather": (st, [H, S]),
        "roast_grad_exchange_p2p2": (st, [H, ctypes.POINTER(roast_opt_config_t), I64, S]),
        "roast_nvls_supported": (st, [I32, ctypes.POINTER(I32)]),
        "roast_nvls_create": (st, [H, I32, ctypes.POINTER(I32)]),
        "roast_nvls_import": (st, [H, I32, I32]),
        "roast_nvls_add_device": (st, [H]),
        "roast_nvls_bind": (st, [H, I32]),
        "roast_nvls_bound": (st, [H, ctypes.POINTER(I32)]),
        "roast_nvls_reset": (st, [H]),
        "roast_layernorm_fwd": (st, [P, P, P, P, P, P, P, P, I64, I32, ctypes.c_float, ctypes.c_int, ctypes.c_int, S]),
        "roast_layernorm_bwd": (st, [P, P, P, P, P, P, P, P, I64, I32, ctypes.c_int, ctypes.c_int, S]),
        "roast_get_error": (st, [H]),
        "roast_status_str": (ctypes.c_char_p, [st]),
        "roast_last_error": (ctypes.c_char_p, []),
        "roast_debug_tile_map": (st, [H, I32, P, P]),
        "roast_debug_chunk_map": (st, [H, I32, P, I64, P, P, S]),
        "roast_debug_materialize": (st, [H, I32, ctypes.c_int, P, S]),
        "roast_launch_count": (I64, [H]),
        "roast_debug_hash_host": (st, [U64, I32, P, I64, I64, I64, I32, I32, P, P]),
        "roast_lms_segments": (st, [P, I32, I64, I32, P, P]),
        "roast_debug_opt_state": (st, [H, I32, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _check(status, where):
    if status != OK:
        raise RoastError(status, where)


# ---- same-name functions (thin) ----------------------------------------------------------
def roast_config_default():
    cfg = roast_config_t()
    _lib.roast_config_default(ctypes.byref(cfg))
    return cfg


def roast_create(mem_size, seed, z1, z2, cfg=None):
    h = ctypes.c_void_p()
    if cfg is None:
        _check(_lib.roast_create(ctypes.byref(h), mem_size, seed, roast_tile_t(z1, z2)), "roast_create")
    else:
        _check(_lib.roast_create_ex(ctypes.byref(h), mem_size, seed, roast_tile_t(z1, z2), ctypes.byref(cfg)),
               "roast_create_ex")
    return h


def roast_destroy(h):
    _check(_lib.roast_destroy(h), "roast_destroy")


def roast_bind(h, M_ptr, dM_ptr, stream=0):
    _check(_lib.roast_bind(h, M_ptr, dM_ptr, stream), "roast_bind")


def roast_register_linear(h, in_features, out_features):
    i = ctypes.c_int32()
    _check(_lib.roast_register_linear(h, in_features, out_features, ctypes.byref(i)), "roast_register_linear")
    return i.value


def roast_register_embedding(h, num_rows, dim, chunk, fan_in=0.0):
    i = ctypes.c_int32()
    _check(_lib.roast_register_embedding(h, num_rows, dim, chunk, fan_in, ctypes.byref(i)),
           "roast_register_embedding")
    return i.value


def roast_register_linear_seg(h, in_features, out_features, seg_base, seg_size):
    i = ctypes.c_int32()
    _check(_lib.roast_register_linear_seg(h, in_features, out_features, seg_base, seg_size, ctypes.byref(i)),
           "roast_register_linear_seg")
    return i.value


def roast_register_embedding_seg(h, num_rows, dim, chunk, fan_in, seg_base, seg_size):
    i = ctypes.c_int32()
    _check(_lib.roast_register_embedding_seg(h, num_rows, dim, chunk, fan_in, seg_base, seg_size, ctypes.byref(i)),
           "roast_register_embedding_seg")
    return i.value


TUNE_OFF, TUNE_INFERENCE, TUNE_TRAINING = 0, 1, 2


def roast_set_autotune(h, strategy):
    _check(_lib.roast_set_autotune(h, strategy), "roast_set_autotune")


def roast_get_tuned(h, mid, kernel, tokens):
    """(WM, split-K) the autotuner cached for kernel 0 fwd / 1 dX / 2 dM, or None."""
    wm, sp = ctypes.c_int32(), ctypes.c_int32()
    if _lib.roast_get_tuned(h, mid, kernel, tokens, ctypes.byref(wm), ctypes.byref(sp)) != 0:
        return None
    return wm.value, sp.value


def roast_set_tuned(h, mid, kernel, tokens, wm, splits):
    _check(_lib.roast_set_tuned(h, mid, kernel, tokens, wm, splits), "roast_set_tuned")


def lms_segments(sizes, mem_size, align=8):
    """LMS memories from the library's roast_lms_segments: piece i of
    sizes[i] parameters gets |M_i| = floor(f_i |M|), f_i = n_i / n, aligned down to
    `align`, the remainder to the last piece (R23).  Returns [(seg_base,
    seg_size)] for roast_register_*_seg / Roast.linear(segment=)."""
    import numpy as np
    sz = np.ascontiguousarray([int(x) for x in sizes], dtype=np.int64)
    base = np.empty(len(sz), dtype=np.int64)
    size = np.empty(len(sz), dtype=np.int64)
    _check(_lib.roast_lms_segments(sz.ctypes.data, len(sz), int(mem_size), int(align), base.ctypes.data,
                                   size.ctypes.data), "roast_lms_segments")
    return [(int(b), int(s)) for b, s in zip(base, size)]


def roast_linear_fwd_bias(h, mid, X_ptr, Y_ptr, tokens, dtype, bias_ptr, stream=0):
    _check(_lib.roast_linear_fwd_bias(h, mid, X_ptr, Y_ptr, tokens, dtype, bias_ptr, stream), "roast_linear_fwd_bias")


ACT_NONE, ACT_GELU_TANH, ACT_RESIDUAL = 0, 1, 2
ERR_UNSUPPORTED = 9


def roast_linear_fwd_act(h, mid, X_ptr, Y_ptr, A_ptr, tokens, dtype, bias_ptr=None, act=ACT_GELU_TANH, stream=0):
    _check(_lib.roast_linear_fwd_act(h, mid, X_ptr, Y_ptr, A_ptr, tokens, dtype, bias_ptr, act, stream),
           "roast_linear_fwd_act")


def roast_linear_bwd_dx_act(h, mid, dY_ptr, U_ptr, dX_ptr, tokens, dtype, act=ACT_GELU_TANH, stream=0):
    _check(_lib.roast_linear_bwd_dx_act(h, mid, dY_ptr, U_ptr, dX_ptr, tokens, dtype, act, stream),
           "roast_linear_bwd_dx_act")


def roast_linear_fwd_chain_act(h, id_a, id_b, X_ptr, U_ptr, A_ptr, Yb_ptr, tokens, dtype, bias_a=None, bias_b=None,
                               act=ACT_GELU_TANH, stream=0):
    _check(_lib.roast_linear_fwd_chain_act(h, id_a, id_b, X_ptr, U_ptr, A_ptr, Yb_ptr, tokens, dtype, bias_a, bias_b,
                                           act, stream), "roast_linear_fwd_chain_act")


def roast_linear_bwd_chain_act(h, id_a, id_b, Xa_ptr, A_ptr, U_ptr, dYb_ptr, dU_ptr, dXa_ptr, tokens, dtype,
                               act=ACT_GELU_TANH, stream=0):
    _check(_lib.roast_linear_bwd_chain_act(h, id_a, id_b, Xa_ptr, A_ptr, U_ptr, dYb_ptr, dU_ptr, dXa_ptr, tokens,
                                           dtype, act, stream), "roast_linear_bwd_chain_act")


def roast_linear_fwd_chain(h, id_a, id_b, X_ptr, Ya_ptr, Yb_ptr, tokens, dtype, bias_a=None, bias_b=None, stream=0):
    _check(_lib.roast_linear_fwd_chain(h, id_a, id_b, X_ptr, Ya_ptr, Yb_ptr, tokens, dtype, bias_a, bias_b, stream),
           "roast_linear_fwd_chain")


def roast_linear_bwd_chain(h, id_a, id_b, Xa_ptr, Ya_ptr, dYb_ptr, dYa_ptr, dXa_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_linear_bwd_chain(h, id_a, id_b, Xa_ptr, Ya_ptr, dYb_ptr, dYa_ptr, dXa_ptr, tokens, dtype, stream),
           "roast_linear_bwd_chain")


def roast_linear_bwd_dx_chain(h, id_a, id_b, dYb_ptr, dYa_ptr, dX_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_linear_bwd_dx_chain(h, id_a, id_b, dYb_ptr, dYa_ptr, dX_ptr, tokens, dtype, stream),
           "roast_linear_bwd_dx_chain")


def roast_bias_fwd(h, bias_id, b_ptr, stream=0):
    _check(_lib.roast_bias_fwd(h, bias_id, b_ptr, stream), "roast_bias_fwd")


def roast_bias_bwd(h, bias_id, dY_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_bias_bwd(h, bias_id, dY_ptr, tokens, dtype, stream), "roast_bias_bwd")


def roast_bias_bwd_ld(h, bias_id, dY_ptr, tokens, ld, dtype, stream=0):
    _check(_lib.roast_bias_bwd_ld(h, bias_id, dY_ptr, tokens, ld, dtype, stream), "roast_bias_bwd_ld")


def roast_colsum(dY_ptr, tokens, n, ld, dtype, db_ptr, stream=0):
    _check(_lib.roast_colsum(dY_ptr, tokens, n, ld, dtype, db_ptr, stream), "roast_colsum")


def roast_colsum_ex(dY_ptr, tokens, n, ld, dtype, db_ptr, accumulate, stream=0):
    _check(_lib.roast_colsum_ex(dY_ptr, tokens, n, ld, dtype, db_ptr, int(accumulate), stream), "roast_colsum_ex")


def roast_register_linear_concat(h, ids):
    arr = (ctypes.c_int32 * len(ids))(*ids)
    out = ctypes.c_int32()
    _check(_lib.roast_register_linear_concat(h, arr, len(ids), ctypes.byref(out)), "roast_register_linear_concat")
    return out.value


def roast_linear_fwd(h, mid, X_ptr, Y_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_linear_fwd(h, mid, X_ptr, Y_ptr, tokens, dtype, stream), "roast_linear_fwd")


def roast_linear_bwd(h, mid, X_ptr, dY_ptr, dX_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_linear_bwd(h, mid, X_ptr, dY_ptr, dX_ptr, tokens, dtype, stream), "roast_linear_bwd")


def roast_linear_bwd_fused(h, mid, X_ptr, dY_ptr, dX_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_linear_bwd_fused(h, mid, X_ptr, dY_ptr, dX_ptr, tokens, dtype, stream), "roast_linear_bwd_fused")


def roast_linear_bwd_dx(h, mid, dY_ptr, dX_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_linear_bwd_dx(h, mid, dY_ptr, dX_ptr, tokens, dtype, stream), "roast_linear_bwd_dx")


def roast_linear_bwd_dm(h, mid, X_ptr, dY_ptr, tokens, dtype, stream=0):
    _check(_lib.roast_linear_bwd_dm(h, mid, X_ptr, dY_ptr, tokens, dtype, stream), "roast_linear_bwd_dm")


def roast_embedding_fwd(h, mid, idx_ptr, n, out_ptr, stream=0):
    _check(_lib.roast_embedding_fwd(h, mid, idx_ptr, n, out_ptr, stream), "roast_embedding_fwd")


def roast_embedding_bwd(h, mid, idx_ptr, n, dout_ptr, stream=0):
    _check(_lib.roast_embedding_bwd(h, mid, idx_ptr, n, dout_ptr, stream), "roast_embedding_bwd")


def _ids(ids):
    return (ctypes.c_int32 * len(ids))(*ids), len(ids)


def roast_embedding_fwd_multi(h, ids, idx_ptr, n, out_ptr, stream=0):
    arr, nt = _ids(ids)
    _check(_lib.roast_embedding_fwd_multi(h, arr, nt, idx_ptr, n, out_ptr, stream), "roast_embedding_fwd_multi")


def roast_embedding_bwd_multi(h, ids, idx_ptr, n, dout_ptr, stream=0):
    arr, nt = _ids(ids)
    _check(_lib.roast_embedding_bwd_multi(h, arr, nt, idx_ptr, n, dout_ptr, stream), "roast_embedding_bwd_multi")


def roast_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.roast_comm_unique_id(buf), "roast_comm_unique_id")
    return buf.raw


def roast_comm_init(h, rank, world, uid: bytes):
    _check(_lib.roast_comm_init(h, rank, world, uid), "roast_comm_init")


def roast_grad_allreduce(h, stream=0):
    _check(_lib.roast_grad_allreduce(h, stream), "roast_grad_allreduce")


EXCHANGE_AUTO, EXCHANGE_DENSE, EXCHANGE_TOUCHED = 0, 1, 2


def roast_set_exchange(h, mode):
    _check(_lib.roast_set_exchange(h, mode), "roast_set_exchange")


def roast_touched_size(h):
    """(elements, intervals) of the touched set the exchange moves."""
    n, k = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.roast_touched_size(h, ctypes.byref(n), ctypes.byref(k)), "roast_touched_size")
    return n.value, k.value


def roast_touched_intervals(starts, span):
    """Host utility: merged [s, s + span) intervals -> (starts, lengths) int64 arrays (no GPU)."""
    import numpy as np
    s = np.ascontiguousarray(starts, dtype=np.int64)
    cap = max(1, len(s))
    out_s = np.empty(cap, dtype=np.int64)
    out_l = np.empty(cap, dtype=np.int64)
    cnt = ctypes.c_int64()
    _check(_lib.roast_touched_intervals(s.ctypes.data, len(s), span, out_s.ctypes.data, out_l.ctypes.data, cap,
                                        ctypes.byref(cnt)), "roast_touched_intervals")
    return out_s[:cnt.value].copy(), out_l[:cnt.value].copy()


def roast_debug_exchange(h, scale, stream=0):
    _check(_lib.roast_debug_exchange(h, scale, stream), "roast_debug_exchange")


def roast_zero_grad(h, stream=0):
    _check(_lib.roast_zero_grad(h, stream), "roast_zero_grad")


def roast_sync_shadow(h, stream=0):
    _check(_lib.roast_sync_shadow(h, stream), "roast_sync_shadow")


def roast_sgd_step(h, lr, stream=0):
    _check(_lib.roast_sgd_step(h, lr, stream), "roast_sgd_step")


def roast_optimizer_step(h, kind, lr, step=1, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, zero_grad=True,
                         stream=0, touched_only=False):
    cfg = roast_opt_config_t(kind, lr, beta1, beta2, eps, weight_decay, int(zero_grad), int(touched_only))
    _check(_lib.roast_optimizer_step(h, ctypes.byref(cfg), step, stream), "roast_optimizer_step")


def roast_grad_exchange_step(h, kind, lr, step=1, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                             zero_grad=True, stream=0, touched_only=False):
    cfg = roast_opt_config_t(kind, lr, beta1, beta2, eps, weight_decay, int(zero_grad), int(touched_only))
    _check(_lib.roast_grad_exchange_step(h, ctypes.byref(cfg), step, stream), "roast_grad_exchange_step")


def roast_p2p_window(h):
    """(device address, bytes) of this handle's exchange window (allocated on first call)."""
    ptr, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(_lib.roast_p2p_window(h, ctypes.byref(ptr), ctypes.byref(n)), "roast_p2p_window")
    return int(ptr.value or 0), int(n.value)


def roast_p2p_ipc_handle(h):
    buf = ctypes.create_string_buffer(64)
    _check(_lib.roast_p2p_ipc_handle(h, buf), "roast_p2p_ipc_handle")
    return buf.raw


def roast_p2p_open(h, rank, world, handles: bytes):
    assert len(handles) == 64 * world
    _check(_lib.roast_p2p_open(h, rank, world, handles), "roast_p2p_open")


def roast_p2p_attach(h, rank, world, windows):
    arr = (ctypes.c_void_p * world)(*[int(w) for w in windows])
    _check(_lib.roast_p2p_attach(h, rank, world, arr), "roast_p2p_attach")


def roast_p2p_post(h, stream=0):
    _check(_lib.roast_p2p_post(h, stream), "roast_p2p_post")


def roast_p2p_finish(h, kind, lr, step=1, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, zero_grad=True,
                     stream=0):
    cfg = roast_opt_config_t(kind, lr, beta1, beta2, eps, weight_decay, int(zero_grad), 1)
    _check(_lib.roast_p2p_finish(h, ctypes.byref(cfg), step, stream), "roast_p2p_finish")


def roast_grad_exchange_p2p(h, kind, lr, step=1, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                            zero_grad=True, stream=0):
    cfg = roast_opt_config_t(kind, lr, beta1, beta2, eps, weight_decay, int(zero_grad), 1)
    _check(_lib.roast_grad_exchange_p2p(h, ctypes.byref(cfg), step, stream), "roast_grad_exchange_p2p")


def roast_p2p_reduce(h, kind, lr, step=1, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, stream=0):
    cfg = roast_opt_config_t(kind, lr, beta1, beta2, eps, weight_decay, 1, 1)
    _check(_lib.roast_p2p_reduce(h, ctypes.byref(cfg), step, stream), "roast_p2p_reduce")


def roast_p2p_gather(h, stream=0):
    _check(_lib.roast_p2p_gather(h, stream), "roast_p2p_gather")


def roast_grad_exchange_p2p2(h, kind, lr, step=1, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, stream=0):
    cfg = roast_opt_config_t(kind, lr, beta1, beta2, eps, weight_decay, 1, 1)
    _check(_lib.roast_grad_exchange_p2p2(h, ctypes.byref(cfg), step, stream), "roast_grad_exchange_p2p2")


def roast_nvls_supported(device):
    v = ctypes.c_int32()
    _check(_lib.roast_nvls_supported(device, ctypes.byref(v)), "roast_nvls_supported")
    return bool(v.value)


def roast_nvls_create(h, world):
    fd = ctypes.c_int32(-1)
    _check(_lib.roast_nvls_create(h, world, ctypes.byref(fd)), "roast_nvls_create")
    return int(fd.value)


def roast_nvls_import(h, world, fd):
    _check(_lib.roast_nvls_import(h, world, fd), "roast_nvls_import")


def roast_nvls_add_device(h):
    _check(_lib.roast_nvls_add_device(h), "roast_nvls_add_device")


def roast_nvls_bind(h, rank):
    _check(_lib.roast_nvls_bind(h, rank), "roast_nvls_bind")


def roast_layernorm_fwd(x, r, gamma, beta, y, s_out, mean, rstd, rows, n, eps, dt, pdt, stream=0):
    _check(_lib.roast_layernorm_fwd(x, r, gamma, beta, y, s_out, mean, rstd, rows, n, eps, dt, pdt, stream),
           "roast_layernorm_fwd")


def roast_layernorm_bwd(dy, s, gamma, mean, rstd, ds, dgamma, dbeta, rows, n, dt, pdt, stream=0):
    _check(_lib.roast_layernorm_bwd(dy, s, gamma, mean, rstd, ds, dgamma, dbeta, rows, n, dt, pdt, stream),
           "roast_layernorm_bwd")


def roast_nvls_reset(h):
    _check(_lib.roast_nvls_reset(h), "roast_nvls_reset")


def roast_nvls_bound(h):
    v = ctypes.c_int32()
    _check(_lib.roast_nvls_bound(h, ctypes.byref(v)), "roast_nvls_bound")
    return bool(v.value)


def roast_get_error(h):
    return _lib.roast_get_error(h)


def roast_debug_tile_map(h, mid, off_ptr, sgn_ptr):
    _check(_lib.roast_debug_tile_map(h, mid, off_ptr, sgn_ptr), "roast_debug_tile_map")


def roast_debug_chunk_map(h, mid, rows_ptr, n, off_ptr, sgn_ptr, stream=0):
    _check(_lib.roast_debug_chunk_map(h, mid, rows_ptr, n, off_ptr, sgn_ptr, stream), "roast_debug_chunk_map")


def roast_debug_materialize(h, mid, dtype, W_ptr, stream=0):
    _check(_lib.roast_debug_materialize(h, mid, dtype, W_ptr, stream), "roast_debug_materialize")


def roast_launch_count(h):
    return _lib.roast_launch_count(h)


def roast_debug_hash_host(seed, module, keys, mem_size, span, align=8, use_sign=True):
    """(offsets, signs) of the library hash evaluated on the host (no GPU needed)."""
    import numpy as np
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    off = np.empty(len(keys), dtype=np.int64)
    sgn = np.empty(len(keys), dtype=np.int8)
    _check(_lib.roast_debug_hash_host(seed, module, keys.ctypes.data, len(keys), mem_size, span, align,
                                      int(use_sign), off.ctypes.data, sgn.ctypes.data), "roast_debug_hash_host")
    return off, sgn


# ---- torch convenience wrapper --------------------------------------------------------------
class Roast:
    """One handle + its caller-owned M / dM (torch fp32 CUDA tensors)."""

    def __init__(self, M, z1, z2, seed=0x5EED, C=1.0, align=8, tile_layout=ROW_MAJOR, mapping=MAP_HASH,
                 use_sign=True, deterministic=False, dM=None, simt_bf16=False):
        import torch
        assert M.is_cuda and M.dtype == torch.float32 and M.is_contiguous()
        self.torch = torch
        self.M = M
        self.dM = torch.zeros_like(M) if dM is None else dM
        cfg = roast_config_default()
        cfg.C, cfg.align_elems, cfg.tile_layout = C, align, tile_layout
        cfg.mapping, cfg.use_sign, cfg.deterministic = mapping, int(use_sign), int(deterministic)
        cfg.simt_bf16 = int(simt_bf16)   # bf16 off the tcgen05 path: error unless opted in
        self.mem_size = M.numel()
        self.z1, self.z2 = z1, z2
        self.h = roast_create(self.mem_size, seed, z1, z2, cfg)
        self.dims = {}
        roast_bind(self.h, M.data_ptr(), self.dM.data_ptr(), self._s())
        # biases via L (registered with bias()): with batch_biases, every bias is recovered by one
        # multi-table lookup per (dim, chunk) group per parameter generation, and their
        # gradients are column sums collected into one buffer and scattered by one multi-table
        # L backward at flush time (exchange / update / flush_bias_grads) — not ~4 small
        # kernels per bias per step
        self.batch_biases = False
        self._biases = []
        self._gen = 0
        self._bias_gen = -1
        self._bias_groups = None
        self._bias_pending = False

    def _s(self, stream=None):
        s = stream if stream is not None else self.torch.cuda.current_stream()
        return s.cuda_stream

    def close(self):
        if self.h:
            roast_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def linear(self, in_features, out_features, segment=None):
        """segment = (seg_base, seg_size): LMS memory of this module (None = GMS)."""
        mid = (roast_register_linear(self.h, in_features, out_features) if segment is None else
               roast_register_linear_seg(self.h, in_features, out_features, *segment))
        self.dims[mid] = ("linear", in_features, out_features)
        return mid

    def linear_concat(self, mids):
        """One GEMM over linears sharing in_features: W = [W_1 | ... | W_n] (their own tiles)."""
        gid = roast_register_linear_concat(self.h, list(mids))
        self.dims[gid] = ("linear", self.dims[mids[0]][1], sum(self.dims[m][2] for m in mids))
        return gid

    def set_autotune(self, strategy):
        roast_set_autotune(self.h, strategy)

    def tuned(self, mid, kernel, tokens):
        return roast_get_tuned(self.h, mid, kernel, tokens)

    def set_tuned(self, mid, kernel, tokens, wm, splits=1):
        roast_set_tuned(self.h, mid, kernel, tokens, wm, splits)

    def embedding(self, num_rows, dim, chunk, fan_in=0.0, segment=None):
        mid = (roast_register_embedding(self.h, num_rows, dim, chunk, fan_in) if segment is None else
               roast_register_embedding_seg(self.h, num_rows, dim, chunk, fan_in, *segment))
        self.dims[mid] = ("embedding", num_rows, dim, chunk)
        return mid

    # ---- biases via L (reading R24) ---------------------------------------------------
    def bias(self, n, fan_in, chunk=64):
        """Register a bias of n elements recovered with L (a 1 x n ROAST embedding)."""
        mid = self.embedding(1, n, chunk, fan_in)
        self._biases.append(mid)
        self._bias_groups = None
        return mid

    def _groups(self):
        if self._bias_groups is None:
            torch = self.torch
            by = {}
            for m in self._biases:
                by.setdefault((self.dims[m][2], self.dims[m][3]), []).append(m)
            self._bias_groups = []
            for (dim, chunk), mids in by.items():
                vals = torch.empty(len(mids), dim, dtype=torch.float32, device=self.M.device)
                grads = torch.zeros(len(mids), dim, dtype=torch.float32, device=self.M.device)
                idx = torch.zeros(len(mids), dtype=torch.int64, device=self.M.device)
                slot = {m: i for i, m in enumerate(mids)}
                self._bias_groups.append((mids, vals, grads, idx, slot))
            self._bias_gen = -1
        return self._bias_groups

    def bias_vector(self, mid, stream=None):
        """The recovered bias (fp32 [n]); batched: a view into its group's buffer, refreshed
        once per parameter generation by one multi-table lookup per group."""
        if not self.batch_biases:
            return self.bias_fwd(mid, stream=stream)
        groups = self._groups()
        if self._bias_gen != self._gen:
            for mids, vals, _, idx, _ in groups:
                roast_embedding_fwd_multi(self.h, mids, idx.data_ptr(), 1, vals.data_ptr(), self._s(stream))
            self._bias_gen = self._gen
        for mids, vals, _, _, slot in groups:
            if mid in slot:
                return vals[slot[mid]]
        raise KeyError(mid)

    def bias_grad(self, mid, dY, stream=None):
        """Bias backward; batched: only the column sums now (into the group buffer), the L
        scatter of every bias at flush_bias_grads()."""
        if not self.batch_biases:
            return self.bias_bwd(mid, dY, stream=stream)
        n = self.dims[mid][2]
        if dY.dim() != 2:
            dY = dY.reshape(-1, n)
        ld = dY.stride(0) if dY.shape[0] > 1 else n
        for _, _, grads, _, slot in self._groups():
            if mid in slot:
                # accumulate: a bias whose layer runs backward twice before the flush (micro-batch
                # accumulation, a shared module) keeps both contributions; flush / zero_grad clear it
                roast_colsum_ex(dY.data_ptr(), dY.shape[0], n, ld, self._dt(dY), grads[slot[mid]].data_ptr(), 1,
                                self._s(stream))
                self._bias_pending = True
                return
        raise KeyError(mid)

    def flush_bias_grads(self, stream=None):
        """dM += every collected bias gradient (one multi-table L backward per group)."""
        if not self._bias_pending:
            return
        s = self._stream_obj(stream)
        for mids, _, grads, idx, _ in self._groups():
            roast_embedding_bwd_multi(self.h, mids, idx.data_ptr(), 1, grads.data_ptr(), self._s(stream))
            with self.torch.cuda.stream(s):     # zero after the scatter has read them (same stream)
                grads.zero_()
        self._bias_pending = False

    def _stream_obj(self, stream):
        """torch stream object for `stream` (None = the current stream; a raw handle is wrapped)."""
        torch = self.torch
        if stream is None:
            return torch.cuda.current_stream()
        if isinstance(stream, torch.cuda.Stream):
            return stream
        return torch.cuda.ExternalStream(int(stream))

    @staticmethod
    def _dt(t):
        import torch
        return BF16 if t.dtype == torch.bfloat16 else FP32

    def fwd(self, mid, X, Y=None, stream=None, bias=None):
        """Y = lambda X W~ (+ bias: fp32 [out] vector added in the epilogue)."""
        _, H, O = self.dims[mid]
        assert X.is_contiguous() and X.shape[-1] == H
        T = X.numel() // H
        if Y is None:
            Y = self.torch.empty(*X.shape[:-1], O, dtype=X.dtype, device=X.device)
        if bias is None:
            roast_linear_fwd(self.h, mid, X.data_ptr(), Y.data_ptr(), T, self._dt(X), self._s(stream))
        else:
            assert bias.dtype == self.torch.float32 and bias.numel() == O and bias.is_contiguous()
            roast_linear_fwd_bias(self.h, mid, X.data_ptr(), Y.data_ptr(), T, self._dt(X), bias.data_ptr(),
                                  self._s(stream))
        return Y

    def fwd_chain(self, a, b, X, Ya=None, Yb=None, stream=None, bias_a=None, bias_b=None):
        """Y_a = X W~_a (+bias_a), Y_b = Y_a W~_b (+bias_b) in one launch; returns (Y_a, Y_b)."""
        _, H, O = self.dims[a]
        _, H2, O2 = self.dims[b]
        T = X.numel() // H
        Ya = self.torch.empty(T, O, dtype=X.dtype, device=X.device) if Ya is None else Ya
        Yb = self.torch.empty(T, O2, dtype=X.dtype, device=X.device) if Yb is None else Yb
        ptr = (lambda t: None if t is None else t.data_ptr())   # noqa: E731
        roast_linear_fwd_chain(self.h, a, b, X.data_ptr(), Ya.data_ptr(), Yb.data_ptr(), T, self._dt(X),
                               ptr(bias_a), ptr(bias_b), self._s(stream))
        return Ya, Yb

    def bwd_dx_chain(self, a, b, dYb, dYa=None, dX=None, stream=None):
        """dY_a = dY_b W~_b^T, dX = dY_a W~_a^T in one launch; returns (dY_a, dX)."""
        _, H, O = self.dims[a]
        _, H2, O2 = self.dims[b]
        T = dYb.numel() // O2
        dYa = self.torch.empty(T, H2, dtype=dYb.dtype, device=dYb.device) if dYa is None else dYa
        dX = self.torch.empty(T, H, dtype=dYb.dtype, device=dYb.device) if dX is None else dX
        roast_linear_bwd_dx_chain(self.h, a, b, dYb.data_ptr(), dYa.data_ptr(), dX.data_ptr(), T, self._dt(dYb),
                                  self._s(stream))
        return dYa, dX

    def bwd_chain(self, a, b, Xa, Ya, dYb, dYa=None, dXa=None, stream=None):
        """The backward of fwd_chain(a, b): dY_a = dY_b W~_b^T, dM += b(Y_a, dY_b), dX_a = dY_a W~_a^T,
        dM += a(X_a, dY_a) — on the tcgen05 path one persistent launch; returns (dY_a, dX_a)."""
        _, H, O = self.dims[a]
        _, H2, O2 = self.dims[b]
        T = dYb.numel() // O2
        dYa = self.torch.empty(T, H2, dtype=dYb.dtype, device=dYb.device) if dYa is None else dYa
        dXa = self.torch.empty(T, H, dtype=dYb.dtype, device=dYb.device) if dXa is None else dXa
        roast_linear_bwd_chain(self.h, a, b, Xa.data_ptr(), Ya.data_ptr(), dYb.data_ptr(), dYa.data_ptr(),
                               dXa.data_ptr(), T, self._dt(dYb), self._s(stream))
        return dYa, dXa

    def bias_fwd(self, bias_mid, out=None, stream=None):
        """The bias vector (row 0 of a 1 x n embedding registered for it) recovered with L."""
        n = self.dims[bias_mid][2]
        if out is None:
            out = self.torch.empty(n, dtype=self.torch.float32, device=self.M.device)
        roast_bias_fwd(self.h, bias_mid, out.data_ptr(), self._s(stream))
        return out

    def bias_bwd(self, bias_mid, dY, stream=None):
        """dM += lambda g * (column sums of dY) scattered through the bias's L mapping.  dY may be
        a column slice of a wider row-major matrix (rows dY.stride(0) elements apart)."""
        n = self.dims[bias_mid][2]
        if dY.dim() != 2:
            dY = dY.reshape(-1, n)
        assert dY.shape[-1] == n and (dY.shape[0] == 0 or dY.stride(-1) == 1)
        ld = dY.stride(0) if dY.shape[0] > 1 else n
        roast_bias_bwd_ld(self.h, bias_mid, dY.data_ptr(), dY.shape[0], ld, self._dt(dY), self._s(stream))

    def bwd(self, mid, X, dY, dX=None, need_dx=True, stream=None):
        _, H, O = self.dims[mid]
        T = X.numel() // H
        assert dY.numel() == T * O and X.dtype == dY.dtype
        if need_dx and dX is None:
            dX = self.torch.empty_like(X)
        roast_linear_bwd(self.h, mid, X.data_ptr(), dY.data_ptr(), dX.data_ptr() if need_dx else None, T,
                         self._dt(X), self._s(stream))
        return dX

    def bwd_fused(self, mid, X, dY, dX=None, stream=None):
        """dX and dM += in one co-scheduled launch where that pays (roast_linear_bwd_fused)."""
        _, H, O = self.dims[mid]
        T = X.numel() // H
        assert dY.numel() == T * O and X.dtype == dY.dtype
        dX = self.torch.empty_like(X) if dX is None else dX
        roast_linear_bwd_fused(self.h, mid, X.data_ptr(), dY.data_ptr(), dX.data_ptr(), T, self._dt(X), self._s(stream))
        return dX

    def fwd_act(self, mid, X, Y=None, A=None, bias=None, act=ACT_GELU_TANH, stream=None):
        """Y = lambda X W~ (+ bias) and A = act(Y) in the same epilogue (roast_linear_fwd_act)."""
        _, H, O = self.dims[mid]
        assert X.is_contiguous() and X.shape[-1] == H
        T = X.numel() // H
        Y = self.torch.empty(*X.shape[:-1], O, dtype=X.dtype, device=X.device) if Y is None else Y
        A = self.torch.empty_like(Y) if A is None else A
        if bias is not None:
            assert bias.dtype == self.torch.float32 and bias.numel() == O and bias.is_contiguous()
        roast_linear_fwd_act(self.h, mid, X.data_ptr(), Y.data_ptr(), A.data_ptr(), T, self._dt(X),
                             bias.data_ptr() if bias is not None else None, act, self._s(stream))
        return Y, A

    def fwd_chain_act(self, a, b, X, bias_a=None, bias_b=None, act=ACT_GELU_TANH, stream=None):
        """U = a(X), A = act(U), Y_b = b(A) in one launch (roast_linear_fwd_chain_act); returns (U, A, Y_b)."""
        _, H, O = self.dims[a]
        _, H2, O2 = self.dims[b]
        T = X.numel() // H
        U = self.torch.empty(T, O, dtype=X.dtype, device=X.device)
        A = self.torch.empty_like(U)
        Yb = self.torch.empty(T, O2, dtype=X.dtype, device=X.device)
        ptr = (lambda t: None if t is None else t.data_ptr())   # noqa: E731
        roast_linear_fwd_chain_act(self.h, a, b, X.data_ptr(), U.data_ptr(), A.data_ptr(), Yb.data_ptr(), T,
                                   self._dt(X), ptr(bias_a), ptr(bias_b), act, self._s(stream))
        return U, A, Yb

    def bwd_chain_act(self, a, b, Xa, A, U, dYb, act=ACT_GELU_TANH, stream=None):
        """The backward of fwd_chain_act (roast_linear_bwd_chain_act): dM += both layers' scatters;
        returns (dU, dX_a)."""
        _, H, O = self.dims[a]
        _, H2, O2 = self.dims[b]
        T = dYb.numel() // O2
        dU = self.torch.empty(T, H2, dtype=dYb.dtype, device=dYb.device)
        dXa = self.torch.empty(T, H, dtype=dYb.dtype, device=dYb.device)
        roast_linear_bwd_chain_act(self.h, a, b, Xa.data_ptr(), A.data_ptr(), U.data_ptr(), dYb.data_ptr(),
                                   dU.data_ptr(), dXa.data_ptr(), T, self._dt(dYb), act, self._s(stream))
        return dU, dXa

    def bwd_dx_act(self, mid, dY, U, dX=None, act=ACT_GELU_TANH, stream=None):
        """dX = (lambda dY W~^T) * act'(U) in the dX GEMM's epilogue (roast_linear_bwd_dx_act)."""
        _, H, O = self.dims[mid]
        T = dY.numel() // O
        dX = self.torch.empty(T, H, dtype=dY.dtype, device=dY.device) if dX is None else dX
        roast_linear_bwd_dx_act(self.h, mid, dY.data_ptr(), U.data_ptr(), dX.data_ptr(), T, self._dt(dY), act,
                                self._s(stream))
        return dX

    def bwd_dx(self, mid, dY, dX, stream=None):
        _, H, O = self.dims[mid]
        roast_linear_bwd_dx(self.h, mid, dY.data_ptr(), dX.data_ptr(), dY.numel() // O, self._dt(dY),
                            self._s(stream))
        return dX

    def bwd_dm(self, mid, X, dY, stream=None):
        _, H, O = self.dims[mid]
        roast_linear_bwd_dm(self.h, mid, X.data_ptr(), dY.data_ptr(), X.numel() // H, self._dt(X),
                            self._s(stream))

    def emb_fwd(self, mid, idx, out=None, stream=None):
        _, rows, dim, chunk = self.dims[mid]
        if out is None:
            out = self.torch.empty(idx.numel(), dim, dtype=self.torch.float32, device=idx.device)
        roast_embedding_fwd(self.h, mid, idx.data_ptr(), idx.numel(), out.data_ptr(), self._s(stream))
        return out

    def emb_bwd(self, mid, idx, dout, stream=None):
        roast_embedding_bwd(self.h, mid, idx.data_ptr(), idx.numel(), dout.data_ptr(), self._s(stream))

    def emb_fwd_multi(self, mids, idx, out=None, stream=None):
        """idx: ntables x n (table-major); returns (ntables n) x dim."""
        _, rows, dim, chunk = self.dims[mids[0]]
        n = idx.numel() // len(mids)
        if out is None:
            out = self.torch.empty(idx.numel(), dim, dtype=self.torch.float32, device=idx.device)
        roast_embedding_fwd_multi(self.h, list(mids), idx.data_ptr(), n, out.data_ptr(), self._s(stream))
        return out

    def emb_bwd_multi(self, mids, idx, dout, stream=None):
        roast_embedding_bwd_multi(self.h, list(mids), idx.data_ptr(), idx.numel() // len(mids), dout.data_ptr(),
                                  self._s(stream))

    def zero_grad(self, stream=None):
        roast_zero_grad(self.h, self._s(stream))
        if self._bias_pending:            # collected-but-unscattered bias gradients are discarded too
            with self.torch.cuda.stream(self._stream_obj(stream)):
                for _, _, grads, _, _ in self._groups():
                    grads.zero_()
            self._bias_pending = False

    def sync_shadow(self, stream=None):
        roast_sync_shadow(self.h, self._s(stream))
        self._gen += 1

    def sgd(self, lr, stream=None):
        self.flush_bias_grads(stream)
        roast_sgd_step(self.h, lr, self._s(stream))
        self._gen += 1

    def optimizer_step(self, kind, lr, step=1, stream=None, **kw):
        self.flush_bias_grads(stream)
        roast_optimizer_step(self.h, kind, lr, step, stream=self._s(stream), **kw)
        self._gen += 1

    def exchange_step(self, kind, lr, step=1, stream=None, **kw):
        self.flush_bias_grads(stream)
        roast_grad_exchange_step(self.h, kind, lr, step, stream=self._s(stream), **kw)
        self._gen += 1

    # ---- one-shot P2P exchange fused with the update (include/roast.h, p2p.cu)
    def p2p_window(self):
        return roast_p2p_window(self.h)

    def p2p_init(self, group=None):
        """Map every rank's exchange window (CUDA IPC; handles exchanged with
        torch.distributed all_gather_object on `group`).  World 1: this rank alone."""
        import torch.distributed as dist
        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
            w, _ = roast_p2p_window(self.h)
            roast_p2p_attach(self.h, 0, 1, [w])
            return
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        mine = roast_p2p_ipc_handle(self.h)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        roast_p2p_open(self.h, rank, world, b"".join(allh))

    def exchange_init(self, group=None, prefer="auto"):
        """Set up the fused exchange + update path (include/roast.h: NVLS, p2p).  NVLS when every
        rank's device reports switch multicast and every driver step succeeds (NVSwitch systems),
        else the CUDA-IPC P2P window (p2p_init).  prefer: "auto" | "nvls" (raise instead of
        falling back) | "p2p".  Returns and records (self.exchange_path) "nvls" or "p2p"; the
        reason for a fallback is kept in self.exchange_fallback."""
        self.exchange_fallback = None
        if prefer != "p2p":
            try:
                self._nvls_init(group)
                self.exchange_path = "nvls"
                return "nvls"
            except (RoastError, OSError) as e:
                if prefer == "nvls":
                    raise
                self.exchange_fallback = repr(e)
                roast_nvls_reset(self.h)
        self.p2p_init(group)
        self.exchange_path = "p2p"
        return "p2p"

    def _nvls_init(self, group):
        """Every rank in the same order: probe, create (rank 0) / import (fd over a unix socket),
        add device, bind; a failure on any rank makes every rank raise (all_gather of the status
        after each step), so all fall back together."""
        import socket
        import uuid
        torch = self.torch
        import torch.distributed as dist
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        rank = dist.get_rank(group) if multi else 0
        world = dist.get_world_size(group) if multi else 1

        def agree(ok, what):
            oks = [None] * world
            if multi:
                dist.all_gather_object(oks, ok, group=group)
            else:
                oks = [ok]
            if not all(o is True for o in oks):
                bad = [f"rank {r}: {o}" for r, o in enumerate(oks) if o is not True]
                raise RoastError(9, f"nvls {what} ({'; '.join(bad)})")

        def attempt(fn):
            try:
                fn()
                return True
            except (RoastError, OSError) as e:
                return repr(e)

        sup = roast_nvls_supported(self.M.device.index or 0)
        agree(True if sup else "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0", "probe")
        fd_box = [-1]
        agree(attempt(lambda: fd_box.__setitem__(0, roast_nvls_create(self.h, world))) if rank == 0 else True,
              "create")
        try:
            if multi:   # the descriptor travels over an abstract unix socket (SCM_RIGHTS)
                name = [("\0roast-nvls-" + uuid.uuid4().hex) if rank == 0 else None]
                dist.broadcast_object_list(name, src=0, group=group)
                if rank == 0:
                    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
                    srv.bind(name[0])
                    srv.listen(world)
                    dist.barrier(group=group)
                    for _ in range(world - 1):
                        conn, _ = srv.accept()
                        socket.send_fds(conn, [b"f"], [fd_box[0]])
                        conn.close()
                    srv.close()
                    ok = True
                else:
                    dist.barrier(group=group)
                    cl = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
                    cl.connect(name[0])
                    _, fds, _, _ = socket.recv_fds(cl, 1, 1)
                    cl.close()
                    ok = attempt(lambda: roast_nvls_import(self.h, world, fds[0]))
                    os.close(fds[0])
                agree(ok, "import")
        finally:
            if fd_box[0] >= 0:
                os.close(fd_box[0])
        agree(attempt(lambda: roast_nvls_add_device(self.h)), "add_device")
        agree(attempt(lambda: roast_nvls_bind(self.h, rank)), "bind")
        if multi:
            dist.barrier(group=group)

    def exchange_fused(self, kind, lr, step=1, stream=None, **kw):
        """The set-up path's two-shot exchange + update (NVLS or P2P; M stays replicated bit for
        bit on both): dM summed over the ranks, optimizer, shadow refresh, dM zeroed."""
        self.exchange_p2p2(kind, lr, step, stream=stream, **kw)

    def p2p_attach(self, rank, windows):
        roast_p2p_attach(self.h, rank, len(windows), windows)

    def p2p_post(self, stream=None):
        self.flush_bias_grads(stream)
        roast_p2p_post(self.h, self._s(stream))

    def p2p_finish(self, kind, lr, step=1, stream=None, **kw):
        roast_p2p_finish(self.h, kind, lr, step, stream=self._s(stream), **kw)
        self._gen += 1

    def exchange_p2p(self, kind, lr, step=1, stream=None, **kw):
        self.flush_bias_grads(stream)
        roast_grad_exchange_p2p(self.h, kind, lr, step, stream=self._s(stream), **kw)
        self._gen += 1

    def p2p_reduce(self, kind, lr, step=1, stream=None, **kw):
        roast_p2p_reduce(self.h, kind, lr, step, stream=self._s(stream), **kw)

    def p2p_gather(self, stream=None):
        roast_p2p_gather(self.h, self._s(stream))
        self._gen += 1

    def exchange_p2p2(self, kind, lr, step=1, stream=None, **kw):
        self.flush_bias_grads(stream)
        roast_grad_exchange_p2p2(self.h, kind, lr, step, stream=self._s(stream), **kw)
        self._gen += 1

    def allreduce(self, stream=None):
        self.flush_bias_grads(stream)
        roast_grad_allreduce(self.h, self._s(stream))

    def set_exchange(self, mode):
        roast_set_exchange(self.h, mode)

    def touched_size(self):
        return roast_touched_size(self.h)

    def tile_map(self, mid):
        import numpy as np
        _, H, O = self.dims[mid]
        n = (H // self.z1) * (O // self.z2)
        off = np.zeros(n, dtype=np.int64)
        sgn = np.zeros(n, dtype=np.int8)
        roast_debug_tile_map(self.h, mid, off.ctypes.data, sgn.ctypes.data)
        return off.reshape(H // self.z1, O // self.z2), sgn.reshape(H // self.z1, O // self.z2)

    def chunk_map(self, mid, rows):
        _, nrows, dim, chunk = self.dims[mid]
        q = -(-dim // chunk)
        off = self.torch.empty(rows.numel(), q, dtype=self.torch.int64, device=rows.device)
        sgn = self.torch.empty(rows.numel(), q, dtype=self.torch.int8, device=rows.device)
        roast_debug_chunk_map(self.h, mid, rows.data_ptr(), rows.numel(), off.data_ptr(), sgn.data_ptr(),
                              self._s())
        return off, sgn

    def materialize(self, mid, dtype):
        _, H, O = self.dims[mid]
        W = self.torch.empty(H, O, dtype=dtype, device=self.M.device)
        roast_debug_materialize(self.h, mid, self._dt(W), W.data_ptr(), self._s())
        return W

    def check(self):
        _check(roast_get_error(self.h), "roast_get_error")

    def opt_state(self, which):
        """Host copy (numpy fp32) of optimizer state array `which` (0: Adagrad G / Adam m; 1: Adam v)."""
        import numpy as np
        out = np.empty(self.mem_size, dtype=np.float32)
        _check(_lib.roast_debug_opt_state(self.h, int(which), out.ctypes.data), "roast_debug_opt_state")
        return out

    def launch_count(self):
        return roast_launch_count(self.h)
