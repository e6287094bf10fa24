"""ctypes declarations for libtlp.so (include/tlp.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TLP_LIB_PATH") or os.path.join(_HERE, "libtlp.so")  # override: A/B timing of builds

TLP_STATUS = {0: "OK", -1: "ERR_ARG", -2: "ERR_SHAPE", -3: "ERR_EMPTY_SEQ",
              -4: "ERR_UNKNOWN_TYPE", -5: "ERR_NONFINITE", -6: "ERR_NAN_LOSS",
              -7: "ERR_NO_LABELS", -8: "ERR_CUDA", -9: "ERR_NCCL", -10: "ERR_STATE",
              -11: "ERR_UNSUPPORTED"}

# Every symbol include/tlp.h declares (checked by tests/test_boundary.py).
EXPORTS = ("tlp_create", "tlp_destroy", "tlp_last_error", "tlp_default_config",
           "tlp_set_token_table", "tlp_set_norm_scales", "tlp_fit_token_table", "tlp_fit_norm_scales", "tlp_num_params", "tlp_set_params",
           "tlp_get_params", "tlp_get_grads", "tlp_get_train_scores", "tlp_set_comm", "tlp_broadcast_state", "tlp_get_unique_id", "tlp_encode",
           "tlp_score", "tlp_train_step", "tlp_compute_grads", "tlp_lambdarank", "tlp_mse", "tlp_topk", "tlp_topk_merge",
           "tlp_search_round", "tlp_dedup", "tlp_topk_score", "tlp_normalize_labels", "tlp_sync", "tlp_launch_count", "tlp_debug_umma",
           "tlp_debug_gemm", "tlp_debug_wgrad", "tlp_ga_set_space", "tlp_ga_num_genes", "tlp_ga_batch_size", "tlp_ga_init",
           "tlp_ga_evolve", "tlp_ga_materialize", "tlp_ga_drop_duplicates", "tlp_ga_round")


class tlp_config(C.Structure):
    _fields_ = [("L", C.c_int), ("E", C.c_int), ("T", C.c_int), ("hidden", C.c_int),
                ("up_dims", C.c_int * 4), ("n_up", C.c_int), ("attn_heads", C.c_int),
                ("n_attn", C.c_int), ("n_res", C.c_int), ("head_dim", C.c_int),
                ("n_tasks", C.c_int), ("precision", C.c_int), ("lr", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("seed", C.c_ulonglong), ("loss", C.c_int), ("attn_mask", C.c_int), ("pos_enc", C.c_int),
                ("backbone", C.c_int)]


class tlp_seq_batch(C.Structure):
    _fields_ = [("seq_off", C.c_void_p), ("prim_type", C.c_void_p), ("arg_off", C.c_void_p),
                ("arg_kind", C.c_void_p), ("arg_num", C.c_void_p), ("arg_name", C.c_void_p),
                ("str_blob", C.c_void_p), ("str_off", C.c_void_p), ("P", C.c_int64),
                ("A", C.c_int64), ("U", C.c_int32)]


class tlp_ga_space(C.Structure):
    _fields_ = [("tmpl", tlp_seq_batch), ("S", C.c_int32), ("knob_off", C.c_void_p),
                ("knob_arg", C.c_void_p), ("knob_grp", C.c_void_p), ("dom_off", C.c_void_p),
                ("dom_num", C.c_void_p), ("dom_name", C.c_void_p), ("id_base", C.c_int32)]


_lib = None


def load() -> C.CDLL:
    """Load libtlp.so; raise loudly if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("libtlp.so not built: run `python -m paper_2211_03578_b200.build` "
                           "(there is no CPU or eager fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "tlp_create": (C.c_int, [C.POINTER(tlp_config), C.c_int, C.POINTER(vp)]),
        "tlp_destroy": (None, [vp]),
        "tlp_last_error": (C.c_char_p, [vp]),
        "tlp_default_config": (None, [C.POINTER(tlp_config)]),
        "tlp_set_token_table": (C.c_int, [vp, vp, vp, i32]),
        "tlp_set_norm_scales": (C.c_int, [vp, vp]),
        "tlp_fit_token_table": (C.c_int, [vp, C.POINTER(tlp_seq_batch), i64]),
        "tlp_fit_norm_scales": (C.c_int, [vp, C.POINTER(tlp_seq_batch), i64, vp, vp]),
        "tlp_num_params": (i64, [vp]),
        "tlp_set_params": (C.c_int, [vp, vp, i64]),
        "tlp_get_params": (C.c_int, [vp, vp, i64]),
        "tlp_get_grads": (C.c_int, [vp, vp, i64]),
        "tlp_get_train_scores": (C.c_int, [vp, vp, i64]),
        "tlp_set_comm": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "tlp_get_unique_id": (C.c_int, [vp]),
        "tlp_broadcast_state": (C.c_int, [vp, C.c_int, vp]),
        "tlp_encode": (C.c_int, [vp, C.POINTER(tlp_seq_batch), i64, vp, vp]),
        "tlp_score": (C.c_int, [vp, vp, i64, vp, vp]),
        "tlp_train_step": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp]),
        "tlp_compute_grads": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp]),
        "tlp_lambdarank": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp, vp]),
        "tlp_topk": (C.c_int, [vp, vp, i32, i32, vp, i32, i32, i64, vp, vp, vp]),
        "tlp_topk_merge": (C.c_int, [vp, vp, vp, i32, i32, i32, vp, vp, vp]),
        "tlp_mse": (C.c_int, [vp, vp, vp, i32, vp, vp, vp]),
        "tlp_search_round": (C.c_int, [vp, C.POINTER(tlp_seq_batch), i64, vp, i32, i32, i32, i64,
                                       i32, vp, vp, vp]),
        "tlp_dedup": (C.c_int, [vp, vp, i64, i32, vp, i32, vp, vp, vp, vp, vp]),
        "tlp_topk_score": (C.c_int, [vp, vp, i32, i32, vp, vp, vp, i32, i32, vp, vp]),
        "tlp_normalize_labels": (C.c_int, [vp, vp, vp, i32, vp, vp]),
        "tlp_sync": (C.c_int, [vp]),
        "tlp_launch_count": (i64, [vp]),
        "tlp_debug_umma": (C.c_int, [vp, vp, vp, i32, i32, i32, vp]),
        "tlp_debug_gemm": (C.c_int, [vp, i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, vp]),
        "tlp_debug_wgrad": (C.c_int, [vp, i64, i64, i64, vp, i64, vp, i64, vp, vp]),
        "tlp_ga_set_space": (C.c_int, [vp, C.POINTER(tlp_ga_space)]),
        "tlp_ga_num_genes": (i32, [vp]),
        "tlp_ga_batch_size": (C.c_int, [vp, i64, vp, vp]),
        "tlp_ga_init": (C.c_int, [vp, i32, C.c_uint64, i32, vp, vp]),
        "tlp_ga_evolve": (C.c_int, [vp, vp, vp, i32, i32, C.c_double, C.c_double, C.c_uint64, i32,
                                    i32, vp, vp]),
        "tlp_ga_materialize": (C.c_int, [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]),
        "tlp_ga_drop_duplicates": (C.c_int, [vp, vp, i32, vp, vp]),
        "tlp_ga_round": (C.c_int, [vp, i32, i32, i32, C.c_double, C.c_double, C.c_uint64, i32, i32,
                                   vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib
