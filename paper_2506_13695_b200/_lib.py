"""ctypes binding of liborx.so (include/orx.h).

The library is built in-tree (``paper_2506_13695_b200/liborx.so``) by
``__graft_entry__.build()`` / ``make -C paper_2506_13695_b200/csrc``. There is
no fallback: if the library is missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ORX_LIB_PATH: an alternative in-tree build (A/B timing of two library versions)
LIB_PATH = os.environ.get("ORX_LIB_PATH") or os.path.join(_HERE, "liborx.so")

ORX_OK, ORX_EINVAL, ORX_ERUNTIME, ORX_ECUDA = 0, -1, -2, -3
PRECISION = {"fp32": 0, "bf16": 1}


class orx_config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_layers", "d_model", "ffn_hidden", "n_heads", "moe_enabled", "n_experts", "experts_active",
        "moe_location", "expert_round_multiple", "n_code_layers", "codebook_size", "short_len",
        "positive_len", "lifelong_len", "n_queries", "lifelong_blocks", "vid_vocab", "aid_vocab",
        "uid_vocab", "gender_vocab", "age_vocab", "n_label_flags", "use_sid_history",
        "vid_only_features", "compress_threshold")] + [("moe_bias_update", C.c_double), ("seed", C.c_uint64)]


class orx_records(C.Structure):
    _fields_ = [
        ("offsets", C.POINTER(C.c_int64)), ("vid", C.POINTER(C.c_int64)), ("aid", C.POINTER(C.c_int32)),
        ("tag", C.POINTER(C.c_double)), ("ts", C.POINTER(C.c_double)), ("playtime", C.POINTER(C.c_double)),
        ("duration", C.POINTER(C.c_double)), ("labels", C.POINTER(C.c_uint32)), ("sid", C.POINTER(C.c_int32)),
    ]


class orx_user_batch(C.Structure):
    _fields_ = [
        ("n_users", C.c_int32), ("uid", C.POINTER(C.c_int32)), ("gender", C.POINTER(C.c_int32)),
        ("age_bucket", C.POINTER(C.c_int32)), ("short_seq", orx_records), ("positive_seq", orx_records),
        ("lifelong_seq", orx_records),
    ]


class orx_beam_out(C.Structure):
    _fields_ = [("codes", C.POINTER(C.c_int32)), ("log_prob", C.POINTER(C.c_double)),
                ("n_items", C.POINTER(C.c_int32))]


class orx_trie(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("child_off", C.POINTER(C.c_int32)), ("n_edges", C.c_int64),
                ("child_code", C.POINTER(C.c_int32)), ("child_node", C.POINTER(C.c_int32))]


class orx_records_out(C.Structure):
    _fields_ = [("offsets", C.POINTER(C.c_int64)), ("vid", C.POINTER(C.c_int64)), ("aid", C.POINTER(C.c_int32)),
                ("tag", C.POINTER(C.c_double)), ("ts", C.POINTER(C.c_double)), ("playtime", C.POINTER(C.c_double)),
                ("duration", C.POINTER(C.c_double)), ("labels", C.POINTER(C.c_uint32)), ("sid", C.POINTER(C.c_int32))]


class orx_gemm_args(C.Structure):
    _fields_ = [
        ("A", C.c_void_p), ("lda", C.c_int32), ("B", C.c_void_p), ("ldb", C.c_int32),
        ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32), ("precision", C.c_int32),
        ("bias", C.c_void_p), ("row_scale", C.c_void_p), ("resid", C.c_void_p), ("ld_resid", C.c_int32),
        ("row_map", C.c_void_p), ("out", C.c_void_p), ("ldo", C.c_int32), ("out_bf16", C.c_int32),
        ("act", C.c_int32), ("swiglu", C.c_int32), ("n_out", C.c_int32), ("m_valid", C.c_int32),
        ("col_off", C.c_int32), ("tile_expert", C.c_void_p), ("n_mtiles", C.c_void_p),
        ("b_rows_per_expert", C.c_int32), ("n_groups", C.c_int32), ("tile_rows", C.c_int32),
        ("force_single_cta", C.c_int32),
    ]


class orx_attn_args(C.Structure):
    _fields_ = [
        ("B", C.c_int32), ("max_q", C.c_int32), ("heads", C.c_int32), ("dh", C.c_int32),
        ("Q", C.c_void_p), ("q_rows", C.c_int64), ("ldq", C.c_int32), ("q_col0", C.c_int32),
        ("K", C.c_void_p), ("k_rows", C.c_int64), ("ldk", C.c_int32), ("k_col0", C.c_int32),
        ("V", C.c_void_p), ("ldv", C.c_int32), ("v_col0", C.c_int32),
        ("Vt", C.c_void_p), ("vt_rows", C.c_int64), ("vt_cols", C.c_int64), ("vt_ld", C.c_int32),
        ("vt_user", C.c_void_p), ("O", C.c_void_p), ("ldo", C.c_int32),
        ("q_start", C.c_void_p), ("q_len", C.c_void_p), ("k_start", C.c_void_p), ("k_len", C.c_void_p),
        ("o_start", C.c_void_p), ("q_stride", C.c_int32), ("q_fixed", C.c_int32), ("k_stride", C.c_int32),
        ("k_fixed", C.c_int32), ("o_stride", C.c_int32), ("kernel", C.c_int32),
    ]


# (name, restype, argtypes) for every function declared in include/orx.h
_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_F32P = C.POINTER(C.c_float)
SIGNATURES = [
    ("orx_last_error", C.c_char_p, []),
    ("orx_version", C.c_char_p, []),
    ("orx_config_default", C.c_int, [C.POINTER(orx_config)]),
    ("orx_config_preset", C.c_int, [C.c_char_p, C.POINTER(orx_config)]),
    ("orx_config_enc_seq_len", C.c_int64, [C.POINTER(orx_config)]),
    ("orx_config_expert_hidden", C.c_int64, [C.POINTER(orx_config)]),
    ("orx_weights_create_random", C.c_int, [C.POINTER(orx_config), C.POINTER(_P)]),
    ("orx_weights_create_random_ep", C.c_int, [C.POINTER(orx_config), C.c_int32, C.c_int32, C.POINTER(_P)]),
    ("orx_weights_create_random_ep_placed", C.c_int, [C.POINTER(orx_config), C.c_int32, C.c_int32, _I32P,
                                                      C.POINTER(_P)]),
    ("orx_config_moe_layers", C.c_int32, [C.POINTER(orx_config)]),
    ("orx_weights_load_grcp", C.c_int, [C.c_char_p, C.POINTER(_P)]),
    ("orx_weights_save_grcp", C.c_int, [_P, C.c_char_p]),
    ("orx_weights_config", C.c_int, [_P, C.POINTER(orx_config)]),
    ("orx_weights_count", C.c_int64, [_P]),
    ("orx_weights_entry", C.c_int, [_P, C.c_int64, C.POINTER(C.c_char_p), _I32P, _I32P,
                                    C.POINTER(_F32P)]),
    ("orx_weights_find", C.c_int, [_P, C.c_char_p, C.POINTER(C.c_int64)]),
    ("orx_weights_set", C.c_int, [_P, C.c_char_p, C.POINTER(C.c_float), C.c_int64]),
    ("orx_weights_destroy", None, [_P]),
    ("orx_validate_batch", C.c_int, [C.POINTER(orx_config), C.POINTER(orx_user_batch)]),
    ("orx_engine_create", C.c_int, [_P, C.c_int, C.c_int, C.c_int32, C.c_int32, C.POINTER(_P)]),
    ("orx_engine_destroy", None, [_P]),
    ("orx_ep_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("orx_engine_create_ep", C.c_int, [_P, C.c_int, C.c_int, C.c_int32, C.c_int32, C.POINTER(C.c_uint8), C.c_int32,
                                       C.c_int32, C.POINTER(_P)]),
    ("orx_engine_create_ep_placed", C.c_int, [_P, C.c_int, C.c_int, C.c_int32, C.c_int32, C.POINTER(C.c_uint8),
                                              C.c_int32, C.c_int32, _I32P, C.POINTER(_P)]),
    ("orx_engine_expert_load", C.c_int, [_P, C.POINTER(C.c_int64), C.c_int32]),
    ("orx_ep_place", C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _I32P,
                               C.POINTER(C.c_double)]),
    ("orx_encode", C.c_int, [_P, C.POINTER(orx_user_batch), _F32P]),
    ("orx_next_logits", C.c_int, [_P, _F32P, C.c_int32, C.c_int32, _I32P, _I32P, _I32P, _F32P]),
    ("orx_score_prefixes", C.c_int, [_P, C.POINTER(orx_user_batch), C.c_int32, _I32P, _I32P, _I32P, _F32P]),
    ("orx_beam_search", C.c_int, [_P, C.POINTER(orx_user_batch), C.c_int32, C.POINTER(orx_beam_out)]),
    ("orx_beam_search_submit", C.c_int, [_P, C.POINTER(orx_user_batch), C.c_int32]),
    ("orx_beam_search_collect", C.c_int, [_P, C.POINTER(orx_beam_out)]),
    ("orx_engine_set_trie", C.c_int, [_P, C.POINTER(orx_trie)]),
    ("orx_beam_search_constrained", C.c_int, [_P, C.POINTER(orx_user_batch), C.c_int32, C.POINTER(orx_beam_out)]),
    ("orx_sequence_log_prob", C.c_int, [_P, C.POINTER(orx_user_batch), C.c_int32, _I32P, _I32P,
                                        C.POINTER(C.c_double)]),
    ("orx_sample", C.c_int, [_P, C.POINTER(orx_user_batch), C.c_int32, C.c_double, C.c_int32, C.c_double,
                             C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(orx_beam_out)]),
    ("orx_engine_stage_batch", C.c_int, [_P, C.POINTER(orx_user_batch)]),
    ("orx_beam_search_staged", C.c_int, [_P, C.c_int32, C.POINTER(orx_beam_out)]),
    ("orx_engine_stats", C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("orx_engine_stream", _P, [_P]),
    ("orx_profile_enable", C.c_int, [C.c_int]),
    ("orx_profile_read", C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("orx_debug_gemm", C.c_int, [C.POINTER(orx_gemm_args), _P]),
    ("orx_debug_row_topk", C.c_int, [C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P]),
    ("orx_debug_topk_fallback_rows", C.c_int64, []),
    ("orx_debug_moe_route", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _F32P, _F32P, _F32P, C.c_int32,
                                      _I32P, _F32P]),
    ("orx_debug_attention", C.c_int, [C.POINTER(orx_attn_args), _P]),
    ("orx_debug_ep_plan", C.c_int, [C.c_int32, C.c_int32, C.c_int32, _I32P, _I32P, C.c_int32, C.c_int32,
                                    C.c_int32, _I32P, _I32P, _I32P, _I32P, C.POINTER(C.c_int64)]),
    ("orx_compress_lifelong", C.c_int, [C.c_int, C.c_int32, C.POINTER(orx_records), C.POINTER(C.c_double), C.c_int32,
                                        C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint64),
                                        C.POINTER(orx_records_out)]),
    ("orx_synth_batch_create", C.c_int, [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.POINTER(_P)]),
    ("orx_synth_batch_view", C.c_int, [_P, C.POINTER(orx_user_batch)]),
    ("orx_synth_batch_destroy", None, [_P]),
]

_lib = None


def lib():
    """Load liborx.so once; raise (never fall back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                              "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        ab = "ORX_LIB_PATH" in os.environ  # A/B timing against an older build: skip entry points it lacks
        for name, res, args in SIGNATURES:
            if ab and not hasattr(h, name):
                continue
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


class OrxError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map ORX error codes to the reference's exception types."""
    if rc == ORX_OK:
        return
    msg = lib().orx_last_error().decode()
    if rc == ORX_EINVAL:
        raise ValueError(msg)  # std::invalid_argument (GENREC_REQUIRE)
    raise OrxError(msg)  # std::runtime_error / CUDA
