"""ctypes binding of libmoa.so (include/moa.h) -- argument marshalling only.

Every function of the C ABI is exposed under its own name with ctypes
argtypes/restype.  Loading fails loudly (ImportError) when the in-tree
library is missing: there is no CPU or eager fallback anywhere in this
package.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_uint8, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libmoa.so")

MOA_OK, MOA_ERR_INVALID_ARG, MOA_ERR_SHAPE, MOA_ERR_STATE, MOA_ERR_UNSUPPORTED, MOA_ERR_OOM, MOA_ERR_CUDA = range(7)
STATUS_NAMES = {0: "MOA_OK", 1: "MOA_ERR_INVALID_ARG", 2: "MOA_ERR_SHAPE", 3: "MOA_ERR_STATE",
                4: "MOA_ERR_UNSUPPORTED", 5: "MOA_ERR_OOM", 6: "MOA_ERR_CUDA"}
MOA_BF16, MOA_FP32 = 0, 1
MOA_TILE = 128

# (name, restype, argtypes) of every exported symbol of include/moa.h
_P = c_void_p
_SIGS = [
    ("moa_version", c_char_p, []),
    ("moa_last_error", c_char_p, []),
    ("moa_create", c_int, [POINTER(c_void_p), c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int]),
    ("moa_destroy", c_int, [_P]),
    ("moa_resolve_spans", c_int, [POINTER(c_float), POINTER(c_float), c_int, c_int64, c_int, POINTER(c_int32)]),
    ("moa_set_spans", c_int, [_P, c_int, POINTER(c_int32), c_int, c_int64]),
    ("moa_set_spans_blocked", c_int, [_P, c_int, POINTER(c_int32), c_int, c_int64, c_int]),
    ("moa_set_ragged", c_int, [_P, c_int, c_int, POINTER(c_int64), POINTER(c_int32)]),
    ("moa_cache_bytes", c_int, [_P, c_int, POINTER(c_size_t), POINTER(c_size_t)]),
    ("moa_layer_cache_bytes", c_int, [_P, c_int, c_int, POINTER(c_size_t), POINTER(c_size_t)]),
    ("moa_workspace_bytes", c_int, [_P, c_int, POINTER(c_size_t)]),
    ("moa_bind_cache", c_int, [_P, _P, _P, c_int]),
    ("moa_bind_layer_cache", c_int, [_P, c_int, _P, _P, c_int]),
    ("moa_prefill", c_int, [_P, c_int, _P, _P, _P, _P, c_int64, c_int64, c_int64, c_int, c_int64, c_float,
                            _P, _P, c_size_t, _P]),
    ("moa_prefill_attn", c_int, [_P, c_int, _P, _P, _P, _P, c_int64, c_int64, c_int64, c_int, c_int64, c_float,
                                 _P, _P]),
    ("moa_cache_fill", c_int, [_P, c_int, _P, _P, c_int64, c_int, c_int64, _P]),
    ("moa_kv_append", c_int, [_P, c_int, _P, _P, c_int64, c_int, c_int64, _P]),
    ("moa_decode_step", c_int, [_P, c_int, _P, _P, c_int64, c_int64, c_int, c_int64, c_float, _P, _P,
                                c_size_t, _P]),
    ("moa_decode_step_fused", c_int, [_P, c_int, _P, _P, _P, _P, c_int64, c_int64, c_int64, c_int, c_int64,
                                      c_float, _P, _P, c_size_t, _P]),
    ("moa_advance_pos", c_int, [_P, c_int, c_int64, _P]),
    ("moa_prepare_layers", c_int, [_P]),
    ("moa_set_peer_outputs", c_int, [_P, c_int, POINTER(c_void_p), POINTER(c_void_p), c_int64, c_int64, c_int]),
    ("moa_wait_flag", c_int, [_P, ctypes.c_uint, _P]),
    ("moa_decode_step_fused_layers", c_int, [_P, c_int, c_int, _P, _P, _P, _P, c_int64, c_int64, c_int64, c_int64,
                                             c_int64, c_int64, c_int, c_int64, c_float, _P, c_int64, _P, c_size_t,
                                             _P]),
    ("moa_set_decode_split", c_int, [_P, c_int]),
    ("moa_decode_step_fused_ragged", c_int, [_P, c_int, _P, _P, _P, _P, c_int64, c_int64, c_int64, c_int, _P,
                                             c_float, _P, _P, c_size_t, _P]),
    ("moa_get_window", c_int, [_P, c_int, c_int, POINTER(c_int32)]),
    ("moa_get_group_window", c_int, [_P, c_int, c_int, POINTER(c_int32)]),
    ("moa_slot_of", c_int, [_P, c_int, c_int, c_int64, POINTER(c_int64)]),
    ("moa_cache_region", c_int, [_P, c_int, c_int, c_int, POINTER(c_int64), POINTER(c_int64)]),
    ("moa_layer_offset", c_int, [_P, c_int, c_int, POINTER(c_size_t)]),
    ("moa_prefill_tiles", c_int, [_P, c_int, c_int, c_int, POINTER(c_int32), POINTER(c_uint8), c_int,
                                  POINTER(c_int32)]),
    ("moa_prefill_items", c_int, [_P, c_int, POINTER(c_int32), c_int, POINTER(c_int32)]),
    ("moa_prefill_schedule", c_int, [_P, c_int, POINTER(c_int32), c_int, POINTER(c_int32), c_int,
                                     POINTER(c_int32), POINTER(c_int32)]),
    ("moa_decode_chunks", c_int, [_P, c_int, POINTER(c_int32), c_int, POINTER(c_int32)]),
    ("moa_next_pos", c_int, [_P, c_int, POINTER(c_int64)]),
    ("moa_attention_influence", c_int, [_P, _P, _P, _P, c_int, c_int64, c_int, c_int, c_int, c_int64, c_int64,
                                        c_float, c_int, _P, c_int, _P]),
    ("moa_plan_rules", c_int, [POINTER(c_float), POINTER(c_float), c_int, c_int, c_int, c_float, c_int,
                               POINTER(c_int32), POINTER(c_float), POINTER(c_float)]),
    ("moa_rule_losses", c_int, [_P, c_int, c_int64, c_int, c_int, POINTER(c_float), POINTER(c_float), c_int, _P,
                                _P]),
]
EXPORTED = [s[0] for s in _SIGS]


class MoAError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    path = os.environ.get("MOA_LIB", path)  # diagnostic builds (tools/build_trace.py)
    if not os.path.exists(path):
        raise ImportError(
            f"libmoa.so not found at {path}: build it with `python -m paper_2406_14909_b200.build` "
            "(no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    diagnostic = os.path.abspath(path) != os.path.abspath(LIB_PATH)
    for name, res, args in _SIGS:
        if diagnostic and not hasattr(lib, name):
            continue  # an older diagnostic build (tools A/B runs) may lack newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


def check(status: int, where: str):
    if status != MOA_OK:
        raise MoAError(status, where, lib().moa_last_error().decode())
