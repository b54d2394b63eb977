"""ctypes binding of the C ABI in include/mesw.h (libmesw.so, built in-tree by build.py).

There is no fallback: if the library is missing, importing the package's GPU
paths raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmesw.so")

MAX_SEGMENTS = 64


class LayerView(C.Structure):
    _fields_ = [("m", C.c_uint32), ("n", C.c_uint32), ("bits", C.c_uint32), ("k", C.c_uint32),
                ("idx_off", C.c_uint64), ("rows_off", C.c_uint64), ("steps_off", C.c_uint64),
                ("codes_off", C.c_uint64), ("codes_len", C.c_uint64)]


class ExpertDev(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("steps", C.c_void_p), ("sal_off", C.c_void_p),
                ("sal_idx", C.c_void_p), ("sal_rows", C.c_void_p)]


class LinearArgs(C.Structure):
    _fields_ = [("x", C.c_void_p), ("B", C.c_int32), ("m", C.c_int32), ("n", C.c_int32),
                ("x_layout", C.c_int32), ("w", C.c_void_p), ("expert_table", C.c_void_p),
                ("code_bits", C.c_int32), ("n_segments", C.c_int32),
                ("seg_begin", C.c_int32 * MAX_SEGMENTS), ("seg_end", C.c_int32 * MAX_SEGMENTS),
                ("seg_slot", C.c_int32 * MAX_SEGMENTS), ("y", C.c_void_p), ("y_bf16", C.c_int32),
                ("ldy", C.c_int32), ("residual", C.c_void_p), ("ld_res", C.c_int32),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_uint64),
                ("counters", C.c_void_p), ("num_ctas", C.c_int32), ("activation", C.c_int32),
                ("x_corr", C.c_void_p), ("x_corr_ld", C.c_int32), ("y_rows", C.c_void_p),
                ("swiglu_I", C.c_int32), ("act", C.c_void_p), ("act_np", C.c_int32), ("act_corr", C.c_void_p),
                ("act_corr_ld", C.c_int32)]


class PrefillArgs(C.Structure):
    _fields_ = [("x", C.c_void_p), ("NP", C.c_int32), ("B", C.c_int32), ("m", C.c_int32), ("n", C.c_int32),
                ("w", C.c_void_p), ("expert_table", C.c_void_p), ("code_bits", C.c_int32),
                ("group_slot", C.c_void_p), ("y", C.c_void_p), ("y_bf16", C.c_int32), ("ldy", C.c_int32),
                ("residual", C.c_void_p), ("ld_res", C.c_int32), ("num_ctas", C.c_int32)]


# (name, restype, argtypes) for every symbol declared in include/mesw.h
_SIGNATURES = [
    ("mesw_abi_version", C.c_int, []),
    ("mesw_me_linear_prefill", C.c_int, [C.POINTER(PrefillArgs), C.c_void_p]),
    ("mesw_pack_x_gather", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_int, C.c_void_p]),
    ("mesw_last_error", C.c_char_p, []),
    ("mesw_device_sm_count", C.c_int, []),
    ("mesw_set_pdl", C.c_int, [C.c_int]),
    ("mesw_parse_header", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]),
    ("mesw_parse_layers", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(LayerView)]),
    ("mesw_packed_nbytes", C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32]),
    ("mesw_layer_block_nbytes", C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    ("mesw_device_code_bits", C.c_int, [C.c_uint32]),
    ("mesw_codes_device_bytes", C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32]),
    ("mesw_weight_device_bytes", C.c_uint64, [C.c_uint32, C.c_uint32]),
    ("mesw_repack_codes", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32,
                                    C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]),
    ("mesw_repack_weight", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p,
                                     C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]),
    ("mesw_build_salient_tables", C.c_int, [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.POINTER(C.c_uint64)]),
    ("mesw_unpack_codes_debug", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    ("mesw_dequant_debug", C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                     C.c_void_p]),
    ("mesw_unpack_weight_debug", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_uint32, C.c_void_p, C.c_void_p]),
    ("mesw_pack_x", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_unpack_x", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_linear_workspace_bytes", C.c_uint64, [C.c_int32, C.c_int32]),
    ("mesw_me_linear", C.c_int, [C.POINTER(LinearArgs), C.c_void_p]),
    ("mesw_embed", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_rmsnorm", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_void_p,
                               C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_rope_append", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_float, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_attention_workspace_bytes", C.c_uint64, [C.c_int, C.c_int, C.c_int]),
    ("mesw_attention_decode", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                        C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_attention_decode_rope", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                             C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_void_p, C.c_int,
                                             C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_swiglu", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                              C.c_void_p, C.c_int, C.c_void_p]),
    ("mesw_argmax", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    ("mesw_compress_workspace_bytes", C.c_uint64, [C.c_uint32, C.c_uint32]),
    ("mesw_compress_layer", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                      C.c_void_p]),
    ("mesw_ste_reconstruct", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mesw_ste_step_grad", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mesw_adam_step", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_float, C.c_void_p]),
    ("mesw_quantize_pack", C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    ("mesw_router_classify", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mesw_advance_positions", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]),
]

SYMBOLS = [s[0] for s in _SIGNATURES]

_lib = None


def lib():
    """Load libmesw.so (once).  Raises RuntimeError if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library not built: {LIB_PATH} missing (run `python build.py`)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_STATUS_EXC = {
    1: errors.BadMagicError,
    2: errors.UnsupportedVersionError,
    3: errors.TruncatedArtifactError,
    4: ValueError,
    5: RuntimeError,
    6: NotImplementedError,
    7: IndexError,
}


def check(status: int) -> None:
    """Map a mesw_status to the reference's exception taxonomy (errors.py:19-56)."""
    if status == 0:
        return
    msg = lib().mesw_last_error().decode("utf-8", "replace")
    raise _STATUS_EXC.get(status, RuntimeError)(msg)
