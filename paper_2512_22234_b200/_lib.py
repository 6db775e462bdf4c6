"""ctypes loader for libbdattn.so (the C-ABI library; include/bd_attn.h).

Argument marshalling only.  There is no fallback: if the library is missing
or fails to load, every op raises.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbdattn.so")

BD_OK = 0


class BdProblem(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32),
        ("prompt_len", ctypes.c_int32),
        ("response_len", ctypes.c_int32),
        ("block_size", ctypes.c_int32),
        ("n_q_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("repeat_prompt", ctypes.c_int32),
        ("softmax_scale", ctypes.c_float),
        ("n_copies", ctypes.c_int32),
        ("seq_prompt_len", ctypes.POINTER(ctypes.c_int32)),
        ("seq_response_len", ctypes.POINTER(ctypes.c_int32)),
        ("q_row_heads", ctypes.c_int32),
        ("kv_row_heads", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_F = ctypes.c_float
_PROB = ctypes.POINTER(BdProblem)

# name -> (restype, argtypes); must match include/bd_attn.h
SIGNATURES = {
    "bd_packed_len": (_I64, [_PROB]),
    "bd_attn_workspace_bytes": (_SZ, [_PROB, ctypes.c_int]),
    "bd_attn_fwd": (ctypes.c_int, [_PROB, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "bd_attn_bwd": (ctypes.c_int, [_PROB, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "bd_logprob": (ctypes.c_int, [_I64, _I32, _P, _I64, _P, _P, _P, _P, _P, _I64, _P]),
    "bd_logprob_bwd": (ctypes.c_int, [_I64, _I32, _P, _I64, _P, _P, _P, _P, _I64, _P]),
    "bd_launch_count": (_I64, []),
    "bd_dipo_group_stats":(ctypes.c_int, [_I32, _P, _P, _P, _I32, _P, _P]),
    "bd_dipo_token_loss": (ctypes.c_int, [_I64, _P, _P, _P, _I32, _P, _P, _P, _I32, _I32, _F, _P, _P, _P]),
    "bd_tilemap_dump": (ctypes.c_int, [_PROB, ctypes.POINTER(_I32), _SZ, ctypes.POINTER(_I64)]),
    "bd_tilemap_stats": (ctypes.c_int, [_PROB, ctypes.POINTER(_I64)]),
    "bd_tilemap_entries_bound": (_I64, [_PROB]),
    "bd_tilemap_selfcheck": (ctypes.c_int, [_PROB, ctypes.POINTER(_I64)]),
    "bd_mask_dump": (ctypes.c_int, [_PROB, _I32, _I64, _I64, _P, _SZ, ctypes.POINTER(_I64)]),
    "bd_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "bd_last_error": (ctypes.c_char_p, []),
    "bd_selftest_mma": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "bd_lmhead_workspace_bytes": (_SZ, [_I64, _I32, _I32, ctypes.c_int, _I64]),
    "bd_lmhead_logprob": (ctypes.c_int, [_I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "bd_lmhead_logprob_bwd": (ctypes.c_int, [_I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _SZ, _P]),
    "bd_decode_workspace_bytes": (_SZ, [_I32, _I32, _I32, _I32, _I32, _I32]),
    "bd_decode_attn": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _F, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "bd_decode_select": (ctypes.c_int, [_I32, _I32, _I32, _P, _P, _F, _P, _P, _P, _P]),
    "bd_selftest_gemm": (ctypes.c_int, [_I32, _I32, _I32, _P, ctypes.c_int, _P, ctypes.c_int, _P, _P]),
}

_lib = None


class BdError(RuntimeError):
    pass


def lib():
    """Load the library once; raise (never fall back) if it is unavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BdError(f"{LIB_PATH} not built: run python -m paper_2512_22234_b200.build "
                          "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code, what):
    if code != BD_OK:
        L = lib()
        raise BdError(f"{what} failed: {L.bd_error_string(code).decode()}: {L.bd_last_error().decode()}")
