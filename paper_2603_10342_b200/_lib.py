"""ctypes binding of libagentserve_b200.so (the C ABI declared in include/*.h).

The product path has no Python fallback: if the shared library is missing or fails to
load this module raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libagentserve_b200.so"


class AsbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "ok", 1: "invalid_argument", 2: "validation_error", 3: "protocol_error",
           4: "io_error", 5: "no_data", 6: "infeasible", 7: "cuda_error"}


class Segment(C.Structure):
    _fields_ = [("session", C.c_uint32), ("n_tokens", C.c_int32), ("want_logits", C.c_int32)]


_lib = None

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I = C.c_int
U32 = C.c_uint32
U64 = C.c_uint64
I64 = C.c_int64
CP = C.c_char_p
I32P = C.POINTER(C.c_int32)
U32P = C.POINTER(C.c_uint32)
U16P = C.POINTER(C.c_uint16)
FP = C.POINTER(C.c_float)

# name: (restype, argtypes)
SIGNATURES = {
    # ---- agentserve_b200.h (device seam)
    "asb_last_error": (CP, []),
    "asb_status_name": (CP, [I]),
    "asb_string_free": (None, [P]),
    "asb_build_info": (CP, []),
    "asb_model_create": (I, [CP, U64, I, I, PP]),
    "asb_model_describe": (I, [P, C.POINTER(C.c_void_p)]),
    "asb_model_free": (None, [P]),
    "asb_kv_create": (I, [P, I, PP]),
    "asb_kv_free": (None, [P]),
    "asb_kv_block_tokens": (I, []),
    "asb_kv_free_blocks": (I, [P]),
    "asb_kv_begin_write": (I, [P, U32]),
    "asb_kv_commit": (I, [P, U32, I]),
    "asb_kv_append": (I, [P, U32, I]),
    "asb_kv_require_sealed": (I, [P, U32]),
    "asb_kv_sealed": (I, [P, U32]),
    "asb_kv_prefix": (I, [P, U32]),
    "asb_kv_length": (I, [P, U32]),
    "asb_kv_block_table": (I, [P, U32, I32P, I, C.POINTER(C.c_int)]),
    "asb_kv_release": (I, [P, U32]),
    "asb_kv_read_token": (I, [P, U32, I, U16P, U16P]),
    "asb_lane_create": (I, [P, I, I, P, PP]),
    "asb_lane_free": (None, [P]),
    "asb_lane_set_stream": (I, [P, P]),
    "asb_lane_stream": (P, [P]),
    "asb_lane_query": (I, [P]),
    "asb_lane_wait": (I, [P]),
    "asb_lane_last_ms": (C.c_float, [P]),
    "asb_forward": (I, [P, P, C.POINTER(Segment), I, I32P]),
    "asb_lane_fetch": (I, [P, I32P, I, FP]),
    "asb_prefill_launch": (I, [P, P, U32, I32P, I]),
    "asb_decode_launch": (I, [P, P, U32P, I32P, I, I64, I32P, I]),
    "asb_slots_create": (I, [I, I, I, PP]),
    "asb_slots_free": (None, [P]),
    "asb_slots_levels": (I, [P]),
    "asb_slots_green": (I, [P]),
    "asb_slots_bind": (I, [P, I, PP, PP]),
    "asb_slots_sm_counts": (I, [P, I, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "asb_debug_gemm": (I, [P, P, P, P, P, I, I, I, I, I, I, P]),
    "asb_debug_gemm_bench": (I, [P, P, P, I, I, I, I, I, I, I, P, FP]),
    "asb_lane_profile": (I, [P, I]),
    "asb_lane_stats": (I, [P, I, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64), I]),
    "asb_lane_set_sms": (I, [P, I]),
    "asb_debug_attn_timeline": (I, [P, C.POINTER(C.c_ulonglong), I]),
    "asb_lane_counters": (I, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64), I]),
}


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2603_10342_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().asb_last_error()
        raise AsbError(status, msg.decode() if msg else "")


def exported_symbols() -> list[str]:
    """Names from SIGNATURES that the loaded library actually exports."""
    L = lib()
    return [n for n in SIGNATURES if getattr(L, n, None) is not None]
