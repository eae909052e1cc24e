"""Thin Python handles over the asb_* device seam (include/agentserve_b200.h).

Model / KvPool / Lane own the C handles; all compute happens in libagentserve_b200.so.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from ._lib import Segment, check, lib


class Model:
    def __init__(self, spec: str = "tiny", seed: int = 13, device: int = 0, max_context: int = 16384):
        h = C.c_void_p()
        check(lib().asb_model_create(spec.encode(), seed, device, max_context, C.byref(h)))
        self.h = h
        out = C.c_void_p()
        check(lib().asb_model_describe(h, C.byref(out)))
        self.info = json.loads(C.string_at(out.value).decode())
        lib().asb_string_free(out)
        self.seed = seed

    @property
    def vocab(self) -> int:
        return self.info["vocab"]

    def close(self):
        if self.h:
            lib().asb_model_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class KvPool:
    def __init__(self, model: Model, num_blocks: int):
        h = C.c_void_p()
        check(lib().asb_kv_create(model.h, num_blocks, C.byref(h)))
        self.h = h
        self.model = model

    def block_table(self, session: int) -> list[int]:
        n = C.c_int()
        check(lib().asb_kv_block_table(self.h, session, None, 0, C.byref(n)))
        buf = (C.c_int32 * max(1, n.value))()
        check(lib().asb_kv_block_table(self.h, session, buf, n.value, C.byref(n)))
        return list(buf[: n.value])

    def length(self, session: int) -> int:
        return lib().asb_kv_length(self.h, session)

    def prefix(self, session: int) -> int:
        return lib().asb_kv_prefix(self.h, session)

    def free_blocks(self) -> int:
        return lib().asb_kv_free_blocks(self.h)

    def begin_write(self, s):
        check(lib().asb_kv_begin_write(self.h, s))

    def commit(self, s, new_prefix):
        check(lib().asb_kv_commit(self.h, s, new_prefix))

    def append(self, s, n):
        check(lib().asb_kv_append(self.h, s, n))

    def require_sealed(self, s):
        check(lib().asb_kv_require_sealed(self.h, s))

    def release(self, s):
        check(lib().asb_kv_release(self.h, s))

    def read_token(self, session: int, pos: int) -> tuple[np.ndarray, np.ndarray]:
        info = self.model.info
        n = info["layers"] * info["n_kv_heads"] * info["head_dim"]
        k = np.zeros(n, dtype=np.uint16)
        v = np.zeros(n, dtype=np.uint16)
        check(lib().asb_kv_read_token(self.h, session, pos,
                                      k.ctypes.data_as(C.POINTER(C.c_uint16)),
                                      v.ctypes.data_as(C.POINTER(C.c_uint16))))
        return k, v

    def close(self):
        if self.h:
            lib().asb_kv_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Lane:
    def __init__(self, model: Model, max_tokens: int = 4096, max_segments: int = 128, stream=None):
        h = C.c_void_p()
        check(lib().asb_lane_create(model.h, max_tokens, max_segments, stream, C.byref(h)))
        self.h = h
        self.model = model

    def forward(self, kv: KvPool, segs: list[tuple[int, int, int]], tokens) -> None:
        arr = (Segment * len(segs))(*[Segment(s, n, w) for (s, n, w) in segs])
        toks = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        check(lib().asb_forward(self.h, kv.h, arr, len(segs),
                                toks.ctypes.data_as(C.POINTER(C.c_int32))))

    def fetch(self, n: int, logits: bool = False):
        ids = np.zeros(max(1, n), dtype=np.int32)
        lg = np.zeros((n, self.model.vocab), dtype=np.float32) if logits else None
        check(lib().asb_lane_fetch(self.h, ids.ctypes.data_as(C.POINTER(C.c_int32)), n,
                                   lg.ctypes.data_as(C.POINTER(C.c_float)) if logits else None))
        return (ids[:n], lg) if logits else ids[:n]

    def wait(self):
        check(lib().asb_lane_wait(self.h))

    def done(self) -> bool:
        return bool(lib().asb_lane_query(self.h))

    def last_ms(self) -> float:
        return float(lib().asb_lane_last_ms(self.h))

    def set_stream(self, stream) -> None:
        check(lib().asb_lane_set_stream(self.h, stream))

    def set_sms(self, sms: int) -> None:
        """SM count the lane sizes its grids for (the partition its stream runs on)."""
        check(lib().asb_lane_set_sms(self.h, sms))

    CATS = ("decode_attn", "prefill_attn", "decode_gemm", "prefill_gemm", "forward", "decode_step")

    def profile(self, on: bool = True) -> None:
        check(lib().asb_lane_profile(self.h, 1 if on else 0))

    def stats(self, reset: bool = True) -> dict:
        """{category: (ms, units, launches)} since the last reset (CUDA-event timed)."""
        out = {}
        for i, name in enumerate(self.CATS):
            ms, u, n = C.c_double(), C.c_double(), C.c_int64()
            check(lib().asb_lane_stats(self.h, i, C.byref(ms), C.byref(u), C.byref(n), 1 if reset else 0))
            out[name] = (ms.value, u.value, n.value)
        return out

    def close(self):
        if self.h:
            lib().asb_lane_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Slots:
    """Green Context SM partitions (asb_slots_*): level l gives decode l*g SMs and prefill the
    complement; level == levels() is the shared full device."""

    def __init__(self, device: int = 0, levels: int = 9, granularity: int = 16):
        h = C.c_void_p()
        check(lib().asb_slots_create(device, levels, granularity, C.byref(h)))
        self.h = h

    def levels(self) -> int:
        return lib().asb_slots_levels(self.h)

    def green(self) -> bool:
        return lib().asb_slots_green(self.h) == 1

    def bind(self, level: int):
        """(decode_stream, prefill_stream) raw cudaStream_t handles of one level."""
        d, p = C.c_void_p(), C.c_void_p()
        check(lib().asb_slots_bind(self.h, level, C.byref(d), C.byref(p)))
        return d.value, p.value

    def sm_counts(self, level: int) -> tuple[int, int]:
        d, p = C.c_int(), C.c_int()
        check(lib().asb_slots_sm_counts(self.h, level, C.byref(d), C.byref(p)))
        return d.value, p.value

    def close(self):
        if self.h:
            lib().asb_slots_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def debug_gemm(x, w, out, tokens, n_out, k, epi, bias=None, resid=None, force_path=-1, splits=0,
               stream=None):
    """Device-pointer GEMM hook for tests (torch tensors' data_ptr())."""
    check(lib().asb_debug_gemm(x, w, bias, resid, out, tokens, n_out, k, epi, force_path, splits,
                               stream))
