"""ctypes wrapper of the CPU fp32 forward oracle (oracle/forward.c). TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libforward_oracle.so"


class Spec(C.Structure):
    _fields_ = [("layers", C.c_int), ("d", C.c_int), ("hq", C.c_int), ("hkv", C.c_int),
                ("hd", C.c_int), ("ffn", C.c_int), ("vocab", C.c_int), ("tied", C.c_int),
                ("qkv_bias", C.c_int), ("theta", C.c_double), ("eps", C.c_float),
                ("rope_llama3", C.c_int), ("rope_factor", C.c_double), ("rope_lo", C.c_double),
                ("rope_hi", C.c_double), ("rope_orig", C.c_double)]


_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE), "forward"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.fo_create.restype = C.c_void_p
        L.fo_create.argtypes = [C.POINTER(Spec), C.c_uint64, C.c_int, C.c_int]
        L.fo_free.argtypes = [C.c_void_p]
        L.fo_weight_bits.restype = C.c_uint16
        L.fo_weight_bits.argtypes = [C.c_uint64, C.c_char_p, C.c_int64, C.c_float, C.c_float]
        L.fo_tensor.restype = C.POINTER(C.c_float)
        L.fo_tensor.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.POINTER(C.c_int64)]
        L.fo_session_new.restype = C.c_void_p
        L.fo_session_new.argtypes = [C.c_void_p]
        L.fo_session_free.argtypes = [C.c_void_p]
        L.fo_session_len.restype = C.c_int
        L.fo_session_len.argtypes = [C.c_void_p]
        L.fo_forward.restype = C.c_int
        L.fo_forward.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_int,
                                 C.POINTER(C.c_float)]
        L.fo_read_kv.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_uint16),
                                 C.POINTER(C.c_uint16)]
        L.fo_substream.restype = C.c_uint64
        L.fo_substream.argtypes = [C.c_uint64, C.c_char_p]
        L.fo_next_u64.restype = C.c_uint64
        L.fo_next_u64.argtypes = [C.POINTER(C.c_uint64)]
        L.fo_uniform_int.restype = C.c_uint64
        L.fo_uniform_int.argtypes = [C.POINTER(C.c_uint64), C.c_uint64]
        _lib = L
    return _lib


# Model presets — must match paper_2603_10342_b200/csrc/runtime.cu spec_preset().
PRESETS = {
    "tiny": dict(layers=2, d=256, hq=4, hkv=2, hd=64, ffn=704, vocab=4096, tied=1, qkv_bias=0,
                 theta=10000.0, eps=1e-6),
    "qwen2.5-0.5b": dict(layers=24, d=896, hq=14, hkv=2, hd=64, ffn=4864, vocab=151936, tied=1,
                         qkv_bias=1, theta=1e6, eps=1e-6),
    "llama3.2-3b": dict(layers=28, d=3072, hq=24, hkv=8, hd=128, ffn=8192, vocab=128256, tied=1,
                        qkv_bias=0, theta=5e5, eps=1e-5, rope_llama3=1, rope_factor=32.0,
                        rope_lo=1.0, rope_hi=4.0, rope_orig=8192.0),
    "qwen2.5-7b": dict(layers=28, d=3584, hq=28, hkv=4, hd=128, ffn=18944, vocab=152064, tied=0,
                       qkv_bias=1, theta=1e6, eps=1e-6),
    "llama3.1-8b": dict(layers=32, d=4096, hq=32, hkv=8, hd=128, ffn=14336, vocab=128256, tied=0,
                        qkv_bias=0, theta=5e5, eps=1e-5, rope_llama3=1, rope_factor=8.0,
                        rope_lo=1.0, rope_hi=4.0, rope_orig=8192.0),
}


def make_spec(name_or_dict) -> Spec:
    d = dict(PRESETS[name_or_dict]) if isinstance(name_or_dict, str) else dict(name_or_dict)
    s = Spec()
    s.rope_llama3 = 0
    s.rope_factor, s.rope_lo, s.rope_hi, s.rope_orig = 1.0, 1.0, 4.0, 8192.0
    for k, v in d.items():
        setattr(s, k, v)
    return s


class OracleModel:
    def __init__(self, spec="tiny", seed: int = 13, max_ctx: int = 4096, layers_limit: int = 0):
        self.spec = make_spec(spec)
        self.h = lib().fo_create(C.byref(self.spec), seed, max_ctx, layers_limit)
        self.seed = seed

    def tensor(self, name: str, layer: int = -1) -> np.ndarray:
        """Copy of a generated weight tensor (fp32 holding bf16 values), flat."""
        n = C.c_int64(0)
        ptr = lib().fo_tensor(self.h, layer, name.encode(), C.byref(n))
        if not ptr:
            raise KeyError(name)
        return np.ctypeslib.as_array(ptr, shape=(n.value,)).copy()

    def session(self) -> "OracleSession":
        return OracleSession(self)

    def __del__(self):
        if getattr(self, "h", None):
            lib().fo_free(self.h)
            self.h = None


class OracleSession:
    def __init__(self, model: OracleModel):
        self.m = model
        self.h = lib().fo_session_new(model.h)

    def forward(self, tokens, want_logits: bool = True):
        toks = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        lg = np.zeros(self.m.spec.vocab, dtype=np.float32)
        nxt = lib().fo_forward(self.m.h, self.h, toks.ctypes.data_as(C.POINTER(C.c_int32)),
                               len(toks), lg.ctypes.data_as(C.POINTER(C.c_float)))
        return nxt, lg

    def read_kv(self, pos: int):
        s = self.m.spec
        n = s.layers * s.hkv * s.hd
        k = np.zeros(n, dtype=np.uint16)
        v = np.zeros(n, dtype=np.uint16)
        lib().fo_read_kv(self.m.h, self.h, pos, k.ctypes.data_as(C.POINTER(C.c_uint16)),
                         v.ctypes.data_as(C.POINTER(C.c_uint16)))
        return k, v

    @property
    def length(self) -> int:
        return lib().fo_session_len(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().fo_session_free(self.h)
            self.h = None


def weight_bits(seed: int, name: str, index: int, offset: float, amp: float) -> int:
    return int(lib().fo_weight_bits(seed, name.encode(), index, offset, amp))


def token_stream(seed: int, name: str, n: int, vocab: int) -> np.ndarray:
    """n uniform token ids from Rng::substream(seed, name).uniform_int(vocab) (rng.hpp:47-50)."""
    st = C.c_uint64(lib().fo_substream(seed, name.encode()))
    return np.array([lib().fo_uniform_int(C.byref(st), vocab) for _ in range(n)], dtype=np.int32)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)
