"""Pins the oracle's splitmix64 named sub-stream restatement (oracle/forward.c) against
golden vectors generated from the REFERENCE's own rng.hpp (tests/golden/make_rng_golden.py).
Weights and synthetic token ids of both the oracle and the device path come from it."""
import json
from pathlib import Path

import ctypes as C

from oracle.forward import lib, token_stream

GOLD = json.loads((Path(__file__).parent / "golden" / "rng_golden.json").read_text())


def test_u64_streams_match_reference_rng():
    L = lib()
    for g in GOLD:
        st = C.c_uint64(L.fo_substream(g["seed"], g["name"].encode()))
        got = [L.fo_next_u64(C.byref(st)) for _ in range(len(g["u64"]))]
        assert got == g["u64"], g["name"]


def test_uniform_int_matches_reference_rng():
    for g in GOLD:
        assert list(token_stream(g["seed"], g["name"], 6, 151936)) == g["below_151936"]


def test_weight_generator_is_bf16_uniform():
    from oracle.forward import weight_bits, bf16_to_f32
    import numpy as np
    bits = np.array([weight_bits(13, "L0/q", i, 0.0, 0.034641016) for i in range(4096)], dtype=np.uint16)
    v = bf16_to_f32(bits)
    assert np.abs(v).max() <= 0.0347
    assert 0.017 < v.std() < 0.023
    norm = np.array([weight_bits(13, "L0/attn_norm", i, 1.0, 0.1) for i in range(512)], dtype=np.uint16)
    nv = bf16_to_f32(norm)
    assert 0.89 < nv.min() and nv.max() < 1.11
