"""Bisect decode attention on a 1-layer model: python scripts/debug_decode.py hq hkv hd B ctx"""
import json, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200.device import KvPool, Lane, Model  # noqa: E402
hq, hkv, hd, B, ctx = map(int, sys.argv[1:6])
spec = json.dumps({"name": "dbg", "layers": 1, "d_model": 256, "n_heads": hq, "n_kv_heads": hkv,
                   "head_dim": hd, "ffn": 256, "vocab": 1024, "tied": True, "qkv_bias": False,
                   "rope_theta": 10000.0, "rms_eps": 1e-5})
m = Model(spec, seed=1, max_context=ctx + 64)
kv = KvPool(m, num_blocks=B * ((ctx + 63) // 64 + 1) + 8)
lane = Lane(m, max_tokens=4096, max_segments=B + 2)
rng = np.random.default_rng(0)
for s in range(B):
    lane.forward(kv, [(s, ctx - 1, 0)], rng.integers(0, 1024, ctx - 1))
lane.wait()
for _ in range(3):
    lane.forward(kv, [(s, 1, 1) for s in range(B)], rng.integers(0, 1024, B))
    lane.wait()
print("ok", lane.last_ms(), flush=True)
