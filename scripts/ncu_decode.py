"""Minimal decode-step workload for ncu: Llama-3.1-8B shape, B sessions at ctx tokens,
N decode steps.  python scripts/ncu_decode.py [model] [B] [ctx] [steps]"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200.device import KvPool, Lane, Model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3.1-8b"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
m = Model(name, seed=13, max_context=ctx + 64)
kv = KvPool(m, num_blocks=B * ((ctx + 63) // 64 + 1) + 8)
lane = Lane(m, max_tokens=4096, max_segments=B + 2)
rng = np.random.default_rng(0)
for s in range(B):
    done = 0
    while done < ctx - 1:
        n = min(4096, ctx - 1 - done)
        lane.forward(kv, [(s, n, 0)], rng.integers(0, m.vocab, n))
        done += n
lane.wait()
for _ in range(steps):
    lane.forward(kv, [(s, 1, 1) for s in range(B)], rng.integers(0, m.vocab, B))
    lane.wait()
print("done", lane.last_ms())
