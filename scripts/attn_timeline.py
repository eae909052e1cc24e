"""Per-CTA timeline of one decode-attention launch (ASB_ATTN_TIMELINE=1), last layer of a decode
step.  python scripts/attn_timeline.py [model] [B] [ctx] [--level=L]"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

os.environ["ASB_ATTN_TIMELINE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200._lib import check, lib  # noqa: E402
from paper_2603_10342_b200.device import KvPool, Lane, Model, Slots  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "qwen2.5-0.5b"
B = int(args[1]) if len(args) > 1 else 2
ctx = int(args[2]) if len(args) > 2 else 2300
level = int([a for a in sys.argv if a.startswith("--level=")][0].split("=")[1]) if any(
    a.startswith("--level=") for a in sys.argv) else 0
m = Model(name, seed=13, max_context=ctx + 256)
kv = KvPool(m, num_blocks=B * ((ctx + 63) // 64 + 2) + 8)
lane = Lane(m, max_tokens=2048, max_segments=B + 4)
rng = np.random.default_rng(0)
for s in range(B):
    done = 0
    while done < ctx - 1:
        n = min(2048, ctx - 1 - done)
        lane.forward(kv, [(s, n, 0)], rng.integers(0, m.vocab, n))
        done += n
lane.wait()
if level:
    slots = Slots(0, levels=9, granularity=16)
    d, _ = slots.bind(level)
    lane.set_stream(d)
    lane.set_sms(slots.sm_counts(level)[0])
for _ in range(4):
    lane.forward(kv, [(s, 1, 1) for s in range(B)], rng.integers(0, m.vocab, B))
    lane.wait()
buf = (C.c_ulonglong * (1024 * 8))()
check(lib().asb_debug_attn_timeline(lane.h, buf, 1024 * 8))
t = np.array(buf[:], dtype=np.float64).reshape(1024, 8)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["entry", "pdl_wait done", "1st K/V", "consumers done", "partial written", "exit(last/single)"]
print(f"{name} B={B} ctx={ctx} level={level}: {len(t)} CTAs; kernel span {(np.nanmax(np.where(t > 0, t, np.nan)) - t0) / 1e3:.1f} us")
for k, nm in enumerate(names):
    v = t[:, k]
    v = v[v > 0]
    if len(v):
        r = (v - t0) / 1e3
        print(f"  {nm:18s} n={len(v):4d} min {r.min():6.1f}  med {np.median(r):6.1f}  max {r.max():6.1f} us")
