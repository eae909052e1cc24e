"""Per-phase timeline of the persistent decode-step kernel (ASB_MK_TIMELINE=1).

  python scripts/mk_timeline.py [model] [B] [ctx] [--level=L]

Prints, per phase kind (qkv / attn / o / gate_up / down / lm_head), the summed duration over
layers of (latest CTA start of the next phase - latest CTA start of this phase), i.e. the
time from one grid barrier to the next, plus embed and total.
"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

os.environ["ASB_MK_TIMELINE"] = "1"
os.environ["ASB_MEGA"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200._lib import check, lib  # noqa: E402
from paper_2603_10342_b200.device import KvPool, Lane, Model, Slots  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "qwen2.5-0.5b"
B = int(args[1]) if len(args) > 1 else 8
ctx = int(args[2]) if len(args) > 2 else 2048
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
sms = 148
if level:
    slots = Slots(0, levels=9, granularity=16)
    d, _ = slots.bind(level)
    lane.set_stream(d)
    sms = slots.sm_counts(level)[0]
    lane.set_sms(sms)
for _ in range(5):
    lane.forward(kv, [(s, 1, 1) for s in range(B)], rng.integers(0, m.vocab, B))
    lane.wait()
buf = (C.c_ulonglong * (148 * 256))()
check(lib().asb_debug_mk_timeline(lane.h, buf, 148 * 256))
t = np.array(buf[:], dtype=np.float64).reshape(148, 256)[:sms]
ends = t[:, 255]
t = t[:, :255]
K = int((t[0] > 0).sum())
start = t[:, :K].max(axis=0)  # phase k begins for the last CTA
t0 = t[:, 0].min()
kinds = ["qkv", "attn", "o", "gate_up", "down"]
tot = {k: 0.0 for k in kinds + ["lm_head"]}
for k in range(K):
    nxt = start[k + 1] if k + 1 < K else ends.max()
    kind = "lm_head" if k == K - 1 else kinds[k % 5]
    tot[kind] += (nxt - start[k]) / 1000.0
print(f"{name} B={B} ctx={ctx} sms={sms} phases={K}: step {(ends.max() - t0) / 1000.0:.1f} us "
      f"(first phase starts +{(start[0] - t0) / 1000.0:.1f} us; CTA start spread {(t[:, 0].max() - t[:, 0].min()) / 1000.0:.1f} us)")
print("  per kind (us, summed over layers):", {k: round(v, 1) for k, v in tot.items()})
print("  lane event ms:", round(lane.last_ms(), 3))
