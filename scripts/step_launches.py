"""Decode-step anatomy: wall/event time of one decode step vs the sum of its kernels.

  python scripts/step_launches.py [model] [B] [ctx]          # timing
  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --csv \
      python scripts/step_launches.py ... --ncu                # per-launch durations
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200.device import KvPool, Lane, Model, Slots  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "qwen2.5-0.5b"
B = int(args[1]) if len(args) > 1 else 8
ctx = int(args[2]) if len(args) > 2 else 2048
ncu = "--ncu" in sys.argv
level = int([a for a in sys.argv if a.startswith("--level=")][0].split("=")[1]) if any(
    a.startswith("--level=") for a in sys.argv) else 0
chunk = int([a for a in sys.argv if a.startswith("--chunk=")][0].split("=")[1]) if any(
    a.startswith("--chunk=") for a in sys.argv) else 0  # admitted resume chunk rows per step
m = Model(name, seed=13, max_context=ctx + 256 + 30 * chunk)
kv = KvPool(m, num_blocks=(B + 1) * ((ctx + 30 * chunk + 63) // 64 + 2) + 8)
lane = Lane(m, max_tokens=2048, max_segments=B + 4)
rng = np.random.default_rng(0)
for s in range(B + (1 if chunk else 0)):
    done = 0
    while done < ctx - 1:
        n = min(2048, ctx - 1 - done)
        lane.forward(kv, [(s, n, 0)], rng.integers(0, m.vocab, n))
        done += n
lane.wait()
if level:  # decode on a green-context partition of level*16 SMs, as the AgentServe engine does
    slots = Slots(0, levels=9, granularity=16)
    dstream, _ = slots.bind(level)
    lane.set_stream(dstream)
    lane.set_sms(slots.sm_counts(level)[0])
steps = 2 if ncu else 20
times = []
for i in range(steps):
    toks = rng.integers(0, m.vocab, B)
    if ncu and i == steps - 1:
        torch.cuda.nvtx.range_push("step")
    t0 = time.perf_counter()
    segs = [(s, 1, 1) for s in range(B)] + ([(B, chunk, 1)] if chunk else [])
    toks = np.concatenate([toks, rng.integers(0, m.vocab, chunk)]) if chunk else toks
    lane.forward(kv, segs, toks)
    t1 = time.perf_counter()
    lane.wait()
    t2 = time.perf_counter()
    if ncu and i == steps - 1:
        torch.cuda.nvtx.range_pop()
    times.append((t1 - t0, t2 - t0, lane.last_ms()))
t = np.array(times[3:] if not ncu else times)
lane_sms = slots.sm_counts(level)[0] if level else 148
if "--prof" in sys.argv:  # per-category device time, one CUDA-event pair per launch (no PDL)
    lane.profile(True)
    lane.stats(reset=True)
    for _ in range(5):
        segs = [(s, 1, 1) for s in range(B)] + ([(B, chunk, 1)] if chunk else [])
        lane.forward(kv, segs, rng.integers(0, m.vocab, B + chunk))
        lane.wait()
    st = lane.stats(reset=True)
    lane.profile(False)
    print("  per step:", {k: f"{v[0]/5*1000:.0f}us/{v[2]//5}" for k, v in st.items() if v[2]})
print(f"{name} B={B}+{chunk} ctx={ctx} sms={lane_sms}: host enqueue {1e3*np.median(t[:,0]):.3f} ms, wall {1e3*np.median(t[:,1]):.3f} ms, "
      f"lane event {np.median(t[:,2]):.3f} ms")
