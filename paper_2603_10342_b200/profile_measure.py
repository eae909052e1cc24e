"""Measured B200 ProfileBundle: the reference's per-phase throughput curves
(`PhaseProfile`, /root/reference/proj/src/profile.cpp:24-39, schema agentsim-profile-v1) measured
with the real kernels on Green Context partitions instead of shaped by hand.

For every slot level l = 1..S/g the forward runs on a partition of l*g SMs (asb_slots decode
stream of that level; the last level is the full device) and we record
  decode_prefill : B decode rows at context `decode_ctx`  -> tokens/s = B / step time
  cold_prefill   : one `cold_len`-token prompt             -> tokens/s = cold_len / forward time
  resume_prefill : `resume_len` tokens appended to a `resume_ctx` context -> tokens/s
exactly the quantities the reference's cost model divides by (decode_step_duration_ms,
executor.cpp:84-97; the prefill rate x length arithmetic, engine.cpp:450-475).  Curves are made
non-decreasing (running max) because the reference validator requires it (profile.cpp:81-128).

    python -m paper_2603_10342_b200.profile_measure --model qwen2.5-0.5b --out profiles/b200_profile_qwen2.5-0.5b.json
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np

from .device import KvPool, Lane, Model, Slots


def _median_ms(lane: Lane, fn, reps: int) -> float:
    ts = []
    for _ in range(reps):
        fn()
        lane.wait()
        ts.append(lane.last_ms())
    return statistics.median(ts)


def measure(model: str = "qwen2.5-0.5b", levels: int = 9, granularity: int = 16, decode_batch: int = 8,
            decode_ctx: int = 2048, cold_len: int = 2048, resume_len: int = 256, resume_ctx: int = 2304,
            reps: int = 5, device: int = 0, seed: int = 13, log=print) -> dict:
    m = Model(model, seed=seed, device=device, max_context=max(decode_ctx + 512, resume_ctx + resume_len + 64,
                                                                 cold_len + 64))
    V = m.vocab
    rng = np.random.default_rng(seed)
    blocks = decode_batch * ((decode_ctx + 64 * levels * (reps + 3)) // 64 + 2) + 2 * ((resume_ctx + resume_len) // 64 + 2) \
        + (cold_len // 64 + 2) + 16
    kv = KvPool(m, num_blocks=blocks)
    chunk = max(2048, cold_len)  # a cold prompt is one forward
    full = Lane(m, max_tokens=chunk, max_segments=max(decode_batch, 8) + 4)

    def prefill(lane: Lane, sid: int, n: int):
        done = 0
        while done < n:
            k = min(chunk, n - done)
            lane.forward(kv, [(sid, k, 1 if done + k == n else 0)], rng.integers(0, V, k))
            done += k

    sessions = list(range(decode_batch))
    for s in sessions:
        prefill(full, s, decode_ctx - 1)
    full.wait()
    slots = Slots(device, levels, granularity)
    S = levels * granularity
    dec, cold, res = [], [], []
    for lvl in range(1, levels + 1):
        sd, _ = slots.bind(lvl)
        dsms, _ = slots.sm_counts(lvl)
        lane = Lane(m, max_tokens=chunk, max_segments=max(decode_batch, 8) + 4, stream=sd)
        lane.set_sms(dsms)
        # decode: B rows, one token each
        step = lambda: lane.forward(kv, [(s, 1, 1) for s in sessions], rng.integers(0, V, decode_batch))
        for _ in range(2):
            step()
        lane.wait()
        d_ms = _median_ms(lane, step, reps)
        # cold prefill
        cid = 1_000_000 + lvl

        def cold_once():
            prefill(lane, cid, cold_len)

        c_ts = []
        for _ in range(reps):
            cold_once()
            lane.wait()
            c_ts.append(lane.last_ms())  # single forward when cold_len <= chunk
            kv.release(cid)
        c_ms = statistics.median(c_ts)
        # resume prefill onto a resume_ctx prefix (prefix built on the full-device lane)
        r_ts = []
        rid = 2_000_000 + lvl
        for _ in range(reps):
            prefill(full, rid, resume_ctx)
            full.wait()
            lane.forward(kv, [(rid, resume_len, 1)], rng.integers(0, V, resume_len))
            lane.wait()
            r_ts.append(lane.last_ms())
            kv.release(rid)
        r_ms = statistics.median(r_ts)
        sms = lvl * granularity
        dec.append([sms, decode_batch * 1000.0 / d_ms])
        cold.append([sms, cold_len * 1000.0 / c_ms])
        res.append([sms, resume_len * 1000.0 / r_ms])
        log(f"level {lvl}: partition {dsms} SMs  decode B={decode_batch} {d_ms:.3f} ms  "
            f"cold {cold_len} {c_ms:.3f} ms  resume {resume_len}@{resume_ctx} {r_ms:.3f} ms")
        lane.close()

    def curve(pts):
        out, run = [], 0.0
        for sms, r in pts:
            run = max(run, r)
            out.append({"sms": sms, "tokens_per_second": round(run, 3)})
        return out

    doc = {"schema": "agentsim-profile-v1", "total_sms": S, "granularity": granularity,
           "decode": curve(dec), "cold_prefill": curve(cold), "resume_prefill": curve(res),
           "measured": {"model": model, "decode_batch": decode_batch, "decode_ctx": decode_ctx,
                        "cold_len": cold_len, "resume_len": resume_len, "resume_ctx": resume_ctx,
                        "reps": reps, "green_contexts": slots.green(),
                        "raw_tokens_per_second": {"decode": dec, "cold_prefill": cold, "resume_prefill": res}}}
    slots.close()
    return doc


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--model", default="qwen2.5-0.5b")
    ap.add_argument("--levels", type=int, default=9)
    ap.add_argument("--granularity", type=int, default=16)
    ap.add_argument("--decode-batch", type=int, default=8)
    ap.add_argument("--decode-ctx", type=int, default=2048)
    ap.add_argument("--cold", type=int, default=2048)
    ap.add_argument("--resume", type=int, default=256)
    ap.add_argument("--resume-ctx", type=int, default=2304)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    doc = measure(a.model, a.levels, a.granularity, a.decode_batch, a.decode_ctx, a.cold, a.resume,
                  a.resume_ctx, a.reps, log=lambda s: print(s, file=sys.stderr, flush=True))
    text = json.dumps(doc, indent=1)
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
