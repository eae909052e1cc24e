"""Kernel rooflines at BASELINE shapes through the asb_* seam (CUDA events per launch inside
the lane; algorithmic bytes / FLOPs per launch).  Writes one JSON object per case.

  python scripts/kernel_bench.py [--models ...] [--out gpurun_out/kernels.json]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200.device import KvPool, Lane, Model  # noqa: E402

PEAKS = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}

CASES = {
    # model: (prefill lengths, decode (B, ctx) list)
    "qwen2.5-0.5b": ([2048], [(8, 2048)]),
    "llama3.2-3b": ([3000], [(32, 3000)]),
    "qwen2.5-7b": ([8192], [(64, 8192)]),
    "llama3.1-8b": ([3000], [(64, 3000)]),
}


def rate(ms, units, kind):
    if ms <= 0:
        return None
    return units / (ms / 1000.0) / (1e9 if kind == "bytes" else 1e12)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", nargs="*", default=list(CASES))
    ap.add_argument("--out", default="gpurun_out/kernels.json")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--decode", nargs="*", default=None, help="override decode cases, e.g. 16x3000 48x3000")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--prefill", type=int, nargs="*", default=None, help="override prefill lengths")
    ap.add_argument("--level", type=int, default=0,
                    help="run the decode cases on the decode partition of this Green Context slot level")
    a = ap.parse_args()
    results = []
    rng = np.random.default_rng(0)
    for name in a.models:
        pls, dcs = CASES[name]
        if a.decode:
            dcs = [tuple(int(v) for v in c.split("x")) for c in a.decode]
        if a.prefill:
            pls = list(a.prefill)
        if a.no_prefill:
            pls = []
        if a.no_decode:
            dcs = []
        max_ctx = max([p for p in pls] + [c for _, c in dcs]) + 256
        pmax = max(pls + [256])
        m = Model(name, seed=13, max_context=max_ctx)
        V = m.vocab
        nb = sum((c + 63) // 64 + 1 for b, c in dcs for _ in range(b)) + 2 * (pmax // 64 + 2)
        kv = KvPool(m, num_blocks=nb)
        lane = Lane(m, max_tokens=pmax, max_segments=80)
        # prefill
        for L in pls:
            for rep in range(a.reps + 1):
                sid = 100000 + rep
                lane.profile(rep > 0)
                lane.forward(kv, [(sid, L, 1)], rng.integers(0, V, L))
                lane.wait()
                kv.release(sid)
            st = lane.stats()
            lane.profile(False)
            g, at = st["prefill_gemm"], st["prefill_attn"]
            results.append({"model": name, "case": f"prefill T={L}",
                            "prefill_gemm_tflops": rate(g[0], g[1], "flops"),
                            "prefill_gemm_frac": rate(g[0], g[1], "flops") / PEAKS["bf16_tflops"],
                            "prefill_attn_tflops": rate(at[0], at[1], "flops"),
                            "forward_ms": st["forward"][0] / a.reps})
            print(json.dumps(results[-1]), flush=True)
        # decode
        dlane, sms = lane, 148
        if a.level:
            from paper_2603_10342_b200.device import Slots
            slots = Slots(0, levels=9, granularity=16)
            sd, _ = slots.bind(a.level)
            sms = slots.sm_counts(a.level)[0]
            dlane = Lane(m, max_tokens=pmax, max_segments=80, stream=sd)
            dlane.set_sms(sms)
        for B, ctx in dcs:
            sess = list(range(B))
            for s in sess:
                done = 0
                while done < ctx - 1:
                    n = min(pmax, ctx - 1 - done)
                    lane.forward(kv, [(s, n, 0)], rng.integers(0, V, n))
                    done += n
            lane.wait()
            for rep in range(2):  # warm
                dlane.forward(kv, [(s, 1, 1) for s in sess], rng.integers(0, V, B))
                dlane.wait()
            dlane.stats()
            dlane.profile(True)
            for rep in range(a.reps):
                dlane.forward(kv, [(s, 1, 1) for s in sess], rng.integers(0, V, B))
                dlane.wait()
            st = dlane.stats()
            dlane.profile(False)
            step_ms = []
            for rep in range(a.reps):  # unprofiled (PDL on)
                dlane.forward(kv, [(s, 1, 1) for s in sess], rng.integers(0, V, B))
                dlane.wait()
                step_ms.append(dlane.last_ms())
            da, dg = st["decode_attn"], st["decode_gemm"]
            results.append({"model": name, "case": f"decode B={B} ctx={ctx}", "sms": sms,
                            "step_ms_unprofiled": float(np.median(step_ms)),
                            "decode_attn_gbs": rate(da[0], da[1], "bytes"),
                            "decode_attn_frac": rate(da[0], da[1], "bytes") / PEAKS["hbm_gbs"],
                            "decode_attn_us_per_layer": 1000 * da[0] / max(1, da[2]),
                            "decode_gemm_gbs": rate(dg[0], dg[1], "bytes"),
                            "decode_gemm_frac": rate(dg[0], dg[1], "bytes") / PEAKS["hbm_gbs"],
                            "step_ms": st["forward"][0] / a.reps})
            print(json.dumps(results[-1]), flush=True)
            for s in sess:
                kv.release(s)
        del dlane, lane, kv, m
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
