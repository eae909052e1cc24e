"""Quick device-time probe of whole forwards (prefill / decode) through the asb_* ABI.
Usage: python scripts/probe_perf.py [model] ; prints ms and derived throughput."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200.device import KvPool, Lane, Model  # noqa: E402

PEAK_TF, PEAK_BW = 1671.0, 6550.4


def main(spec):
    m = Model(spec, seed=13, max_context=16384)
    info = m.info
    L, d, hq, hkv, hd, F, V = (info[k] for k in ("layers", "d_model", "n_heads", "n_kv_heads",
                                                  "head_dim", "ffn", "vocab"))
    lin = L * (d * (hq + 2 * hkv) * hd + hq * hd * d + 3 * d * F)
    lm = V * d
    kvb = 2 * L * hkv * hd * 2  # bytes per token
    kv = KvPool(m, num_blocks=3000)
    lane = Lane(m, max_tokens=8192, max_segments=128)
    rng = np.random.default_rng(0)
    for T in (512, 2048, 8192):
        best = 1e9
        for it in range(4):
            s = 1000 + it + T
            lane.forward(kv, [(s, T, 1)], rng.integers(0, V, T))
            lane.wait()
            best = min(best, lane.last_ms())
            kv.release(s)
        fl = 2 * T * lin + 2 * d * V + 4 * L * hq * hd * T * T / 2
        print(f"{spec} prefill T={T}: {best:.3f} ms  {fl / best / 1e9:.1f} TFLOP/s "
              f"({fl / best / 1e9 / PEAK_TF * 100:.1f}% of {PEAK_TF})")
    for B, ctx in ((1, 2048), (8, 2048), (32, 3000), (64, 2048)):
        sess = list(range(B))
        for s in sess:
            kv.release(s)
        # fill contexts with one prefill per session (chunks of up to 4096)
        for s in sess:
            lane.forward(kv, [(s, ctx, 0)], rng.integers(0, V, ctx))
        lane.wait()
        best = 1e9
        for it in range(5):
            lane.forward(kv, [(s, 1, 1) for s in sess], rng.integers(0, V, B))
            lane.wait()
            best = min(best, lane.last_ms())
        byts = 2 * (lin + lm) + B * ctx * kvb
        print(f"{spec} decode B={B} ctx={ctx}: {best:.3f} ms  {byts / best / 1e6:.0f} GB/s "
              f"({byts / best / 1e6 / PEAK_BW * 100:.1f}% of {PEAK_BW})")
        for s in sess:
            kv.release(s)


if __name__ == "__main__":
    for spec in (sys.argv[1:] or ["qwen2.5-0.5b", "llama3.1-8b"]):
        main(spec)
