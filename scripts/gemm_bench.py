"""Decode linear-layer micro-bench: tcgen05 swap-AB (path 1) vs small-batch dgemv (path 2) vs the TMA-ring warp-MMA tgemv (path 3).

Back-to-back launches with PDL (asb_debug_gemm_bench), weights packed once; reports us per
launch and algorithmic GB/s (weights + X + Y bytes) against the measured HBM peak.

  python scripts/gemm_bench.py [--tokens 8 16 32] [--sms 0 32] [--out gpurun_out/gemm_bench.json]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200._lib import check, lib  # noqa: E402
from paper_2603_10342_b200.device import Slots  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6550.0
SHAPES = {
    "qwen2.5-0.5b": [("qkv", 1152, 896, 0), ("o", 896, 896, 1), ("gate_up", 9728, 896, 2), ("down", 896, 4864, 1),
                     ("lm_head", 151936, 896, 3)],
    "llama3.2-3b": [("qkv", 5120, 3072, 0), ("o", 3072, 3072, 1), ("gate_up", 16384, 3072, 2), ("down", 3072, 8192, 1)],
    "llama3.1-8b": [("qkv", 6144, 4096, 0), ("o", 4096, 4096, 1), ("gate_up", 28672, 4096, 2), ("down", 4096, 14336, 1)],
}

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, nargs="+", default=[8, 16, 32])
ap.add_argument("--levels", type=int, nargs="+", default=[0],
                help="green-context decode levels (SMs = level x 16 on B200); 0 = whole device")
ap.add_argument("--models", nargs="+", default=list(SHAPES))
ap.add_argument("--out", default=None)
ap.add_argument("--linears", nargs="*", default=None, help="only these linears (e.g. gate_up)")
ap.add_argument("--paths", type=int, nargs="*", default=None, help="only these paths (1 tcgen05, 2 dgemv, 3 tgemv)")
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--prefill", action="store_true", help="normal (prefill) path 0 at the given token counts; TF/s")
a = ap.parse_args()
dev = torch.device("cuda:0")
slots = Slots(0, levels=9, granularity=16)
res = []
for model in a.models:
    for name, N, K, epi in SHAPES[model]:
        if a.linears and name not in a.linears:
            continue
        w = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
        for T in a.tokens:
            x = torch.randn(T, K, device=dev).bfloat16()
            out = torch.zeros(T, N // 2 if epi == 2 else N, device=dev,
                              dtype=torch.float32 if epi == 3 else torch.bfloat16)
            bytes_ = 2.0 * (N * K + T * K) + T * N * (4 if epi == 3 else 2)
            for lev in a.levels:
                stream, sms = None, 0
                if lev:
                    stream, _ = slots.bind(lev)
                    sms = slots.sm_counts(lev)[0]
                row = {"model": model, "linear": name, "T": T, "N": N, "K": K, "sms": sms or 148}
                paths = (0,) if a.prefill else ((1, 2, 3) if T <= 32 else (1,))
                for path in paths:
                    if a.paths and path not in a.paths:
                        continue
                    us = C.c_float(0)
                    check(lib().asb_debug_gemm_bench(x.data_ptr(), w.data_ptr(), out.data_ptr(), T, N, K, epi, path,
                                                     a.iters, sms, stream, C.byref(us)))
                    row[f"p{path}_us"] = round(us.value, 2)
                    row[f"p{path}_gbs"] = round(bytes_ / (us.value * 1e-6) / 1e9, 1)
                    if a.prefill:
                        row["tflops"] = round(2.0 * T * N * K / (us.value * 1e-6) / 1e12, 1)
                if "p1_gbs" in row:
                    row["p1_frac"] = round(row["p1_gbs"] / PEAK, 3)
                if "p2_gbs" in row:
                    row["p2_frac"] = round(row["p2_gbs"] / PEAK, 3)
                if "p3_gbs" in row:
                    row["p3_frac"] = round(row["p3_gbs"] / PEAK, 3)
                res.append(row)
                print(json.dumps(row), flush=True)
        del w
if a.out:
    Path(a.out).write_text(json.dumps(res, indent=1))
