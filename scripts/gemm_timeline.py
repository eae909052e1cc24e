"""Per-CTA timeline of one GEMM launch (ASB_GEMM_TIMELINE=1) at decode shapes.

Prints, per phase, min/median/max over CTAs of globaltimer stamps relative to the first CTA
start: start, MMA issue done (warp 1), epilogue done (warp 2), exit.
"""
import ctypes as C, os, sys
from pathlib import Path
os.environ["ASB_GEMM_TIMELINE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch  # noqa
from paper_2603_10342_b200._lib import lib, check  # noqa
from paper_2603_10342_b200.device import debug_gemm  # noqa

L = lib()
L.asb_debug_gemm_timeline.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
EPI = {"bf16": 0, "resid": 1, "silu": 2, "f32": 3}
SHAPES = {"8b": [("qkv", 6144, 4096, "bf16"), ("o", 4096, 4096, "resid"), ("gate_up", 28672, 4096, "silu"),
                ("down", 4096, 14336, "resid")],
          "3b": [("qkv", 5120, 3072, "bf16"), ("o", 3072, 3072, "resid"), ("gate_up", 16384, 3072, "silu"),
                 ("down", 3072, 8192, "resid")],
          "0.5b": [("qkv", 1152, 896, "bf16"), ("o", 896, 896, "resid"), ("gate_up", 9728, 896, "silu"),
                  ("down", 896, 4864, "resid"), ("lm_head", 151936, 896, "f32")]}
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
shapes = SHAPES[sys.argv[2] if len(sys.argv) > 2 else "8b"]
dev = torch.device("cuda:0")
for name, N, K, epi in shapes:
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
    out = torch.empty(T, N // 2 if epi == "silu" else N, device=dev, dtype=torch.float32 if epi == "f32" else torch.bfloat16)
    resid = torch.randn(out.shape, device=dev).bfloat16() if epi == "resid" else None
    for rep in range(4):
        debug_gemm(x.data_ptr(), w.data_ptr(), out.data_ptr(), T, N, K, EPI[epi],
                   resid=resid.data_ptr() if resid is not None else None)
    buf = (C.c_ulonglong * (148 * 8))()
    check(L.asb_debug_gemm_timeline(None, buf, 148 * 8))
    t = np.array(buf[:], dtype=np.float64).reshape(148, 8)
    t = t[t[:, 0] > 0]
    rel = (t - t[:, 0].min()) / 1000.0
    f = lambda c: "%6.1f/%6.1f/%6.1f" % (rel[:, c].min(), np.median(rel[:, c]), rel[:, c].max())
    print(f"{name:8s} T={T} N={N} K={K} ctas={len(t)}  start {f(0)} tmem {f(6)} 1st-data {f(4)}  mma {f(1)} "
          f"1st-acc {f(5)}  epi {f(2)}  cluster-sync {f(7)}  exit {f(3)}  "
          f"min-bytes-time {N*K*2/6.55e3/1e3:.1f}us")
