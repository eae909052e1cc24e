"""Co-run interference: a decode step on the decode Green Context partition, alone and while the
complementary prefill partition runs back-to-back prefill launch units, with SM clock / power
sampled through NVML during each phase.

  python scripts/corun_probe.py [model] [B] [ctx] [--levels=3,4,6] [--unit=4096] [--chunk=16]
"""
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_10342_b200.device import KvPool, Lane, Model, Slots  # noqa: E402


def opt(key, default):
    for a in sys.argv[1:]:
        if a.startswith(f"--{key}="):
            return a.split("=", 1)[1]
    return default


args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "llama3.2-3b"
B = int(args[1]) if len(args) > 1 else 12
ctx = int(args[2]) if len(args) > 2 else 3000
levels = [int(x) for x in opt("levels", "3,4,6").split(",")]
unit = int(opt("unit", "4096"))
chunk = int(opt("chunk", "0"))
steps = int(opt("steps", "40"))
# what the prefill partition runs: the engine's prefill units, a bf16 cuBLAS GEMM loop (tensor /
# L2 heavy, little HBM) or a 1 GiB device copy loop (HBM heavy)
aggressor = opt("aggressor", "prefill")


class Clocks:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        self.samples = []
        self.on = False

    def _run(self):
        while self.on:
            self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                 self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0,
                                 self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            time.sleep(0.005)

    def start(self):
        self.samples, self.on = [], True
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self):
        self.on = False
        self.t.join()
        a = np.array(self.samples) if self.samples else np.zeros((1, 3))
        names = {0x1: "idle", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal",
                 0x40: "hw_thermal", 0x80: "hw_power_brake"}
        seen = 0
        for r in a[:, 2].astype(np.int64):
            seen |= int(r)
        why = ",".join(v for k, v in names.items() if seen & k) or "-"
        return (f"sm {np.median(a[:, 0]):.0f} MHz (min {a[:, 0].min():.0f}), power {np.median(a[:, 1]):.0f} W, "
                f"reasons {why} (0x{seen:x})")


grow = (2 * steps + 10) * len(levels) * max(1, chunk)  # tokens a session gains over the run
m = Model(name, seed=13, max_context=max(ctx + grow + 512, unit + 64))
blocks_dec = (B + 1) * ((ctx + grow + 63) // 64 + 4)
kv = KvPool(m, num_blocks=blocks_dec + 2 * (unit // 64 + 2) + 8)
dlane = Lane(m, max_tokens=max(2048, B + chunk), max_segments=B + 4)
plane = Lane(m, max_tokens=unit, max_segments=4)
rng = np.random.default_rng(0)
for s in range(B + (1 if chunk else 0)):
    done = 0
    while done < ctx - 1:
        n = min(2048, ctx - 1 - done)
        dlane.forward(kv, [(s, n, 0)], rng.integers(0, m.vocab, n))
        done += n
dlane.wait()
slots = Slots(0, levels=9, granularity=16)
clk = Clocks()
psid = [1000]
agg = {}


def aggressor_next():
    """Keep the prefill partition busy with the chosen aggressor."""
    if aggressor == "prefill":
        if plane.done():
            prefill_next()
        return
    import torch
    ev = agg.get("ev")
    if ev is not None and not ev.query():
        return
    with torch.cuda.stream(agg["stream"]):
        for _ in range(40 if aggressor == "gemm" else 24):  # ~10 ms of work per enqueue
            if aggressor == "gemm":
                torch.matmul(agg["a"], agg["b"], out=agg["c"])
            else:
                agg["y"].copy_(agg["x"])
        agg["ev"] = torch.cuda.Event()
        agg["ev"].record()


def aggressor_wait():
    if aggressor == "prefill":
        plane.wait()
    elif agg.get("ev") is not None:
        agg["ev"].synchronize()


def prefill_next():
    """Start the next cold prefill unit on the prefill lane (previous session released)."""
    if psid[0] > 1000:
        kv.release(psid[0] - 1)
    plane.forward(kv, [(psid[0], unit, 1)], rng.integers(0, m.vocab, unit))
    psid[0] += 1


def decode_steps(n, corun):
    out = []
    for _ in range(n):
        if corun:
            aggressor_next()
        segs = [(s, 1, 1) for s in range(B)] + ([(B, chunk, 1)] if chunk else [])
        dlane.forward(kv, segs, rng.integers(0, m.vocab, B + chunk))
        dlane.wait()
        out.append(dlane.last_ms())
    return np.array(out)


for lv in levels:
    dstream, pstream = slots.bind(lv)
    dsms, psms = slots.sm_counts(lv)
    dlane.set_stream(dstream)
    dlane.set_sms(dsms)
    plane.set_stream(pstream)
    plane.set_sms(psms)
    if aggressor != "prefill":
        import torch
        agg["stream"] = torch.cuda.ExternalStream(pstream)
        if "a" not in agg:
            agg["a"] = torch.randn(unit, 3072, device="cuda", dtype=torch.bfloat16)
            agg["b"] = torch.randn(3072, 8192, device="cuda", dtype=torch.bfloat16)
            agg["c"] = torch.empty(unit, 8192, device="cuda", dtype=torch.bfloat16)
            agg["x"] = torch.empty(1 << 29, device="cuda", dtype=torch.float16)
            agg["y"] = torch.empty(1 << 29, device="cuda", dtype=torch.float16)
    decode_steps(5, False)
    clk.start()
    iso = decode_steps(steps, False)
    ci = clk.stop()
    pt = [0.0]
    if aggressor == "prefill":  # prefill alone on its partition: unit time
        plane.wait()
        pt = []
        for _ in range(3):
            prefill_next()
            plane.wait()
            pt.append(plane.last_ms())
    aggressor_next()
    decode_steps(5, True)
    clk.start()
    co = decode_steps(steps, True)
    cc = clk.stop()
    aggressor_wait()
    print(f"{name} B={B}+{chunk} ctx={ctx} decode {dsms} SMs | {aggressor} {psms} SMs x {unit} tok "
          f"({np.median(pt):.1f} ms/unit alone): step alone {np.median(iso):.3f} ms [{ci}], "
          f"co-run p50 {np.median(co):.3f} p90 {np.percentile(co, 90):.3f} ms "
          f"(x{np.median(co) / np.median(iso):.2f}) [{cc}]", flush=True)
