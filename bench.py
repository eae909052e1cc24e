#!/usr/bin/env python3
"""AgentServe hot-path benchmark on B200 (driver contract: one JSON line on rank 0).

A *step* is one full serving episode of a BASELINE.json configuration (default C3, the
north_star target: a Llama-3.2-3B-shaped random-init SLM serving 32 concurrent ReAct agents per
GPU, mixed cold/resume/decode arrivals), scheduled by the AgentServe policy (TPOT controller +
resume-prefill budget + Green Context partitions) and executed for real on the B200 through
the drop-in agsv_* C ABI.  The same episodes are then served by the unpartitioned FCFS policy
(`mixed_fcfs`, the llama.cpp archetype) on the same kernels, and both are reported in the line.

metric  : served decode tokens / s (the reference's throughput_tps, metrics.cpp:144-155),
          whole job over all GPUs; p50/p95/p99 TTFT and TPOT (the reference's definitions,
          metrics.cpp:71-92, pooled over all timed episodes) for both policies.
value   : AgentServe emitted tokens / episode time on the engine's clock (device completions),
          slowest rank.
e2e     : the same tokens / wall time around the agsv_simulate C-ABI call from this host
          client (config JSON in, trace out; token ids and block tables H2D and greedy ids D2H
          every forward, counted by the lanes).
roofline: dominant kernel category by device time, timed with CUDA events on the lane stream
          (backend.profile_kernels) during one profiled replay of the same episode right after
          the timed ones, against MEASURED_PEAKS.json; `traffic` from the committed ncu capture
          of the same config (profiles/ncu_traffic_<config>.json, scripts/ncu_traffic.py).
cpu_baseline / --impl reference: the CPU fp32 oracle forward (oracle/forward.c) on the box's
          host cores executing a real slice of the same episode (see cpu_slice).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl mine|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2603_10342_b200 import workloads  # noqa: E402

METRIC = "served decode tokens/s per GPU under the agent trace (p50/p99 TTFT & TPOT ms; decode-attn HBM GB/s)"


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": d.get("hbm_gbs", 6650.0), "bf16": d.get("bf16_tflops", 1590.0),
                "bf16_sust": d.get("bf16_tflops_sustained", 1380.0), "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sust": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.out, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict | None:
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.out.flush()
        rows = [r.split(",") for r in Path(self.out.name).read_text().splitlines() if r.strip()]
        sms, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sms.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not sms:
            return None
        busy = [s for s in sms if s > 0.5 * mx] or sms
        busy.sort()
        return {"sm_mhz": busy[len(busy) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def pct(xs: list[float], p: float) -> float | None:
    """nearest-rank percentile (metrics.cpp:45-59)"""
    if not xs:
        return None
    s = sorted(xs)
    k = max(1, math.ceil(p / 100.0 * len(s)))
    return s[min(k, len(s)) - 1]


def episode_stats(recs: list[dict], metrics: dict) -> dict:
    """Counts, per-gap TPOT samples and TTFTs of one episode trace (the reference's
    collect_tokens walk, metrics.cpp:71-92: gap chains break at decode-phase starts)."""
    foot = recs[-1]
    steps = [r for r in recs if r.get("k") == "step_done"]
    gaps, prev = [], {}
    for r in recs:
        if r.get("k") == "issue" and r.get("req") == "decode":
            prev[r["s"]] = None
        elif r.get("k") == "step_done":
            for s in r["emit"]:
                if prev.get(s) is not None:
                    gaps.append(r["t"] - prev[s])
                prev[s] = r["t"]
    return {"tokens": sum(len(s["emit"]) for s in steps), "end_ms": foot["end_ms"],
            "device": foot.get("device", {}), "n_steps": len(steps),
            "gaps": gaps, "ttft": [s["ttft_ms"] for s in metrics["sessions"] if s["ttft_ms"] >= 0],
            "slo": metrics.get("slo_attainment", metrics.get("joint_slo_attainment")),
            "step_sms": [(s.get("sms", 0), s.get("dev_ms", 0.0)) for s in steps]}


# ------------------------------------------------------------------------------- CPU baseline
class CpuSlice:
    """The CPU fp32 oracle (oracle/forward.c, OpenMP over all host cores) serving a REAL slice
    of the same episode: the trace's Q_P prefills (cold prompts, resumes over budget) and
    decode steps (every stream's row + the admitted-resume chunk) are executed in trace order
    with the config's full-width model truncated to 2 and to 1 decoder layers (same events
    on both), for a wall-time budget.  Per-forward and per-layer costs separate from the two
    runs: full-depth cost = base + L * per_layer, with base = 2*T1 - T2 and per_layer =
    T2 - T1 over the same events.  The episode estimate prices the unexecuted rest of the
    trace at the slice's measured per-token (prefill) and per-row (decode) rates.  State
    persists across calls, so repeated steps extend one slice."""

    def __init__(self, cfg_name: str, recs: list[dict], seed: int = 13):
        from oracle.forward import OracleModel, PRESETS
        self.cfg_name = cfg_name
        self.model = workloads.CONFIGS[cfg_name]["model"]
        self.layers = PRESETS[self.model]["layers"]
        self.seed = seed
        self.recs = recs
        self.work = self._work_items(recs)
        tot = {}  # tokens each session accumulates over the episode -> the oracle's KV capacity
        for kind, s, n, _, r in self.work:
            if kind == "prefill":
                tot[s] = tot.get(s, 0) + n
                continue
            for e in r["emit"]:
                tot[e] = tot.get(e, 0) + 1
            if r.get("chunk"):
                tot[r["chunk_s"]] = tot.get(r["chunk_s"], 0) + int(r["chunk"])
        max_ctx = max(tot.values(), default=0)
        self.m2 = OracleModel(self.model, seed=seed, max_ctx=max_ctx + 64, layers_limit=min(2, self.layers))
        self.m1 = OracleModel(self.model, seed=seed, max_ctx=max_ctx + 64, layers_limit=1)
        self.s2, self.s1 = {}, {}
        self.done = 0  # work items executed
        self.t2 = {"prefill": 0.0, "step": 0.0}
        self.t1 = {"prefill": 0.0, "step": 0.0}
        self.cnt = {"prefill_tokens": 0, "step_rows": 0, "steps": 0}

    @staticmethod
    def _work_items(recs):
        """(kind, session, tokens, rows, record) in trace order: 'prefill' = one Q_P job (cold
        prompt or resume over budget); 'step' = one decode step (rows = its single-token
        streams, tokens = rows + the admitted-resume chunk)."""
        out = []
        for r in recs:
            k = r.get("k")
            if k == "prefill_done" and r.get("ctx") != "decode":
                out.append(("prefill", r["s"], int(r["len"]), 0, r))
            elif k == "step_done":
                rows = len(r["emit"])
                out.append(("step", -1, rows + int(r.get("chunk", 0)), rows, r))
        return out

    def _exec(self, model, sess, item):
        import numpy as np
        kind, s, n, rows, r = item
        V = model.spec.vocab
        if kind == "prefill":
            ss = sess.setdefault(s, model.session())
            ss.forward(np.random.default_rng(s).integers(0, V, n, dtype=np.int32))
            return
        for e in r["emit"]:
            sess.setdefault(e, model.session()).forward(np.array([1 + e % (V - 1)], dtype=np.int32))
        chunk = int(r.get("chunk", 0))
        if chunk > 0:
            cs = r["chunk_s"]
            sess.setdefault(cs, model.session()).forward(
                np.random.default_rng(cs).integers(0, V, chunk, dtype=np.int32))

    def run(self, budget_s: float) -> None:
        t_end = time.perf_counter() + budget_s
        while self.done < len(self.work) and time.perf_counter() < t_end:
            item = self.work[self.done]
            t0 = time.perf_counter()
            self._exec(self.m2, self.s2, item)
            t1 = time.perf_counter()
            self._exec(self.m1, self.s1, item)
            t2 = time.perf_counter()
            self.t2[item[0]] += t1 - t0
            self.t1[item[0]] += t2 - t1
            if item[0] == "prefill":
                self.cnt["prefill_tokens"] += item[2]
            else:
                self.cnt["step_rows"] += item[2]
                self.cnt["steps"] += 1
            self.done += 1

    def estimate(self) -> dict:
        L = self.layers

        def full(kind):
            t2, t1 = self.t2[kind], self.t1[kind]
            per_layer = max(t2 - t1, 0.0)
            base = max(t1 - per_layer, 0.0)
            return base + L * per_layer

        t_pf, t_st = full("prefill"), full("step")
        rest_pf = sum(w[2] for w in self.work[self.done:] if w[0] == "prefill")
        rest_rows = sum(w[2] for w in self.work[self.done:] if w[0] == "step")
        rate_pf = t_pf / self.cnt["prefill_tokens"] if self.cnt["prefill_tokens"] else None
        rate_row = t_st / self.cnt["step_rows"] if self.cnt["step_rows"] else None
        if rate_row is None and rate_pf is not None:
            rate_row = rate_pf  # a decode row costs at least a prefill token
        if rate_pf is None and rate_row is not None:
            rate_pf = rate_row
        t_total = t_pf + t_st + (rest_pf * rate_pf if rate_pf else 0.0) + (rest_rows * rate_row if rate_row else 0.0)
        tokens = sum(len(r["emit"]) for r in self.recs if r.get("k") == "step_done")
        return {"value": tokens / t_total if t_total > 0 else 0.0, "unit": "tokens/s",
                "cores": os.cpu_count(), "kind": "port",
                "sample": (f"CPU fp32 oracle (oracle/forward.c, OpenMP {os.cpu_count()} threads) executed the first "
                           f"{self.done} of {len(self.work)} work items of the {self.cfg_name.upper()} episode trace in "
                           f"order ({self.cnt['prefill_tokens']} Q_P prefill tokens, {self.cnt['steps']} decode steps / "
                           f"{self.cnt['step_rows']} rows) on the full-width {self.model} truncated to 2 and 1 of {L} "
                           f"layers; full depth = base + {L} x per-layer cost; the rest of the episode "
                           f"({rest_pf} prefill tokens, {rest_rows} step rows) priced at the slice's measured rates; "
                           f"episode estimate {t_total:.1f} s for {tokens} tokens")}


# ------------------------------------------------------------------------------- harness
def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 1, 0, None
    import torch.distributed as dist
    # sessions never exchange data: the harness's barrier / max / gather are host plumbing,
    # kept off NCCL by default (north_star: no NCCL)
    dist.init_process_group(backend=os.environ.get("BENCH_BACKEND", "gloo"))
    return ws, dist.get_rank(), dist


def _reduce(dist, vals: list[float], op: str) -> list[float]:
    if dist is None:
        return vals
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.cpu().tolist()


def _gather(dist, xs: list) -> list:
    if dist is None:
        return xs
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, xs)
    return [v for part in out for v in part]


def device_index() -> tuple[int, int]:
    """(CUDA ordinal in this process, physical GPU index for nvidia-smi) of this rank: one rank
    per GPU.  A launcher that pins one device per process through CUDA_VISIBLE_DEVICES leaves
    ordinal 0; otherwise the rank's LOCAL_RANK selects the device."""
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cvd = [x.strip() for x in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if x.strip()]
    if len(cvd) == 1:
        return 0, int(cvd[0]) if cvd[0].isdigit() else local
    if cvd and local < len(cvd) and cvd[local].isdigit():
        return local, int(cvd[local])
    return local, local


def policy_summary(stats: list[dict], dist, tokens_all: float, t_max_ms: float) -> dict:
    gaps = _gather(dist, [g for s in stats for g in s["gaps"]])
    ttft = _gather(dist, [t for s in stats for t in s["ttft"]])
    slo = _gather(dist, [s["slo"] for s in stats if s["slo"] is not None])
    return {"tokens_per_s": round(tokens_all / (t_max_ms / 1000.0), 2) if t_max_ms > 0 else 0.0,
            "ttft_ms": {f"p{p}": round(pct(ttft, p), 3) if ttft else None for p in (50, 95, 99)},
            "tpot_ms": {f"p{p}": round(pct(gaps, p), 3) if gaps else None for p in (50, 95, 99)},
            "slo_attainment": round(sum(slo) / len(slo), 4) if slo else None,
            "sessions": len(ttft), "tpot_gaps": len(gaps)}


def run_mine(args) -> None:
    n_gpus, rank, dist = _dist()
    import torch
    dev_idx, phys_idx = device_index()
    clock = "virtual" if args.virtual else "wall"
    if clock == "wall":
        torch.cuda.set_device(dev_idx)
    from paper_2603_10342_b200.agsv import Agsv
    api = Agsv()

    def cfg_of(policy, profile_kernels=False):
        c = workloads.run_config(args.config, clock=clock, policy=policy, n_shards=n_gpus, shard=rank,
                                 device=dev_idx, profile_kernels=profile_kernels)
        if args.horizon_ms:  # profiling runs only (ncu launch lists): cut every episode
            c["horizon_ms"] = args.horizon_ms
        return c

    cfg = cfg_of(args.policy)
    td = tempfile.mkdtemp()

    def episode(c):
        t0 = time.perf_counter()
        tr = api.run(c)
        recs = [json.loads(x) for x in tr.jsonl(td).splitlines()]
        m = tr.metrics()
        return recs, m, time.perf_counter() - t0

    for _ in range(args.warmup):
        episode(cfg)
    if dist is not None:
        dist.barrier()
    if clock == "wall":
        torch.cuda.synchronize()
        sampler = ClockSampler(phys_idx)
        sampler.start()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    t_wall0 = time.perf_counter()
    eps = [episode(cfg) for _ in range(args.steps)]
    t_wall = time.perf_counter() - t_wall0
    if clock == "wall":
        ev1.record()
        torch.cuda.synchronize()
        span_ms = ev0.elapsed_time(ev1)
        clocks = sampler.stop()
    else:
        span_ms, clocks = t_wall * 1000.0, None
    if dist is not None:
        dist.barrier()
    stats = [episode_stats(r, m) for r, m, _ in eps]

    # the unpartitioned FCFS arm on the same kernels and the same episodes
    cmp_stats = []
    if args.compare != "none":
        ccfg = cfg_of(args.compare)
        episode(ccfg)  # warm
        cmp_stats = [episode_stats(r, m) for r, m, _ in (episode(ccfg) for _ in range(max(1, args.steps)))]

    # profiled replay (per-launch CUDA events) for the kernel breakdown / roofline
    prof_stats = None
    if clock == "wall":
        r, m, _ = episode(cfg_of(args.policy, profile_kernels=True))
        prof_stats = episode_stats(r, m)

    tokens = sum(s["tokens"] for s in stats)
    engine_ms = sum(s["end_ms"] for s in stats)
    e2e_s = sum(w for _, _, w in eps)
    io = {"kernel_launches": 0, "h2d_bytes": 0, "d2h_bytes": 0}
    for s in stats:
        for kk in io:
            io[kk] += s["device"].get("io", {}).get(kk, 0)
    cats = {}
    if prof_stats:
        for name, lanes in prof_stats["device"].get("kernels", {}).items():
            c = cats.setdefault(name, {"ms": 0.0, "units": 0.0, "launches": 0, "unit": lanes.get("unit")})
            for ln in ("decode_lane", "prefill_lane"):
                if ln in lanes:
                    c["ms"] += lanes[ln]["ms"]
                    c["units"] += lanes[ln]["units"]
                    c["launches"] += lanes[ln]["launches"]
    c_tokens = sum(s["tokens"] for s in cmp_stats)
    c_ms = sum(s["end_ms"] for s in cmp_stats)
    red = _reduce(dist, [float(tokens), float(c_tokens)], "sum")
    mx = _reduce(dist, [float(engine_ms), float(e2e_s), float(span_ms), float(c_ms)], "max")
    main_sum = policy_summary(stats, dist, red[0], mx[0])
    cmp_sum = policy_summary(cmp_stats, dist, red[1], mx[3]) if cmp_stats else None
    rebinds = _gather(dist, [s["device"].get("rebind_us", {}) for s in stats])
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peaks = _peaks()
    value = red[0] / (mx[0] / 1000.0) if mx[0] > 0 else 0.0  # whole job / slowest rank
    e2e_value = red[0] / mx[1] if mx[1] > 0 else 0.0
    label = workloads.CONFIGS[args.config]["label"]
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mx[2] / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights from named splitmix64 sub-streams; synthetic token ids)",
        "config": {"workload": label, "config": args.config.upper(),
                   "model": workloads.CONFIGS[args.config]["model"],
                   "agents_per_gpu": workloads.CONFIGS[args.config]["agents"], "policy": args.policy,
                   "compare_policy": args.compare, "clock": clock,
                   "parallelism": f"session-sharded replicas x{n_gpus} (no collective)",
                   "slo": cfg.get("slo"), "controller": cfg.get("controller"),
                   "lend_idle_prefill": cfg.get("backend", {}).get("lend_idle_prefill"),
                   "profile": str(workloads.profile_path(workloads.CONFIGS[args.config]["model"]).relative_to(ROOT)),
                   "l2": "weights and KV exceed the 126 MB L2; no flush needed"},
        "latency_ms": {"ttft": main_sum["ttft_ms"], "tpot": main_sum["tpot_ms"],
                       "sessions": main_sum["sessions"], "tpot_gaps": main_sum["tpot_gaps"]},
        "policies": {args.policy: main_sum, **({args.compare: cmp_sum} if cmp_sum else {})},
        "e2e": {"value": round(e2e_value, 3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(io["h2d_bytes"] / max(1, args.steps)),
                "d2h_bytes_per_step": int(io["d2h_bytes"] / max(1, args.steps))},
        "gpu_launches": int(io["kernel_launches"]),
    }
    if cmp_sum:
        def ratio(a, b):
            return round(a / b, 4) if a is not None and b else None
        line["tails_vs_" + args.compare] = {
            f"{k}_{p}": ratio(main_sum[k + "_ms"][p], cmp_sum[k + "_ms"][p])
            for k in ("ttft", "tpot") for p in ("p50", "p95", "p99")}
    rb = [r for r in rebinds if r and r.get("n", 0) > 0]
    if rb:
        line["rebind_us"] = {"p50_max_over_episodes": max(r["p50"] for r in rb),
                             "p99_max_over_episodes": max(r["p99"] for r in rb),
                             "max": max(r["max"] for r in rb), "rebinds": sum(r["n"] for r in rb),
                             "target": "< 50 us (PAPER.md:453)"}
    if clocks:
        line["clocks"] = clocks
    kern = {k: v for k, v in cats.items() if k != "forward" and v["ms"] > 0}
    if kern:
        dom_name, dom = max(kern.items(), key=lambda kv: kv[1]["ms"])
        hbm = dom["unit"] == "bytes"
        achieved = dom["units"] / (dom["ms"] / 1000.0) / (1e9 if hbm else 1e12)
        peak = peaks["hbm"] if hbm else peaks["bf16_sust"]
        traffic, traffic_ratio = None, None
        tf = ROOT / "profiles" / f"ncu_traffic_{args.config}.json"
        if tf.exists():
            tdoc = json.loads(tf.read_text())
            traffic = tdoc.get(dom_name)
            alg = tdoc.get(f"_algorithmic_{dom_name}_per_launch")
            if traffic and alg:
                traffic_ratio = round(traffic / alg, 4)
        line["roofline"] = {"kernel": dom_name, "bound": "hbm" if hbm else "tensor",
                            "achieved": round(achieved, 2), "peak": peak,
                            "unit": "GB/s" if hbm else "TFLOP/s", "frac": round(achieved / peak, 4),
                            "traffic": round(traffic) if traffic else None,
                            "traffic_over_algorithmic": traffic_ratio, "peak_source": peaks["src"],
                            "avg_launch_us": round(1000.0 * dom["ms"] / max(1, dom["launches"]), 2),
                            "share_of_device_time": round(dom["ms"] / sum(v["ms"] for v in kern.values()), 3),
                            "measured": "profiled replay of the timed episode (CUDA events per launch)"}
        sms_w = [(n, ms) for s in stats for n, ms in s.get("step_sms", []) if n > 0 and ms > 0]
        if sms_w and hbm:
            mean_sms = sum(n * ms for n, ms in sms_w) / sum(ms for _, ms in sms_w)
            line["roofline"]["decode_sms_mean"] = round(mean_sms, 1)
        da = cats.get("decode_attn")
        if da and da["ms"] > 0:
            gbs = da["units"] / (da["ms"] / 1000.0) / 1e9
            line["decode_attn"] = {"achieved_gbs": round(gbs, 1), "frac_of_hbm": round(gbs / peaks["hbm"], 4),
                                   "launches": da["launches"],
                                   "avg_launch_us": round(1000.0 * da["ms"] / max(1, da["launches"]), 2)}
        line["kernels"] = {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                               "achieved": round(v["units"] / (v["ms"] / 1000.0) / (1e9 if v["unit"] == "bytes" else 1e12), 2),
                               "unit": "GB/s" if v["unit"] == "bytes" else "TFLOP/s"}
                           for k, v in kern.items()}
    if n_gpus == 1 and not args.no_cpu and clock == "wall":
        cs = CpuSlice(args.config, eps[0][0])
        cs.run(args.cpu_budget)
        line["cpu_baseline"] = cs.estimate()
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args) -> None:
    """Reference arm: the reference has no forward, so its CPU implementation of
    this path is the oracle port (oracle/forward.c) on the host cores, executing the same
    episode: the trace of the config comes from the compiled reference simulator
    (oracle/_ref/libagentsim.so, agsv_simulate) on the same workload config, and each bench
    step extends one real slice of it (CpuSlice) by a bounded budget."""
    n, rank, dist = _dist()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    from paper_2603_10342_b200.agsv import Agsv
    from tests.ref_oracle import REF_LIB
    api = Agsv(REF_LIB) if REF_LIB.exists() else Agsv()
    cfg = workloads.run_config(args.config, clock="virtual", policy=args.policy)
    td = tempfile.mkdtemp()
    recs = [json.loads(x) for x in api.run(cfg).jsonl(td).splitlines()]
    cs = CpuSlice(args.config, recs)
    per_step = max(2.0, args.ref_budget / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cs.run(per_step)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cs.run(per_step)
    wall = time.perf_counter() - t0
    base = cs.estimate()
    v = base["value"]
    label = workloads.CONFIGS[args.config]["label"]
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "tokens/s",
            "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000 * wall / max(1, args.steps), 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": label, "config": args.config.upper(),
                                            "trace": "reference simulator (oracle/_ref/libagentsim.so), same workload config",
                                            "policy": args.policy},
            "cpu_baseline": {**base, "value": round(v, 4),
                             "reference_simulator": "agsv_simulate of the compiled reference produced the episode trace"},
            "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mine", "reference"], default="mine")
    ap.add_argument("--config", choices=sorted(workloads.CONFIGS), default="c3")
    ap.add_argument("--policy", default="agentserve")
    ap.add_argument("--compare", default="mixed_fcfs", help="second policy on the same kernels ('none': skip)")
    ap.add_argument("--sim-clock", dest="virtual", action="store_true", help="virtual clock (CPU-only test mode)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU slice for cpu_baseline")
    ap.add_argument("--ref-budget", type=float, default=150.0, help="reference arm: total CPU seconds over all steps")
    ap.add_argument("--horizon-ms", type=float, default=None,
                    help="cut every episode at this engine time (ncu launch-list captures only; not a bench line)")
    args = ap.parse_args()
    if args.warmup < 3 and not args.virtual:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
