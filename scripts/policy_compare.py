"""The paper's policy ablation on real B200 kernels (the reference's CLI
`compare` sweep, /root/reference/proj/tools/agentsim_main.cpp:171-259, run in wall-clock mode):
every policy (and the static Green Context split sweep) serves the same synthetic agent trace
through agsv_simulate; we record TTFT/TPOT p50/p95/p99 pooled over reps, throughput, SLO
attainment, rebind latency and the competitive-ratio verification summary.

  python scripts/policy_compare.py --config c3 --reps 3 \
      --runs agentserve mixed_fcfs agentserve:lend=0 agentserve:slack=2 static_partition:k=4 \
      --out profiles/r2_policy_compare_c3.json

A run spec is policy[:key=value,...] with keys lend (0/1), slack, tlow (theta_low / tau), thigh (theta_high / tau),
calib (0/1: measured-curve calibration vs the reference's factor-8), k (static decode slots),
unit (prefill launch-unit tokens), dt (control interval ms), r0 / rbase (initial / base
decode slots), b0 / bmin (initial / minimum resume-prefill budget tokens), dr (slots per controller move), early (backend.early_tick_steps), thnc (backend.theta_high_no_cold_ms / tau).
"""
import argparse
import json
import math
import statistics
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_10342_b200 import workloads  # noqa: E402
from paper_2603_10342_b200.agsv import Agsv  # noqa: E402


def pct(xs, p):
    if not xs:
        return None
    s = sorted(xs)
    k = max(1, math.ceil(p / 100.0 * len(s)))
    return s[min(k, len(s)) - 1]


def gaps_and_ttft(recs, metrics):
    """Per-gap TPOT samples (the reference's collect_tokens, metrics.cpp:71-92) and TTFTs."""
    gaps, prev = [], {}
    for r in recs:
        if r.get("k") == "issue" and r.get("req") == "decode":
            prev[r["s"]] = None
        elif r.get("k") == "step_done":
            for s in r["emit"]:
                if prev.get(s) is not None:
                    gaps.append(r["t"] - prev[s])
                prev[s] = r["t"]
    ttft = [s["ttft_ms"] for s in metrics["sessions"] if s["ttft_ms"] >= 0]
    return gaps, ttft


def parse_spec(spec):
    pol, _, rest = spec.partition(":")
    kw = {}
    for item in filter(None, rest.split(",")):
        k, v = item.split("=")
        kw[k] = float(v) if "." in v else int(v)
    return pol, kw


def run_spec(api, cfg_name, spec, reps, td, horizon=None):
    pol, kw = parse_spec(spec)
    cfg = workloads.run_config(cfg_name, policy=pol, lend=bool(kw.get("lend", 1)),
                               calibrated=bool(kw.get("calib", 1)), slack=float(kw.get("slack", workloads.SLACK)),
                               theta_low_frac=float(kw.get("tlow", workloads.THETA_LOW_FRAC)),
                               theta_high_frac=float(kw.get("thigh", workloads.THETA_HIGH_FRAC)),
                               theta_high_no_cold_frac=float(kw.get("thnc", workloads.THETA_HIGH_NO_COLD_FRAC)),
                               static_slots=kw.get("k"), unit_tokens=int(kw.get("unit", workloads.UNIT_TOKENS)))
    if "dt" in kw:
        cfg.setdefault("controller", {})["delta_t_ms"] = float(kw["dt"])
    if "r0" in kw:
        cfg.setdefault("controller", {})["initial_r_slots"] = int(kw["r0"])
    if "rbase" in kw:
        cfg.setdefault("controller", {})["r_base_slots"] = int(kw["rbase"])
    if "early" in kw:
        cfg.setdefault("backend", {})["early_tick_steps"] = int(kw["early"])
    if "dr" in kw:
        cfg.setdefault("controller", {})["delta_r_slots"] = int(kw["dr"])
    if "b0" in kw:
        cfg.setdefault("controller", {})["initial_b_tokens"] = int(kw["b0"])
    if "bmin" in kw:
        cfg.setdefault("controller", {})["b_min_tokens"] = int(kw["bmin"])
    if horizon:
        cfg["horizon_ms"] = horizon
    gaps, ttft, tps, att, reb, ends, tokens = [], [], [], [], [], [], 0
    ver = None
    for _ in range(reps):
        t = api.run(cfg)
        m = t.metrics()
        recs = [json.loads(x) for x in t.jsonl(td).splitlines()]
        g, tt = gaps_and_ttft(recs, m)
        gaps += g
        ttft += tt
        tps.append(m["throughput_tps"])
        att.append(m.get("slo_attainment", m.get("joint_slo_attainment")))
        dev = recs[-1].get("device", {})
        reb.append(dev.get("rebind_us", {}))
        ends.append(recs[-1]["end_ms"])
        tokens += sum(len(r["emit"]) for r in recs if r.get("k") == "step_done")
        ver = json.loads(t.verify()[0])
    row = {"run": spec, "policy": pol, **{k: v for k, v in kw.items()},
           "tokens_per_s": round(1000.0 * tokens / sum(ends), 1),
           "ttft_ms": {p: round(pct(ttft, p), 3) for p in (50, 95, 99)},
           "tpot_ms": {p: round(pct(gaps, p), 3) for p in (50, 95, 99)},
           "slo_attainment": statistics.mean(a for a in att if a is not None) if any(a is not None for a in att) else None,
           "rebind_us": reb[-1],
           "slo": cfg.get("slo"), "controller": cfg.get("controller"),
           "verify": {"checked": ver["checked"], "vacuous": ver["vacuous"], "violations": ver["violations"],
                      "min_rho": ver["min_rho"], "assumptions_met": ver["assumptions_met"]},
           "samples": {"sessions": len(ttft), "tpot_gaps": len(gaps)}}
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(workloads.CONFIGS), default="c3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--runs", nargs="*", default=None)
    ap.add_argument("--static-sweep", action="store_true")
    ap.add_argument("--horizon-ms", type=float, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    api = Agsv()
    td = tempfile.mkdtemp()
    runs = a.runs or ["agentserve", "mixed_fcfs", "chunked_prefill", "agentserve_no_slots"]
    if a.static_sweep:
        prof, _ = workloads.load_profile(workloads.CONFIGS[a.config]["model"])
        runs += [f"static_partition:k={k}" for k in range(1, prof["total_sms"] // prof["granularity"])]
    rows = []
    sys.path.insert(0, str(ROOT))
    from bench import ClockSampler  # nvidia-smi clocks / throttle reasons during each run
    for spec in runs:
        sampler = ClockSampler(0)
        sampler.start()
        row = run_spec(api, a.config, spec, a.reps, td, a.horizon_ms)
        row["clocks"] = sampler.stop()
        rows.append(row)
        print(json.dumps(row), flush=True)
    doc = {"config": a.config, "label": workloads.CONFIGS[a.config]["label"], "reps": a.reps,
           "clock": "wall (B200, Green Context partitions)", "runs": rows}
    if a.out:
        Path(a.out).write_text(json.dumps(doc, indent=1) + "\n")


if __name__ == "__main__":
    main()
