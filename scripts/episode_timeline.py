"""Timeline of one wall-clock serving episode: per control interval the decode slot level,
measured TPOT, decode batch and step time, Q_P backlog and prefill throughput; then every
session's cold arrival -> prefill start / done -> first emission (TTFT) in arrival order.

  python scripts/episode_timeline.py --config c3 --spec agentserve[:key=val,...] [--clock wall]
"""
import argparse
import json
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
from paper_2603_10342_b200 import workloads  # noqa: E402
from paper_2603_10342_b200.agsv import Agsv  # noqa: E402
from policy_compare import parse_spec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--spec", default="agentserve")
ap.add_argument("--clock", default="wall")
ap.add_argument("--warm", type=int, default=1)
a = ap.parse_args()
pol, kw = parse_spec(a.spec)
cfg = workloads.run_config(a.config, clock=a.clock, policy=pol, lend=bool(kw.get("lend", 1)),
                           calibrated=bool(kw.get("calib", 1)), slack=float(kw.get("slack", workloads.SLACK)),
                           theta_low_frac=float(kw.get("tlow", 0.5)), static_slots=kw.get("k"),
                           unit_tokens=int(kw.get("unit", workloads.UNIT_TOKENS)))
for key, ck in (("dt", "delta_t_ms"), ("r0", "initial_r_slots"), ("rbase", "r_base_slots"),
                ("b0", "initial_b_tokens"), ("bmin", "b_min_tokens")):
    if key in kw:
        cfg.setdefault("controller", {})[ck] = kw[key]
api = Agsv()
for _ in range(a.warm):
    api.run(cfg)
t = api.run(cfg)
recs = [json.loads(x) for x in t.jsonl(tempfile.mkdtemp()).splitlines()]
m = t.metrics()
print("config", json.dumps({k: cfg.get(k) for k in ("slo", "controller")}))
ticks = [r for r in recs if r.get("k") == "tick"]
steps = [r for r in recs if r.get("k") == "step_done"]
issues = [r for r in recs if r.get("k") == "issue"]
pdone = [r for r in recs if r.get("k") == "prefill_done"]
print(f"{'t1':>7} {'dsl':>3} {'psl':>3} {'tpot':>6} {'steps':>5} {'B_avg':>5} {'step_ms':>7} {'qp':>3} {'cold_tok':>8} {'res_p':>6} {'res_d':>6}")
for tk in ticks:
    s = tk["summary"]
    st = [x for x in steps if s["t0"] <= x["t"] < s["t1"]]
    qp = sum(1 for x in issues if x["q"] == "QP" and x["t"] < s["t1"]) - sum(1 for x in pdone if x["t"] < s["t1"] and x.get("ctx") != "decode")
    b = sum(len(x["emit"]) for x in st) / max(1, len(st))
    sm = sum(x["t"] - x["start"] for x in st) / max(1, len(st))
    print(f"{s['t1']:7.0f} {s['dslots']:3d} {s['pslots']:3d} {s['tpot']:6.2f} {len(st):5d} {b:5.1f} {sm:7.2f} {qp:3d} "
          f"{s['cold_tok']:8.0f} {s['res_tok_p']:6.0f} {s['res_tok_d']:6.0f}")
arr = {r["s"]: r["t"] for r in recs if r.get("k") == "arrival"}
cold = {r["s"]: r for r in pdone if r.get("req") == "cold"}
first = {}
for x in steps:
    for s in x["emit"]:
        first.setdefault(s, x["t"])
print(f"{'s':>3} {'arrive':>7} {'pstart':>7} {'pdone':>7} {'first':>7} {'ttft':>7}")
for s in sorted(arr, key=arr.get):
    c = cold.get(s, {})
    print(f"{s:3d} {arr[s]:7.1f} {c.get('start', -1):7.1f} {c.get('t', -1):7.1f} {first.get(s, -1):7.1f} "
          f"{first.get(s, -1) - arr[s]:7.1f}")
print("metrics", json.dumps({k: m.get(k) for k in ("ttft_p50_ms", "ttft_p95_ms", "ttft_p99_ms", "tpot_p50_ms",
                                                    "tpot_p95_ms", "tpot_p99_ms", "throughput_tps")}))
# where the TPOT tail comes from: step duration by decode SM count and admitted-chunk presence
import collections
by = collections.defaultdict(list)
for x in steps:
    by[(x.get("sms", 0), int(x.get("chunk", 0)) > 0)].append((x["t"] - x["start"], x.get("dev_ms", -1.0)))
# host = launch -> completion seen by the host; dev = the lane's CUDA-event time of the step
print(f"{'sms':>4} {'chunk':>5} {'steps':>5} {'host50':>6} {'host95':>6} {'dev50':>6} {'dev95':>6} {'B_avg':>5}")
for (sms, ch), v in sorted(by.items()):
    h = sorted(a for a, _ in v)
    d = sorted(b for _, b in v)
    bs = [len(x["emit"]) for x in steps if x.get("sms", 0) == sms and (int(x.get("chunk", 0)) > 0) == ch]
    print(f"{sms:4d} {str(ch):>5} {len(v):5d} {h[len(h) // 2]:6.2f} {h[int(0.95 * (len(h) - 1))]:6.2f} "
          f"{d[len(d) // 2]:6.2f} {d[int(0.95 * (len(d) - 1))]:6.2f} {sum(bs) / len(bs):5.1f}")
# consecutive decode steps: idle time between one step's completion and the next step's launch
idle = [b["start"] - a["t"] for a, b in zip(steps, steps[1:])]
idle.sort()
print("decode lane idle between steps (ms): p50 %.3f p90 %.3f p99 %.3f" % (
    idle[len(idle) // 2], idle[int(0.9 * (len(idle) - 1))], idle[int(0.99 * (len(idle) - 1))]))
gaps = []
prev = {}
for r in recs:
    if r.get("k") == "issue" and r.get("req") == "decode":
        prev[r["s"]] = None
    elif r.get("k") == "step_done":
        for s_ in r["emit"]:
            if prev.get(s_) is not None:
                # stalled: the gap holds more than this step (a prefill unit or another step ran between)
                gaps.append((r["t"] - prev[s_], r.get("sms", 0), int(r.get("chunk", 0)) > 0, r["t"],
                             (r["t"] - prev[s_]) > (r["t"] - r["start"]) + 0.5))
            prev[s_] = r["t"]
gaps.sort()
print("TPOT gap percentiles:", {p: round(gaps[int(p / 100 * (len(gaps) - 1))][0], 2)
                                for p in (50, 80, 85, 90, 92, 94, 95, 96, 98, 99)})
for lo in (4.5, 5.0, 6.0):
    sl = [g for g in gaps if g[0] >= lo]
    print(f"gaps >= {lo} ms: {len(sl) / len(gaps):.3f} of all; stalled {sum(g[4] for g in sl)}, by (sms, chunk):",
          dict(collections.Counter((g[1], g[2]) for g in sl)))
p95 = gaps[int(0.95 * (len(gaps) - 1))][0]
tail = [g for g in gaps if g[0] >= p95]
print(f"TPOT gaps {len(gaps)}, p95 {p95:.2f} ms; gaps >= p95: by (sms, chunk):",
      dict(collections.Counter((g[1], g[2]) for g in tail)),
      "time range", round(min(g[3] for g in tail)), "-", round(max(g[3] for g in tail)))
