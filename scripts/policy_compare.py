"""The paper's policy ablation on real B200 kernels (the reference's CLI
`compare` sweep, /root/reference/proj/tools/agentsim_main.cpp:171-259, run in wall-clock mode):
every policy and the static Green Context split sweep serve the same synthetic agent trace
through agsv_simulate, and we record TTFT/TPOT percentiles, throughput and the
competitive-ratio verification summary.

  python scripts/policy_compare.py [--config c2|c3] [--reps 2] [--out profiles/r1_policy_compare_c2.json]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2603_10342_b200.agsv import Agsv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", choices=["c2", "c3", "c4"], default="c2")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--out", default=None)
ap.add_argument("--policies", nargs="*", default=None, help="subset, e.g. agentserve mixed_fcfs static_partition:3")
ap.add_argument("--horizon-ms", type=float, default=None)
a = ap.parse_args()
api = Agsv()

if a.config == "c2":
    doc, src = bench.profile_doc(api)
    base = bench.workload_config(1, 0, "wall", "agentserve", doc)
elif a.config == "c4":  # C4: Qwen2.5-7B-shaped, 64 agents, 8k system prompts
    prof = ROOT / "profiles" / "b200_profile_qwen2.5-7b.json"
    d = json.loads(prof.read_text())
    d.pop("measured", None)
    base = {"workload": {"paradigm": "react", "model": "qwen2.5-7b", "concurrency": 64,
                         "cold": {"min": 8192, "max": 8192, "mean": 8192},
                         "resume": {"min": 256, "max": 256, "mean": 256}},
            "slo": {"factor": 8.0, "tpot_stat": "p95"}, "policy": "agentserve", "seed": 13,
            "profile": {"inline": d},
            "backend": {"clock": "wall", "model": "qwen2.5-7b", "device": 0, "prefill_unit_tokens": 2048}}
    src = str(prof.relative_to(ROOT))
else:  # C3: Llama-3.2-3B-shaped, 32 ReAct agents
    prof = ROOT / "profiles" / "b200_profile_llama3.2-3b.json"
    d = json.loads(prof.read_text())
    d.pop("measured", None)
    base = {"workload": {"paradigm": "react", "model": "qwen2.5-3b", "concurrency": 32},
            "slo": {"factor": 8.0, "tpot_stat": "p95"}, "policy": "agentserve", "seed": 13,
            "profile": {"inline": d},
            "backend": {"clock": "wall", "model": "llama3.2-3b", "device": 0, "prefill_unit_tokens": 2048}}
    src = str(prof.relative_to(ROOT))

slots = json.loads(json.dumps(base["profile"]["inline"]))["total_sms"] // json.loads(json.dumps(base["profile"]["inline"]))["granularity"]
runs = [("agentserve", None), ("mixed_fcfs", None), ("chunked_prefill", None), ("agentserve_no_slots", None)]
runs += [("static_partition", k) for k in range(1, slots)]
if a.policies:
    want = [(x.split(":")[0], int(x.split(":")[1]) if ":" in x else None) for x in a.policies]
    runs = [r for r in runs if r in want]
rows = []
for pol, k in runs:
    cfg = json.loads(json.dumps(base))
    cfg["policy"] = pol
    if k is not None:
        cfg["static_decode_slots"] = k
    if a.horizon_ms:
        cfg["horizon_ms"] = a.horizon_ms
    ms = []
    for _ in range(a.reps):
        t = api.run(cfg)
        ms.append((t.metrics(), t))
    m0 = ms[-1][0]
    ver = json.loads(ms[-1][1].verify()[0])
    row = {"policy": pol, "static_decode_slots": k,
           "throughput_tps": round(statistics.median(m["throughput_tps"] for m, _ in ms), 1),
           "ttft_p50_ms": round(statistics.median(m["ttft_p50_ms"] for m, _ in ms), 3),
           "ttft_p99_ms": round(statistics.median(m["ttft_p99_ms"] for m, _ in ms), 3),
           "tpot_p50_ms": round(statistics.median(m["tpot_p50_ms"] for m, _ in ms), 3),
           "tpot_p99_ms": round(statistics.median(m["tpot_p99_ms"] for m, _ in ms), 3),
           "slo_attainment": m0.get("slo_attainment", m0.get("joint_slo_attainment")),
           "verify": {"checked": ver["checked"], "vacuous": ver["vacuous"], "violations": ver["violations"],
                      "min_rho": ver["min_rho"], "assumptions_met": ver["assumptions_met"]}}
    rows.append(row)
    print(json.dumps(row), flush=True)
doc = {"config": a.config, "profile": src, "reps": a.reps, "clock": "wall (B200, Green Context partitions)",
       "runs": rows}
if a.out:
    Path(a.out).write_text(json.dumps(doc, indent=1))
