"""Anatomy of one bench.py serving episode (C2, wall clock, AgentServe policy).

Prints the decode-step device time by batch composition, the decode SM level over time, the
prefill units, and how TPOT gaps split into device time vs host/scheduling time.

  python scripts/episode_stats.py [--policy agentserve] [--episodes 2]
"""
import argparse
import collections
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2603_10342_b200.agsv import Agsv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--policy", default="agentserve")
ap.add_argument("--episodes", type=int, default=2)
ap.add_argument("--calibrated-slo", action="store_true", help="SLO from the profile (calibrate_slo, factor 8)")
a = ap.parse_args()
api = Agsv()
doc, _ = bench.profile_doc(api)
cfg = bench.workload_config(1, 0, "wall", a.policy, doc)
if a.calibrated_slo:
    cfg["slo"] = {"factor": 8.0, "tpot_stat": "p95"}
td = tempfile.mkdtemp()
for ep in range(a.episodes):
    tr = api.run(cfg)
    recs = [json.loads(x) for x in tr.jsonl(td).splitlines()]
m = tr.metrics()
kinds = collections.Counter(r.get("k") for r in recs)
print("record kinds:", dict(kinds))
for k in ("step_done", "prefill_done", "tick", "rebind"):
    ex = [r for r in recs if r.get("k") == k][:1]
    if ex:
        print(f"example {k}:", json.dumps(ex[0])[:400])
steps = [r for r in recs if r.get("k") == "step_done"]
by = collections.defaultdict(list)
for r in steps:
    b = len(r.get("emit", []))
    ch = 1 if r.get("chunk_session", r.get("chunk", -1)) not in (-1, None) else 0
    by[(b, ch)].append(r.get("dev_ms", float("nan")))
print("decode steps by (rows emitted, has chunk): n, dev_ms p50/p90")
for key in sorted(by):
    v = np.array(by[key], dtype=float)
    print(f"  {key}: n={len(v)} p50={np.nanmedian(v):.3f} p90={np.nanpercentile(v, 90):.3f}")
dev = np.array([r.get("dev_ms", np.nan) for r in steps], dtype=float)
t = np.array([r["t"] for r in steps], dtype=float)
gaps = np.diff(t)
print(f"steps={len(steps)} device ms total {np.nansum(dev):.1f}; step spacing p50 {np.median(gaps):.3f} ms; "
      f"dev p50 {np.nanmedian(dev):.3f} ms; episode end {m.get('end_ms', t[-1] if len(t) else 0):.1f} ms")
print("metrics:", {k: m[k] for k in m if k.endswith("_ms") or k in ("throughput_tps",)})
foot = recs[-1]
ticks = [r["summary"] for r in recs if r.get("k") == "tick"]
print("ticks (t1, dslots, tpot, b):", [(round(x["t1"]), x["dslots"], round(x["tpot"], 2) if x.get("tpot") else None, x["b"]) for x in ticks])
