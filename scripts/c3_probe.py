"""C3-shaped wall-clock episode (Llama-3.2-3B, ReAct qwen2.5-3b row) at a given concurrency,
for diagnosing episode length/scaling.  python scripts/c3_probe.py N [policy] [model]"""
import faulthandler
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_10342_b200.agsv import Agsv  # noqa: E402

if os.environ.get("C3_DUMP_AFTER"):  # print the Python stack if the run is still going
    faulthandler.dump_traceback_later(float(os.environ["C3_DUMP_AFTER"]))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
pol = sys.argv[2] if len(sys.argv) > 2 else "agentserve"
model = sys.argv[3] if len(sys.argv) > 3 else "llama3.2-3b"
d = json.loads((ROOT / "profiles" / "b200_profile_llama3.2-3b.json").read_text())
d.pop("measured", None)
cfg = {"workload": {"paradigm": "react", "model": "qwen2.5-3b", "concurrency": n},
       "slo": {"factor": 8.0, "tpot_stat": "p95"}, "policy": pol, "seed": 13, "profile": {"inline": d},
       "backend": {"clock": "wall", "model": model, "device": 0, "prefill_unit_tokens": 2048}}
t0 = time.time()
tr = Agsv().run(cfg)
m = tr.metrics()
print(json.dumps({"n": n, "policy": pol, "model": model, "wall_s": round(time.time() - t0, 2),
                  **{k: round(v, 3) for k, v in m.items() if isinstance(v, float)}}), flush=True)
