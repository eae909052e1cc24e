"""Episodes for compute-sanitizer (memcheck / racecheck / synccheck): a lockstep C1 episode
(every decode step and prefill unit executed on the device in the simulator's order) and a
short wall-clock episode per policy (decode and prefill lanes co-running on complementary
Green Context partitions over one shared KV pool, rebinds in flight).

  compute-sanitizer --tool memcheck python scripts/sanitize_episode.py [--quick]
"""
import json
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_10342_b200 import workloads  # noqa: E402
from paper_2603_10342_b200.agsv import Agsv  # noqa: E402

quick = "--quick" in sys.argv
api = Agsv()
td = tempfile.mkdtemp()

c1 = workloads.run_config("c1", clock="lockstep", policy="agentserve")
if quick:
    c1["workload"]["cold"] = {"min": 300, "max": 300, "mean": 300}
    c1["workload"]["decode"] = {"min": 8, "max": 8, "mean": 8}
t = api.run(c1)
st, rep = t.replay()
print(json.dumps({"episode": "c1 lockstep agentserve", "replay_status": st,
                  "tokens": t.metrics()["throughput_tps"]}), flush=True)

wall = {"workload": {"paradigm": "react", "concurrency": 4, "stagger_ms": 5.0, "steps_per_session": 2,
                     "cold": {"min": 400, "max": 400, "mean": 400},
                     "resume": {"min": 300, "max": 300, "mean": 300},
                     "decode": {"min": 6, "max": 10, "mean": 8},
                     "tool_delay": {"kind": "fixed", "ms": 3.0}},
        "slo": {"tau_tpot_ms": 20.0, "tau_ttft_ms": 2000.0}, "seed": 13,
        "controller": {"delta_t_ms": 20.0},
        "backend": {"clock": "wall", "model": "tiny", "prefill_unit_tokens": 128, "lend_idle_prefill": True}}
for pol in (["agentserve"] if quick else ["agentserve", "mixed_fcfs", "static_partition"]):
    cfg = json.loads(json.dumps(wall))
    cfg["policy"] = pol
    if pol == "static_partition":
        cfg["static_decode_slots"] = 3
    t = api.run(cfg)
    st, rep = t.replay()
    foot = json.loads(t.jsonl(td).splitlines()[-1])
    print(json.dumps({"episode": f"wall {pol}", "replay_status": st, "green_contexts": foot["device"]["green_contexts"],
                      "rebinds": foot["device"].get("rebind_us", {}).get("n")}), flush=True)
print("sanitize episodes done")
