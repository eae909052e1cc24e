"""Multi-GPU = session-sharded replicas with no collective.  Sharding must
partition the global workload exactly (plans are independent of the shard count because
every session draws from its own named sub-stream), and bench.py under torchrun (gloo,
world size 2, virtual clock on CPU) must aggregate into one whole-job JSON line."""
import json
import os
import socket
import subprocess
import sys
import tempfile
from pathlib import Path

import pytest

from paper_2603_10342_b200.agsv import Agsv

ROOT = Path(__file__).resolve().parents[1]


def _sessions(api, cfg):
    td = tempfile.mkdtemp()
    return [json.loads(x) for x in api.run(cfg).jsonl(td).splitlines() if '"rec":"session"' in x]


def test_shards_partition_the_global_workload(built_lib):
    api = Agsv()
    base = {"workload": {"paradigm": "react", "concurrency": 12}, "policy": "agentserve", "seed": 13}
    full = _sessions(api, base)
    for n in (2, 3, 4):
        seen = {}
        for r in range(n):
            cfg = json.loads(json.dumps(base))
            cfg["workload"].update({"shard_index": r, "shard_count": n})
            for k, s in enumerate(_sessions(api, cfg)):
                gid = r + k * n
                seen[gid] = s
        assert sorted(seen) == list(range(12))
        for gid, s in seen.items():
            g = full[gid]
            for key in ("arrival", "cold_len", "decode_lens", "resume_lens", "tool_delays", "rounds"):
                assert s[key] == g[key], (n, gid, key)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun_bench(n, extra):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    env.pop("BENCH_BACKEND", None)  # the harness defaults to gloo (sessions exchange nothing)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", str(n), "--steps", "1", "--warmup", "1", "--sim-clock", "--no-cpu", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_torchrun_gloo_two_ranks(built_lib):
    d = _torchrun_bench(2, [])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["config"] == "C3"
    assert d["latency_ms"]["sessions"] == 64  # 32 agents per rank, both ranks counted
    assert d["value"] > 0
    # both policies of the same episodes in one line, pooled over ranks
    assert set(d["policies"]) == {"agentserve", "mixed_fcfs"}
    assert d["policies"]["mixed_fcfs"]["sessions"] == 64
    assert d["tails_vs_mixed_fcfs"]["tpot_p99"] is not None


def test_bench_torchrun_gloo_eight_ranks_c5(built_lib):
    """C5: Llama-3.1-8B-shaped, 64 agents per GPU as session-sharded replicas; world size 8 on
    gloo (the driver's 8-GPU scaling launch), whole-job aggregation on rank 0."""
    d = _torchrun_bench(8, ["--config", "c5", "--compare", "none"])
    assert d["n_gpus"] == 8 and d["config"]["config"] == "C5"
    assert d["config"]["agents_per_gpu"] == 64
    assert d["latency_ms"]["sessions"] == 512
    assert d["value"] > 0 and d["policies"]["agentserve"]["tpot_gaps"] > 0


@pytest.mark.parametrize("env,want", [
    ({"LOCAL_RANK": "3"}, (3, 3)),                                  # torchrun, all GPUs visible
    ({"LOCAL_RANK": "3", "CUDA_VISIBLE_DEVICES": "5"}, (0, 5)),     # launcher pins one GPU per rank
    ({"LOCAL_RANK": "1", "CUDA_VISIBLE_DEVICES": "4,6"}, (1, 6)),   # a visible subset
    ({}, (0, 0)),
])
def test_bench_device_index(monkeypatch, env, want):
    """One rank per GPU: the CUDA ordinal the rank binds (and the physical index nvidia-smi
    samples) for the launch patterns the driver may use."""
    import bench
    for k in ("LOCAL_RANK", "CUDA_VISIBLE_DEVICES"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    assert bench.device_index() == want
