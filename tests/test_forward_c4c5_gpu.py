"""Device forward at the C4 / C5 head layouts against the CPU fp32 oracle, full width,
layer-truncated, at the configs' context lengths (BASELINE configs[3], configs[4]; model rows
/root/reference/proj/src/workload.cpp:153-156):

  C4 Qwen2.5-7B  : d 3584, 28 q heads / 4 KV heads (GQA group 7 -> 126 of 128 packed MMA rows),
                   hd 128, q/k/v bias (fused bias + RoPE + paged append epilogue), untied
                   152064-token head; 8192-token cold prompt + a 3000-token one
  C5 Llama-3.1-8B: d 4096, 32 / 8 heads (GQA 4), hd 128, Llama-3 RoPE scaling, untied head;
                   3000 + 2500-token prompts

Prefill runs the way the engine runs a Q_P job: launch units of 2048 tokens, so every unit
after the first is a resume-style prefill over the session's cached context (prefix P > 0),
and the two sessions' units share ragged batches.  Then decode steps with three rows (the
two long contexts + a short third session) and a 16-token admitted-resume chunk riding along
(SURVEY §8(a) A1), teacher-forced with the device's ids.  Tolerances are those of
tests/test_forward_gpu.py; the near-tie count is printed (north_star: greedy ids bit-exact,
a mismatch is only accepted where the oracle's own top-2 margin is inside the measured
error, and at most a fifth of the ids per test; measured on a B200: C4 0 / 15, C5 2 / 15).

Every decode split-merge path and both prefill-attention decompositions are re-run at the C4
layout (G = 7, hd 128; one layer, 5000-token context) in a fresh process each, as tests/test_attn_paths_gpu.py
does at GQA 3.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle.forward import OracleModel, token_stream
from tests.test_forward_gpu import _cmp_logits, _kv_check

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
UNIT = 2048

# case -> (preset, decoder layers kept, context lengths)
CASES = {
    "c4": ("qwen2.5-7b", 2, (8192, 3000, 40)),
    "c5": ("llama3.1-8b", 2, (3000, 2500, 40)),
    # the merge-path re-runs: one layer (the CPU oracle dominates their cost), 5k context
    "c4_paths": ("qwen2.5-7b", 1, (5000, 1200, 40)),
}


def _ids_ok(dev_id, cpu_logits, err, stats):
    cpu_id = int(np.argmax(cpu_logits))
    if dev_id == cpu_id:
        stats["match"] += 1
        return
    top2 = np.sort(cpu_logits)[-2:]
    assert top2[1] - top2[0] <= 2 * err + 1e-6, f"greedy id {dev_id} vs oracle {cpu_id}, margin {top2[1] - top2[0]}"
    stats["near_tie"] += 1


@pytest.mark.parametrize("case", sorted(CASES))
def test_full_width_truncated_matches_oracle(case):
    from paper_2603_10342_b200.device import KvPool, Lane, Model

    name, LAYERS, lens = CASES[case]
    seed = 13
    steps = 4
    max_ctx = max(lens) + 128
    m = Model('{"preset":"%s","layers":%d}' % (name, LAYERS), seed=seed, max_context=max_ctx)
    assert m.info["layers"] == LAYERS and m.info["head_dim"] == 128
    blocks = sum((n + 64 + 63) // 64 for n in lens) + 8
    kv = KvPool(m, num_blocks=blocks)
    lane = Lane(m, max_tokens=UNIT * len(lens), max_segments=8)
    om = OracleModel(name, seed=seed, max_ctx=max_ctx, layers_limit=LAYERS)
    V = m.vocab
    osess = [om.session() for _ in lens]
    stats = {"match": 0, "near_tie": 0}
    worst = [0.0, 0.0]

    def track(dev, cpu, what):
        err = _cmp_logits(dev, cpu, what)
        scale = float(np.abs(cpu).max())
        worst[0] = max(worst[0], err / scale)
        worst[1] = max(worst[1], float(np.linalg.norm(dev - cpu) / np.linalg.norm(cpu)))
        return err

    # 1. prefill in 2048-token launch units; units of different sessions share a batch
    prompts = [token_stream(seed, f"tok/{i}/cold", n, V) for i, n in enumerate(lens)]
    done = [0] * len(lens)
    nxt = [None] * len(lens)
    while any(d < n for d, n in zip(done, lens)):
        segs, toks, last = [], [], []
        for i, n in enumerate(lens):
            if done[i] >= n:
                continue
            k = min(UNIT, n - done[i])
            fin = done[i] + k == n
            segs.append((i, k, 1 if fin else 0))
            toks.append(prompts[i][done[i]:done[i] + k])
            if fin:
                last.append(i)
            done[i] += k
        lane.forward(kv, segs, np.concatenate(toks))
        if last:
            ids, lg = lane.fetch(len(last), logits=True)
            for r, i in enumerate(last):
                _, clg = osess[i].forward(prompts[i])
                err = track(lg[r], clg, f"{case} prefill s{i}")
                _ids_ok(int(ids[r]), clg, err, stats)
                nxt[i] = int(ids[r])
        else:
            lane.wait()
    for i, n in enumerate(lens):
        assert kv.length(i) == n

    # 2. decode steps: every session one row; a 16-token resume chunk for session 2 in steps 1-2
    chunk = token_stream(seed, "tok/2/resume/0", 32, V)
    cpos = 0
    for step in range(steps):
        segs, toks = [], []
        for i in range(len(lens)):
            if i == 2 and 1 <= step < 3:
                segs.append((i, 16, 1))
                toks += list(chunk[cpos:cpos + 16])
                cpos += 16
            else:
                segs.append((i, 1, 1))
                toks.append(nxt[i])
        lane.forward(kv, segs, np.asarray(toks, dtype=np.int32))
        ids, lg = lane.fetch(len(segs), logits=True)
        off = 0
        for r, (s, n, _) in enumerate(segs):
            _, clg = osess[s].forward(toks[off:off + n])
            off += n
            err = track(lg[r], clg, f"{case} step {step} s{s}")
            _ids_ok(int(ids[r]), clg, err, stats)
            nxt[s] = int(ids[r])
    for i in range(len(lens)):
        assert kv.length(i) == osess[i].length
    # 3. KV contents: block and launch-unit boundaries, the newest decode tokens (the
    #    layer-limited oracle's KV readout spans the preset's full depth; keep the live layers)
    per = m.info["n_kv_heads"] * 128

    class _Live:
        def __init__(self, sess):
            self.sess = sess

        def read_kv(self, p):
            k, v = self.sess.read_kv(p)
            return k[:LAYERS * per], v[:LAYERS * per]

    for i in range(2):
        L = kv.length(i)
        pos = sorted(p for p in {0, 63, 64, UNIT - 1, UNIT, lens[i] - 1, L - 2, L - 1} if p < L)
        _kv_check(kv, i, _Live(osess[i]), pos, LAYERS, per)
    n = stats["match"] + stats["near_tie"]
    print(f"{case} {name} x{LAYERS} layers, contexts {lens}: {n} greedy ids, near-ties {stats['near_tie']}, "
          f"worst max-err frac {worst[0]:.4f}, rel-L2 {worst[1]:.4f}")
    # random-init 2-layer models have flat logits (top-2 margins of ~1e-3 of max|logit| are
    # common at 128-152k vocab); every mismatch above was checked to sit inside the measured
    # error, and at most a fifth of the ids may be such near-ties
    assert stats["near_tie"] <= max(1, n // 5), stats


@pytest.mark.parametrize("env", [
    {"ASB_DECODE_SPLITS": "3"},
    {"ASB_ATTN_NO_CLUSTER": "1", "ASB_DECODE_SPLITS": "16"},
    {"ASB_ATTN_COMBINE": "1", "ASB_ATTN_NO_CLUSTER": "1"},
    {"ASB_DECODE_MAX_SPLITS": "1"},
    {"ASB_PREFILL_UNITS": "0"},
    {"ASB_PREFILL_UNITS": "0", "ASB_PREFILL_SPLITS": "3"},
    {"ASB_DECODE_PERSIST": "1"},
    {"ASB_TGEMV": "1"},
    {"ASB_CHUNK_AS_DECODE": "0"},
], ids=["cluster3", "last_arriver16", "combine", "single", "prefill_uniform", "prefill_uniform3", "persistent",
        "tgemv_all", "chunk_as_prefill"])
def test_c4_layout_merge_paths(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-s", "-p", "no:cacheprovider",
                        "tests/test_forward_c4c5_gpu.py::test_full_width_truncated_matches_oracle[c4_paths]"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "1 passed" in r.stdout
    print([ln for ln in r.stdout.splitlines() if "near-ties" in ln])
