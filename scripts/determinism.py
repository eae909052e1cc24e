"""Run-to-run determinism of the decode forward: the same prompts prefilled into fresh sessions,
then the same decode steps, N times; every run's logits must be bit-identical to the first (all
reductions are fixed-order).  A mismatch is a race.  Env switches select the paths under test.

  python scripts/determinism.py [model] [trials] [steps]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.forward import token_stream  # noqa: E402
from paper_2603_10342_b200.device import KvPool, Lane, Model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3.2-3b"
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 6
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
lens = (3000, 500)
m = Model(name, seed=13, max_context=4096)
kv = KvPool(m, num_blocks=(trials + 1) * 2 * (4096 // 64))
lane = Lane(m, max_tokens=4096, max_segments=8)
V = m.vocab
prompts = [token_stream(13, f"hfpin/{i}", n, V) for i, n in enumerate(lens)]
ref = None
fed = []  # the token rows trial 0 fed at each decode step (its own greedy ids); later trials replay them
bad = 0
for tr in range(trials):
    sids = [100 * (tr + 1) + i for i in range(len(lens))]
    lane.forward(kv, [(s, n, 1) for s, n in zip(sids, lens)], np.concatenate(prompts))
    ids, lg = lane.fetch(len(lens), logits=True)
    outs = [lg.copy()]
    for k in range(steps):
        if tr == 0:
            fed.append([int(x) for x in ids])
        lane.forward(kv, [(s, 1, 1) for s in sids], fed[k])
        ids, lg = lane.fetch(len(lens), logits=True)
        outs.append(lg.copy())
    if ref is None:
        ref = outs
    else:
        for k, (a, b) in enumerate(zip(ref, outs)):
            d = float(np.abs(a - b).max())
            if d != 0.0:
                bad += 1
                print(f"trial {tr} step {k}: max |diff| {d:.4g} (rows differing: "
                      f"{[int(i) for i in np.where(np.abs(a - b).max(axis=1) > 0)[0]]})")
    if "--keep" not in sys.argv:
        for s in sids:
            kv.release(s)
print(f"{name}: {trials} trials x {steps} decode steps, {bad} mismatching steps")
