"""Device vs transformers logits error by model / prompt length (diagnostic for
tests/test_device_vs_hf_gpu.py).  python scripts/hf_diag.py name len1 [len2 ...]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.forward import OracleModel, token_stream  # noqa: E402
from paper_2603_10342_b200.device import KvPool, Lane, Model  # noqa: E402
from tests.test_oracle_pin_hf import _hf_model  # noqa: E402

name = sys.argv[1]
lens = [int(x) for x in sys.argv[2:]]
om = OracleModel(name, seed=13, max_ctx=4096)
hf = _hf_model(om, device="cuda")
m = Model(name, seed=13, max_context=4096)
for n in lens:
    kv = KvPool(m, num_blocks=4096 // 64 + 8)
    lane = Lane(m, max_tokens=4096, max_segments=4)
    p = token_stream(13, f"diag/{n}", n, m.vocab)
    lane.forward(kv, [(0, n, 1)], p)
    ids, lg = lane.fetch(1, logits=True)
    with torch.no_grad():
        ref = hf(torch.tensor(p, device="cuda")[None]).logits[0, -1].float().cpu().numpy()
    d = lg[0]
    print(f"{name} T={n}: max err frac {np.abs(d-ref).max()/np.abs(ref).max():.4f} rel-L2 {np.linalg.norm(d-ref)/np.linalg.norm(ref):.4f} "
          f"max|ref| {np.abs(ref).max():.3f} argmax dev {int(np.argmax(d))} ref {int(np.argmax(ref))}", flush=True)
    # oracle on short prompts only (CPU)
    if n <= 256:
        _, ol = om.session().forward(p)
        print(f"   oracle vs hf: max err frac {np.abs(ol-ref).max()/np.abs(ref).max():.4f} rel-L2 {np.linalg.norm(ol-ref)/np.linalg.norm(ref):.4f}; "
              f"dev vs oracle {np.abs(d-ol).max()/np.abs(ol).max():.4f} / {np.linalg.norm(d-ol)/np.linalg.norm(ol):.4f}", flush=True)
    del lane, kv
