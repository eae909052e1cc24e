"""The device forward at full model shape against transformers' modelling code in fp32 on the
same GPU, with the same generated weights, at the BASELINE configs' context lengths (two
prompts in one ragged prefill batch, then teacher-forced decode steps of both rows):
  C2 Qwen2.5-0.5B (24 layers, GQA 7, hd 64, q/k/v bias, tied 151936-token head), 2300 + 700;
  C3 Llama-3.2-3B (28 layers, GQA 3, hd 128, Llama-3 RoPE scaling, tied head), 3000 + 500.

This exercises the paths the small oracle cases cannot: long-context split-KV decode
attention, multi-tile GQA-packed prefill attention, and the decode GEMM paths the real
model's shapes select.  Tolerances are the device-vs-oracle ones of tests/test_forward_gpu.py
(bf16 storage against an fp32 reference); measured on a B200: max error 1.45% of max|logit|,
rel-L2 1.39% (0.5B); 4.86% / 4.60% (3B, see TOL); greedy ids identical in both.
"""
import numpy as np
import pytest

from oracle.forward import OracleModel, token_stream

torch = pytest.importorskip("torch")
pytest.importorskip("transformers")

pytestmark = pytest.mark.gpu

# (max |err| / max |logit|, rel-L2).  3B: the CPU oracle — the device's own bf16 rounding
# points, fp32 accumulation — is itself 2.8-3.8% from transformers' fp32 forward at every
# prompt length (64-3000 tokens, scripts/hf_diag.py, profiles/r1_hf_diag.txt): bf16
# activation rounding amplified through 28 random-weight layers.  The device sits at the same
# distance (3.6-4.3%), so the 3B bound is that noise floor plus margin, not a looser kernel.
TOL = {"qwen2.5-0.5b": (0.03, 0.02), "llama3.2-3b": (0.06, 0.06)}


@pytest.mark.parametrize("name,lens", [("qwen2.5-0.5b", (2300, 700)), ("llama3.2-3b", (3000, 500))])
def test_device_matches_transformers_at_config_lengths(name, lens):
    LOGIT_ATOL_FRAC, LOGIT_RL2 = TOL[name]
    from paper_2603_10342_b200.device import KvPool, Lane, Model
    from tests.test_oracle_pin_hf import _hf_model

    seed = 13
    steps = 4
    om = OracleModel(name, seed=seed, max_ctx=4096)
    hf = _hf_model(om, device="cuda")
    del om
    m = Model(name, seed=seed, max_context=4096)
    kv = KvPool(m, num_blocks=2 * (4096 // 64) + 8)
    lane = Lane(m, max_tokens=4096, max_segments=8)
    V = m.vocab
    prompts = [token_stream(seed, f"hfpin/{i}", n, V) for i, n in enumerate(lens)]
    lane.forward(kv, [(i, n, 1) for i, n in enumerate(lens)], np.concatenate(prompts))
    ids, lg = lane.fetch(len(lens), logits=True)
    seqs = [list(p) for p in prompts]
    dev_logits = [[lg[i]] for i in range(len(lens))]
    for _ in range(steps):
        nxt = [int(x) for x in ids]
        for i in range(len(lens)):
            seqs[i].append(nxt[i])
        lane.forward(kv, [(i, 1, 1) for i in range(len(lens))], nxt)
        ids, lg = lane.fetch(len(lens), logits=True)
        for i in range(len(lens)):
            dev_logits[i].append(lg[i])
    near_ties = 0
    worst = [0.0, 0.0]
    with torch.no_grad():
        for i, n in enumerate(lens):
            ref = hf(torch.tensor(seqs[i], device="cuda")[None]).logits[0].float().cpu().numpy()
            for k, dl in enumerate(dev_logits[i]):
                r = ref[n - 1 + k]
                err = np.abs(dl - r).max()
                assert err <= LOGIT_ATOL_FRAC * np.abs(r).max(), (i, k, err, np.abs(r).max())
                rl2 = np.linalg.norm(dl - r) / np.linalg.norm(r)
                assert rl2 <= LOGIT_RL2, (i, k, rl2)
                worst = [max(worst[0], err / np.abs(r).max()), max(worst[1], rl2)]
                # the device's greedy id (fed back as the next token) must be the reference's
                # argmax unless the reference's top-2 margin is within the measured error
                dev_id = seqs[i][n + k] if k < steps else int(np.argmax(dl))
                if dev_id != int(np.argmax(r)):
                    top2 = np.sort(r)[-2:]
                    assert top2[1] - top2[0] <= 2 * err, (i, k, dev_id, int(np.argmax(r)))
                    near_ties += 1
    print(f"worst max-err frac {worst[0]:.4f}, rel-L2 {worst[1]:.4f}, near-ties {near_ties}")
    assert near_ties <= 1
