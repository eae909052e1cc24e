"""Pins the forward oracle (oracle/forward.c) to an independent implementation of the same
decoder math: HuggingFace transformers' Llama / Qwen2 modelling code (transformers 5.5.0 as
installed in the image), run in fp32 on CPU with the oracle's own generated weights.

The reference has no model inside (its executor is a latency model), so the
forward oracle cannot be pinned to it; this test pins the decoder conventions the oracle and
the device kernels share — RMSNorm, rotate-half RoPE (default and Llama-3 frequency scaling),
GQA head grouping, Qwen2 q/k/v bias, SwiGLU, tied / untied LM heads — to a public
implementation.  The oracle rounds activations to bf16 at the device's rounding points and
transformers stays in fp32, so logits agree to bf16 noise (measured: max error 0.3-0.5% of
max|logit|, rel-L2 0.4-0.5%); the bound is 1%, tighter than the device test's 3% / 2%, and a
wrong RoPE theta or a mis-grouped KV head exceeds it (1.2-8.7%).  Greedy ids must match
except at near-ties.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

from oracle.forward import OracleModel, token_stream  # noqa: E402

LOGIT_ATOL_FRAC = 0.01
LOGIT_RL2 = 0.01

SPECS = {
    # Llama layout, hd 64, GQA 2, tied head
    "tiny": "tiny",
    # Qwen2 layout: q/k/v bias, theta 1e6, untied head
    "qwen_bias": dict(layers=2, d=256, hq=4, hkv=2, hd=64, ffn=512, vocab=4096, tied=0, qkv_bias=1,
                      theta=1e6, eps=1e-6),
    # Llama-3.2 layout: hd 128, GQA 3, Llama-3 RoPE frequency scaling
    "llama3_rope": dict(layers=2, d=384, hq=6, hkv=2, hd=128, ffn=512, vocab=4096, tied=1, qkv_bias=0,
                        theta=5e5, eps=1e-5, rope_llama3=1, rope_factor=32.0, rope_lo=1.0, rope_hi=4.0,
                        rope_orig=8192.0),
}


def _hf_model(om: OracleModel, device: str = "cpu"):
    s = om.spec
    rope = {"rope_type": "default", "rope_theta": float(s.theta)}
    if s.rope_llama3:
        rope = {"rope_type": "llama3", "rope_theta": float(s.theta), "factor": float(s.rope_factor),
                "low_freq_factor": float(s.rope_lo), "high_freq_factor": float(s.rope_hi),
                "original_max_position_embeddings": int(s.rope_orig)}
    common = dict(vocab_size=s.vocab, hidden_size=s.d, intermediate_size=s.ffn, num_hidden_layers=s.layers,
                  num_attention_heads=s.hq, num_key_value_heads=s.hkv, head_dim=s.hd,
                  rms_norm_eps=float(s.eps), rope_parameters=rope, tie_word_embeddings=bool(s.tied),
                  max_position_embeddings=131072 if s.rope_llama3 else 4096)
    with torch.device(device):
        if s.qkv_bias:
            cfg = transformers.Qwen2Config(**common)
            model = transformers.Qwen2ForCausalLM(cfg)
        else:
            cfg = transformers.LlamaConfig(attention_bias=False, mlp_bias=False, **common)
            model = transformers.LlamaForCausalLM(cfg)
    cfg._attn_implementation = "eager"
    model = model.float().eval()

    def t(name, shape, layer=-1):
        return torch.from_numpy(om.tensor(name, layer).reshape(shape))

    qd, kvd = s.hq * s.hd, s.hkv * s.hd
    with torch.no_grad():
        model.model.embed_tokens.weight.copy_(t("embed", (s.vocab, s.d)))
        model.model.norm.weight.copy_(t("final_norm", (s.d,)))
        if not s.tied:
            model.lm_head.weight.copy_(t("lm_head", (s.vocab, s.d)))
        for l, layer in enumerate(model.model.layers):
            a, m = layer.self_attn, layer.mlp
            layer.input_layernorm.weight.copy_(t("attn_norm", (s.d,), l))
            layer.post_attention_layernorm.weight.copy_(t("mlp_norm", (s.d,), l))
            a.q_proj.weight.copy_(t("q", (qd, s.d), l))
            a.k_proj.weight.copy_(t("k", (kvd, s.d), l))
            a.v_proj.weight.copy_(t("v", (kvd, s.d), l))
            a.o_proj.weight.copy_(t("o", (s.d, qd), l))
            if s.qkv_bias:
                a.q_proj.bias.copy_(t("q_bias", (qd,), l))
                a.k_proj.bias.copy_(t("k_bias", (kvd,), l))
                a.v_proj.bias.copy_(t("v_bias", (kvd,), l))
            m.gate_proj.weight.copy_(t("gate", (s.ffn, s.d), l))
            m.up_proj.weight.copy_(t("up", (s.ffn, s.d), l))
            m.down_proj.weight.copy_(t("down", (s.d, s.ffn), l))
    if s.tied:
        assert model.lm_head.weight.data_ptr() == model.model.embed_tokens.weight.data_ptr()
    return model


@pytest.mark.parametrize("spec", list(SPECS))
def test_oracle_matches_transformers(spec):
    seed = 13
    om = OracleModel(SPECS[spec], seed=seed, max_ctx=2048)
    model = _hf_model(om)
    V = om.spec.vocab
    prompt = token_stream(seed, f"pin/{spec}", 1200, V)
    extra = token_stream(seed, f"pin/{spec}/decode", 4, V)
    seq = np.concatenate([prompt, extra])
    with torch.no_grad():
        hf = model(torch.from_numpy(seq.astype(np.int64))[None]).logits[0].float().numpy()
    sess = om.session()
    outs = [sess.forward(prompt)]
    for tok in extra[:-1]:
        outs.append(sess.forward([tok]))
    near_ties = 0
    for i, (nxt, lg) in enumerate(outs):
        ref = hf[len(prompt) - 1 + i]
        err = np.abs(lg - ref).max()
        assert err <= LOGIT_ATOL_FRAC * np.abs(ref).max(), (spec, i, err, np.abs(ref).max())
        assert np.linalg.norm(lg - ref) / np.linalg.norm(ref) <= LOGIT_RL2, (spec, i)
        if nxt != int(np.argmax(ref)):
            top2 = np.sort(ref)[-2:]
            assert top2[1] - top2[0] <= 2 * err, (spec, i, nxt, int(np.argmax(ref)))
            near_ties += 1
    assert near_ties <= 1
