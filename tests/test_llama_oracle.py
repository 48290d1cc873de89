"""Pin the LM oracle (oracle/llama.py) to the published algorithm: [3P] transformers
5.5.0 LlamaForCausalLM / Qwen2ForCausalLM loaded with the oracle's own weights.

The oracle restates the Llama / Qwen2 decoder with the GPU's rounding points (bf16
GEMM inputs).  With those rounding points switched off (bf16_round -> identity) it
must reproduce transformers' fp64 forward to fp32 accuracy -- RoPE convention
(rotate_half), GQA grouping, RMSNorm, SiLU-gated MLP, q|k|v bias, tied head;
with them on, the difference is the bf16 activation rounding only.  CPU only.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

import oracle.llama as ol  # noqa: E402
from oracle.weights import BackboneWeights  # noqa: E402
from paper_2602_00269_b200.config import tiny, tiny_cosy  # noqa: E402


def _hf_model(cfg, w):
    common = dict(vocab_size=cfg.vocab, hidden_size=cfg.d_model, intermediate_size=cfg.d_ff,
                  num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                  num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.rms_eps,
                  rope_theta=cfg.rope_theta, tie_word_embeddings=True, max_position_embeddings=cfg.max_ctx)
    if cfg.qkv_bias:
        mcfg = transformers.Qwen2Config(**common)
        model = transformers.Qwen2ForCausalLM(mcfg)
    else:
        mcfg = transformers.LlamaConfig(attention_bias=False, mlp_bias=False, **common)
        model = transformers.LlamaForCausalLM(mcfg)
    model = model.double().eval()
    H, KV, hd, dff = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_ff
    t = lambda a: torch.from_numpy(np.asarray(a, np.float64))  # noqa: E731
    with torch.no_grad():
        model.model.embed_tokens.weight.copy_(t(w.emb))
        for l, L in enumerate(w.layers):
            lay = model.model.layers[l]
            qkv = L["qkv"]
            lay.self_attn.q_proj.weight.copy_(t(qkv[: H * hd]))
            lay.self_attn.k_proj.weight.copy_(t(qkv[H * hd:(H + KV) * hd]))
            lay.self_attn.v_proj.weight.copy_(t(qkv[(H + KV) * hd:]))
            if cfg.qkv_bias:
                b = L["qkv_bias"]
                lay.self_attn.q_proj.bias.copy_(t(b[: H * hd]))
                lay.self_attn.k_proj.bias.copy_(t(b[H * hd:(H + KV) * hd]))
                lay.self_attn.v_proj.bias.copy_(t(b[(H + KV) * hd:]))
            lay.self_attn.o_proj.weight.copy_(t(L["o"]))
            lay.mlp.gate_proj.weight.copy_(t(L["gu"][:dff]))
            lay.mlp.up_proj.weight.copy_(t(L["gu"][dff:]))
            lay.mlp.down_proj.weight.copy_(t(L["down"]))
            lay.input_layernorm.weight.copy_(t(L["norm_attn"]))
            lay.post_attention_layernorm.weight.copy_(t(L["norm_mlp"]))
        model.model.norm.weight.copy_(t(w.norm_final))
    return model


@pytest.mark.parametrize("family", ["llama", "qwen2"])
def test_oracle_matches_transformers(family, monkeypatch):
    # config-1 geometry (a reduced vocabulary keeps the CPU test small)
    base = tiny() if family == "llama" else tiny_cosy()
    cfg = base.with_capacity(vocab=6000, text_vocab=5000, audio_base=-1, max_ctx=128)
    w = BackboneWeights(cfg, seed=77)
    model = _hf_model(cfg, w)
    rng = np.random.default_rng(3)
    toks = rng.integers(0, cfg.text_vocab, size=40)
    with torch.no_grad():
        ref = model(torch.from_numpy(toks[None])).logits[0].numpy()

    # rounding points off: the same algorithm, fp32 vs transformers' fp64
    monkeypatch.setattr(ol, "bf16_round", lambda a: np.asarray(a, np.float32))
    exact, _ = ol.LlamaOracle(cfg, 77, weights=w).forward("r", toks, np.arange(len(toks)))
    err = np.abs(exact - ref).max() / np.abs(ref).max()
    assert err < 1e-4, err
    monkeypatch.undo()

    # the GPU's rounding points (bf16 GEMM inputs): bf16-level deviation only
    got, _ = ol.LlamaOracle(cfg, 77, weights=w).forward("r", toks, np.arange(len(toks)))
    rel = np.sqrt(np.mean((got - ref) ** 2) / np.mean(ref ** 2))
    assert rel < 3e-2, rel
    agree = np.mean(got.argmax(-1) == ref.argmax(-1))
    assert agree > 0.9, agree
