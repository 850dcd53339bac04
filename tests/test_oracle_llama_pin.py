"""Pin of the oracle's layer COMPOSITION (oracle/model.py layer_forward / forward_chain) against an
implementation written by someone else: `transformers`' LlamaForCausalLM, run in fp64.

What this pins (R19): residual placement (h1 = h + O-proj,
h2 = h1 + MLP(RMSNorm(h1))), the MLP input (ffn_norm of h1, not of h), SwiGLU order
(silu(gate) * up, gate rows first), the final norm on h2, GQA head mapping (q head hq -> kv head
hq // G), rotate_half RoPE at absolute positions, causal attention over cache + chain, the
q | k | v row split of wqkv, the untied lm-head, and that the cache the oracle keeps (post-RoPE K)
reproduces a full-sequence forward.

How: the oracle's bf16 rounding points (`round_bf16`, a design decision of S10, pinned on its own
in test_oracle_numerics.py) are switched to the identity, and both sides get the same fp64 RoPE
table (HF computes its angles in fp32; the table itself is pinned by test_oracle_model.py). Then
both compute the same real-number function. HF upcasts its RMSNorm and its softmax to fp32 even in
an fp64 model, so the two agree to fp32 rounding (~1e-7 of the logit scale; bound 2e-6), while any
composition slip moves logits by > 1e-3 of the scale (test_composition_slips_are_detected). The oracle
builds its cache by running the prompt through forward_chain itself; HF runs the whole sequence
(prompt + chain) in one causal forward.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import model

transformers = pytest.importorskip("transformers")
TOL = 2e-6          # HF's fp32 RMSNorm / softmax inside an fp64 model


def _hf_model(cfg, w):
    from transformers import LlamaConfig, LlamaForCausalLM
    hc = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model, intermediate_size=max(cfg.ffn_dim, 1),
                     num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_q_heads,
                     num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.norm_eps,
                     rope_theta=cfg.rope_theta, max_position_embeddings=cfg.max_pos, attention_bias=False,
                     mlp_bias=False, tie_word_embeddings=False, hidden_act="silu")
    hc._attn_implementation = "eager"
    m = LlamaForCausalLM(hc).to(torch.float64).eval()
    t = {k: v.to(torch.float64) for k, v in w.items()}
    nq, nk = cfg.n_q_heads * cfg.head_dim, cfg.n_kv_heads * cfg.head_dim
    F = cfg.ffn_dim
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(t["embed"])
        for i, lyr in enumerate(m.model.layers):
            lyr.input_layernorm.weight.copy_(t["attn_norm"][i])
            lyr.self_attn.q_proj.weight.copy_(t["wqkv"][i][:nq])
            lyr.self_attn.k_proj.weight.copy_(t["wqkv"][i][nq:nq + nk])
            lyr.self_attn.v_proj.weight.copy_(t["wqkv"][i][nq + nk:])
            lyr.self_attn.o_proj.weight.copy_(t["wo"][i])
            lyr.post_attention_layernorm.weight.copy_(t["ffn_norm"][i])
            if F > 0:
                lyr.mlp.gate_proj.weight.copy_(t["w_gate_up"][i][:F])
                lyr.mlp.up_proj.weight.copy_(t["w_gate_up"][i][F:])
                lyr.mlp.down_proj.weight.copy_(t["w_down"][i])
            else:                                   # ffn_dim = 0: no MLP (an exact zero branch)
                lyr.mlp.down_proj.weight.zero_()
        m.model.norm.weight.copy_(t["final_norm"])
        m.lm_head.weight.copy_(t["lm_head"])
    return m


class _Rotary(torch.nn.Module):
    """HF rotary-embedding stand-in returning the fp64 table (cos, sin duplicated over both halves,
    HF's rotate_half layout) at the requested positions."""

    def __init__(self, cos, sin):
        super().__init__()
        self.cos = torch.from_numpy(np.concatenate([cos, cos], axis=-1))
        self.sin = torch.from_numpy(np.concatenate([sin, sin], axis=-1))

    def forward(self, x, position_ids):
        return self.cos[position_ids].to(x.dtype), self.sin[position_ids].to(x.dtype)


def _fp64_table(cfg):
    m = np.arange(cfg.head_dim // 2, dtype=np.float64)
    ang = np.arange(cfg.max_pos, dtype=np.float64)[:, None] / np.power(float(cfg.rope_theta), 2.0 * m / cfg.head_dim)
    return np.cos(ang), np.sin(ang)


@pytest.mark.parametrize("name,layers", [("toy", 1), ("toy_mlp", 1), ("toy_mlp", 2), ("gqa", 2)])
def test_forward_chain_matches_transformers_llama(monkeypatch, name, layers):
    if name == "gqa":      # GQA (G = 4), head_dim 64, norm gains != 1, an MLP: every composition path
        cfg = synth.TOY_MLP.with_(n_q_heads=8, n_kv_heads=2, d_model=256, ffn_dim=192, n_layers=layers)
    else:
        cfg = synth.CONFIGS[name].with_(n_layers=layers)
    w = synth.model_weights(cfg, seed=7, norm_one=False, std=0.08)
    monkeypatch.setattr(model, "round_bf16", lambda x: np.asarray(x, dtype=np.float64))
    cos, sin = _fp64_table(cfg)
    wnp = {k: v.to(torch.float64).numpy() for k, v in w.items()}

    rng = np.random.default_rng(layers * 31 + len(name))
    n_prompt, k = 23, 5
    seq = [int(t) for t in rng.integers(0, cfg.vocab, size=n_prompt + k + 1)]
    # oracle: the prompt with an empty cache, then the chain [pending, d_1..d_k] over that cache
    empty = [(np.zeros((0, cfg.n_kv_heads, cfg.head_dim)),) * 2 for _ in range(cfg.n_layers)]
    _, lp, kv = model.forward_chain(wnp, seq[:n_prompt], np.arange(n_prompt), empty, cfg, cos, sin)
    caches = [(kk, vv) for kk, vv in kv]
    pos = np.arange(n_prompt, n_prompt + k + 1)
    _, lc, _ = model.forward_chain(wnp, seq[n_prompt:], pos, caches, cfg, cos, sin)

    hf = _hf_model(cfg, w)
    hf.model.rotary_emb = _Rotary(cos, sin)
    with torch.no_grad():
        ref = hf(torch.tensor([seq]), use_cache=False).logits[0].numpy()
    scale = np.abs(ref).max()
    assert np.max(np.abs(lp - ref[:n_prompt])) <= TOL * scale
    assert np.max(np.abs(lc - ref[n_prompt:])) <= TOL * scale


def test_composition_slips_are_detected(monkeypatch):
    """The pin has power: plausible slips in the composition (a dropped attention residual, gate and
    up swapped in SwiGLU) move the logits far outside the TOL band."""
    cfg = synth.TOY_MLP
    w = synth.model_weights(cfg, seed=3, norm_one=False, std=0.08)
    monkeypatch.setattr(model, "round_bf16", lambda x: np.asarray(x, dtype=np.float64))
    cos, sin = _fp64_table(cfg)
    wnp = {k: v.to(torch.float64).numpy() for k, v in w.items()}
    seq = list(range(3, 14))
    empty = [(np.zeros((0, cfg.n_kv_heads, cfg.head_dim)),) * 2]
    hf = _hf_model(cfg, w)
    hf.model.rotary_emb = _Rotary(cos, sin)
    with torch.no_grad():
        ref = hf(torch.tensor([seq]), use_cache=False).logits[0].numpy()

    def err():
        _, lg, _ = model.forward_chain(wnp, seq, np.arange(len(seq)), empty, cfg, cos, sin)
        return np.max(np.abs(lg - ref)) / np.abs(ref).max()

    assert err() <= TOL
    with monkeypatch.context() as m:
        m.setattr(model, "attn_out", lambda h, o, wo: np.asarray(o, dtype=np.float64) @ np.asarray(wo).T)
        assert err() > 1e-3
    with monkeypatch.context() as m:
        F = cfg.ffn_dim
        m.setattr(model, "swiglu", lambda b, wgu: (lambda W: model.silu(b @ W[F:].T) * (b @ W[:F].T))(
            np.asarray(wgu, dtype=np.float64)))
        assert err() > 1e-3
