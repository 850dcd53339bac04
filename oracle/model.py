"""Stage functions of the single Llama-shaped decoder layer + lm-head, in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The model is SURVEY.md §8(c) step 1 ("Model forward"), the "bf16 operands,
fp32 accumulation" model of north_star evaluated exactly (fp64) from bf16
operands, with bf16 rounding exactly where the GPU path stores bf16 (MMA
operands and the KV cache). Each function below is one stage so that parity
can be graded teacher-forced: the test feeds each
stage the GPU's own inputs to that stage.

    step 1.1  h = E[c]
    step 1.2  a = bf16(RMSNorm(h) * g_attn),  RMSNorm(x) = x / sqrt(mean(x^2) + eps)
    step 1.3  q, k, v = a Wq^T, a Wk^T, a Wv^T
    step 1.4  RoPE (rotate_half) at absolute position P, then q,k,v <- bf16(.)
    step 1.5  softmax(q k^T / sqrt(d_h)) over cache keys 0..L-1 and chain keys 0..j
    step 1.6  o <- bf16(o); h <- h + o Wo^T
    step 1.7  b = bf16(RMSNorm(h) g_ffn); u = bf16(silu(b Wg^T) * (b Wu^T)); h <- h + u Wd^T
    step 1.8  z = bf16(RMSNorm(h) g_final); logits = z W_lm^T (fp64, unrounded)

RoPE frequencies theta^(-2m/d_h), m = 0..d_h/2-1 (Llama/HF rotate_half); the
cos/sin table is computed in fp64 and stored as fp32 (SURVEY.md §8(c) "Model
details fixed for both paths").

Pinned by tests/test_oracle_model.py: attention vs torch
scaled_dot_product_attention (fp64, causal on a dense copy), softmax vs
torch.log_softmax, RMSNorm and RoPE closed forms (constant vectors,
position-0 identity, pair norms, relative-position property), silu closed form;
and the layer COMPOSITION (layer_forward / forward_chain: residual placement, MLP input,
final norm, GQA mapping, cache semantics) by tests/test_oracle_llama_pin.py against
transformers' LlamaForCausalLM in fp64 with the bf16 rounding points switched off.
"""
import numpy as np

from .numerics import round_bf16


def rope_table(max_pos, head_dim, theta):
    """cos/sin [max_pos][head_dim/2] fp32 from fp64 angles pos * theta^(-2m/d_h)."""
    m = np.arange(head_dim // 2, dtype=np.float64)
    inv_freq = 1.0 / np.power(float(theta), 2.0 * m / head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv_freq[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def rmsnorm(x, g, eps):
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope(x, pos, cos, sin):
    """rotate_half RoPE on x [R, H, d_h] at positions pos [R] (fp64 result)."""
    half = x.shape[-1] // 2
    c = np.asarray(cos, dtype=np.float64)[pos][:, None, :]
    s = np.asarray(sin, dtype=np.float64)[pos][:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x):
    return x / (1.0 + np.exp(-x))


def softmax(x, axis=-1):
    m = np.max(x, axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / np.sum(e, axis=axis, keepdims=True)


# ---------------------------------------------------------------- stages

def embed(E, tokens):
    """step 1.1: h0 = E[c] (rows of the bf16 embedding, exact in fp64)."""
    return np.asarray(E, dtype=np.float64)[np.asarray(tokens, dtype=np.int64)]


def attn_norm(h, g_attn, eps):
    """step 1.2: a = bf16(RMSNorm(h) * g)."""
    return round_bf16(rmsnorm(h, g_attn, eps))


def qkv_rope(a, wqkv, pos, cos, sin, n_q_heads, n_kv_heads, head_dim):
    """steps 1.3-1.4: q,k,v from bf16 a; RoPE on q,k; all rounded to bf16.

    wqkv rows: [q heads | k heads | v heads] x head_dim (the ABI layout).
    Returns q [R,Hq,dh], k [R,Hkv,dh], v [R,Hkv,dh] (fp64 arrays of bf16 values).
    """
    R = a.shape[0]
    y = a @ np.asarray(wqkv, dtype=np.float64).T
    nq = n_q_heads * head_dim
    nk = n_kv_heads * head_dim
    q = y[:, :nq].reshape(R, n_q_heads, head_dim)
    k = y[:, nq:nq + nk].reshape(R, n_kv_heads, head_dim)
    v = y[:, nq + nk:].reshape(R, n_kv_heads, head_dim)
    pos = np.asarray(pos, dtype=np.int64)
    return (round_bf16(rope(q, pos, cos, sin)), round_bf16(rope(k, pos, cos, sin)),
            round_bf16(v))


def verify_attention(q, cache_k, cache_v, chain_k, chain_v):
    """step 1.5-1.6a for one request: chain row j attends cache keys 0..L-1 and chain keys 0..j.

    q [R,Hq,dh]; cache_k/v [L,Hkv,dh]; chain_k/v [R,Hkv,dh] (R = k_i + 1).
    GQA: q head hq uses kv head hq // G. Scale 1/sqrt(d_h). Softmax in fp64.
    Returns O [R, Hq*dh] rounded to bf16.
    """
    R, Hq, dh = q.shape
    Hkv = chain_k.shape[1]
    G = Hq // Hkv
    L = cache_k.shape[0]
    out = np.zeros((R, Hq, dh))
    for j in range(R):
        keys = np.concatenate([cache_k[:L], chain_k[: j + 1]], axis=0)      # [L+j+1, Hkv, dh]
        vals = np.concatenate([cache_v[:L], chain_v[: j + 1]], axis=0)
        for hq in range(Hq):
            hk = hq // G
            s = keys[:, hk, :] @ q[j, hq, :] / np.sqrt(dh)
            p = softmax(s)
            out[j, hq, :] = p @ vals[:, hk, :]
    return round_bf16(out.reshape(R, Hq * dh))


def attn_out(h, o, wo):
    """step 1.6b: h1 = h + o Wo^T (fp64, never rounded)."""
    return h + np.asarray(o, dtype=np.float64) @ np.asarray(wo, dtype=np.float64).T


def ffn_norm(h1, g_ffn, eps):
    """step 1.7a: b = bf16(RMSNorm(h1) * g_ffn)."""
    return round_bf16(rmsnorm(h1, g_ffn, eps))


def swiglu(b, w_gate_up):
    """step 1.7b: u = bf16(silu(b Wg^T) * (b Wu^T)); w_gate_up rows [gate F | up F]."""
    F = w_gate_up.shape[0] // 2
    W = np.asarray(w_gate_up, dtype=np.float64)
    gate = b @ W[:F].T
    up = b @ W[F:].T
    return round_bf16(silu(gate) * up)


def down_residual(h1, u, w_down):
    """step 1.7c: h2 = h1 + u Wd^T."""
    return h1 + np.asarray(u, dtype=np.float64) @ np.asarray(w_down, dtype=np.float64).T


def final_norm(h, g_final, eps):
    """step 1.8a: z = bf16(RMSNorm(h) * g_final)."""
    return round_bf16(rmsnorm(h, g_final, eps))


def lm_head(z, w_lm, chunk=16384):
    """step 1.8b: logits = z W_lm^T in fp64 (not rounded). Vocab processed in
    chunks only to bound host memory (no reordering of any sum)."""
    z = np.asarray(z, dtype=np.float64)
    V = w_lm.shape[0]
    out = np.empty((z.shape[0], V))
    for c0 in range(0, V, chunk):
        out[:, c0:c0 + chunk] = z @ np.asarray(w_lm[c0:c0 + chunk], dtype=np.float64).T
    return out


def tile_stats(logits, tile=256):
    """Per (row, vocab tile) statistics the GPU lm-head epilogue emits:
    max, sum exp(l - max), argmax (lowest index). Plain loop over tiles."""
    R, V = logits.shape
    nt = (V + tile - 1) // tile
    mx = np.zeros((R, nt))
    se = np.zeros((R, nt))
    am = np.zeros((R, nt), dtype=np.int64)
    for t in range(nt):
        blk = logits[:, t * tile:(t + 1) * tile]
        mx[:, t] = blk.max(axis=1)
        am[:, t] = t * tile + np.argmax(blk, axis=1)     # numpy argmax: first occurrence
        se[:, t] = np.exp(blk - mx[:, t:t + 1]).sum(axis=1)
    return mx, se, am


# ---------------------------------------------------------------- full forward

def layer_forward(w, layer, h, pos, cache_k, cache_v, cfg, cos, sin, taps=None):
    """One decoder layer for one request's chain rows (h [R,D], pos [R]).

    cache_k/v: this layer's dense cache [L,Hkv,dh]. Returns (h_out, chain_k, chain_v).
    """
    a = attn_norm(h, np.asarray(w["attn_norm"][layer], dtype=np.float64), cfg.norm_eps)
    q, k, v = qkv_rope(a, w["wqkv"][layer], pos, cos, sin,
                       cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim)
    o = verify_attention(q, cache_k, cache_v, k, v)
    h1 = attn_out(h, o, w["wo"][layer])
    if cfg.ffn_dim > 0:
        b = ffn_norm(h1, np.asarray(w["ffn_norm"][layer], dtype=np.float64), cfg.norm_eps)
        u = swiglu(b, w["w_gate_up"][layer])
        h2 = down_residual(h1, u, w["w_down"][layer])
    else:
        b = u = None
        h2 = h1
    if taps is not None:
        taps.append(dict(a=a, q=q, k=k, v=v, o=o, h1=h1, b=b, u=u, h2=h2))
    return h2, k, v


def forward_chain(w, tokens, pos, caches, cfg, cos, sin, taps=None):
    """Full model on one request's chain. caches: list over layers of (K [L,Hkv,dh], V).

    Returns (z [R,D] bf16, logits [R,V] fp64, chain_kv list over layers of (k, v)).
    """
    h = embed(w["embed"], tokens)
    chain_kv = []
    for layer in range(cfg.n_layers):
        ck, cv = caches[layer]
        h, k, v = layer_forward(w, layer, h, pos, ck, cv, cfg, cos, sin, taps)
        chain_kv.append((k, v))
    z = final_norm(h, np.asarray(w["final_norm"], dtype=np.float64), cfg.norm_eps)
    return z, lm_head(z, w["lm_head"]), chain_kv
