"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no norm, attention, softmax,
sampling or commit logic): only model shapes, seeded random tensors and the
input recipes of DESIGN.md §"Input recipe". Both ``oracle`` and the tests /
bench that drive the CUDA library take their inputs from here.

Shapes follow BASELINE.json ``configs`` and SURVEY.md §8 "Fixed definitions"
(Llama-3-8B-shaped layer: D=4096, 32 q / 8 kv heads, d_h=128, V=128256,
F=14336, RoPE theta 500000, eps 1e-5).
"""
from dataclasses import dataclass, replace, asdict

import numpy as np
import torch


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int
    d_model: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    ffn_dim: int            # 0 = no MLP
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    page_size: int = 64
    n_pages: int = 64
    max_slots: int = 8
    max_batch: int = 8
    max_depth: int = 8
    max_pos: int = 1024

    def with_(self, **kw):
        return replace(self, **kw)

    def as_dict(self):
        return asdict(self)

    @property
    def qkv_rows(self):
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim


# BASELINE.json configs[0]: toy verify (1 layer, 2 q / 2 kv heads x 64, vocab 512)
TOY = ModelConfig(n_layers=1, d_model=128, n_q_heads=2, n_kv_heads=2, head_dim=64,
                  vocab=512, ffn_dim=0, n_pages=128, max_slots=8, max_batch=8,
                  max_depth=8, max_pos=2048)
# coverage variant with the MLP on (SURVEY.md §8 "toy+mlp")
TOY_MLP = TOY.with_(ffn_dim=256)
# BASELINE.json configs[1] (and north-star): Llama-3-8B-shaped single layer + lm-head
LLAMA = ModelConfig(n_layers=1, d_model=4096, n_q_heads=32, n_kv_heads=8, head_dim=128,
                    vocab=128256, ffn_dim=14336, n_pages=4608, max_slots=128,
                    max_batch=128, max_depth=8, max_pos=8192 + 64)

CONFIGS = {"toy": TOY, "toy_mlp": TOY_MLP, "llama": LLAMA}


def _gen(seed, device="cpu"):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def model_weights(cfg, seed=0, std=0.02, embed_std=1.0, norm_one=True, device="cpu"):
    """Random-init weights, bf16, [out, in] row-major, layer-stacked.

    fp32 N(0, std^2) draws rounded once to bf16 by torch's cast (SURVEY.md §8(c)
    S19: identical values are fed to both paths). Norm gains are 1 (or
    1 + N(0, 0.1^2) with norm_one=False, to exercise the gain multiply).
    """
    g = _gen(seed, device)
    L, D, V, F = cfg.n_layers, cfg.d_model, cfg.vocab, cfg.ffn_dim
    hd = cfg.n_q_heads * cfg.head_dim

    def rn(*shape, s):
        out = torch.empty(*shape, dtype=torch.bfloat16, device=device)
        flat = out.view(shape[0], -1)
        for i in range(shape[0]):            # per leading index: bounded fp32 scratch for big models
            flat[i] = (torch.randn(flat.shape[1], generator=g, dtype=torch.float32, device=device) * s).to(torch.bfloat16)
        return out

    def norm(*shape):
        if norm_one:
            return torch.ones(*shape, dtype=torch.bfloat16, device=device)
        return (1.0 + 0.1 * torch.randn(*shape, generator=g, device=device)).to(torch.bfloat16)

    w = {
        "embed": rn(V, D, s=embed_std),
        "attn_norm": norm(L, D),
        "wqkv": rn(L, cfg.qkv_rows, D, s=std),
        "wo": rn(L, D, hd, s=std),
        "ffn_norm": norm(L, D),
        "w_gate_up": rn(L, 2 * F, D, s=std) if F > 0 else torch.zeros(L, 0, D, dtype=torch.bfloat16, device=device),
        "w_down": rn(L, D, F, s=std) if F > 0 else torch.zeros(L, D, 0, dtype=torch.bfloat16, device=device),
        "final_norm": norm(D),
        "lm_head": rn(V, D, s=std),
    }
    return w


def context_kv(cfg, n_tokens, seed, std=1.0, device="cpu"):
    """Synthetic post-RoPE context K/V for one request: [n_layers][n][H_kv][d_h] bf16."""
    g = _gen(seed, device)
    shape = (cfg.n_layers, n_tokens, cfg.n_kv_heads, cfg.head_dim)
    k = (torch.randn(*shape, generator=g, device=device) * std).to(torch.bfloat16)
    v = (torch.randn(*shape, generator=g, device=device) * std).to(torch.bfloat16)
    return k, v


def random_tokens(n, vocab, seed):
    g = _gen(seed)
    return torch.randint(0, vocab, (n,), generator=g, dtype=torch.int32)


def depths_uniform(batch, kmin, kmax, seed):
    g = _gen(seed)
    return torch.randint(kmin, kmax + 1, (batch,), generator=g, dtype=torch.int32)


def draft_probs_dense(n_rows, vocab, seed, sharpness=3.0):
    """Dense draft distributions q [n_rows][V] fp32 (rows sum to 1 in fp64 before the cast).

    q = w / sum(w) with w = exp-distributed weights raised to `sharpness`
    (a heavy-tailed random simplex point; no softmax involved).
    """
    g = _gen(seed)
    e = -torch.log(torch.rand(n_rows, vocab, generator=g, dtype=torch.float64).clamp_min(1e-300))
    w = e ** sharpness
    q = w / w.sum(dim=1, keepdim=True)
    return q.to(torch.float32)


def draft_tokens_from(q_rows, seed):
    """Draw one draft token per row from q (inverse-CDF on fp64 uniforms)."""
    g = _gen(seed)
    q = q_rows.to(torch.float64)
    cdf = torch.cumsum(q, dim=1)
    u = torch.rand(q.shape[0], 1, generator=g, dtype=torch.float64) * cdf[:, -1:]
    tok = torch.searchsorted(cdf, u).clamp_max(q.shape[1] - 1)
    return tok.view(-1).to(torch.int32)


def planted_successor(cfg, weights, seed, beta):
    """Planted-successor fixture (SURVEY.md §8(d) "Acceptance control").

    Picks a permutation f of the vocab and adds beta * E[t]/||E[t]|| to
    lm_head row f(t), so the model's argmax continuation of t is f(t) with a
    margin set by beta. Returns (new_weights, f as int32 tensor).
    """
    g = _gen(seed)
    V = cfg.vocab
    f = torch.randperm(V, generator=g).to(torch.int64)
    E = weights["embed"].to(torch.float32)
    En = E / E.norm(dim=1, keepdim=True)
    lm = weights["lm_head"].to(torch.float32).clone()
    lm[f.to(lm.device)] += beta * En
    w = dict(weights)
    w["lm_head"] = lm.to(torch.bfloat16)
    return w, f.to(torch.int32)


@dataclass(frozen=True)
class Workload:
    """A bench / parity workload."""
    name: str
    cfg: ModelConfig
    batch: int
    ctx: tuple            # (min, max) context length at start, uniform
    kmin: int
    kmax: int
    mode: str             # "greedy" | "sample"
    alpha: float          # planted drafter: probability each draft follows the planted successor
    embed_std: float = 8.0
    beta: float = 0.3     # planted-successor strength (logit margin ~ beta * sqrt(D))
    temperature: float = 1.0
    controller: bool = False   # depths from the SpecuStream controller (NEXT-1) instead of U{kmin..kmax}
    gen_on_device: bool = False  # draw weights / context KV with a CUDA generator (multi-GB models)
    alpha_sigma: float = 0.0   # per-request acceptance follows AR(1) around alpha with this stationary std
    tree: tuple = ()           # NEXT-4 token trees (R30): every request drafts this tree (parents of nodes 1..k)
    top_k: int = 0             # NEXT-4 filtered targets (R31), SAMPLE only
    top_p: float = 1.0


def workload(name, steps_budget=64):
    """Named workloads. `steps_budget` sizes the page pool for that many verify steps."""
    def pool(batch, ctx_max, kmax, page=64):
        per_req = (ctx_max + (kmax + 1) * steps_budget + page - 1) // page + 1
        return batch * per_req, ctx_max + (kmax + 1) * steps_budget + 64
    if name == "ns":          # north-star: bs64, k = 8, 4k context (BASELINE metric's verify-step config)
        n_pages, max_pos = pool(64, 4096, 8)
        cfg = LLAMA.with_(n_pages=n_pages, max_slots=64, max_batch=64, max_pos=max_pos)
        return Workload("ns", cfg, 64, (4096, 4096), 8, 8, "greedy", 0.8)
    if name == "ns32":        # NEXT-4: the north-star batch through all 32 Llama-3-8B layers
        n_pages, max_pos = pool(64, 4096, 8)
        cfg = LLAMA.with_(n_layers=32, n_pages=n_pages, max_slots=64, max_batch=64, max_pos=max_pos)
        return Workload("ns32", cfg, 64, (4096, 4096), 8, 8, "greedy", 0.8, gen_on_device=True)
    if name == "c2":          # BASELINE configs[1]: bs64, adaptive k 1-8, ALPACA-like 256-token prompts
        n_pages, max_pos = pool(64, 256, 8)
        cfg = LLAMA.with_(n_pages=n_pages, max_slots=64, max_batch=64, max_pos=max_pos)
        return Workload("c2", cfg, 64, (256, 256), 1, 8, "sample", 0.75)
    if name == "c3":          # BASELINE configs[2]: bs128, context 1k-2k, sampled
        n_pages, max_pos = pool(128, 2048, 8)
        cfg = LLAMA.with_(n_pages=n_pages, max_slots=128, max_batch=128, max_pos=max_pos)
        return Workload("c3", cfg, 128, (1024, 2048), 5, 8, "sample", 0.72, controller=True, alpha_sigma=0.10)
    if name == "c4":          # BASELINE configs[3] decode lane: bs32, 8k prompts
        n_pages, max_pos = pool(32, 8192, 8)
        cfg = LLAMA.with_(n_pages=n_pages, max_slots=32, max_batch=32, max_pos=max_pos)
        return Workload("c4", cfg, 32, (8192, 8192), 8, 8, "greedy", 0.85)
    if name == "ns_tree":     # NEXT-4: the north-star batch drafting 8-node token trees (R30)
        n_pages, max_pos = pool(64, 4096, 8)
        cfg = LLAMA.with_(n_pages=n_pages, max_slots=64, max_batch=64, max_pos=max_pos)
        return Workload("ns_tree", cfg, 64, (4096, 4096), 8, 8, "greedy", 0.7, tree=(0, 0, 1, 1, 2, 3, 5, 7))
    if name == "c2_filter":   # NEXT-4: configs[1] sampled with a top-k 50 / top-p 0.9 filtered target (R31)
        n_pages, max_pos = pool(64, 256, 8)
        cfg = LLAMA.with_(n_pages=n_pages, max_slots=64, max_batch=64, max_pos=max_pos)
        return Workload("c2_filter", cfg, 64, (256, 256), 1, 8, "sample", 0.75, top_k=50, top_p=0.9)
    if name == "toy":         # BASELINE configs[0]
        n_pages, max_pos = pool(4, 128, 4)
        cfg = TOY.with_(n_pages=n_pages, max_slots=4, max_batch=4, max_pos=max_pos)
        return Workload("toy", cfg, 4, (128, 128), 1, 4, "sample", 0.7, embed_std=1.0, beta=0.0)
    raise KeyError(name)


def ctx_lengths(wl, seed):
    g = _gen(seed)
    lo, hi = wl.ctx
    return [int(x) for x in torch.randint(lo, hi + 1, (wl.batch,), generator=g)]


def planted_masks(n_steps, rows, alpha, vocab, seed):
    """Per-step deviation masks (1 with probability 1 - alpha) and replacement tokens."""
    g = _gen(seed)
    m = (torch.rand(n_steps, rows, generator=g) >= alpha).to(torch.uint8)
    t = torch.randint(0, vocab, (n_steps, rows), generator=g, dtype=torch.int32)
    return m, t


def ar1_alphas(n_steps, batch, p0, sigma, rho, seed):
    """Per-request planted acceptance probabilities [n_steps][batch]: AR(1) around p0 with
    stationary std sigma and coefficient rho ("order-1 autoregressive process"),
    clipped to [0, 1]."""
    g = _gen(seed)
    a = torch.empty(n_steps, batch, dtype=torch.float64)
    x = p0 + sigma * torch.randn(batch, generator=g, dtype=torch.float64)
    innov = sigma * (1.0 - rho * rho) ** 0.5
    for i in range(n_steps):
        a[i] = x.clamp(0.0, 1.0)
        x = p0 + rho * (x - p0) + innov * torch.randn(batch, generator=g, dtype=torch.float64)
    return a


def planted_masks_req(n_steps, batch, kmax, alphas, vocab, seed):
    """Per-step, per-request deviation masks [n_steps][batch][kmax] (1 with probability
    1 - alphas[step][request]) and replacement tokens of the same shape."""
    g = _gen(seed)
    u = torch.rand(n_steps, batch, kmax, generator=g, dtype=torch.float64)
    m = (u >= alphas[:, :, None]).to(torch.uint8)
    t = torch.randint(0, vocab, (n_steps, batch, kmax), generator=g, dtype=torch.int32)
    return m, t


def as_f64(t):
    """bf16/fp32 torch tensor -> numpy fp64 (exact)."""
    return t.detach().to("cpu").to(torch.float64).numpy()


# ---------------------------------------------------------------- config 5: mixed serving trace
# BASELINE configs[4] / SURVEY.md §8(d) config 5: 80 queries each of ALPACA (prompt 256), GSM8K and
# HUMANEVAL (prompt U[1k, 2k]) and SUM (prompt 8k); output lengths lognormal with the SPEC.md:420
# medians 60 / 150 / 220 / 90 and sigma 0.5 (our choice); planted acceptance profiles
# p0 = 0.70 / 0.72 / 0.75 / 0.85. Seeded; no method arithmetic.
TRACE_PROFILES = {            # dataset: (prompt_lo, prompt_hi, output median, acceptance p0)
    "ALPACA": (256, 256, 60, 0.70),
    "GSM8K": (1024, 2048, 150, 0.72),
    "HUMANEVAL": (1024, 2048, 220, 0.75),
    "SUM": (8192, 8192, 90, 0.85),
}


def mixed_trace(n_per_dataset=80, seed=0, sigma=0.5, max_out=1024):
    """The 320-query trace as a list of dicts (qid, dataset, prompt_len, out_len, alpha, prompt_seed),
    datasets interleaved in a seeded random order."""
    g = _gen(seed)
    qs = []
    for name, (lo, hi, med, p0) in TRACE_PROFILES.items():
        plen = torch.randint(lo, hi + 1, (n_per_dataset,), generator=g)
        z = torch.randn(n_per_dataset, generator=g, dtype=torch.float64)
        out = torch.clamp((med * torch.exp(sigma * z)).round(), 1, max_out).to(torch.int64)
        for i in range(n_per_dataset):
            qs.append(dict(dataset=name, prompt_len=int(plen[i]), out_len=int(out[i]), alpha=p0))
    order = torch.randperm(len(qs), generator=g).tolist()
    trace = [qs[i] for i in order]
    for qid, q in enumerate(trace):
        q["qid"] = qid
        q["prompt_seed"] = 1_000_003 * (seed + 1) + qid
    return trace
