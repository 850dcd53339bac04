"""NEXT-4 fp32-SIMT exactness instantiation (sv_exact_forward): the verify
step's model arithmetic with fp32 operands and no bf16 rounding, against the fp64 oracle with its
bf16 rounding points switched to the identity (the same switch tests/test_oracle_llama_pin.py uses to
pin the oracle's composition against transformers' LlamaForCausalLM), fed identical fp32 weights,
caches and RoPE table. What remains is fp32 accumulation error: dot products of length K carry
~sqrt(K) * 2^-24 relative error (K = 4096 / 14336 at Llama shape), so the logits must agree to
1e-6 of the row's scale at toy shape and 1e-5 at Llama shape; greedy decisions on the exact logits
(sv_verify_logits) equal the oracle's except at a top-2 gap below twice the row's error."""
import numpy as np
import pytest
import torch

import synth
from oracle import model, verify as ov
from paper_2604_09562_b200 import sv

pytestmark = pytest.mark.gpu


def _case(cfg, ctx, depths, seed, monkeypatch):
    w = synth.model_weights(cfg, seed=seed, norm_one=False)
    wf = {k: v.float().contiguous().cuda() for k, v in w.items()}
    wnp = {k: v.double().numpy() for k, v in w.items()}
    B = len(ctx)
    max_ctx = max(1, max(ctx))
    g = torch.Generator().manual_seed(seed + 1)
    ck = torch.randn(cfg.n_layers, B, max_ctx, cfg.n_kv_heads, cfg.head_dim, generator=g)
    cv = torch.randn(cfg.n_layers, B, max_ctx, cfg.n_kv_heads, cfg.head_dim, generator=g)
    toks = synth.random_tokens(sum(depths) + B, cfg.vocab, seed=seed + 2)
    row_off = [0]
    for k in depths:
        row_off.append(row_off[-1] + k + 1)
    logits, ws = sv.exact_forward(cfg, wf, row_off, toks.cuda(), ctx, ck.cuda(), cv.cuda())
    torch.cuda.synchronize()
    lg = logits.cpu().double().numpy()
    monkeypatch.setattr(model, "round_bf16", lambda x: np.asarray(x, dtype=np.float64))
    cos, sin = model.rope_table(cfg.max_pos, cfg.head_dim, cfg.rope_theta)
    worst, refs = 0.0, []
    for b in range(B):
        L = ctx[b]
        caches = [(ck[l, b, :L].double().numpy(), cv[l, b, :L].double().numpy()) for l in range(cfg.n_layers)]
        rows = slice(row_off[b], row_off[b + 1])
        pos = np.arange(L, L + depths[b] + 1)
        _, ref, _ = model.forward_chain(wnp, [int(t) for t in toks[rows]], pos, caches, cfg, cos, sin)
        err = np.abs(lg[rows] - ref).max(axis=1) / np.maximum(1.0, np.abs(ref).max(axis=1))
        worst = max(worst, float(err.max()))
        refs.append((ref, err))
    return lg, refs, toks, row_off, worst


def _greedy_matches(cfg, lg, refs, toks, row_off, depths, ctx):
    lane = sv.Lane(cfg.with_(max_batch=len(depths), max_slots=len(depths)),
                   {k: v.cuda() for k, v in synth.model_weights(cfg, seed=0).items()})
    e = torch.empty(cfg.n_layers, 0, cfg.n_kv_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    for b in range(len(depths)):                 # greedy decisions read only the logits
        lane.append_kv(b, 900 + b, e, e, int(toks[row_off[b]]))
    drafts = torch.cat([toks[row_off[b] + 1:row_off[b + 1]] for b in range(len(depths))])
    acc, tok = lane.verify_logits(list(range(len(depths))), depths, drafts.cuda(),
                                  torch.from_numpy(lg.astype(np.float32)).cuda(), mode="greedy")
    torch.cuda.synchronize()
    acc, tok = acc.cpu().numpy(), tok.cpu().numpy()
    for b, (ref, err) in enumerate(refs):
        dr = [int(t) for t in toks[row_off[b] + 1:row_off[b + 1]]]
        r = ov.verify_request(ref, dr, None, 0, 900 + b, 0, ov.GREEDY)
        if acc[b] != r["a"] or list(tok[b][:acc[b] + 1]) != r["emitted"]:
            j = min(int(acc[b]), r["a"])
            top2 = np.sort(ref[j])[-2:]
            assert top2[1] - top2[0] < 2 * err[j] * max(1.0, np.abs(ref[j]).max()), (b, acc[b], r)


@pytest.mark.parametrize("name,layers", [("toy", 1), ("toy_mlp", 2)])
def test_exact_toy(name, layers, monkeypatch):
    cfg = synth.CONFIGS[name].with_(n_layers=layers)
    ctx, depths = [128, 0, 5, 300], [1, 2, 3, 4]
    lg, refs, toks, row_off, worst = _case(cfg, ctx, depths, 31 + layers, monkeypatch)
    print(name, layers, "worst relative logit error", worst)
    assert worst <= 1e-6, worst
    _greedy_matches(cfg, lg, refs, toks, row_off, depths, ctx)


def test_exact_llama_shape(monkeypatch):
    cfg = synth.LLAMA.with_(max_batch=3, max_slots=3, n_pages=32, max_pos=1024)
    ctx, depths = [200, 64, 1], [4, 8, 0]
    lg, refs, toks, row_off, worst = _case(cfg, ctx, depths, 41, monkeypatch)
    print("llama worst relative logit error", worst)
    assert worst <= 1e-5, worst
    _greedy_matches(cfg, lg, refs, toks, row_off, depths, ctx)
