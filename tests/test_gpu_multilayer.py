"""n_layers > 1, free-running against the oracle lane (oracle/lane.py, the whole model in fp64):
two verify + commit steps of a 3-layer toy+mlp model, so each layer's chain K/V reaches its own
pages and the second step attends over committed multi-layer KV.

Tolerance. Free-running, the GPU rounds a, q, k, v, O, b, u, z to bf16 at every layer (relative
2^-9 each) while the oracle keeps fp64; across 3 layers these perturb the logits by a few 1e-3 of
their scale (measured 1e-3). The test allows 5e-3 * max(1, max|l|) per row, and excuses a greedy decision only
where the oracle's top-2 logit gap is below 2 * the row's max |dl| (SURVEY.md S13 rule)."""
import numpy as np
import pytest
import torch

import synth
from oracle.lane import OracleLane
from oracle import verify as ov
from paper_2604_09562_b200 import sv

from gpu_util import f64

pytestmark = pytest.mark.gpu

REL = 5e-3


def _excused(lrow_ref, err):
    top2 = np.sort(lrow_ref)[-2:]
    return (top2[1] - top2[0]) < 2 * err


def test_three_layers_two_steps():
    cfg = synth.TOY_MLP.with_(n_layers=3, n_pages=64)
    w = synth.model_weights(cfg, seed=21, norm_one=False)
    gpu = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
    orc = OracleLane(cfg, {k: v.to(torch.float32).numpy() for k, v in w.items()})
    ctx = [(100, 7), (37, 11), (250, 300)]
    for s, (n, pend) in enumerate(ctx):
        k, v = synth.context_kv(cfg, n, seed=60 + s)
        rid = 5000 + s
        gpu.append_kv(s, rid, k.cuda(), v.cuda(), pend)
        orc.append_kv(s, rid, k.to(torch.float32).numpy(), v.to(torch.float32).numpy(), pend)
    worst = 0.0
    for step, depths in enumerate(([4, 2, 6], [3, 5, 1])):
        drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=70 + step)
        T = sum(depths) + len(depths)
        lo = torch.empty(T, cfg.vocab, device="cuda")
        acc, tok = gpu.verify([0, 1, 2], depths, drafts.cuda(), None, seed=9, mode="greedy", logits_out=lo)
        torch.cuda.synchronize()
        acc, tok, lo = acc.cpu().numpy(), tok.cpu().numpy(), f64(lo)
        oa, oe, ol = orc.verify([0, 1, 2], depths, drafts.numpy(), None, 9, ov.GREEDY)
        r0 = 0
        for b, k in enumerate(depths):
            ref = ol[b]
            err = np.abs(lo[r0:r0 + k + 1] - ref).max(axis=1)
            scale = np.maximum(1.0, np.abs(ref).max(axis=1))
            worst = max(worst, float((err / scale).max()))
            assert (err / scale).max() <= REL, (step, b, (err / scale).max())
            if acc[b] != oa[b] or list(tok[b][:acc[b] + 1]) != oe[b]:
                # a flip is excused only at a near-tie of the oracle's top-2 on the deciding row
                j = min(acc[b], oa[b])
                assert _excused(ref[j], err[j]), (step, b, acc[b], oa[b])
            r0 += k + 1
        # keep both lanes on the same sequence: commit the oracle's decisions on both sides
        n_keep = torch.tensor([a + 1 for a in oa], dtype=torch.int32, device="cuda")
        if all(acc[b] == oa[b] for b in range(3)):
            gpu.commit()
        else:
            gpu.commit(n_keep)
        orc.commit()
    print("worst relative logit error", worst)


def test_two_llama_layers_two_steps():
    """The same free-running check at Llama-3-8B shape with 2 layers (GQA 32/8 heads x 128, F = 14336,
    V = 128256): contexts of 1..3 pages per layer, two verify + commit steps. Free-running drift at this
    shape is larger (SURVEY.md S11 measured 2.5e-3 row-normalised for one layer from the bf16 rounding
    cascade), so the bound is 1e-2 * max(1, max|l|) per row; decisions with the S13 excuse rule."""
    cfg = synth.LLAMA.with_(n_layers=2, n_pages=48, max_slots=3, max_batch=3, max_pos=1024)
    w = synth.model_weights(cfg, seed=22, norm_one=False)
    gpu = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
    orc = OracleLane(cfg, {k: v.to(torch.float32).numpy() for k, v in w.items()})
    ctx = [(100, 7), (37, 11), (190, 300)]
    for s, (n, pend) in enumerate(ctx):
        k, v = synth.context_kv(cfg, n, seed=80 + s)
        rid = 6000 + s
        gpu.append_kv(s, rid, k.cuda(), v.cuda(), pend)
        orc.append_kv(s, rid, k.to(torch.float32).numpy(), v.to(torch.float32).numpy(), pend)
    worst = 0.0
    for step, depths in enumerate(([4, 2, 6], [3, 5, 1])):
        drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=90 + step)
        T = sum(depths) + len(depths)
        lo = torch.empty(T, cfg.vocab, device="cuda")
        acc, tok = gpu.verify([0, 1, 2], depths, drafts.cuda(), None, seed=9, mode="greedy", logits_out=lo)
        torch.cuda.synchronize()
        acc, tok, lo = acc.cpu().numpy(), tok.cpu().numpy(), f64(lo)
        oa, oe, ol = orc.verify([0, 1, 2], depths, drafts.numpy(), None, 9, ov.GREEDY)
        r0 = 0
        for b, k in enumerate(depths):
            ref = ol[b]
            err = np.abs(lo[r0:r0 + k + 1] - ref).max(axis=1)
            scale = np.maximum(1.0, np.abs(ref).max(axis=1))
            worst = max(worst, float((err / scale).max()))
            assert (err / scale).max() <= 1e-2, (step, b, (err / scale).max())
            if acc[b] != oa[b] or list(tok[b][:acc[b] + 1]) != oe[b]:
                j = min(acc[b], oa[b])
                assert _excused(ref[j], err[j]), (step, b, acc[b], oa[b])
            r0 += k + 1
        n_keep = torch.tensor([a + 1 for a in oa], dtype=torch.int32, device="cuda")
        if all(acc[b] == oa[b] for b in range(3)):
            gpu.commit()
        else:
            gpu.commit(n_keep)
        orc.commit()
    print("llama 2 layers: worst relative logit error", worst)
