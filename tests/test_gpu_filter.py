"""Top-k / top-p filtered targets on the GPU (sv_set_filter; NEXT-4, R31) against the
oracle (oracle/verify.py filtered_target): decisions on exact logits for chains and trees, ties at
the threshold, top_k = 1 = greedy, the filtered law by chi-square on the device's own draws, and a
full-model sampled verify with filtering. Borderline: an accept test within 1e-5 (S12), or a row
whose top-p cut sits within 1e-5 of a cumulative sum (the kept set is decided in fp32 / fixed point
on the GPU, fp64 in the oracle)."""
import numpy as np
import pytest
import torch
from scipy import stats

import synth
from oracle import tree, verify
from oracle.philox import uniform_accept

from gpu_util import Setup, f64

pytestmark = pytest.mark.gpu


def _top_p_borderline(lrow, temperature, top_p):
    if top_p >= 1.0:
        return False
    v = np.asarray(lrow, dtype=np.float32).astype(np.float64) * np.float64(np.float32(1.0 / temperature))
    p = np.exp(v - v.max())
    p /= p.sum()
    order = np.lexsort((np.arange(len(p)), -v))
    cum = np.cumsum(p[order])
    return bool(np.min(np.abs(cum - top_p)) < 1e-5)


def _chain_decisions(S, slots, depths, drafts, probs, logits, seed, temperature, top_k, top_p):
    out, r0, off = [], 0, 0
    for s, k in zip(slots, depths):
        c = S.ctx[s]
        lrow = logits[r0:r0 + k + 1]
        dr = [int(t) for t in drafts[off:off + k]]
        qr = None if probs is None else f64(probs[off:off + k])
        r = verify.verify_request(lrow, dr, qr, seed, c["rid"], c["L"], verify.SAMPLE, temperature, top_k, top_p)
        p = verify.filtered_probs(lrow, temperature, top_k, top_p)
        bl = any(_top_p_borderline(lrow[j], temperature, top_p) for j in range(k + 1))
        for j in range(1, k + 1):
            u = uniform_accept(seed, c["rid"], c["L"] + j)
            qd = 1.0 if qr is None else qr[j - 1][dr[j - 1]]
            if qd > 0 and abs(u - p[j - 1][dr[j - 1]] / qd) < 1e-5:
                bl = True
        r["borderline"] = bl
        out.append(r)
        r0 += k + 1
        off += k
    return out


def _logits_with_ties(T, V, rng):
    """Random logits rounded to a coarse grid, so equal values (ties) are common near the top."""
    return np.round(rng.standard_normal((T, V)) * 2.5 * 4) / 4


@pytest.mark.parametrize("top_k,top_p", [(5, 1.0), (0, 0.9), (40, 0.7), (3, 0.95), (1, 1.0), (0, 0.3)])
@pytest.mark.parametrize("dense", [True, False])
def test_filtered_chain_decisions_on_exact_logits(top_k, top_p, dense):
    _filtered_chain_case(top_k, top_p, dense, synth.TOY.vocab)


@pytest.mark.parametrize("top_k,top_p", [(5, 1.0), (0, 0.9), (40, 0.7)])
@pytest.mark.parametrize("dense", [True, False])
def test_filtered_chain_decisions_odd_vocab(top_k, top_p, dense):
    """V % 4 != 0 (GPT-2-like odd vocabularies): the filter's scalar row pass and the race's
    scalar loads (the float4 paths need V % 4 == 0) against the oracle."""
    _filtered_chain_case(top_k, top_p, dense, 509)


def _filtered_chain_case(top_k, top_p, dense, vocab):
    cfg = synth.TOY.with_(max_batch=16, max_slots=16, vocab=vocab)
    S = Setup(cfg, [10 + 9 * i for i in range(16)], seed=1)
    S.lane.set_filter(top_k, top_p)
    rng = np.random.default_rng(top_k * 7 + int(100 * top_p) + dense)
    V = cfg.vocab
    for rep in range(3):
        depths = [int(x) for x in rng.integers(0, cfg.max_depth + 1, size=16)]
        T = sum(depths) + 16
        lg = (_logits_with_ties(T, V, rng) if rep == 2 else rng.standard_normal((T, V)) * 2.5).astype(np.float32)
        probs = synth.draft_probs_dense(sum(depths), V, seed=10 + rep) if dense else None
        # drafts near the top of the target so that tests accept often
        drafts, r0 = [], 0
        for k in depths:
            for j in range(k):
                top = np.argsort(-lg[r0 + j], kind="stable")
                drafts.append(int(top[int(rng.integers(0, 4))]))
            r0 += k + 1
        drafts = torch.tensor(drafts, dtype=torch.int32)
        acc, tok = S.lane.verify_logits(list(range(16)), depths, drafts.cuda(), torch.from_numpy(lg).cuda(),
                                        None if probs is None else probs.cuda(), seed=50 + rep, mode="sample",
                                        temperature=0.8)
        torch.cuda.synchronize()
        acc, tok = acc.cpu().numpy(), tok.cpu().numpy()
        res = _chain_decisions(S, list(range(16)), depths, drafts, probs, lg.astype(np.float64), 50 + rep, 0.8,
                               top_k, top_p)
        n_bl = 0
        for b, r in enumerate(res):
            if not (acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"]):
                assert r["borderline"], (rep, b, acc[b], tok[b], r)
                n_bl += 1
        print(top_k, top_p, dense, rep, "borderline", n_bl, "accepted", int(acc.sum()))


def test_top_k_one_sampled_equals_greedy_on_the_gpu():
    cfg = synth.TOY.with_(max_batch=16, max_slots=16)
    S = Setup(cfg, [20 + 5 * i for i in range(16)], seed=2)
    rng = np.random.default_rng(9)
    depths = [int(x) for x in rng.integers(0, cfg.max_depth + 1, size=16)]
    T = sum(depths) + 16
    lg = torch.from_numpy((rng.standard_normal((T, cfg.vocab)) * 2).astype(np.float32)).cuda()
    top = lg.argmax(1).cpu().numpy()
    drafts, r0 = [], 0
    for k in depths:
        drafts += [int(top[r0 + j]) if rng.random() < 0.7 else int(rng.integers(cfg.vocab)) for j in range(k)]
        r0 += k + 1
    drafts = torch.tensor(drafts, dtype=torch.int32).cuda()
    probs = synth.draft_probs_dense(len(drafts), cfg.vocab, seed=3).cuda()
    ga, gt = (x.clone() for x in S.lane.verify_logits(list(range(16)), depths, drafts, lg, mode="greedy"))
    S.lane.set_filter(1, 1.0)
    sa, st = S.lane.verify_logits(list(range(16)), depths, drafts, lg, probs, seed=4, mode="sample", temperature=1.3)
    torch.cuda.synchronize()
    assert torch.equal(ga, sa) and torch.equal(gt, st)


@pytest.mark.parametrize("top_k,top_p", [(4, 1.0), (0, 0.8)])
def test_filtered_first_token_law_chi_square(top_k, top_p):
    """Many requests verify the same row with different request ids (independent Philox streams):
    the first emitted token must follow the filtered target p' (Leviathan with target p')."""
    cfg = synth.TOY.with_(max_batch=64, max_slots=64, n_pages=128)
    S = Setup(cfg, [3] * 64, seed=5)
    S.lane.set_filter(top_k, top_p)
    V = cfg.vocab
    rng = np.random.default_rng(11)
    row = (rng.standard_normal(V) * 1.5).astype(np.float32)
    row[:6] += 4.0                                        # a few dominant tokens
    p = verify.filtered_target(verify.target_probs(row.astype(np.float64), 1.0), row.astype(np.float64), top_k, top_p)
    q = torch.tensor(np.maximum(p, 0) * 0.5 + 0.5 / V, dtype=torch.float32)   # a proposal overlapping p'
    q = q / q.sum()
    counts = np.zeros(V)
    n_calls = 150
    lg = torch.from_numpy(np.stack([row, row] * 64)).cuda()                  # k = 1: two rows per request
    for call in range(n_calls):
        drafts = torch.multinomial(q, 64, replacement=True, generator=torch.Generator().manual_seed(call)).to(torch.int32)
        probs = q[None].repeat(64, 1)
        acc, tok = S.lane.verify_logits(list(range(64)), [1] * 64, drafts.cuda(), lg, probs.cuda(), seed=1000 + call,
                                        mode="sample")
        for t in tok[:, 0].cpu().numpy():
            counts[t] += 1
    n = counts.sum()
    assert counts[p == 0].sum() == 0
    e = p[p > 0] * n
    assert stats.chisquare(counts[p > 0], e * n / e.sum()).pvalue > 0.01


def test_filtered_tree_decisions_on_exact_logits():
    cfg = synth.TOY.with_(max_depth=12, max_batch=16, max_slots=16)
    S = Setup(cfg, [10 + 13 * i for i in range(16)], seed=2)
    S.lane.set_filter(20, 0.9)
    V = cfg.vocab
    rng = np.random.default_rng(21)
    trees = [[int(rng.integers(0, max(1, min(n, 3)))) for n in range(1, int(rng.integers(0, 13)) + 1)]
             for _ in range(16)]
    depths = [len(t) for t in trees]
    T = sum(depths) + 16
    lg = (rng.standard_normal((T, V)) * 2.5).astype(np.float32)
    probs = synth.draft_probs_dense(sum(depths), V, seed=3)
    drafts, r0 = [], 0
    for t in trees:
        for n, par in enumerate(t, start=1):
            drafts.append(int(np.argsort(-lg[r0 + par], kind="stable")[int(rng.integers(0, 3))]))
        r0 += len(t) + 1
    drafts = torch.tensor(drafts, dtype=torch.int32)
    par_dev = torch.tensor([p for t in trees for p in t], dtype=torch.int32).cuda()
    acc, tok, nodes = S.lane.verify_tree_logits(list(range(16)), depths, par_dev, drafts.cuda(),
                                                torch.from_numpy(lg).cuda(), probs.cuda(), seed=5, mode="sample",
                                                temperature=0.9)
    torch.cuda.synchronize()
    acc, tok, nodes = acc.cpu().numpy(), tok.cpu().numpy(), nodes.cpu().numpy()
    r0, off, n_bl = 0, 0, 0
    for b, t in enumerate(trees):
        k = len(t)
        c = S.ctx[b]
        lrow = lg[r0:r0 + k + 1].astype(np.float64)
        r = tree.verify_tree(lrow, [int(x) for x in drafts[off:off + k]], t, f64(probs[off:off + k]), 5, c["rid"],
                             c["L"], verify.SAMPLE, 0.9, 20, 0.9)
        bl = any(abs(u - rt) < 1e-5 for _, u, rt in r["tests"] if np.isfinite(rt)) or \
            any(_top_p_borderline(lrow[j], 0.9, 0.9) for j in range(k + 1))
        if not (acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"] and
                list(nodes[b][: r["a"] + 1]) == r["path"]):
            assert bl, (b, acc[b], tok[b], nodes[b], r)
            n_bl += 1
        r0 += k + 1
        off += k
    print("borderline", n_bl, "accepted", acc.tolist())


def test_full_model_sampled_verify_with_filter():
    """Toy+mlp lane: sampled verify with top-k/top-p, decisions teacher-forced on the GPU logits."""
    cfg = synth.TOY_MLP
    S = Setup(cfg, [128, 40, 300, 7], seed=8)
    S.lane.set_filter(30, 0.85)
    depths = [4, 0, 8, 2]
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=9)
    probs = synth.draft_probs_dense(sum(depths), cfg.vocab, seed=10)
    T = sum(depths) + 4
    lg = torch.empty(T, cfg.vocab, device="cuda")
    acc, tok = S.lane.verify([0, 1, 2, 3], depths, drafts.cuda(), probs.cuda(), seed=11, mode="sample",
                             temperature=0.7, logits_out=lg)
    torch.cuda.synchronize()
    res = _chain_decisions(S, [0, 1, 2, 3], depths, drafts, probs, f64(lg), 11, 0.7, 30, 0.85)
    acc, tok = acc.cpu().numpy(), tok.cpu().numpy()
    for b, r in enumerate(res):
        if not (acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"]):
            assert r["borderline"], (b, acc[b], tok[b], r)
    S.lane.commit()
    with pytest.raises(Exception):
        S.lane.set_filter(-1, 0.5)
    with pytest.raises(Exception):
        S.lane.set_filter(3, 0.0)


@pytest.mark.parametrize("filt", [(0, 1.0), (30, 0.85)])
def test_full_model_sampled_verify_odd_vocab(filt):
    """Toy+mlp lane with V = 509 (ragged last vocab tile, V % 4 != 0): lm-head logits within the
    north_star tolerance of the fp64 product of the GPU's z, and sampled decisions (dense q, with and
    without a filter) teacher-forced on the GPU logits."""
    from oracle import model
    cfg = synth.TOY_MLP.with_(vocab=509)
    S = Setup(cfg, [128, 40, 300, 7], seed=18)
    S.lane.set_filter(*filt)
    depths = [4, 0, 8, 2]
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=19)
    probs = synth.draft_probs_dense(sum(depths), cfg.vocab, seed=20)
    T = sum(depths) + 4
    lg = torch.empty(T, cfg.vocab, device="cuda")
    acc, tok = S.lane.verify([0, 1, 2, 3], depths, drafts.cuda(), probs.cuda(), seed=21, mode="sample",
                             temperature=0.9, logits_out=lg)
    torch.cuda.synchronize()
    z = S.tap("z", torch.bfloat16, (T, cfg.d_model))
    ref = model.lm_head(f64(z), S.wnp["lm_head"])
    err = np.abs(f64(lg) - ref).max(axis=1) / np.maximum(1.0, np.abs(ref).max(axis=1))
    assert err.max() <= 2e-3, err.max()
    res = _chain_decisions(S, [0, 1, 2, 3], depths, drafts, probs, f64(lg), 21, 0.9, *filt)
    acc, tok = acc.cpu().numpy(), tok.cpu().numpy()
    for b, r in enumerate(res):
        if not (acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"]):
            assert r["borderline"], (b, acc[b], tok[b], r)
    S.lane.commit()
