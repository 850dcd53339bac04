"""Token-tree verify (NEXT-4, R30) through the C ABI against oracle/tree.py.

Stage parity is teacher-forced as in tests/test_gpu_parity.py (each oracle stage fed the GPU's
own inputs to it, same tolerances): RoPE positions follow node depth, attention uses the ancestor
mask, decisions walk the tree. Covered on the rows-on-lanes (toy, d_h = 64), keys-on-lanes
(Llama shape, G = 4) and SIMT attention kernels; plus chain-shaped trees = sv_verify bit for bit,
free-running verify_tree + commit against the oracle lane, decision-only trees up to 16 nodes on
exact logits (dense and one-hot q), and the bad-parent device error.
"""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import model, tree, verify
from oracle.lane import OracleLane
from paper_2604_09562_b200 import sv

from gpu_util import Setup, f64
from test_gpu_parity import LOGIT_REL, _cmp_bf16, _cmp_resid

pytestmark = pytest.mark.gpu

# per-request trees (parents of nodes 1..k): chain, star, two-level, deep-with-branches, root only
TREES = [[0, 1, 2], [0, 0, 0, 0], [0, 0, 1, 1, 2, 2], [0, 1, 1, 2, 3, 3, 5, 0], []]


def _flat(trees):
    return [p for t in trees for p in t]


def _tree_tolerance(q, ck, cv, kc, vc, parents):
    """tests/test_gpu_parity.attention_tolerance with node n's visible chain keys = its root path."""
    R, Hq, dh = q.shape
    G = Hq // kc.shape[1]
    L = ck.shape[0]
    tol = np.zeros((R, Hq, dh))
    for n in range(R):
        vis = sorted(tree.path(parents, n))
        keys = np.concatenate([ck[:L], kc[vis]])
        vals = np.concatenate([cv[:L], vc[vis]])
        for hq in range(Hq):
            w = model.softmax(keys[:, hq // G, :] @ q[n, hq] / np.sqrt(dh))
            v = vals[:, hq // G, :]
            o = w @ v
            sig = 2.0 ** -8 / np.sqrt(3.0) * np.sqrt((w[:, None] ** 2 * (v - o[None]) ** 2).sum(axis=0))
            tol[n, hq] = 6 * sig + 2.0 ** -7 * np.abs(o) + 1e-6 * np.abs(v).max()
    return tol


def _tree_decisions(S, slots, trees, drafts, probs, logits, seed, mode, temperature):
    """Oracle tree decisions on the given logits; borderline = an accept test within 1e-5 or a race
    whose top-2 scores are within 1e-5 relative."""
    out, r0, off = [], 0, 0
    m = verify.GREEDY if mode == "greedy" else verify.SAMPLE
    for s, par in zip(slots, trees):
        c = S.ctx[s] if hasattr(S, "ctx") else S[s]
        k = len(par)
        lrow = logits[r0:r0 + k + 1]
        dr = [int(t) for t in drafts[off:off + k]]
        qr = None if probs is None else f64(probs[off:off + k])
        r = tree.verify_tree(lrow, dr, par, qr, seed, c["rid"], c["L"], m, temperature)
        r["borderline"] = m == verify.SAMPLE and any(np.isfinite(rt) and abs(u - rt) < 1e-5 for _, u, rt in r["tests"])
        out.append(r)
        r0 += k + 1
        off += k
    return out


def run_tree_and_check(S, slots, trees, drafts, mode, seed=99, temperature=1.0, probs=None):
    cfg, lane = S.cfg, S.lane
    depths = [len(t) for t in trees]
    par_dev = torch.tensor(_flat(trees), dtype=torch.int32).cuda()
    acc, tok, nodes = lane.verify_tree(slots, depths, par_dev, drafts.cuda(),
                                       None if probs is None else probs.cuda(), seed=seed, mode=mode,
                                       temperature=temperature)
    torch.cuda.synchronize()
    acc, tok, nodes = acc.cpu().numpy(), tok.cpu().numpy(), nodes.cpu().numpy()
    T = sum(k + 1 for k in depths)
    D, V, Hq, Hkv, dh = cfg.d_model, cfg.vocab, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
    report = {}
    toks, pos, off = [], [], 0
    for s, par in zip(slots, trees):
        c = S.ctx[s]
        toks += [c["pending"]] + [int(t) for t in drafts[off:off + len(par)]]
        pos += [c["L"] + dp for dp in tree.depths(par)]
        off += len(par)
    toks, pos = np.array(toks), np.array(pos)
    W = S.wnp
    h0 = S.tap("h0", torch.float32, (T, D))
    assert np.array_equal(f64(h0), model.embed(W["embed"], toks))
    a = S.tap("a", torch.bfloat16, (T, D))
    cos = S.tap("rope_cos", torch.float32, (cfg.max_pos, dh // 2)).numpy()
    sin = S.tap("rope_sin", torch.float32, (cfg.max_pos, dh // 2)).numpy()
    q, k, v = model.qkv_rope(f64(a), W["wqkv"][0], pos, cos, sin, Hq, Hkv, dh)   # positions L + depth
    gq = S.tap("q", torch.bfloat16, (T, Hq, dh))
    Tmax = cfg.max_batch * (cfg.max_depth + 1)
    gk = S.tap("kc", torch.bfloat16, (cfg.n_layers, Tmax, Hkv, dh))[0, :T]
    gv = S.tap("vc", torch.bfloat16, (cfg.n_layers, Tmax, Hkv, dh))[0, :T]
    _cmp_bf16("q", gq, q, report)
    _cmp_bf16("k", gk, k, report)
    _cmp_bf16("v", gv, v, report)
    go = S.tap("o", torch.bfloat16, (T, Hq * dh))
    worst, r0 = 0.0, 0
    for s, par in zip(slots, trees):
        c = S.ctx[s]
        R = len(par) + 1
        q_, ck, cv = f64(gq[r0:r0 + R]), f64(c["k"][0]), f64(c["v"][0])
        kc_, vc_ = f64(gk[r0:r0 + R]), f64(gv[r0:r0 + R])
        ref = tree.tree_attention(q_, ck, cv, kc_, vc_, par).reshape(R, Hq, dh)
        g = f64(go[r0:r0 + R]).reshape(R, Hq, dh)
        worst = max(worst, float((np.abs(g - ref) / _tree_tolerance(q_, ck, cv, kc_, vc_, par)).max()))
        r0 += R
    report["o_err_over_tol"] = worst
    assert worst <= 1.0, worst
    h1 = S.tap("h1", torch.float32, (T, D))
    _cmp_resid("h1", f64(h1), model.attn_out(f64(h0), f64(go), W["wo"][0]), report)
    lg = S.tap("logits", torch.float32, (T, V))
    z = S.tap("z", torch.bfloat16, (T, D))
    ref_l = model.lm_head(f64(z), W["lm_head"])
    row_err = np.abs(f64(lg) - ref_l).max(axis=1) / np.maximum(1.0, np.abs(ref_l).max(axis=1))
    assert row_err.max() <= LOGIT_REL, row_err.max()
    res = _tree_decisions(S, slots, trees, drafts, probs, f64(lg), seed, mode, temperature)
    borderline = 0
    K1 = cfg.max_depth + 1
    for b, r in enumerate(res):
        ok = acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"] and \
            list(nodes[b][: r["a"] + 1]) == r["path"]
        if not ok:
            assert mode == "sample" and r["borderline"], (b, acc[b], tok[b], nodes[b], r)
            borderline += 1
        assert all(t == -1 for t in tok[b][acc[b] + 1:K1]) and all(t == -1 for t in nodes[b][acc[b] + 1:K1])
    report["borderline"] = borderline
    report["accepted"] = acc.tolist()
    return report, acc, tok, nodes


def _planted_toy(seed=0, beta=0.3):
    cfg = synth.TOY_MLP
    w = synth.model_weights(cfg, seed=seed, norm_one=False)
    w, f = synth.planted_successor(cfg, w, seed=seed + 1, beta=beta)
    return cfg, w, f


def _greedy_tree_drafts(S, slots, trees, f, rng):
    """Node tokens: the planted successor of the parent's token (accepted) with probability 0.7,
    else a random token (rejected), so the walks go several levels deep and branch."""
    out = []
    for s, par in zip(slots, trees):
        toks = [S.ctx[s]["pending"]]
        for p in par:
            t = int(f[toks[p]]) if rng.random() < 0.7 else int(rng.integers(S.cfg.vocab))
            toks.append(t)
        out += toks[1:]
    return torch.tensor(out, dtype=torch.int32)


@pytest.mark.parametrize("mode", ["greedy", "sample"])
def test_tree_stages_toy(mode):
    """rows-on-lanes attention (d_h = 64, G = 1); planted model so greedy walks go deep."""
    cfg, w, f = _planted_toy()
    S = Setup(cfg, [128, 77, 300, 5, 64], seed=3, weights=w)
    rng = np.random.default_rng(4)
    slots = [0, 1, 2, 3, 4]
    drafts = _greedy_tree_drafts(S, slots, TREES, f, rng)
    probs = synth.draft_probs_dense(len(drafts), cfg.vocab, seed=8) if mode == "sample" else None
    rep, acc, _, _ = run_tree_and_check(S, slots, TREES, drafts, mode, probs=probs, temperature=0.9)
    print(mode, rep)
    if mode == "greedy":
        assert max(acc) >= 2                     # the planted drafts make the walk go deep somewhere


@pytest.mark.parametrize("env", [{}, {"SV_ATTN": "simt"}, {"SV_ATTN": "tc1"}])
def test_tree_stages_llama_shape(env):
    """keys-on-lanes attention (default; G = 4, (k+1) G <= 64), the SIMT and rows-on-lanes paths."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        cfg = synth.LLAMA.with_(n_pages=128, max_slots=6, max_batch=6, max_pos=2048)
        S = Setup(cfg, [300, 1100, 64, 700, 1], seed=23)
        slots = [0, 1, 2, 3, 4]
        drafts = synth.random_tokens(len(_flat(TREES)), cfg.vocab, seed=24)
        rep, _, _, _ = run_tree_and_check(S, slots, TREES, drafts, "greedy")
        print(env, rep)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("mode", ["greedy", "sample"])
def test_chain_shaped_tree_equals_sv_verify_bitwise(mode):
    cfg, w, f = _planted_toy(seed=5)
    S1 = Setup(cfg, [128, 40, 200], seed=6, weights=w)
    S2 = Setup(cfg, [128, 40, 200], seed=6, weights=w)
    depths = [3, 0, 6]
    rng = np.random.default_rng(1)
    trees = [list(range(k)) for k in depths]
    drafts = _greedy_tree_drafts(S1, [0, 1, 2], trees, f, rng).cuda()
    probs = synth.draft_probs_dense(len(drafts), cfg.vocab, seed=2).cuda() if mode == "sample" else None
    T = sum(depths) + 3
    l1 = torch.empty(T, cfg.vocab, device="cuda")
    l2 = torch.empty(T, cfg.vocab, device="cuda")
    for step in range(2):
        a1, t1 = (x.clone() for x in S1.lane.verify([0, 1, 2], depths, drafts, probs, seed=7, mode=mode,
                                                     temperature=0.8, logits_out=l1))
        par = torch.tensor(_flat(trees), dtype=torch.int32).cuda()
        a2, t2, n2 = S2.lane.verify_tree([0, 1, 2], depths, par, drafts, probs, seed=7, mode=mode, temperature=0.8,
                                          logits_out=l2)
        torch.cuda.synchronize()
        assert torch.equal(a1, a2) and torch.equal(t1, t2) and torch.equal(l1, l2)
        for b in range(3):
            a = int(a2[b])
            assert n2[b, : a + 1].tolist() == list(range(a + 1))
        S1.lane.commit()
        S2.lane.commit()
    s1, s2 = S1.lane.stats(), S2.lane.stats()
    assert s1 == s2


def test_tree_free_running_against_the_oracle_lane():
    """Three verify_tree + commit steps (greedy, planted toy+mlp): accepted paths, emitted tokens and
    the committed KV (seen through the next step's logits) follow the fp64 oracle lane."""
    cfg, w, f = _planted_toy(seed=9)
    gpu = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
    orc = OracleLane(cfg, {k: v.to(torch.float32).numpy() for k, v in w.items()})
    ctx = [(100, 7), (37, 11), (250, 300)]
    state = []
    for s, (n, pend) in enumerate(ctx):
        k, v = synth.context_kv(cfg, n, seed=60 + s)
        gpu.append_kv(s, 5000 + s, k.cuda(), v.cuda(), pend)
        orc.append_kv(s, 5000 + s, k.to(torch.float32).numpy(), v.to(torch.float32).numpy(), pend)
        state.append(dict(pending=pend))
    rng = np.random.default_rng(3)
    trees = [[0, 0, 1, 1, 3], [0, 1, 2, 0], [0, 0, 0, 1, 2, 3, 4, 4]]
    total = 0
    for step in range(3):
        drafts = []
        for s, par in enumerate(trees):
            toks = [orc.slots[s]["pending"]]
            for p in par:
                toks.append(int(f[toks[p]]) if rng.random() < 0.75 else int(rng.integers(cfg.vocab)))
            drafts += toks[1:]
        T = sum(len(t) + 1 for t in trees)
        lg = torch.empty(T, cfg.vocab, device="cuda")
        par = torch.tensor(_flat(trees), dtype=torch.int32).cuda()
        acc, tok, nodes = gpu.verify_tree([0, 1, 2], [len(t) for t in trees], par,
                                          torch.tensor(drafts, dtype=torch.int32).cuda(), seed=1, mode="greedy",
                                          logits_out=lg)
        oacc, oem, olg, opaths = orc.verify_tree([0, 1, 2], [len(t) for t in trees], _flat(trees), drafts, None, 1,
                                                 verify.GREEDY)
        torch.cuda.synchronize()
        lg = f64(lg)
        r0 = 0
        for b, par_b in enumerate(trees):
            R = len(par_b) + 1
            ref = olg[b]
            err = np.abs(lg[r0:r0 + R] - ref).max()
            assert err <= 5e-3 * max(1.0, np.abs(ref).max()), (step, b, err)
            assert int(acc[b]) == oacc[b] and tok[b, : oacc[b] + 1].tolist() == oem[b], (step, b)
            assert nodes[b, : oacc[b] + 1].tolist() == opaths[b]
            total += oacc[b]
            r0 += R
        gpu.commit()
        orc.commit()
    assert total >= 6                          # the walks did accept several levels
    st = gpu.stats()
    assert st["accepted"] == orc.stats["accepted"] and st["accepted_independent"] == orc.stats["accepted_independent"]
    for s in range(3):
        assert int(gpu.tap("len", torch.int32, (cfg.max_slots,))[s]) == orc.length(s)


@pytest.mark.parametrize("dense", [True, False])
def test_tree_decisions_on_exact_logits(dense):
    """sv_verify_tree_logits on random logits: trees of up to 16 nodes, many siblings (several
    rejections and residual passes per node), sampled mode; decisions = oracle except borderline."""
    cfg = synth.TOY.with_(max_depth=16, max_batch=16, max_slots=16)
    V = cfg.vocab
    S = Setup(cfg, [10 + 13 * i for i in range(16)], seed=2)
    rng = np.random.default_rng(5 + dense)
    for rep in range(3):
        trees = []
        for b in range(16):
            k = int(rng.integers(0, 17))
            trees.append([int(rng.integers(0, max(1, min(n, 3)))) if rng.random() < 0.6 else int(rng.integers(0, n))
                          for n in range(1, k + 1)])
        depths = [len(t) for t in trees]
        T = sum(depths) + 16
        logits = torch.randn(T, V, dtype=torch.float64) * 2.5
        logits32 = logits.to(torch.float32)
        probs = synth.draft_probs_dense(sum(depths), V, seed=30 + rep) if dense else None
        # drafts drawn from q (dense) or near the target's top tokens (one-hot) so tests accept often
        if dense:
            drafts = synth.draft_tokens_from(probs, seed=40 + rep)
        else:
            drafts, off, r0 = [], 0, 0
            for t in trees:
                for n, p in enumerate(t, start=1):
                    top = torch.argsort(logits32[r0 + p], descending=True)
                    drafts.append(int(top[int(rng.integers(0, 3))]))
                r0 += len(t) + 1
            drafts = torch.tensor(drafts, dtype=torch.int32)
        par = torch.tensor(_flat(trees), dtype=torch.int32).cuda()
        acc, tok, nodes = S.lane.verify_tree_logits(list(range(16)), depths, par, drafts.cuda(), logits32.cuda(),
                                                    None if probs is None else probs.cuda(), seed=77 + rep,
                                                    mode="sample", temperature=1.1)
        torch.cuda.synchronize()
        acc, tok, nodes = acc.cpu().numpy(), tok.cpu().numpy(), nodes.cpu().numpy()
        res = _tree_decisions(S, list(range(16)), trees, drafts, probs, logits32.to(torch.float64).numpy(), 77 + rep,
                              "sample", 1.1)
        bad = 0
        for b, r in enumerate(res):
            if not (acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"]
                    and list(nodes[b][: r["a"] + 1]) == r["path"]):
                assert r["borderline"], (rep, b, acc[b], tok[b], nodes[b], r)
                bad += 1
        print("borderline", bad, "accepted", acc.tolist())
        assert sum(acc) > 0


def test_bad_parent_sets_the_device_error():
    cfg = synth.TOY
    S = Setup(cfg, [20, 30], seed=1)
    par = torch.tensor([0, 0, 3, 0, 1], dtype=torch.int32).cuda()      # request 0: node 3's parent is 3
    drafts = synth.random_tokens(5, cfg.vocab, seed=3).cuda()
    acc, tok, nodes = S.lane.verify_tree([0, 1], [3, 2], par, drafts, mode="greedy")
    torch.cuda.synchronize()
    assert int(acc[0]) == -1 and int(acc[1]) >= 0
    assert tok[0].tolist() == [-1] * (cfg.max_depth + 1)
    S.lane.commit()
    with pytest.raises(sv.SvError):
        S.lane.stats()
    assert int(S.lane.tap("len", torch.int32, (cfg.max_slots,))[0]) == 20
