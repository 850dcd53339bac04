"""Token trees (R30) and top-k / top-p filtering (R31) at the north-star size: workload `ns`
(64 requests x 4096-token contexts, Llama-3-8B-shaped layer + lm-head, planted-successor
weights), each request drafting an 8-node tree. Checked on what the oracle computes one by one:

* attention of sampled requests (all split-KV items, all 32 heads) with the ancestor mask, teacher-
  forced on the GPU's Q / chain K,V (tree tolerance of tests/test_gpu_tree.py);
* greedy tree walks of ALL 64 requests, bit-exact against oracle/tree.py on the GPU's fp32 logits;
* a sampled tree verify with top-k 50 / top-p 0.9 over the full 128256-token vocabulary: all 64
  requests' walks against the oracle on the GPU's logits (borderline excused and counted);
* commit of the accepted paths: the next verify's attention sees the committed rows."""
import numpy as np
import pytest
import torch

import bench
import synth
from oracle import tree, verify

from gpu_util import f64
from test_gpu_filter import _top_p_borderline
from test_gpu_tree import _tree_tolerance

pytestmark = pytest.mark.gpu

PARENTS = [0, 0, 1, 1, 2, 3, 5, 7]            # 8 nodes: two branches at the root, depth up to 5
K = len(PARENTS)


def _drafts(reqs, succ, rng, alpha):
    out = []
    for c in reqs:
        toks = [c["pending"]]
        for p in PARENTS:
            toks.append(int(succ[toks[p]]) if rng.random() < alpha else int(rng.integers(len(succ))))
        out += toks[1:]
    return out


@pytest.fixture(scope="module")
def lane_setup():
    wl = synth.workload("ns", steps_budget=4)
    dev = torch.device("cuda:0")
    lane, w, succ, reqs = bench.build_lane(wl, 0, dev)
    lane.set_taps(True)
    return wl, lane, w, succ, reqs


def _tap(lane, n, dt, sh):
    return lane.tap(n, dt, sh).cpu().clone()


def test_tree_greedy_full_size_then_filtered_sampled(lane_setup):
    wl, lane, w, succ, reqs = lane_setup
    cfg, B = wl.cfg, wl.batch
    rng = np.random.default_rng(0)
    depths = [K] * B
    par = torch.tensor(PARENTS * B, dtype=torch.int32).cuda()
    drafts = _drafts(reqs, succ.tolist(), rng, 0.7)
    acc, tok, nodes = lane.verify_tree(list(range(B)), depths, par, torch.tensor(drafts, dtype=torch.int32).cuda(),
                                       seed=1234, mode="greedy")
    torch.cuda.synchronize()
    T = B * (K + 1)
    Tmax = cfg.max_batch * (cfg.max_depth + 1)
    q = _tap(lane, "q", torch.bfloat16, (T, cfg.n_q_heads, cfg.head_dim))
    kc = _tap(lane, "kc", torch.bfloat16, (cfg.n_layers, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T]
    vc = _tap(lane, "vc", torch.bfloat16, (cfg.n_layers, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T]
    o = _tap(lane, "o", torch.bfloat16, (T, cfg.n_q_heads * cfg.head_dim))
    lg = _tap(lane, "logits", torch.float32, (T, cfg.vocab)).numpy().astype(np.float64)
    R = K + 1
    worst = 0.0
    for b in (0, 37, 63):
        r0 = b * R
        q_, kc_, vc_ = f64(q[r0:r0 + R]), f64(kc[r0:r0 + R]), f64(vc[r0:r0 + R])
        ck, cv = f64(reqs[b]["k"][0]), f64(reqs[b]["v"][0])
        ref = tree.tree_attention(q_, ck, cv, kc_, vc_, PARENTS).reshape(R, cfg.n_q_heads, cfg.head_dim)
        g = f64(o[r0:r0 + R]).reshape(R, cfg.n_q_heads, cfg.head_dim)
        worst = max(worst, float((np.abs(g - ref) / _tree_tolerance(q_, ck, cv, kc_, vc_, PARENTS)).max()))
    assert worst <= 1.0, worst
    acc, tok, nodes = acc.cpu().numpy(), tok.cpu().numpy(), nodes.cpu().numpy()
    for b in range(B):
        c = reqs[b]
        r = tree.verify_tree(lg[b * R:(b + 1) * R], drafts[b * K:(b + 1) * K], PARENTS, None, 1234, c["rid"], c["L"],
                             verify.GREEDY)
        assert (int(acc[b]), tok[b][:r["a"] + 1].tolist(), nodes[b][:r["a"] + 1].tolist()) == \
            (r["a"], r["emitted"], r["path"]), b
    assert acc.mean() > 1.0                   # the planted drafts are accepted several levels deep
    lane.commit()
    for b in range(B):
        reqs[b]["L"] += int(acc[b]) + 1
        reqs[b]["pending"] = int(tok[b][acc[b]])

    # sampled + filtered, full vocabulary, on the committed state
    lane.set_filter(50, 0.9)
    drafts = _drafts(reqs, succ.tolist(), rng, 0.6)
    probs = None
    acc, tok, nodes = lane.verify_tree(list(range(B)), depths, par, torch.tensor(drafts, dtype=torch.int32).cuda(),
                                       probs, seed=77, mode="sample", temperature=0.8)
    torch.cuda.synchronize()
    lg = _tap(lane, "logits", torch.float32, (T, cfg.vocab)).numpy().astype(np.float64)
    acc, tok, nodes = acc.cpu().numpy(), tok.cpu().numpy(), nodes.cpu().numpy()
    n_bl = 0
    for b in range(B):
        c = reqs[b]
        rows = lg[b * R:(b + 1) * R]
        r = tree.verify_tree(rows, drafts[b * K:(b + 1) * K], PARENTS, None, 77, c["rid"], c["L"], verify.SAMPLE, 0.8,
                             50, 0.9)
        if (int(acc[b]), tok[b][:r["a"] + 1].tolist(), nodes[b][:r["a"] + 1].tolist()) != \
                (r["a"], r["emitted"], r["path"]):
            bl = any(abs(u - rt) < 1e-5 for _, u, rt in r["tests"] if np.isfinite(rt)) or \
                any(_top_p_borderline(rows[j], 0.8, 0.9) for j in range(R))
            assert bl, (b, acc[b], tok[b], nodes[b], r)
            n_bl += 1
    print("filtered sampled: borderline", n_bl, "mean accepted", acc.mean())
    lane.commit()
    lane.set_filter(0, 1.0)
