"""Pins for oracle/tree.py (token-tree drafts, NEXT-4, R30).

Every expected value comes from something other than oracle/tree.py itself: the already pinned
chain verifier and chain attention (a chain is a tree of only-children; a tree row is the last
row of its root path), torch's scaled_dot_product_attention with an explicit ancestor mask,
enumeration of root paths, and the losslessness theorem of speculative sampling (the emitted
tokens follow the target's autoregressive law), checked by chi-square.
"""
import copy

import numpy as np
import pytest
import torch
import torch.nn.functional as F
from scipy import stats

import synth
from oracle import model, tree, verify
from oracle.lane import OracleLane
from oracle.numerics import round_bf16
from oracle.philox import uniform_accept, uniform_accept_rank

ALPHA = 0.01


def _chisq(observed, expected_p):
    obs = np.asarray(observed, dtype=np.float64)
    n = obs.sum()
    exp = np.asarray(expected_p, dtype=np.float64) * n
    assert obs[exp == 0].sum() == 0               # nothing emitted outside the support
    big = exp >= 5
    if exp[~big].sum() == 0:
        big = exp > 0
    o = list(obs[big]) + ([obs[~big].sum()] if (~big).any() else [])
    e = list(exp[big]) + ([exp[~big].sum()] if (~big).any() else [])
    o, e = np.array(o), np.array(e)
    o, e = o[e > 0], e[e > 0]
    e *= o.sum() / e.sum()
    return stats.chisquare(o, e).pvalue


def _simplex(rng, V, sharp=2.0, zeros=0):
    w = rng.exponential(size=V) ** sharp
    if zeros:
        w[rng.choice(V, zeros, replace=False)] = 0.0
    return w / w.sum()


def _log(p):
    return np.log(np.where(p > 0, p, 1e-300))


# ------------------------------------------------------------------ structure + RNG

def test_rank_zero_uniform_is_the_chain_uniform():
    for seed, rid, z in [(0, 0, 0), (11, 5, 1), (2 ** 40 + 3, 2 ** 33 + 7, 4095)]:
        assert uniform_accept_rank(seed, rid, z, 0) == uniform_accept(seed, rid, z)
    # distinct ranks draw distinct words (lanes 1..3 and the next counter block)
    us = {uniform_accept_rank(5, 9, 100, s) for s in range(12)}
    assert len(us) == 12


def test_parent_validation_and_depths():
    tree.check_parents([0, 0, 1, 1, 3])
    assert tree.depths([0, 0, 1, 1, 3]) == [0, 1, 1, 2, 2, 3]
    assert tree.path([0, 0, 1, 1, 3], 5) == [0, 1, 3, 5]
    for bad in ([1], [0, 2], [0, -1]):
        with pytest.raises(ValueError):
            tree.check_parents(bad)


# ------------------------------------------------------------------ chain reduction

@pytest.mark.parametrize("mode", [verify.GREEDY, verify.SAMPLE])
@pytest.mark.parametrize("dense", [True, False])
def test_chain_shaped_tree_equals_chain_verifier(mode, dense):
    rng = np.random.default_rng(5 + 2 * mode + dense)
    V, k = 16, 5
    for trial in range(300):
        logits = rng.standard_normal((k + 1, V)) * 2
        q = np.stack([_simplex(rng, V, zeros=2) for _ in range(k)]) if dense else None
        if mode == verify.GREEDY:
            top = logits.argmax(1)
            drafts = [int(top[j]) if rng.random() < 0.7 else int(rng.integers(V)) for j in range(k)]
        else:
            drafts = [int(rng.choice(V, p=q[j])) if dense else int(rng.integers(V)) for j in range(k)]
        want = verify.verify_request(logits, drafts, q, 31, trial, 50, mode, 0.9)
        got = tree.verify_tree(logits, drafts, list(range(k)), q, 31, trial, 50, mode, 0.9)
        assert (got["a"], got["emitted"], got["indep"]) == (want["a"], want["emitted"], want["indep"])
        assert got["path"] == list(range(got["a"] + 1))


# ------------------------------------------------------------------ attention

def test_tree_attention_matches_torch_sdpa_with_ancestor_mask():
    rng = np.random.default_rng(1)
    parents = [0, 0, 1, 1, 2, 0, 6]
    R, L, Hq, Hkv, dh = len(parents) + 1, 29, 8, 2, 16
    q = rng.standard_normal((R, Hq, dh))
    ck, cv = rng.standard_normal((L, Hkv, dh)), rng.standard_normal((L, Hkv, dh))
    kk, vv = rng.standard_normal((R, Hkv, dh)), rng.standard_normal((R, Hkv, dh))
    got = tree.tree_attention(q, ck, cv, kk, vv, parents)
    # mask[n][m]: m is n or an ancestor of n, by following parent pointers here
    mask = torch.zeros(R, L + R, dtype=torch.bool)
    mask[:, :L] = True
    for n in range(R):
        m = n
        while True:
            mask[n, L + m] = True
            if m == 0:
                break
            m = parents[m - 1]
    K = torch.tensor(np.concatenate([ck, kk])).permute(1, 0, 2).repeat_interleave(Hq // Hkv, dim=0)
    Vt = torch.tensor(np.concatenate([cv, vv])).permute(1, 0, 2).repeat_interleave(Hq // Hkv, dim=0)
    ref = F.scaled_dot_product_attention(torch.tensor(q).permute(1, 0, 2), K, Vt, attn_mask=mask)
    ref = ref.permute(1, 0, 2).reshape(R, Hq * dh).numpy()
    assert np.max(np.abs(got - round_bf16(ref))) <= 2.0 ** -7 * np.max(np.abs(ref))
    assert np.mean(got == round_bf16(ref)) > 0.999


def test_tree_attention_row_is_chain_attention_on_its_path():
    rng = np.random.default_rng(2)
    parents = [0, 1, 0, 3, 3, 1]
    R, L, Hq, Hkv, dh = len(parents) + 1, 17, 4, 2, 8
    q = rng.standard_normal((R, Hq, dh))
    ck, cv = rng.standard_normal((L, Hkv, dh)), rng.standard_normal((L, Hkv, dh))
    kk, vv = rng.standard_normal((R, Hkv, dh)), rng.standard_normal((R, Hkv, dh))
    got = tree.tree_attention(q, ck, cv, kk, vv, parents)
    for n in range(R):
        pth = tree.path(parents, n)
        ref = model.verify_attention(q[pth], ck, cv, kk[pth], vv[pth])
        assert np.array_equal(got[n], ref[-1])


@pytest.mark.parametrize("cfgname", ["toy", "toy_mlp"])
def test_tree_forward_equals_chain_forward_on_every_root_path(cfgname):
    cfg = synth.CONFIGS[cfgname]
    w = {k: synth.as_f64(v) for k, v in synth.model_weights(cfg, seed=3, norm_one=False).items()}
    cos, sin = model.rope_table(cfg.max_pos, cfg.head_dim, cfg.rope_theta)
    k_, v_ = synth.context_kv(cfg, 21, seed=4)
    caches = [(synth.as_f64(k_)[l], synth.as_f64(v_)[l]) for l in range(cfg.n_layers)]
    parents = [0, 0, 1, 2, 2, 0]
    toks = [5, 17, 17, 90, 3, 44, 200]
    L = 21
    _, lg, kv = tree.forward_tree(w, toks, parents, L, caches, cfg, cos, sin)
    leaves = [n for n in range(len(toks)) if not tree.children(parents, n)]
    for leaf in leaves:
        pth = tree.path(parents, leaf)
        _, lc, kvc = model.forward_chain(w, [toks[n] for n in pth], L + np.arange(len(pth)), caches, cfg, cos, sin)
        assert np.allclose(lg[pth], lc, rtol=0, atol=1e-9 * np.abs(lc).max())
        for layer in range(cfg.n_layers):
            assert np.array_equal(kv[layer][0][pth], kvc[layer][0])
            assert np.array_equal(kv[layer][1][pth], kvc[layer][1])


# ------------------------------------------------------------------ greedy

def test_greedy_walk_equals_brute_force_path_enumeration():
    rng = np.random.default_rng(7)
    V = 6
    for trial in range(400):
        k = int(rng.integers(1, 10))
        parents = [int(rng.integers(0, n)) for n in range(1, k + 1)]
        logits = rng.standard_normal((k + 1, V))
        top = logits.argmax(1)
        drafts = [int(top[parents[n - 1]]) if rng.random() < 0.6 else int(rng.integers(V))
                  for n in range(1, k + 1)]
        r = tree.verify_tree(logits, drafts, parents, None, 0, trial, 10, verify.GREEDY)
        # brute force: every root path all of whose tokens are their parent's argmax; the walk
        # takes the lowest-index matching child, i.e. the lexicographically first such path
        best = [0]
        for n in range(k + 1):
            pth = tree.path(parents, n)
            if all(drafts[m - 1] == top[parents[m - 1]] for m in pth[1:]):
                if len(pth) > len(best) or (len(pth) == len(best) and pth < best):
                    best = pth
        walk = r["path"]
        match = lambda m: drafts[m - 1] == top[parents[m - 1]]
        assert walk[0] == 0 and all(parents[walk[i] - 1] == walk[i - 1] and match(walk[i]) for i in range(1, len(walk)))
        assert not any(match(c) for c in tree.children(parents, walk[-1]))      # maximal
        for i in range(1, len(walk)):                                           # lowest matching child
            assert walk[i] == min(c for c in tree.children(parents, walk[i - 1]) if match(c))
        assert r["a"] == len(walk) - 1
        assert r["emitted"] == [drafts[m - 1] for m in walk[1:]] + [int(top[walk[-1]])]
        assert len(walk) <= len(best)
        if len(set(drafts)) == k:                    # distinct tokens: the matching path is unique
            assert walk == best


# ------------------------------------------------------------------ sampled: losslessness

def _target_table(rng, V, depth):
    """A target 'model': p(. | prefix) for every token prefix up to `depth` (a dict)."""
    table = {}

    def rec(prefix):
        table[prefix] = _simplex(rng, V, zeros=1)
        if len(prefix) < depth:
            for x in range(V):
                rec(prefix + (x,))
    rec(())
    return table


@pytest.mark.parametrize("dense", [True, False])
def test_sampled_tree_emits_the_target_law(dense):
    """Root with 3 children, each child with 2 children (9 nodes): drafts drawn i.i.d. per parent
    from q (dense), or the distinct top tokens of q (one-hot). The first two emitted tokens
    must follow p(x) p(y | x) whatever the drafts."""
    rng = np.random.default_rng(11 + dense)
    V = 5
    table = _target_table(rng, V, 2)
    parents = [0, 0, 0, 1, 1, 2, 2, 3, 3]
    n = 12000
    first = np.zeros(V)
    pair = np.zeros((V, V))
    qtab = {pre: _simplex(rng, V) for pre in table}
    for rid in range(n):
        toks = {0: ()}
        drafts, qrows = [], []
        for node, par in enumerate(parents, start=1):
            pre = toks[par]
            q = qtab[pre]
            if dense:
                d = int(rng.choice(V, p=q))
            else:                                     # distinct siblings: the parent's m-th best
                m = tree.children(parents, par).index(node)
                d = int(np.argsort(-q, kind="stable")[m])
            drafts.append(d)
            qrows.append(q)
            toks[node] = pre + (d,)
        logits = np.stack([_log(table[toks[nd]]) if len(toks[nd]) <= 2 else np.zeros(V)
                           for nd in range(len(parents) + 1)])
        r = tree.verify_tree(logits, drafts, parents, np.array(qrows) if dense else None,
                             1234, rid, 30, verify.SAMPLE)
        em = r["emitted"]
        first[em[0]] += 1
        if len(em) >= 2:
            pair[em[0], em[1]] += 1
    assert _chisq(first, table[()]) > ALPHA
    for x in range(V):
        if pair[x].sum() > 500:
            assert _chisq(pair[x], table[(x,)]) > ALPHA


def test_two_sibling_residual_closed_form():
    """Root children c1, c2 with one-hot q: P(accept c1) = p(c1); P(accept c2) =
    (1 - p(c1)) p(c2) / (1 - p(c1)) = p(c2); resample from p with both removed otherwise."""
    p = np.array([0.1, 0.2, 0.3, 0.4])
    logits = np.stack([np.log(p)] * 3)
    counts = {}
    n = 20000
    for rid in range(n):
        r = tree.verify_tree(logits, [3, 1], [0, 0], None, 8, rid, 0, verify.SAMPLE)
        key = (tuple(r["path"]), r["emitted"][0])
        counts[key] = counts.get(key, 0) + 1
        if r["path"] == [0]:
            assert r["emitted"][0] in (0, 2)
    want = {((0, 1), 3): 0.4, ((0, 2), 1): 0.2, ((0,), 0): 0.1, ((0,), 2): 0.3}
    keys = sorted(want)
    assert set(counts) == set(want)
    assert _chisq([counts[k] for k in keys], [want[k] for k in keys]) > ALPHA


def test_duplicate_sibling_is_rejected_with_one_hot_q():
    p = np.array([0.5, 0.5])
    logits = np.stack([np.log(p)] * 3)
    for rid in range(200):
        r = tree.verify_tree(logits, [1, 1], [0, 0], None, 3, rid, 0, verify.SAMPLE)
        assert r["path"] != [0, 2]                 # the second copy has zero residual mass
        assert r["emitted"][0] in (0, 1)


# ------------------------------------------------------------------ lane: commit keeps the path

def test_lane_tree_commit_keeps_the_accepted_path():
    cfg = synth.TOY_MLP
    w = {k: synth.as_f64(v) for k, v in synth.model_weights(cfg, seed=0, norm_one=False).items()}
    lane = OracleLane(cfg, w)
    k_, v_ = synth.context_kv(cfg, 30, seed=1)
    lane.append_kv(0, 77, synth.as_f64(k_), synth.as_f64(v_), pending_token=9)
    # greedy continuation of the pending token, by plain decode steps
    ref = copy.deepcopy(lane)
    cont = []
    for _ in range(3):
        _, em, _ = ref.verify([0], [0], [], None, 0, verify.GREEDY)
        ref.commit()
        cont.append(em[0][0])
    wrong = [(t + 1) % cfg.vocab for t in cont]
    # tree: root -> {wrong0, cont0}; cont0 -> {wrong1, cont1}; a decoy under wrong0
    parents = [0, 0, 2, 2, 1]
    drafts = [wrong[0], cont[0], wrong[1], cont[1], cont[1]]
    acc, em, _, paths = lane.verify_tree([0], [5], parents, drafts, None, 0, verify.GREEDY)
    assert acc == [2] and paths == [[0, 2, 4]] and em[0] == cont[:3]
    lane.commit()
    assert lane.length(0) == 33
    for layer in range(cfg.n_layers):
        assert np.array_equal(lane.slots[0]["K"][layer][:33], ref.slots[0]["K"][layer][:33])
        assert np.array_equal(lane.slots[0]["V"][layer][:33], ref.slots[0]["V"][layer][:33])
    assert lane.slots[0]["pending"] == cont[2]
