"""Tree-structured drafts (EAGLE-2-style token trees), in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper names tree drafting only as related work (EAGLE's draft trees; its own
SpecuStream drafts chains). The generalisation below is DESIGN.md reading R30, written out in
this order:

  tree     node 0 = the pending token x (the chain head), nodes 1..k = drafts d_1..d_k;
           parent(n) in [0, n-1] (topological order); depth(0) = 0, depth(n) = depth(parent) + 1;
           anc*(n) = {n} and the ancestors of n.
  forward  node n sits at absolute position L + depth(n); its query attends the cache keys
           0..L-1 and the chain keys of anc*(n) (model step 1.5 with the causal chain mask
           replaced by the ancestor mask). A chain (parent(n) = n - 1) is the verify chain.
  GREEDY   cur = 0: y = argmax l_cur (lowest id); the first child c of cur (ascending node
           index) with d_c = y becomes cur; stop when none. a = depth(cur), emitted = the
           path's tokens, then y.
  SAMPLE   recursive rejection over siblings (multi-draft speculative sampling, SpecInfer):
           at cur, r = p_cur = softmax(l_cur / T); for its children c_0, c_1, ... in index
           order (sibling rank s): u = U(seed, rid, L + depth(cur) + 1, ACCEPT, s);
           accept c_s iff u < r(d_c) / q_c(d_c) (+inf when q_c(d_c) = 0; R3);
           on acceptance cur = c_s and r = p_cur afresh; on rejection
           r <- max(0, r - q_c) / Z (Z = its sum; Z = 0 keeps r, R4); q_c = one-hot at d_c when
           draft_probs is NULL. When cur has no child left, y is drawn from r by the exponential
           race at z = L + depth(cur) + 1 (R5). Each c_s is drawn from q_c independently of its
           siblings, so every step is a Leviathan step against the current r and the emitted
           sequence follows the target (pinned below by chi-square).
  commit   the path's rows (node 0, n_1, ..., n_a) land at positions L .. L + a (their RoPE
           positions), everything else is dropped.
  a7       indep = sum over nodes of the node's own test against its parent's unmodified
           target: [d_n = argmax l_parent] (GREEDY) or [U(z_n, rank_n) < p_parent(d_n)/q_n(d_n)]
           (SAMPLE). For a chain all of this is verify.verify_request.

Pinned by tests/test_oracle_tree.py: a chain-shaped tree equals the pinned chain verifier in
both modes (same uniforms: rank 0 is the chain's counter); tree attention row n equals the
pinned chain attention on the root-to-n path; the tree forward equals forward_chain on every
root-to-leaf path; greedy walk = brute-force enumeration of root paths; sampled emission law =
the target's autoregressive law (chi-square, dense q with i.i.d. siblings and one-hot q with
distinct siblings); accept/reject and residual closed forms on a two-sibling example.
"""
import numpy as np

from . import model
from .numerics import round_bf16
from .philox import uniform_accept_rank, uniform_race
from .verify import GREEDY, SAMPLE, argmax_lowest, filtered_probs


def check_parents(parents):
    """parents[n-1] = parent of node n (n = 1..k); raises on a non-topological entry."""
    for n, p in enumerate(parents, start=1):
        if not (0 <= int(p) < n):
            raise ValueError(f"node {n}: parent {p} not in [0, {n - 1}]")


def depths(parents):
    dep = [0]
    for p in parents:
        dep.append(dep[int(p)] + 1)
    return dep


def path(parents, n):
    """Node indices root..n (root first)."""
    out = [n]
    while n != 0:
        n = int(parents[n - 1])
        out.append(n)
    return out[::-1]


def children(parents, n):
    return [c for c in range(1, len(parents) + 1) if int(parents[c - 1]) == n]


def tree_attention(q, cache_k, cache_v, chain_k, chain_v, parents):
    """Model step 1.5 with the ancestor mask: node n attends cache keys 0..L-1 and chain keys
    anc*(n) (ascending node order; the softmax is order free). Shapes as model.verify_attention."""
    R, Hq, dh = q.shape
    Hkv = chain_k.shape[1]
    G = Hq // Hkv
    L = cache_k.shape[0]
    out = np.zeros((R, Hq, dh))
    for n in range(R):
        vis = sorted(path(parents, n))
        keys = np.concatenate([cache_k[:L], chain_k[vis]], axis=0)
        vals = np.concatenate([cache_v[:L], chain_v[vis]], axis=0)
        for hq in range(Hq):
            hk = hq // G
            s = keys[:, hk, :] @ q[n, hq, :] / np.sqrt(dh)
            out[n, hq, :] = model.softmax(s) @ vals[:, hk, :]
    return round_bf16(out.reshape(R, Hq * dh))


def forward_tree(w, tokens, parents, L, caches, cfg, cos, sin):
    """Model forward (model steps 1.1-1.8) of one request's token tree. tokens [k+1] = [x, d_1..].

    Returns (z, logits [k+1][V], chain_kv per layer of (k, v) [k+1][Hkv][dh]).
    """
    pos = L + np.asarray(depths(parents), dtype=np.int64)
    h = model.embed(w["embed"], tokens)
    chain_kv = []
    for layer in range(cfg.n_layers):
        ck, cv = caches[layer]
        a = model.attn_norm(h, np.asarray(w["attn_norm"][layer], dtype=np.float64), cfg.norm_eps)
        q, k, v = model.qkv_rope(a, w["wqkv"][layer], pos, cos, sin, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim)
        o = tree_attention(q, ck, cv, k, v, parents)
        h = model.attn_out(h, o, w["wo"][layer])
        if cfg.ffn_dim > 0:
            b = model.ffn_norm(h, np.asarray(w["ffn_norm"][layer], dtype=np.float64), cfg.norm_eps)
            h = model.down_residual(h, model.swiglu(b, w["w_gate_up"][layer]), w["w_down"][layer])
        chain_kv.append((k, v))
    z = model.final_norm(h, np.asarray(w["final_norm"], dtype=np.float64), cfg.norm_eps)
    return z, model.lm_head(z, w["lm_head"]), chain_kv


def verify_tree(logits, drafts, parents, q_rows, seed, rid, L, mode, temperature=1.0, top_k=0, top_p=1.0):
    """Decide one request's token tree. logits [k+1][V] (row n = node n); drafts [k] (d_n =
    drafts[n-1]); parents [k]; q_rows [k][V] (row n-1 = the distribution d_n was drawn from) or
    None (one-hot). Returns dict(a, emitted, path, indep, tests) where tests lists the sampled
    accept tests made on the walk as (node, u, ratio) (for borderline analysis)."""
    logits = np.asarray(logits, dtype=np.float64)
    k = len(drafts)
    assert logits.shape[0] == k + 1 and len(parents) == k
    check_parents(parents)
    dep = depths(parents)
    kids = [children(parents, n) for n in range(k + 1)]
    rank = {c: s for n in range(k + 1) for s, c in enumerate(kids[n])}
    if mode == GREEDY:
        top = [argmax_lowest(logits[n]) for n in range(k + 1)]
        cur, walk = 0, [0]
        while True:
            nxt = [c for c in kids[cur] if int(drafts[c - 1]) == top[cur]]
            if not nxt:
                break
            cur = nxt[0]
            walk.append(cur)
        indep = sum(1 for n in range(1, k + 1) if int(drafts[n - 1]) == top[int(parents[n - 1])])
        return dict(a=dep[cur], emitted=[int(drafts[n - 1]) for n in walk[1:]] + [top[cur]], path=walk,
                    indep=indep, tests=[])
    assert mode == SAMPLE
    p = filtered_probs(logits, temperature, top_k, top_p)     # R31 filtering (NEXT-4)
    V = p.shape[1]

    def qrow(c):
        if q_rows is None:
            e = np.zeros(V)
            e[int(drafts[c - 1])] = 1.0
            return e
        return np.asarray(q_rows[c - 1], dtype=np.float64)

    def ratio(r, c):
        d = int(drafts[c - 1])
        qd = qrow(c)[d]
        return np.inf if qd == 0.0 else r[d] / qd

    indep = 0
    for n in range(1, k + 1):
        par = int(parents[n - 1])
        u = uniform_accept_rank(seed, rid, L + dep[par] + 1, rank[n])
        indep += int(u < ratio(p[par], n))
    cur, walk, tests = 0, [0], []
    r = p[0]
    while True:
        z = L + dep[cur] + 1
        nxt = None
        for s, c in enumerate(kids[cur]):
            u = uniform_accept_rank(seed, rid, z, s)
            rt = ratio(r, c)
            tests.append((c, u, rt))
            if u < rt:
                nxt = c
                break
            R = np.maximum(0.0, r - qrow(c))
            if R.sum() > 0.0:
                r = R / R.sum()
        if nxt is None:
            break
        cur = nxt
        walk.append(cur)
        r = p[cur]
    E = -np.log(uniform_race(seed, rid, L + dep[cur] + 1, V))
    y = argmax_lowest(np.where(r > 0, r / E, -np.inf))
    return dict(a=dep[cur], emitted=[int(drafts[n - 1]) for n in walk[1:]] + [y], path=walk, indep=indep,
                tests=tests)
