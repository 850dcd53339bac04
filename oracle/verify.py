"""Speculative verification decisions and lane acceptance counters, in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper relies on but never defines the verification step (PAPER.md:37
"verifying multiple predicted tokens in parallel", PAPER.md:65 Leviathan
"preserving output distribution"). Our reading (R1-R9,
SURVEY.md §8(c) steps 2-5 and S1-S9, S14, S20) is Leviathan rejection sampling
with a bonus token, or a greedy prefix match, written out here in that order:

  step 2  p_{j+1} = softmax(l_j / temperature), j = 0..k (row j of the chain), then optionally
          top-k / top-p filtered (filtered_target, R31; NEXT-4) before everything below
  step 3  GREEDY: a = largest m <= k with d_j = argmax l_{j-1} for all j <= m
          (ties -> lowest id); emit d_1..d_a, y = argmax l_a
  step 4  SAMPLE: for j = 1..k
            u_j = U(seed, rid, L + j, ACCEPT)
            r_j = p_j(d_j) / q_j(d_j)   (+inf if q_j(d_j) = 0)
            accept iff u_j < r_j (strict); first failure ends the prefix: a = j-1
          if a < k: R = max(0, p_{a+1} - q_{a+1}); if sum R = 0: R = p_{a+1}
          else      R = p_{k+1}
          y = argmax_{x: R(x) > 0} R(x) / E_x,  E_x = -ln U(seed, rid, L + a + 1, RACE, x)
          (exponential race; P(y = x) = R(x) / sum R; ties -> lowest x)
          q NULL (one-hot at d_j): r_j = p_j(d_j); residual = p with d_{a+1} zeroed
  step 5  outputs a in [0, k], emitted = d_1..d_a, y
  PREFILL (NEXT-3, R29): a = k, y = argmax l_k (a prompt chunk whose KV is all kept; no counters)
  a7      lane counters: steps, rows, drafted, accepted,
          emitted, accepted_independent (sum over ALL j of [u_j < r_j], or of
          [d_j == argmax l_{j-1}] in greedy), hist_accepted[a],
          drafted_by_k[k] += k, accepted_by_k[k] += a.

Pinned by tests/test_oracle_verify.py: P1 (first emitted token ~ p_1 for any
q, chi-square), P2 (brute-force joint law of (a, emitted) on V <= 8, k <= 3),
P3 (truncated-geometric accepted length + SPEC.md:325 closed form), P4 (greedy
= argmax chain), P5 (bounds), P8 (multi-step sequence law under the RNG
layout), P10 (hand-derived worked example, tests/golden/verify_worked.json).
"""
import numpy as np

from .philox import uniform_accept, uniform_race
from .model import softmax

GREEDY = 0
SAMPLE = 1
PREFILL = 2    # NEXT-3 chunked prefill (R29): the "drafts" are prompt tokens, all kept
MAXK = 32


def argmax_lowest(row):
    """argmax with ties to the lowest index (numpy's first occurrence)."""
    return int(np.argmax(row))


def target_probs(logits, temperature):
    """step 2: p = softmax(l / temperature), fp64."""
    return softmax(np.asarray(logits, dtype=np.float64) / float(temperature), axis=-1)


def filtered_target(p_row, logits_row, top_k=0, top_p=1.0):
    """Top-k / top-p filtered target (reading R31), fp64:

      order the tokens by (scaled logit descending, token id ascending);
      n_k = top_k if 0 < top_k < V else V;
      n_p = V if top_p >= 1 else the smallest n with p(o_1) + ... + p(o_n) >= top_p
            (cumulative sum in that order);
      keep the first min(n_k, n_p) tokens; p' = p * [kept] / sum of the kept p.

    Temperature is applied before filtering (p = softmax(l / T), the logits row given here is
    l / T). top_k = 0 and top_p >= 1 return p unchanged."""
    p_row = np.asarray(p_row, dtype=np.float64)
    V = p_row.shape[0]
    n_k = top_k if 0 < top_k < V else V
    if n_k == V and top_p >= 1.0:
        return p_row
    ids = np.arange(V)
    order = np.lexsort((ids, -np.asarray(logits_row, dtype=np.float64)))
    if top_p >= 1.0:
        n_p = V
    else:
        cum = np.cumsum(p_row[order])
        n_p = int(np.argmax(cum >= top_p)) + 1 if (cum >= top_p).any() else V
    keep = order[:min(n_k, n_p)]
    out = np.zeros(V)
    out[keep] = p_row[keep]
    return out / out.sum()


def filtered_probs(logits, temperature, top_k=0, top_p=1.0):
    """Rows of softmax(l / T), each filtered by filtered_target."""
    lg = np.asarray(logits, dtype=np.float64) / float(temperature)
    p = softmax(lg, axis=-1)
    if top_k <= 0 and top_p >= 1.0:
        return p
    return np.stack([filtered_target(p[j], lg[j], top_k, top_p) for j in range(p.shape[0])])


def verify_request(logits, drafts, q_rows, seed, rid, L, mode, temperature=1.0, top_k=0, top_p=1.0):
    """Decide one request. logits [k+1][V]; drafts [k] ints; q_rows [k][V] or None.

    L is the request's cache length at verify time (the chain head sits at
    sequence index L). Returns dict(a, emitted, indep).
    """
    logits = np.asarray(logits, dtype=np.float64)
    k = len(drafts)
    assert logits.shape[0] == k + 1
    if mode == PREFILL:
        # eq:prefill_computation: the chain is a chunk of the prompt, every
        # row's KV is kept (a = k); y = argmax l_k is the model's next token after the chunk
        y = argmax_lowest(logits[k])
        return dict(a=k, emitted=list(drafts) + [y], indep=0, prefill=True)
    if mode == GREEDY:
        top = [argmax_lowest(logits[j]) for j in range(k + 1)]
        a = 0
        while a < k and drafts[a] == top[a]:
            a += 1
        indep = sum(1 for j in range(k) if drafts[j] == top[j])
        y = top[a]
        return dict(a=a, emitted=list(drafts[:a]) + [y], indep=indep)

    p = filtered_probs(logits, temperature, top_k, top_p)   # p[j] = p_{j+1} (R31 filtering)
    V = p.shape[1]
    a = k
    indep = 0
    for j in range(1, k + 1):
        d = int(drafts[j - 1])
        u = uniform_accept(seed, rid, L + j)
        qd = 1.0 if q_rows is None else float(q_rows[j - 1][d])
        r = np.inf if qd == 0.0 else p[j - 1][d] / qd
        acc = u < r
        indep += int(acc)
        if not acc and a == k:
            a = j - 1
    if a < k:
        pj = p[a]
        if q_rows is None:
            qj = np.zeros(V)
            qj[int(drafts[a])] = 1.0
        else:
            qj = np.asarray(q_rows[a], dtype=np.float64)
        R = np.maximum(0.0, pj - qj)
        if R.sum() == 0.0:
            R = pj
    else:
        R = p[k]
    E = -np.log(uniform_race(seed, rid, L + a + 1, V))
    score = np.where(R > 0, R / E, -np.inf)
    y = argmax_lowest(score)
    return dict(a=a, emitted=list(int(t) for t in drafts[:a]) + [y], indep=indep)


def race_scores(logits_row, q_row, d_reject, seed, rid, z, temperature, residual, top_k=0, top_p=1.0):
    """The race scores R(x)/E_x used for one selected row (for borderline analysis)."""
    p = filtered_probs(np.asarray(logits_row)[None], temperature, top_k, top_p)[0]
    V = p.shape[0]
    if residual:
        if q_row is None:
            q = np.zeros(V)
            q[int(d_reject)] = 1.0
        else:
            q = np.asarray(q_row, dtype=np.float64)
        R = np.maximum(0.0, p - q)
        if R.sum() == 0.0:
            R = p
    else:
        R = p
    E = -np.log(uniform_race(seed, rid, z, V))
    return np.where(R > 0, R / E, -np.inf)


def new_stats():
    return dict(steps=0, rows=0, drafted=0, accepted=0, emitted=0, accepted_independent=0,
                hist_accepted=[0] * (MAXK + 1), drafted_by_k=[0] * (MAXK + 1),
                accepted_by_k=[0] * (MAXK + 1))


def accumulate_stats(stats, depths, results):
    """a7: fold one verify call's per-request results into the lane counters."""
    if any(r.get("prefill") for r in results):      # prefill chunks are not speculation
        return stats
    stats["steps"] += 1
    for k, r in zip(depths, results):
        a = r["a"]
        stats["rows"] += k + 1
        stats["drafted"] += k
        stats["accepted"] += a
        stats["emitted"] += a + 1
        stats["accepted_independent"] += r["indep"]
        stats["hist_accepted"][a] += 1
        stats["drafted_by_k"][k] += k
        stats["accepted_by_k"][k] += a
    return stats
