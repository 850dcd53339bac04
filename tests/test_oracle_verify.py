"""Pins for oracle/verify.py: distribution laws, brute force, closed forms, worked example.

SURVEY.md §8(c) pins P1, P2, P3, P5, P8, P10. Every expected value below comes
from the mathematics (Leviathan's theorem, enumeration, SPEC.md:325's closed
form) or the hand-derived example in tests/golden/verify_worked.json; none
comes from the oracle or the CUDA path.
"""
import itertools
import json
import os

import numpy as np
import pytest
from scipy import stats

from oracle import verify
from oracle.philox import uniform_accept

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "verify_worked.json")))
ALPHA = 0.01


def _chisq(observed, expected_p, n):
    """chi-square p-value, cells with expected count < 5 merged into one."""
    obs = np.asarray(observed, dtype=np.float64)
    exp = np.asarray(expected_p, dtype=np.float64) * n
    big = exp >= 5
    o = list(obs[big]) + ([obs[~big].sum()] if (~big).any() else [])
    e = list(exp[big]) + ([exp[~big].sum()] if (~big).any() else [])
    o, e = np.array(o), np.array(e)
    e *= o.sum() / e.sum()
    return stats.chisquare(o, e).pvalue


def _rand_simplex(rng, V, sharp=2.0, zeros=0):
    w = rng.exponential(size=V) ** sharp
    if zeros:
        w[rng.choice(V, zeros, replace=False)] = 0.0
    return w / w.sum()


# ------------------------------------------------------------------ P10 worked example

def test_worked_example_ratio_and_decisions():
    ex = GOLD["sampled"]
    p, q, d = np.array(ex["p"]), np.array(ex["q"]), ex["draft"]
    logits = np.log(np.stack([p, p]))
    # find request ids whose accept uniform lands near the example's u values
    seen = {"acc": False, "rej": False}
    for rid in range(5000):
        u = uniform_accept(11, rid, 1)          # L = 0 -> d_1 decides index 1
        r = verify.verify_request(logits, [d], [q], 11, rid, 0, verify.SAMPLE)
        assert (r["a"] == 1) == (u < ex["ratio"])
        if abs(u - ex["u_accept_example"]) < 0.01:
            assert r["a"] == 1
            seen["acc"] = True
        if abs(u - ex["u_reject_example"]) < 0.01:
            assert r["a"] == 0
            seen["rej"] = True
    assert seen["acc"] and seen["rej"]


def test_worked_example_residual_law():
    ex = GOLD["sampled"]
    p, q = np.array(ex["p"]), np.array(ex["q"])
    logits = np.log(np.stack([p, p]))
    counts = np.zeros(4)
    for rid in range(6000):
        r = verify.verify_request(logits, [ex["draft"]], [q], 3, rid, 0, verify.SAMPLE)
        if r["a"] == 0:
            counts[r["emitted"][0]] += 1
    assert counts[2] == 0 and counts[3] == 0
    assert _chisq(counts[:2], ex["residual"][:2], counts.sum()) > ALPHA


def test_worked_example_acceptance_probability():
    ex = GOLD["sampled"]
    p, q = np.array(ex["p"]), np.array(ex["q"])
    rng = np.random.default_rng(0)
    logits = np.log(np.stack([p, p]))
    n, acc = 8000, 0
    for rid in range(n):
        d = int(rng.choice(4, p=q))
        acc += verify.verify_request(logits, [d], [q], 5, rid, 0, verify.SAMPLE)["a"]
    assert abs(acc / n - ex["acceptance_probability_draft_from_q"]) < 4 * np.sqrt(0.21 / n)


def test_worked_example_greedy_tie():
    g = GOLD["greedy"]
    logits = np.array([g["logits"]])
    assert verify.verify_request(logits, [], None, 0, 0, 0, verify.GREEDY)["emitted"] == [g["argmax"]]
    two = np.array([g["logits"], g["logits"]])
    assert verify.verify_request(two, [2], None, 0, 0, 0, verify.GREEDY)["a"] == 0
    assert verify.verify_request(two, [1], None, 0, 0, 0, verify.GREEDY) == \
        dict(a=1, emitted=[1, 1], indep=1)


# ------------------------------------------------------------------ P1 Leviathan: first token ~ p_1

@pytest.mark.parametrize("dense", [True, False])
def test_first_emitted_token_follows_target(dense):
    rng = np.random.default_rng(1 if dense else 2)
    V, k, n = 12, 3, 12000
    p = np.stack([_rand_simplex(rng, V, zeros=2) for _ in range(k + 1)])
    q = np.stack([_rand_simplex(rng, V, zeros=3) for _ in range(k)])
    logits = np.log(np.where(p > 0, p, 1e-300))
    counts = np.zeros(V)
    for rid in range(n):
        drafts = [int(rng.choice(V, p=q[j])) for j in range(k)]
        r = verify.verify_request(logits, drafts, q if dense else None, 77, rid, 40, verify.SAMPLE)
        counts[r["emitted"][0]] += 1
    p1 = np.exp(logits[0] - logits[0].max())
    p1 /= p1.sum()
    assert _chisq(counts, p1, n) > ALPHA


@pytest.mark.parametrize("temperature", [0.5, 1.7])
@pytest.mark.parametrize("dense", [True, False])
def test_first_emitted_token_follows_tempered_target(temperature, dense):
    """P1 at T != 1: the first emitted token ~ softmax(l / T). The expected law is written as
    p^(1/T) / sum p^(1/T) with p = softmax(l) (a different route from the oracle's scaled-logit
    softmax), so a temperature applied twice, inverted or dropped fails here."""
    rng = np.random.default_rng(int(10 * temperature) + (5 if dense else 0))
    V, k, n = 10, 2, 12000
    base = np.stack([_rand_simplex(rng, V, sharp=1.0) for _ in range(k + 1)])
    logits = np.log(base) + rng.normal(size=(1, 1))         # a row offset the softmax must ignore
    q = np.stack([_rand_simplex(rng, V, zeros=2) for _ in range(k)])
    counts = np.zeros(V)
    for rid in range(n):
        drafts = [int(rng.choice(V, p=q[j])) for j in range(k)]
        r = verify.verify_request(logits, drafts, q if dense else None, 91, rid, 12, verify.SAMPLE, temperature)
        counts[r["emitted"][0]] += 1
    pT = base[0] ** (1.0 / temperature)
    pT /= pT.sum()
    assert _chisq(counts, pT, n) > ALPHA
    # and the law at T is not the T = 1 law (the test has power to see a dropped temperature)
    p1 = base[0] / base[0].sum()
    assert _chisq(counts, p1, n) < 1e-6


def test_tempered_acceptance_probability_closed_form():
    """With one-hot drafts d ~ q the acceptance probability at T is sum_x q(x) min(1, p_T(x)),
    p_T = p^(1/T) normalised (Leviathan's beta for q = the drafter's law, one-hot verification
    compares p_T(d) against 1)."""
    rng = np.random.default_rng(3)
    V, n, T = 6, 20000, 0.6
    base = _rand_simplex(rng, V, sharp=1.0)
    q = _rand_simplex(rng, V)
    logits = np.log(np.stack([base, base]))
    acc = 0
    for rid in range(n):
        d = int(rng.choice(V, p=q))
        acc += verify.verify_request(logits, [d], None, 17, rid, 3, verify.SAMPLE, T)["a"]
    pT = base ** (1.0 / T)
    pT /= pT.sum()
    beta = float(np.sum(q * np.minimum(1.0, pT)))
    assert abs(acc / n - beta) < 4 * np.sqrt(beta * (1 - beta) / n)


# ------------------------------------------------------------------ P2 brute force

def _exact_law(p, q):
    """Enumerate drafts under q; acceptance min(1, p/q); residual R/sum R; bonus from p_{k+1}."""
    k, V = q.shape
    law = {}

    def resid(j):
        R = np.maximum(0.0, p[j] - q[j])
        return R / R.sum() if R.sum() > 0 else p[j]

    for drafts in itertools.product(range(V), repeat=k):
        w = np.prod([q[j][drafts[j]] for j in range(k)])
        if w == 0:
            continue
        prefix = w
        for j in range(k):
            d = drafts[j]
            acc = min(1.0, p[j][d] / q[j][d])
            rej = prefix * (1 - acc)
            if rej > 0:
                for y in range(V):
                    key = (j, tuple(drafts[:j]) + (y,))
                    law[key] = law.get(key, 0.0) + rej * resid(j)[y]
            prefix *= acc
        for y in range(V):
            key = (k, tuple(drafts) + (y,))
            law[key] = law.get(key, 0.0) + prefix * p[k][y]
    return law


def test_brute_force_joint_law():
    rng = np.random.default_rng(3)
    V, k = 4, 2
    p = np.stack([_rand_simplex(rng, V) for _ in range(k + 1)])
    q = np.stack([_rand_simplex(rng, V, zeros=1) for _ in range(k)])
    law = _exact_law(p, q)
    assert abs(sum(law.values()) - 1) < 1e-12
    # (i) first emitted token has law p_1; P(a >= 1) = sum min(p_1, q_1)
    first = np.zeros(V)
    pa1 = 0.0
    for (a, em), pr in law.items():
        first[em[0]] += pr
        if a >= 1:
            pa1 += pr
    assert np.allclose(first, p[0], atol=1e-12)
    assert abs(pa1 - np.minimum(p[0], q[0]).sum()) < 1e-12
    # (ii) the oracle with its RNG reproduces the enumerated law
    keys = sorted(law)
    idx = {kk: i for i, kk in enumerate(keys)}
    counts = np.zeros(len(keys))
    logits = np.log(p)
    n = 15000
    for rid in range(n):
        drafts = [int(rng.choice(V, p=q[j])) for j in range(k)]
        r = verify.verify_request(logits, drafts, q, 2024, rid, 7, verify.SAMPLE)
        counts[idx[(r["a"], tuple(r["emitted"]))]] += 1
    assert _chisq(counts, [law[kk] for kk in keys], n) > ALPHA


# ------------------------------------------------------------------ P3 accepted-length law

def _iid_pair(rng, V, alpha):
    """p, q on V symbols with sum min(p, q) = alpha exactly (by construction)."""
    base = _rand_simplex(rng, V // 2)
    p = np.concatenate([alpha * base, (1 - alpha) * _rand_simplex(rng, V - V // 2)])
    q = np.concatenate([alpha * base, np.zeros(V - V // 2)])
    q[: V // 2] += (1 - alpha) * _rand_simplex(rng, V // 2)
    # min(p, q) = alpha * base on the first half (q >= p there), 0 on the second
    assert abs(np.minimum(p, q).sum() - alpha) < 1e-12
    return p, q


@pytest.mark.parametrize("alpha", [0.3, 0.7])
def test_accepted_length_truncated_geometric(alpha):
    rng = np.random.default_rng(int(alpha * 10))
    V, k, n = 8, 4, 10000
    p, q = _iid_pair(rng, V, alpha)
    logits = np.log(np.where(p > 0, p, 1e-300))[None].repeat(k + 1, axis=0)
    qr = q[None].repeat(k, axis=0)
    hist = np.zeros(k + 1)
    for rid in range(n):
        drafts = [int(rng.choice(V, p=q)) for _ in range(k)]
        hist[verify.verify_request(logits, drafts, qr, 9, rid, 100, verify.SAMPLE)["a"]] += 1
    law = [alpha ** m * (1 - alpha) for m in range(k)] + [alpha ** k]
    assert _chisq(hist, law, n) > ALPHA
    mean_tokens = (hist * (np.arange(k + 1) + 1)).sum() / n
    closed = (1 - alpha ** (k + 1)) / (1 - alpha)
    assert abs(mean_tokens - closed) / closed < 0.02


def test_emission_degenerate_cases():
    """alpha = 0 -> 1 token/step; alpha = 1 -> k + 1."""
    V, k = 6, 5
    p = np.array([0.5, 0.5, 0, 0, 0, 0])
    q0 = np.array([0, 0, 0.5, 0.5, 0, 0])
    logits = np.log(np.where(p > 0, p, 1e-300))[None].repeat(k + 1, axis=0)
    for rid in range(50):
        r0 = verify.verify_request(logits, [2, 3, 2, 3, 2], q0[None].repeat(k, 0), 1, rid, 0, verify.SAMPLE)
        assert r0["a"] == 0 and len(r0["emitted"]) == 1 and r0["emitted"][0] in (0, 1)
        r1 = verify.verify_request(logits, [0, 1, 1, 0, 0], p[None].repeat(k, 0), 1, rid, 0, verify.SAMPLE)
        assert r1["a"] == k and len(r1["emitted"]) == k + 1


def test_spec_closed_form_golden():
    g = GOLD["speculative_emission"]
    a, k = g["alpha"], g["k"]
    assert abs((1 - a ** (k + 1)) / (1 - a) - g["expected_tokens_per_step"]) < 1e-4


# ------------------------------------------------------------------ P5 bounds, S4/S5 edge readings

def test_bounds_and_counters():
    rng = np.random.default_rng(4)
    V = 10
    st = verify.new_stats()
    for step in range(30):
        depths = [int(x) for x in rng.integers(0, 6, size=5)]
        res = []
        for i, k in enumerate(depths):
            logits = rng.standard_normal((k + 1, V)) * 3
            drafts = [int(x) for x in rng.integers(0, V, size=k)]
            mode = verify.SAMPLE if i % 2 else verify.GREEDY
            r = verify.verify_request(logits, drafts, None, step, i, 50, mode)
            assert 0 <= r["a"] <= k and len(r["emitted"]) == r["a"] + 1
            assert r["emitted"][: r["a"]] == drafts[: r["a"]]
            assert r["a"] <= r["indep"] <= k
            res.append(r)
        verify.accumulate_stats(st, depths, res)
    assert st["steps"] == 30
    assert st["emitted"] == st["accepted"] + sum(st["hist_accepted"])
    assert st["drafted"] == sum(st["drafted_by_k"]) and st["accepted"] == sum(st["accepted_by_k"])


def test_zero_q_accepts_and_zero_p_rejects():
    V = 4
    p = np.array([0.0, 0.5, 0.5, 0.0])
    logits = np.log(np.where(p > 0, p, 1e-300))
    logits[0] = logits[3] = -np.inf
    L2 = np.stack([logits, logits])
    qz = np.array([[0.0, 0.0, 0.5, 0.5]])
    for rid in range(40):
        # q(d) = 0 -> ratio +inf -> accept (S4)
        assert verify.verify_request(L2, [1], qz, 0, rid, 0, verify.SAMPLE)["a"] == 1
        # p(d) = 0 -> always reject; the residual never emits a p = 0 token
        r = verify.verify_request(L2, [3], qz, 0, rid, 0, verify.SAMPLE)
        assert r["a"] == 0 and r["emitted"][0] in (1, 2)


def test_zero_residual_falls_back_to_target():
    """S5: if max(0, p - q) sums to 0 the resample is from p itself."""
    p = np.array([0.25, 0.25, 0.25, 0.25])
    q = np.array([[0.25, 0.25, 0.25, 0.25]])
    logits = np.log(np.stack([p, p]))
    s = verify.race_scores(logits[0], q[0], 0, 1, 2, 3, 1.0, residual=True)
    assert np.all(np.isfinite(s))


def test_prefill_mode_keeps_the_chunk_and_predicts_the_next_token():
    """NEXT-3 reading R29: a = k, emitted = the chunk's tokens + argmax of the last row; equals
    GREEDY when the chunk happens to be the greedy argmax chain; no lane counters."""
    rng = np.random.default_rng(3)
    V, k = 40, 6
    lg = rng.normal(size=(k + 1, V))
    drafts = [int(x) for x in rng.integers(0, V, size=k)]
    r = verify.verify_request(lg, drafts, None, 1, 2, 10, verify.PREFILL)
    assert r["a"] == k and r["emitted"] == drafts + [int(np.argmax(lg[k]))]
    chain = [int(np.argmax(lg[j])) for j in range(k)]
    assert verify.verify_request(lg, chain, None, 1, 2, 10, verify.PREFILL) == \
        dict(verify.verify_request(lg, chain, None, 1, 2, 10, verify.GREEDY), indep=0, prefill=True)
    st = verify.new_stats()
    verify.accumulate_stats(st, [k], [r])
    assert st["steps"] == 0 and st["emitted"] == 0
