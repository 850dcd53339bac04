"""Pins for top-k / top-p filtered targets (oracle/verify.py filtered_target; NEXT-4, DESIGN.md
R31): hand-derived worked values, the top_k = 1 reduction to greedy verification, and the
Leviathan law with the filtered target (first emitted token ~ p', chi-square, p' built here by
a plain sort-and-accumulate loop)."""
import numpy as np
import pytest
from scipy import stats

from oracle import tree, verify

ALPHA = 0.01


def _fv(p, **kw):
    p = np.asarray(p, dtype=np.float64)
    return verify.filtered_target(p, np.log(p), **kw)


def test_worked_values():
    p = [0.5, 0.3, 0.15, 0.05]
    assert np.allclose(_fv(p, top_p=0.75), [0.625, 0.375, 0, 0], atol=1e-15)
    assert np.allclose(_fv(p, top_p=0.81), [0.5 / 0.95, 0.3 / 0.95, 0.15 / 0.95, 0], atol=1e-15)
    assert np.allclose(_fv(p, top_k=3), [0.5 / 0.95, 0.3 / 0.95, 0.15 / 0.95, 0], atol=1e-15)
    assert np.allclose(_fv(p, top_k=3, top_p=0.75), [0.625, 0.375, 0, 0], atol=1e-15)
    assert np.allclose(_fv(p, top_p=0.1), [1, 0, 0, 0])           # the top token alone crosses 0.1
    assert np.array_equal(_fv(p, top_k=4), np.asarray(p))        # k = V: no filtering
    assert np.array_equal(_fv(p, top_k=0, top_p=1.0), np.asarray(p))
    # ties go to the lowest token id
    assert np.allclose(_fv([0.25, 0.25, 0.25, 0.25], top_k=2), [0.5, 0.5, 0, 0])
    assert np.allclose(_fv([0.1, 0.3, 0.3, 0.3], top_k=2), [0, 0.5, 0.5, 0])
    assert np.allclose(_fv([0.1, 0.3, 0.3, 0.3], top_p=0.5), [0, 0.5, 0.5, 0])


@pytest.mark.parametrize("dense", [True, False])
def test_top_k_one_is_greedy(dense):
    rng = np.random.default_rng(3 + dense)
    V, k = 32, 5
    for trial in range(300):
        logits = rng.standard_normal((k + 1, V)) * 2
        top = logits.argmax(1)
        drafts = [int(top[j]) if rng.random() < 0.6 else int(rng.integers(V)) for j in range(k)]
        q = None
        if dense:
            q = rng.exponential(size=(k, V)) ** 2
            q /= q.sum(1, keepdims=True)
        g = verify.verify_request(logits, drafts, None, 0, trial, 9, verify.GREEDY)
        s = verify.verify_request(logits, drafts, q, 17, trial, 9, verify.SAMPLE, 0.7, top_k=1)
        assert (s["a"], s["emitted"]) == (g["a"], g["emitted"])
        par = [int(rng.integers(0, n)) for n in range(1, k + 1)]
        gt = tree.verify_tree(logits, drafts, par, None, 0, trial, 9, verify.GREEDY)
        st = tree.verify_tree(logits, drafts, par, q, 17, trial, 9, verify.SAMPLE, 0.7, top_k=1)
        assert (st["a"], st["emitted"], st["path"]) == (gt["a"], gt["emitted"], gt["path"])


def _filtered_by_loop(p, top_k, top_p):
    items = sorted(range(len(p)), key=lambda x: (-p[x], x))    # p order == logit order here
    keep, acc = [], 0.0
    for x in items:
        if top_k and len(keep) >= top_k:
            break
        if top_p < 1.0 and acc >= top_p:
            break
        keep.append(x)
        acc += p[x]
    out = np.zeros(len(p))
    out[keep] = [p[x] for x in keep]
    return out / out.sum()


@pytest.mark.parametrize("top_k,top_p", [(3, 1.0), (0, 0.6), (4, 0.8)])
def test_first_emitted_token_follows_the_filtered_target(top_k, top_p):
    rng = np.random.default_rng(top_k + int(10 * top_p))
    V, k, n = 10, 3, 12000
    p = rng.exponential(size=(k + 1, V)) ** 2
    p /= p.sum(1, keepdims=True)
    q = rng.exponential(size=(k, V)) ** 2
    q /= q.sum(1, keepdims=True)
    logits = np.log(p)
    want = _filtered_by_loop(p[0], top_k, top_p)
    assert np.allclose(verify.filtered_target(p[0], logits[0], top_k, top_p), want, atol=1e-14)
    counts = np.zeros(V)
    for rid in range(n):
        drafts = [int(rng.choice(V, p=q[j])) for j in range(k)]
        r = verify.verify_request(logits, drafts, q, 5, rid, 30, verify.SAMPLE, 1.0, top_k, top_p)
        counts[r["emitted"][0]] += 1
    assert counts[want == 0].sum() == 0
    e = want[want > 0] * n
    assert stats.chisquare(counts[want > 0], e * counts.sum() / e.sum()).pvalue > ALPHA
