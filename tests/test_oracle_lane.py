"""Pins for oracle/lane.py: greedy = argmax chain (P4), multi-step unbiasedness of the
RNG counter layout (P8), commit/rollback and incremental consistency (P5)."""
import copy
import itertools

import numpy as np
import pytest
from scipy import stats

import synth
from oracle import verify
from oracle.lane import OracleLane


def _np_weights(w):
    return {k: synth.as_f64(v) for k, v in w.items()}


def _lane(cfg, seed=0, ctx=24, slots=(0, 1, 2)):
    w = _np_weights(synth.model_weights(cfg, seed=seed, norm_one=False))
    lane = OracleLane(cfg, w)
    for i, s in enumerate(slots):
        k, v = synth.context_kv(cfg, ctx + 3 * i, seed=100 + i)
        lane.append_kv(s, 1000 + i, synth.as_f64(k), synth.as_f64(v), pending_token=7 * i + 1)
    return lane


def _greedy_chain(lane, slot, n):
    """n plain decode steps (k = 0 verify + commit) on a clone of the lane."""
    c = copy.deepcopy(lane)
    toks, logits = [], []
    for _ in range(n):
        acc, em, lg = c.verify([slot], [0], [], None, 0, verify.GREEDY)
        c.commit()
        toks.append(em[0][0])
        logits.append(lg[0][0])
    return toks, np.array(logits)


@pytest.mark.parametrize("cfgname", ["toy", "toy_mlp"])
def test_greedy_equals_argmax_chain(cfgname):
    cfg = synth.CONFIGS[cfgname]
    lane = _lane(cfg)
    k = 4
    chain, seq_logits = _greedy_chain(lane, 1, k + 1)
    c = copy.deepcopy(lane)
    acc, em, lg = c.verify([1], [k], chain[:k], None, 0, verify.GREEDY)
    assert acc == [k] and em[0] == chain
    # the k+1 verify rows reproduce the k+1 sequential decode steps' logits
    assert np.allclose(lg[0], seq_logits, rtol=0, atol=1e-9 * np.abs(seq_logits).max())
    for m in range(1, k + 1):          # corrupt draft m -> a = m - 1, y = the true token
        bad = list(chain[:k])
        bad[m - 1] = (bad[m - 1] + 1) % cfg.vocab
        c = copy.deepcopy(lane)
        acc, em, _ = c.verify([1], [k], bad, None, 0, verify.GREEDY)
        assert acc == [m - 1] and em[0] == chain[:m]


def test_commit_rollback_and_incremental_consistency():
    cfg = synth.TOY_MLP
    lane = _lane(cfg)
    L0 = lane.length(2)
    drafts = [int(t) for t in synth.random_tokens(3, cfg.vocab, seed=5)]
    acc, em, _ = lane.verify([2], [3], drafts, None, 0, verify.GREEDY)
    lane.commit()
    assert lane.length(2) == L0 + acc[0] + 1          # rejected rows rolled back
    assert lane.slots[2]["pending"] == em[0][-1]
    # a fresh lane with the full committed sequence appended gives identical verify output
    fresh = OracleLane(cfg, lane.w)
    st = lane.slots[2]
    fresh.append_kv(2, st["rid"], np.stack(st["K"]), np.stack(st["V"]), st["pending"])
    d2 = [int(t) for t in synth.random_tokens(4, cfg.vocab, seed=6)]
    a1, e1, l1 = lane.verify([2], [4], d2, None, 99, verify.SAMPLE)
    a2, e2, l2 = fresh.verify([2], [4], d2, None, 99, verify.SAMPLE)
    assert a1 == a2 and e1 == e2 and np.array_equal(l1[0], l2[0])


def test_n_keep_truncation():
    cfg = synth.TOY
    lane = _lane(cfg)
    chain, _ = _greedy_chain(lane, 0, 4)
    L0 = lane.length(0)
    acc, em, _ = lane.verify([0], [3], chain[:3], None, 0, verify.GREEDY)
    assert acc == [3]
    lane.commit(n_keep=[2])
    assert lane.length(0) == L0 + 2 and lane.slots[0]["pending"] == chain[1]


def test_batch_order_and_lane_invariance():
    """Outputs depend on (request_id, position), not on slot, batch order or lane."""
    cfg = synth.TOY
    lane = _lane(cfg)
    d = [int(t) for t in synth.random_tokens(9, cfg.vocab, seed=8)]
    a1, e1, _ = copy.deepcopy(lane).verify([0, 1, 2], [2, 3, 4], d, None, 5, verify.SAMPLE)
    a2, e2, _ = copy.deepcopy(lane).verify([2, 0, 1], [4, 2, 3], d[5:] + d[:5], None, 5, verify.SAMPLE)
    assert a1 == [a2[1], a2[2], a2[0]] and e1 == [e2[1], e2[2], e2[0]]
    solo = copy.deepcopy(lane)
    for s in (0, 2):
        solo.release(s)
    a3, e3, _ = solo.verify([1], [3], d[2:5], None, 5, verify.SAMPLE)
    assert a3[0] == a1[1] and e3[0] == e1[1]


def test_multistep_sequence_law_unbiased():
    """P8 / S7: re-drawing the same (rid, index) counters across steps leaves the
    generated sequence law equal to the target's (Markov target, Markov drafter)."""
    rng = np.random.default_rng(12)
    V, n_tok, runs = 3, 4, 6000
    P = np.array([[0.6, 0.3, 0.1], [0.2, 0.2, 0.6], [0.3, 0.5, 0.2]])
    Q = np.array([[0.3, 0.3, 0.4], [0.5, 0.25, 0.25], [0.1, 0.8, 0.1]])
    x0 = 1
    counts = {}
    for run in range(runs):
        pending, L, gen = x0, 20, []
        while len(gen) < n_tok:
            k = int(rng.integers(0, 5))
            drafts, prev = [], pending
            for _ in range(k):
                prev = int(rng.choice(V, p=Q[prev]))
                drafts.append(prev)
            chain = [pending] + drafts
            logits = np.log(P[chain])
            qrows = Q[chain[:k]] if k else np.zeros((0, V))
            r = verify.verify_request(logits, drafts, qrows, 31337, run, L, verify.SAMPLE)
            gen += r["emitted"]
            L += r["a"] + 1
            pending = r["emitted"][-1]
        key = tuple(gen[:n_tok])
        counts[key] = counts.get(key, 0) + 1
    cells = list(itertools.product(range(V), repeat=n_tok))
    law = []
    for c in cells:
        pr, prev = 1.0, x0
        for t in c:
            pr *= P[prev, t]
            prev = t
        law.append(pr)
    obs = np.array([counts.get(c, 0) for c in cells], dtype=float)
    exp = np.array(law) * runs
    assert stats.chisquare(obs, exp).pvalue > 0.01
