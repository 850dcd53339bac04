"""Pins of oracle/flowguard.py (§3.3, Alg. 2) to SPEC.md's worked values
 and the routing properties of SPEC.md:171-176."""
import math
import random

import pytest

from oracle import flowguard as fg

CFG = fg.RouteConfig()


def W(c=0.0, m=0.0, q=0.0, l=0.0, ts=0):
    return fg.WorkerMetrics(timestamp_ms=ts, cache_hit=c, mem_util=m, queue_depth=q, active_load=l)


def test_score_worked_values():
    assert fg.score(W(c=1, m=0, q=0, l=0), CFG) == 1.0                      # SPEC.md:136 perfect worker
    assert fg.score(W(c=0, m=1, q=100, l=1), CFG) == 0.0                    # SPEC.md:137 no headroom
    # 0.4*0.5 + 0.1*0.6 + 0.3*0.8 + 0.2*0.7 = 0.64
    assert math.isclose(fg.score(W(c=0.5, m=0.4, q=20, l=0.3), CFG), 0.64, rel_tol=1e-15)
    assert fg.score(W(q=1e6), CFG) == fg.score(W(q=100), CFG)               # Q_w clamped at 1


def test_overload_worked_values():
    assert fg.overload_score(W(), CFG) == 0.0
    assert math.isclose(fg.overload_score(W(m=0.5, q=20), CFG), 0.9, rel_tol=1e-15)
    assert fg.overload_score(W(m=0.85), CFG) == 0.85
    assert fg.is_overloaded(W(m=0.5, q=20), CFG)                            # 0.9 > 0.85
    assert not fg.is_overloaded(W(m=0.85), CFG)                             # strict >
    assert not fg.is_overloaded(W(), CFG)


def test_staleness_boundary():
    assert not fg.is_stale(W(ts=500), 500, CFG)
    assert not fg.is_stale(W(ts=0), 1000, CFG)                              # exactly the window: fresh
    assert fg.is_stale(W(ts=0), 1001, CFG)


def test_select_worked_cases():
    healthy, over = W(c=0.5, m=0.4, q=20, l=0.3), W(m=0.9, q=10)
    d = fg.select_worker([healthy, over], None, 0, CFG)
    assert d.chosen == 0 and not d.used_fallback and d.overloaded == (False, True) and d.scores[1] is None
    d = fg.select_worker([W(m=0.9, q=5), W(m=0.9, q=2)], [5, 2], 0, CFG)    # SPEC.md:166 all overloaded
    assert d.chosen == 1 and d.used_fallback
    a, b = W(c=0.5, m=0.4, q=20, l=0.3), W(c=0.6, m=0.4, q=20, l=0.2)     # 0.64; 0.24+0.06+0.24+0.16 = 0.70
    d = fg.select_worker([a, b], None, 0, CFG)
    assert d.chosen == 1 and math.isclose(d.scores[1], 0.70, rel_tol=1e-12)
    # live queue depth replaces the snapshot's (Alg. 2 "load_i.qd <- Q_{P_i}.size()")
    d = fg.select_worker([a, b], [0, 80], 0, CFG)
    assert d.overloaded == (False, True) and d.chosen == 0
    # stale workers are excluded from scoring but stay in the fallback
    d = fg.select_worker([W(ts=0, c=1), W(ts=5000, m=0.9)], [7, 3], 5000, CFG)
    assert d.stale == (True, False) and d.used_fallback and d.chosen == 1


def _rand_worker(rng, now):
    return W(c=rng.random(), m=rng.random(), q=rng.choice([0, 1, 5, 20, 40, 99, 150]) * rng.random(),
             l=rng.random(), ts=now - rng.choice([0, 100, 999, 1000, 1001, 4000]))


def test_properties_random():
    rng = random.Random(5)
    for _ in range(3000):
        now = 10_000
        n = rng.randint(1, 8)
        ws = [_rand_worker(rng, now) for _ in range(n)]
        live = [rng.randint(0, 60) for _ in range(n)]
        d = fg.select_worker(ws, live, now, CFG)
        assert 0 <= d.chosen < n
        if not d.used_fallback:
            assert not d.overloaded[d.chosen] and not d.stale[d.chosen]
            best = max(s for s in d.scores if s is not None)
            assert d.scores[d.chosen] == best
            assert all(d.scores[i] is None or d.scores[i] < best for i in range(d.chosen))   # lowest index
        else:
            assert all(d.overloaded[i] or d.stale[i] for i in range(n))
            assert live[d.chosen] == min(live) and live.index(min(live)) == d.chosen
        if n == 1:
            assert d.chosen == 0
        assert fg.select_worker(ws, live, now, CFG) == d                    # determinism
        # scale-free: weights times k, renormalised, select the same worker
        k = rng.choice([0.5, 3.0, 7.0])
        al = [a * k for a in CFG.alpha]
        s = sum(al)
        cfg2 = fg.RouteConfig(alpha=tuple(a / s for a in al))
        assert fg.select_worker(ws, live, now, cfg2).chosen == d.chosen


def test_score_monotonicity():
    rng = random.Random(8)
    for _ in range(2000):
        base = dict(c=rng.random(), m=rng.random(), q=100 * rng.random(), l=rng.random())
        s0 = fg.score(W(**base), CFG)
        up = dict(base, c=min(1.0, base["c"] + 0.1))
        assert fg.score(W(**up), CFG) >= s0
        for key, step in (("m", 0.1), ("q", 10.0), ("l", 0.1)):
            worse = dict(base)
            worse[key] = base[key] + step if key == "q" else min(1.0, base[key] + step)
            assert fg.score(W(**worse), CFG) <= s0


def test_empty_worker_list_is_an_error():
    with pytest.raises(ValueError):
        fg.select_worker([], None, 0, CFG)
