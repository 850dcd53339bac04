"""The library's FlowGuard router (csrc/flowguard.cpp via include/sv.h) against the oracle
(oracle/flowguard.py, Alg. 2). Host code: runs without a GPU. Same double arithmetic in the same
order: decisions, flags and scores must match exactly."""
import random

import pytest

from oracle import flowguard as fg
from paper_2604_09562_b200 import flowguard as lib_fg
from paper_2604_09562_b200 import sv


def _both(ws, live, now, alpha=None):
    ocfg = fg.RouteConfig() if alpha is None else fg.RouteConfig(alpha=alpha)
    lcfg = lib_fg.RouteConfig.default() if alpha is None else lib_fg.RouteConfig.default(alpha=alpha)
    d = fg.select_worker(ws, live, now, ocfg)
    tup = [(w.timestamp_ms, w.cache_hit, w.mem_util, w.queue_depth, w.active_load) for w in ws]
    return d, lib_fg.select(tup, live, now, lcfg)


def test_matches_oracle_exactly():
    rng = random.Random(11)
    for _ in range(4000):
        now = 50_000
        n = rng.randint(1, 9)
        ws = [fg.WorkerMetrics(now - rng.choice([0, 10, 999, 1000, 1001, 3000]), rng.random(), rng.random(),
                               rng.choice([0, 3, 17, 42, 99, 140]) * rng.random(), rng.random()) for _ in range(n)]
        live = None if rng.random() < 0.3 else [rng.randint(0, 70) for _ in range(n)]
        d, (chosen, scores, flags, fb) = _both(ws, live, now)
        assert chosen == d.chosen and fb == d.used_fallback
        assert scores == list(d.scores)
        assert flags == [(1 if o else 0) | (2 if s else 0) for o, s in zip(d.overloaded, d.stale)]


def test_worked_values_through_the_library():
    chosen, scores, flags, fb = lib_fg.select([(0, 0.5, 0.4, 20, 0.3), (0, 0.0, 0.9, 10, 0.0)])
    assert chosen == 0 and not fb and flags == [0, lib_fg.SV_ROUTE_OVERLOADED] and abs(scores[0] - 0.64) < 1e-15
    chosen, _, _, fb = lib_fg.select([(0, 0, 0.9, 5, 0), (0, 0, 0.9, 2, 0)], live_queue=[5, 2])
    assert chosen == 1 and fb


def test_errors():
    with pytest.raises(sv.SvError):
        lib_fg.select([])
    with pytest.raises(sv.SvError):
        lib_fg.select([(0, 1.5, 0.0, 0, 0.0)])                       # cache hit outside [0, 1]
    with pytest.raises(sv.SvError):
        lib_fg.select([(0, 0.5, 0.0, 0, 0.0)], cfg=lib_fg.RouteConfig.default(alpha=(0.5, 0.5, 0.5, 0.0)))
