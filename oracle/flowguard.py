"""FlowGuard routing (NEXT-2): PAPER.md §3.3 "FlowGuard: Metric-Aware Routing" — the score
eq:flowguard_score, overload detection eq:overload_detection /
eq:overload_score, the fallback eq:fallback_selection and
Alg. 2 "FlowGuard Worker Selection". TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

Written out term by term in the paper's notation, Python floats (IEEE double):

    S_w     = a1 C_w + a2 (1 - M_w) + a3 (1 - Q_w) + a4 (1 - L_w),    Q_w = min(Q_raw / Q_max, 1)
    omega_w = M_w + 2 Q_raw / Q_max                                     (eq:overload_score, M as a fraction)
    Overload(w) = omega_w > tau                                         (strict)
    Alg. 2: workers that are stale or overloaded are excluded; argmax S over the rest (lowest
            index on ties); if none remain, argmin of the live queue depths (lowest index on ties).

Readings (R25-R28, from SPEC.md:110-190 where the paper is silent or at odds):
* Eq. overload_score divides M_w by 100 while Table 2 has M_w in [0, 1]: M enters as a fraction.
* Q_w in the score is Q_raw / Q_max clamped to 1; Alg. 2's live queue depth replaces Q_raw.
* stale  <=>  now - timestamp > staleness window (1000 ms = 2 x the 500 ms collection cadence).
* ties: lowest worker index, for the argmax and for the fallback argmin.

Pinned by tests/test_oracle_flowguard.py: SPEC.md's worked values, and the
properties of SPEC.md:171-176 (monotonicity, scale-free selection, exclusions, single worker,
determinism).
"""
from dataclasses import dataclass
from typing import List, Optional, Sequence


@dataclass(frozen=True)
class RouteConfig:
    alpha: tuple = (0.4, 0.1, 0.3, 0.2)       # cache, memory headroom, queue headroom, load headroom
    tau: float = 0.85
    q_max: float = 100.0
    staleness_ms: int = 1000


@dataclass(frozen=True)
class WorkerMetrics:
    timestamp_ms: int
    cache_hit: float        # C_w in [0, 1]
    mem_util: float         # M_w in [0, 1]
    queue_depth: float      # Q_raw >= 0 (count)
    active_load: float      # L_w in [0, 1]


@dataclass(frozen=True)
class Decision:
    chosen: int
    scores: tuple           # None for excluded workers
    overloaded: tuple
    stale: tuple
    used_fallback: bool


def score(m: WorkerMetrics, cfg: RouteConfig, q_raw: Optional[float] = None) -> float:
    q = m.queue_depth if q_raw is None else q_raw
    qw = min(q / cfg.q_max, 1.0)
    a1, a2, a3, a4 = cfg.alpha
    return a1 * m.cache_hit + a2 * (1.0 - m.mem_util) + a3 * (1.0 - qw) + a4 * (1.0 - m.active_load)


def overload_score(m: WorkerMetrics, cfg: RouteConfig, q_raw: Optional[float] = None) -> float:
    q = m.queue_depth if q_raw is None else q_raw
    return (100.0 * m.mem_util) / 100.0 + 2.0 * (q / cfg.q_max)


def is_overloaded(m: WorkerMetrics, cfg: RouteConfig, q_raw: Optional[float] = None) -> bool:
    return overload_score(m, cfg, q_raw) > cfg.tau


def is_stale(m: WorkerMetrics, now_ms: int, cfg: RouteConfig) -> bool:
    return now_ms - m.timestamp_ms > cfg.staleness_ms


def select_worker(metrics: Sequence[WorkerMetrics], live_queue: Optional[Sequence[float]], now_ms: int,
                  cfg: RouteConfig) -> Decision:
    """Alg. 2. live_queue[i] (the fresh Q_{P_i}.size()) replaces the snapshot's queue depth."""
    if len(metrics) == 0:
        raise ValueError("no workers")
    n = len(metrics)
    qd = [float(live_queue[i]) if live_queue is not None else metrics[i].queue_depth for i in range(n)]
    scores: List[Optional[float]] = [None] * n
    over, stale = [False] * n, [False] * n
    avail = []
    for i in range(n):
        stale[i] = is_stale(metrics[i], now_ms, cfg)
        over[i] = is_overloaded(metrics[i], cfg, qd[i])
        if not stale[i] and not over[i]:
            scores[i] = score(metrics[i], cfg, qd[i])
            avail.append(i)
    if not avail:
        best = 0
        for i in range(1, n):                    # argmin queue depth, lowest index on ties
            if qd[i] < qd[best]:
                best = i
        return Decision(best, tuple(scores), tuple(over), tuple(stale), True)
    best = avail[0]
    for i in avail[1:]:                          # argmax score, lowest index on ties
        if scores[i] > scores[best]:
            best = i
    return Decision(best, tuple(scores), tuple(over), tuple(stale), False)
