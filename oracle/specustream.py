"""SpecuStream depth controller (NEXT-1): PAPER.md §3.5, Alg. 4 "SpecuStream Adaptation"
 with the equations eq:acceptance_gradient ... eq_exponential_smoothing
(PAPER.md:303-366). TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Written out in Alg. 4's step order, in Python floats (IEEE double), one scalar at a time:

    delta <- a - mean(f);  f[idx] <- delta;  idx <- (idx + 1) mod h       (eq:acceptance_gradient)
    mag   <- mean(|f|)                                                    (eq:flow_magnitude)
    scale <- max(1, tau_target / max(t, 1))                               (eq:throughput_scaling)
    adj   <- 1 - min(l, 0.9)                                              (eq:load_adaptation)
    d     <- d_base + (a * mag * gamma) * adj * scale                     (eq:optimal_depth)
    d*    <- clip(d, d_min, d_max)                                        (eq:depth_clipping)
    b     <- max(1, floor(16 * 5 / d*))                                   (eq:microbatch_size)
    t_proj <- t * (1 + a * 0.5)                                           (Alg. 4 line 10)
    tau_recent <- 0.9 * tau_recent + 0.1 * t_proj                         (eq_exponential_smoothing)

Readings (R21-R24, from SPEC.md:221-256 where the paper is silent):
* d* is an integer token count: round-half-up of the clipped value; b uses that integer d*.
* t_proj follows Alg. 4 (measured t); eq:projected_throughput's tau_recent source is the
  `projection_source="smoothed"` toggle.
* mean(f) in delta uses the buffer before the write; mag the buffer after it; both divide by h.
* Initial state: f = 0, idx = 0, tau_recent = tau_target (paper silent).

Pinned by tests/test_oracle_specustream.py: SPEC.md's worked traces, the
invariants of SPEC.md:241-248 (bounds, micro-batch coupling, load monotonicity, scale floor,
flow-buffer replay, smoothing contraction, purity) and closed forms of the cold-start step.
"""
import math
from dataclasses import dataclass, field, replace
from typing import List


@dataclass(frozen=True)
class SpecConfig:
    d_base: float = 5.0
    gamma: float = 5.0
    d_min: float = 2.0
    d_max: float = 20.0
    h: int = 10
    tau_target: float = 400.0
    micro_batch_numerator: float = 80.0      # 16 * 5 (eq:microbatch_size)
    projection_source: str = "measured"      # Alg. 4: t; "smoothed": eq:projected_throughput's tau_recent


@dataclass(frozen=True)
class FlowState:
    f: tuple
    idx: int
    tau_recent: float


@dataclass(frozen=True)
class SpeculationPlan:
    depth: int
    micro_batch: int
    projected: float
    raw_depth: float
    delta: float
    mag: float
    scale: float
    adj: float


def reset(cfg: SpecConfig) -> FlowState:
    return FlowState(f=tuple(0.0 for _ in range(cfg.h)), idx=0, tau_recent=float(cfg.tau_target))


def _mean(xs):
    s = 0.0
    for x in xs:                             # j = 0 .. h-1, in order
        s += x
    return s / len(xs)


def round_half_up(x):
    return int(math.floor(x + 0.5))


def adapt(state: FlowState, a: float, l: float, t: float, cfg: SpecConfig):
    """One Alg. 4 step. Returns (plan, new_state); the input state is not modified."""
    f: List[float] = list(state.f)
    delta = a - _mean(f)                                        # uses f before the write
    f[state.idx] = delta
    idx = (state.idx + 1) % cfg.h
    mag = _mean([abs(x) for x in f])                            # after the write
    scale = max(1.0, cfg.tau_target / max(t, 1.0))
    adj = 1.0 - min(l, 0.9)
    raw = cfg.d_base + (a * mag * cfg.gamma) * adj * scale
    clipped = min(max(raw, cfg.d_min), cfg.d_max)
    depth = round_half_up(clipped)
    micro = max(1, int(math.floor(cfg.micro_batch_numerator / depth)))
    src = t if cfg.projection_source == "measured" else state.tau_recent
    t_proj = src * (1.0 + a * 0.5)
    tau_new = 0.9 * state.tau_recent + 0.1 * t_proj
    plan = SpeculationPlan(depth=depth, micro_batch=micro, projected=t_proj, raw_depth=raw, delta=delta, mag=mag,
                           scale=scale, adj=adj)
    return plan, FlowState(f=tuple(f), idx=idx, tau_recent=tau_new)
