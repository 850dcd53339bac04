"""Pins of oracle/specustream.py (Alg. 4) to values and laws fixed outside it:
SPEC.md's worked traces, the invariants of SPEC.md:241-248, and an
independent history-based formulation of the flow vector (eq:acceptance_gradient)."""
import math
import random

import pytest

from oracle import specustream as ss

CFG = ss.SpecConfig()


def test_trivial_zero_signal_keeps_baseline():
    # SPEC.md:227 [TRIVIAL]: a = 0, f zeros, any l, t = 400 -> delta 0, mag 0, raw 5, d* 5, b 16, t_proj 400
    for l in (0.0, 0.5, 1.0):
        plan, st = ss.adapt(ss.reset(CFG), 0.0, l, 400.0, CFG)
        assert (plan.delta, plan.mag, plan.raw_depth, plan.depth, plan.micro_batch, plan.projected) == \
            (0.0, 0.0, 5.0, 5, 16, 400.0)
        assert st.tau_recent == 400.0


def test_worked_cold_start_trace():
    # SPEC.md:228, 583 [PRIMARY]: a = 0.8, l = 0, t = 400, cold state ->
    # delta 0.8, mag 0.08, scale 1, adj 1, raw 5.32, d* 5, b 16, t_proj 560, tau_recent' 416
    plan, st = ss.adapt(ss.reset(CFG), 0.8, 0.0, 400.0, CFG)
    assert plan.delta == 0.8 and plan.scale == 1.0 and plan.adj == 1.0
    assert math.isclose(plan.mag, 0.08, rel_tol=1e-15)
    assert math.isclose(plan.raw_depth, 5.32, rel_tol=1e-15)
    assert (plan.depth, plan.micro_batch) == (5, 16)
    assert math.isclose(plan.projected, 560.0, rel_tol=1e-15)
    assert math.isclose(st.tau_recent, 416.0, rel_tol=1e-15)
    assert st.idx == 1 and st.f[0] == 0.8 and all(x == 0.0 for x in st.f[1:])


def test_worked_upper_clip_trace():
    # a = 1, f such that mag_after = 1, l = 0, t = 100 -> scale 4, raw 25, d* 20, b 4.
    # f_before = 1.1 everywhere: delta = 1 - 1.1 = -0.1, mag_after = (0.1 + 9 * 1.1) / 10 = 1
    st = ss.FlowState(f=tuple([1.1] * 10), idx=0, tau_recent=400.0)
    plan, _ = ss.adapt(st, 1.0, 0.0, 100.0, CFG)
    assert plan.scale == 4.0
    assert math.isclose(plan.mag, 1.0, rel_tol=1e-14)
    assert math.isclose(plan.raw_depth, 25.0, rel_tol=1e-14)
    assert (plan.depth, plan.micro_batch) == (20, 4)


def test_reset_and_purity():
    a, b = ss.reset(CFG), ss.reset(CFG)
    assert a == b and a.tau_recent == 400.0 and a.idx == 0 and len(a.f) == CFG.h
    p1, s1 = ss.adapt(a, 0.7, 0.3, 250.0, CFG)
    p2, s2 = ss.adapt(a, 0.7, 0.3, 250.0, CFG)
    assert p1 == p2 and s1 == s2 and a == b                  # deterministic; input not mutated


def _history_flow(a_seq, h):
    """f after each step from the history definition: slot j holds the latest delta_m with m = j mod h,
    delta_n = a_n - (1/h) sum over slots of the latest deltas written before step n."""
    deltas, out = [], []
    for n, a in enumerate(a_seq):
        slots = []
        for j in range(h):
            ms = [m for m in range(n) if m % h == j]
            slots.append(deltas[ms[-1]] if ms else 0.0)
        deltas.append(a - sum(slots) / h)
        after = []
        for j in range(h):
            ms = [m for m in range(n + 1) if m % h == j]
            after.append(deltas[ms[-1]] if ms else 0.0)
        out.append(after)
    return out


@pytest.mark.parametrize("h", [1, 3, 10])
def test_flow_buffer_equals_history_replay(h):
    cfg = ss.SpecConfig(h=h)
    rng = random.Random(h)
    a_seq = [rng.random() for _ in range(37)]
    ref = _history_flow(a_seq, h)
    st = ss.reset(cfg)
    for n, a in enumerate(a_seq):
        plan, st = ss.adapt(st, a, 0.2, 300.0, cfg)
        for x, y in zip(st.f, ref[n]):
            assert abs(x - y) <= 1e-12 * max(1.0, abs(y))
        assert math.isclose(plan.mag, sum(abs(y) for y in ref[n]) / h, rel_tol=1e-12, abs_tol=1e-15)


def test_invariants_random_walk():
    rng = random.Random(7)
    st = ss.reset(CFG)
    for _ in range(2000):
        a, l, t = rng.random(), rng.random(), rng.choice([0.0, 0.5, 50.0, 399.0, 400.0, 1e4]) * rng.random()
        plan, st2 = ss.adapt(st, a, l, t, CFG)
        assert CFG.d_min <= plan.depth <= CFG.d_max                              # depth bounds
        assert plan.micro_batch >= 1
        assert plan.micro_batch * plan.depth <= CFG.micro_batch_numerator + plan.depth   # coupling
        assert plan.scale >= 1.0 and (t < CFG.tau_target or plan.scale == 1.0)   # scale floor
        # load monotonicity: raw depth nonincreasing in l with a, t, f fixed
        hi, _ = ss.adapt(st, a, min(1.0, l + 0.3), t, CFG)
        assert hi.raw_depth <= plan.raw_depth
        # smoothing contraction: |tau' - t_proj| = 0.9 |tau - t_proj|
        lhs, rhs = abs(st2.tau_recent - plan.projected), 0.9 * abs(st.tau_recent - plan.projected)
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, rhs)
        st = st2


def test_projection_source_toggle():
    cfg = ss.SpecConfig(projection_source="smoothed")
    st = ss.FlowState(f=tuple([0.0] * 10), idx=0, tau_recent=200.0)
    plan, st2 = ss.adapt(st, 0.5, 0.0, 999.0, cfg)
    assert plan.projected == 200.0 * 1.25 and st2.tau_recent == 0.9 * 200.0 + 0.1 * 250.0


def test_lower_clip_unreachable_with_paper_defaults():
    # d = d_base + (non-negative term) >= 5 > d_min
    rng = random.Random(3)
    st = ss.reset(CFG)
    for _ in range(500):
        plan, st = ss.adapt(st, rng.random(), rng.random(), 1000 * rng.random(), CFG)
        assert plan.raw_depth >= CFG.d_base
