"""The library's SpecuStream controller (csrc/specustream.cpp via include/sv.h) against the oracle
(oracle/specustream.py, Alg. 4). Host code: runs without a GPU. Same double arithmetic in the
same order, so plans and states must match bit for bit."""
import ctypes
import random

import pytest

from oracle import specustream as ss
from paper_2604_09562_b200 import specustream as lib_ss
from paper_2604_09562_b200 import sv


def _oracle_cfg(c):
    return ss.SpecConfig(d_base=c.d_base, gamma=c.gamma, d_min=c.d_min, d_max=c.d_max, h=c.h,
                         tau_target=c.tau_target, micro_batch_numerator=c.micro_batch_numerator,
                         projection_source="measured" if c.projection_source == 0 else "smoothed")


@pytest.mark.parametrize("overrides", [{}, {"h": 1}, {"h": 64, "gamma": 2.5, "d_max": 8.0},
                                       {"projection_source": 1, "tau_target": 2000.0, "d_min": 1.0, "d_base": 1.0}])
def test_matches_oracle_bitwise(overrides):
    cfg = lib_ss.SpecConfig.default(**overrides)
    ocfg = _oracle_cfg(cfg)
    ctl = lib_ss.Controller(cfg)
    ost = ss.reset(ocfg)
    rng = random.Random(hash(tuple(sorted(overrides.items()))) & 0xffff)
    for _ in range(500):
        a, l = rng.random(), rng.random()
        t = rng.choice([0.0, 0.3, 1.0, 123.4, 400.0, 5e4]) * rng.random()
        p = ctl.adapt(a, l, t)
        op, ost = ss.adapt(ost, a, l, t, ocfg)
        assert (p.depth, p.micro_batch) == (op.depth, op.micro_batch)
        for k in ("projected", "raw_depth", "delta", "mag", "scale", "adj"):
            assert getattr(p, k) == getattr(op, k), k
        assert ctl.flow() == list(ost.f) and ctl.state.idx == ost.idx and ctl.state.tau_recent == ost.tau_recent


def test_worked_trace_through_the_library():
    ctl = lib_ss.Controller()
    p = ctl.adapt(0.8, 0.0, 400.0)
    assert (p.depth, p.micro_batch) == (5, 16)
    assert abs(p.raw_depth - 5.32) < 1e-12 and abs(p.projected - 560.0) < 1e-12
    assert abs(ctl.state.tau_recent - 416.0) < 1e-12


def test_step_from_lane_counters():
    """a, t, l from two sv_lane_stats snapshots (R24) then Alg. 4."""
    s0, s1 = sv.LaneStats(), sv.LaneStats()
    s0.drafted, s0.accepted, s0.emitted = 100, 40, 150
    s1.drafted, s1.accepted, s1.emitted = 612, 300, 830
    ctl, ref = lib_ss.Controller(), lib_ss.Controller()
    p = ctl.step(s0, s1, 0.5, 48, 64)
    q = ref.adapt(260 / 512, 48 / 64, 680 / 0.5)
    assert p.as_dict() == q.as_dict()
    empty = lib_ss.Controller().step(s0, s0, 0.5, 0, 64)  # nothing drafted: a = 0 -> baseline
    assert empty.depth == 5 and empty.delta == 0.0


def test_errors():
    lib = lib_ss._lib()
    cfg = lib_ss.SpecConfig.default()
    st, plan = lib_ss.FlowState(), lib_ss.SpecPlan()
    bad = lib_ss.SpecConfig.default(h=0)
    assert lib.sv_spec_reset(ctypes.byref(bad), ctypes.byref(st)) == sv.SV_EINVAL
    bad = lib_ss.SpecConfig.default(d_min=6.0)            # d_min > d_base
    assert lib.sv_spec_reset(ctypes.byref(bad), ctypes.byref(st)) == sv.SV_EINVAL
    assert lib.sv_spec_reset(ctypes.byref(cfg), ctypes.byref(st)) == sv.SV_OK
    for a, l, t in ((1.5, 0.0, 1.0), (0.5, -0.1, 1.0), (0.5, 0.5, -1.0), (float("nan"), 0.0, 1.0)):
        assert lib.sv_spec_adapt(ctypes.byref(cfg), ctypes.byref(st), a, l, t, ctypes.byref(plan),
                                 ctypes.byref(st)) == sv.SV_EINVAL
    st.idx = 10
    assert lib.sv_spec_adapt(ctypes.byref(cfg), ctypes.byref(st), 0.5, 0.5, 1.0, ctypes.byref(plan),
                             ctypes.byref(st)) == sv.SV_EINVAL
