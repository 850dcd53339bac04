"""Host logic of the config-5 serving loop (paper_2604_09562_b200/engine.py) on CPU with a lane double:
the mixed trace (synth.mixed_trace), nearest-rank percentiles, closed-loop admission (never more than
C requests in flight, every request completes with its output length), the 500 ms metrics window
feeding SpecuStream, the per-request metrics of PAPER.md eq:latency/tpot/throughput, and the
FlowGuard-routed two-lane control plane over gloo (world size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2604_09562_b200 import engine, sv
from paper_2604_09562_b200 import specustream as sps


class FakeLane:
    """Same calls as sv.Lane, no device: accepted length ~ Binomial-like by the drafted alpha."""

    def __init__(self, cfg, seed=0):
        self.cfg = cfg
        self.st = sv.LaneStats()
        self.active = set()
        self.rng = np.random.default_rng(seed)
        self.pages = 0
        self.inflight = 0
        self.max_inflight = 0

    def stats_raw(self):
        s = sv.LaneStats()
        for n in ("steps", "drafted", "accepted", "emitted"):
            setattr(s, n, getattr(self.st, n))
        return s

    def prefill(self, slot, rid, prompt, chunk):
        assert slot not in self.active and 1 <= chunk
        self.active.add(slot)
        self.pages += len(prompt) // 64 + 1
        self.max_inflight = max(self.max_inflight, len(self.active))
        return 0

    def release(self, slot):
        self.active.remove(slot)

    def draft_planted(self, slots, depths, succ, mask, dev, out):
        self.masks = mask[: sum(depths)].clone()

    def verify(self, slots, depths, drafts, probs, seed=0, mode="sample", out=None):
        acc = out[0]
        off = 0
        for i, d in enumerate(depths):
            m = self.masks[off:off + d].tolist()
            a = 0
            while a < d and not m[a]:
                a += 1
            acc[i] = a
            self.st.drafted += d
            self.st.accepted += a
            self.st.emitted += a + 1
            off += d
        self.st.steps += 1
        return acc, out[1]

    def commit(self):
        pass

    def occupancy(self):
        return len(self.active), self.cfg.n_pages - min(self.pages, self.cfg.n_pages)


class FakeClock:
    def __init__(self, dt=0.003):
        self.t, self.dt = 0.0, dt

    def __call__(self):
        self.t += self.dt
        return self.t


def _engine(cfg, seed=0, clock=None):
    lane = FakeLane(cfg, seed)
    succ = torch.arange(cfg.vocab, dtype=torch.int32)
    eng = engine.LaneEngine(lane, cfg, succ, 8, lambda r: [0] * r.prompt_len, clock=clock or FakeClock(),
                            controller=sps.Controller(), device="cpu", seed=seed)
    return lane, eng


def test_mixed_trace_shape():
    t = synth.mixed_trace()
    assert len(t) == 320 and len({q["qid"] for q in t}) == 320
    for name, (lo, hi, med, p0) in synth.TRACE_PROFILES.items():
        qs = [q for q in t if q["dataset"] == name]
        assert len(qs) == 80 and all(lo <= q["prompt_len"] <= hi and q["alpha"] == p0 for q in qs)
        assert 0.7 * med <= np.median([q["out_len"] for q in qs]) <= 1.3 * med
    assert t == synth.mixed_trace()                             # seeded


def test_nearest_rank():
    xs = [15, 20, 35, 40, 50]
    assert engine.nearest_rank(xs, 5) == 15 and engine.nearest_rank(xs, 30) == 20
    assert engine.nearest_rank(xs, 40) == 20 and engine.nearest_rank(xs, 50) == 35
    assert engine.nearest_rank(xs, 100) == 50 and engine.nearest_rank([], 50) is None


@pytest.mark.parametrize("C", [1, 7, 64])
def test_closed_loop_completes_trace_within_concurrency(C):
    cfg = synth.LLAMA.with_(max_slots=32, max_batch=32, n_pages=100000, max_pos=16384)
    trace = synth.mixed_trace(n_per_dataset=10, seed=3)
    clock = FakeClock()
    lane, eng = _engine(cfg, clock=clock)
    loop = engine.ClosedLoop(eng, trace, C, clock=clock)
    run = loop.run()
    assert len(eng.done) == len(trace) and not eng.active and not eng.queue
    assert lane.max_inflight <= min(C, cfg.max_slots)
    for r in eng.done:
        assert r.generated >= r.out_len and r.generated <= r.out_len + 8
        assert r.t_submit <= r.t_first <= r.t_end
    rep = engine.level_report(C, [r.report() for r in eng.done], run["seconds"], 1, [eng.trace])
    assert rep["requests"] == len(trace) and rep["latency_s"]["p50"] <= rep["latency_s"]["p99"]
    assert len(eng.trace) >= 2                                  # the 500 ms windows ran
    assert all(1 <= w["depth"] <= 8 for w in eng.trace)
    r0 = eng.done[0].report()
    assert abs(r0["throughput_tps"] - (r0["prompt_len"] + r0["generated"]) / r0["latency_s"]) < 1e-9


def _two_lane_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.LLAMA.with_(max_slots=16, max_batch=16, n_pages=100000, max_pos=16384)
    trace = synth.mixed_trace(n_per_dataset=6, seed=5)
    clock = FakeClock(0.002 + 0.001 * rank)                   # lanes run at different speeds
    lane, eng = _engine(cfg, seed=rank, clock=clock)
    loop = engine.ClosedLoop(eng, trace, 12, rank=rank, world=world, clock=clock, device=torch.device("cpu"))
    loop.run()
    out[rank] = (sorted(r.qid for r in eng.done), loop.routed)
    dist.destroy_process_group()


def test_two_lane_flowguard_routing_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = mp.Manager().dict()
    mp.spawn(_two_lane_worker, args=(2, port, out), nprocs=2, join=True)
    q0, routed0 = out[0]
    q1, routed1 = out[1]
    assert routed0 == routed1                                  # every rank routed the same way
    assert sorted(q0 + q1) == list(range(24)) and not set(q0) & set(q1)
    assert len(q0) > 0 and len(q1) > 0
