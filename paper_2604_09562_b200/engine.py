"""Config 5 serving loop (NEXT-2; BASELINE configs[4]): closed-loop continuous batching of a mixed
request trace over decode lanes, with the paper's control plane around the verify step:

* metrics every 500 ms ("StreamServe collects system metrics at 500-millisecond
  intervals"): each lane's window of sv_stats deltas (acceptance a = accepted / drafted, throughput
  t = emitted tokens / s), load l = active / max_batch, KV memory M = pages in use / pool, queue depth;
* SpecuStream (Alg. 4, in libsv) turns (a, l, t) into the lane's depth for the next window;
* FlowGuard (Alg. 2, in libsv) routes each admitted request to a lane from the published snapshots
  (staleness, overload) and the live queue depths;
* per request: latency = t_end - t_start (eq:latency_computation), TPOT = (t_last - t_first) / l_g
  over the generated tokens (eq:tpot_computation, reading R33), throughput = (l_p + l_g) / latency
  (eq:throughput_computation); nearest-rank percentiles.

One process per GPU (one lane each). All ranks run the same deterministic control plane: at every
control tick they all_gather each lane's (finished, published metrics) and route the same new
requests, so no rank is a separate router process. The data path (prefill, verify, commit) never
crosses ranks. Host-side logic only; every step of the path runs in libsv.
"""
import collections
import math
import time

import numpy as np
import torch

from . import dist as svdist

METRICS_INTERVAL_S = 0.5


def nearest_rank(xs, p):
    """Nearest-rank percentile: the smallest x with at least p % of the values <= x."""
    if not xs:
        return None
    s = sorted(xs)
    k = max(1, math.ceil(p / 100.0 * len(s)))
    return s[k - 1]


class Request:
    __slots__ = ("qid", "dataset", "prompt_len", "out_len", "alpha", "prompt_seed", "rid", "lane", "slot",
                 "t_submit", "t_first", "t_end", "generated", "first_step")

    def __init__(self, q, rid):
        self.qid, self.dataset = q["qid"], q["dataset"]
        self.prompt_len, self.out_len, self.alpha = q["prompt_len"], q["out_len"], q["alpha"]
        self.prompt_seed = q["prompt_seed"]
        self.rid = rid
        self.lane = self.slot = None
        self.t_submit = self.t_first = self.t_end = None
        self.generated = 0

    def report(self):
        lat = self.t_end - self.t_submit
        g = max(1, self.generated)
        return {"qid": self.qid, "dataset": self.dataset, "latency_s": lat,
                "tpot_s": (self.t_end - self.t_first) / g, "throughput_tps": (self.prompt_len + g) / lat,
                "generated": g, "prompt_len": self.prompt_len}


class LaneEngine:
    """One decode lane: local queue, prefill admission into free slots, one verify + commit step over
    all active requests at the lane's current depth, completion, the 500 ms metrics window and the
    SpecuStream depth update. `lane` is an sv.Lane (or a test double with the same methods)."""

    def __init__(self, lane, cfg, succ, kmax, prompt_fn, clock=time.perf_counter, controller=None, chunk=None,
                 device="cuda", seed=0):
        self.lane, self.cfg, self.kmax = lane, cfg, kmax
        self.clock = clock
        self.prompt_fn = prompt_fn
        self.queue = collections.deque()
        self.active = {}
        self.free = list(range(cfg.max_slots))[::-1]
        self.done = []
        self.ctl = controller
        self.depth = kmax if controller is None else min(kmax, int(controller.cfg.d_base))
        self.chunk = chunk or min(cfg.max_batch * (cfg.max_depth + 1), 1024)
        self.device = device
        self.on_gpu = torch.device(device).type == "cuda"
        self.succ_d = succ.to(device) if hasattr(succ, "to") else succ
        self.rng = np.random.default_rng(seed)
        self.steps = 0
        self.s0 = lane.stats_raw()
        self.t_window = clock()
        self.published = None
        self.trace = []
        B = cfg.max_batch
        self.drafts = torch.empty(B * kmax, dtype=torch.int32, device=device)
        self.acc = torch.empty(B, dtype=torch.int32, device=device)
        self.tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=device)
        self.h_mask = torch.zeros(B * kmax, dtype=torch.uint8)
        self.h_dev = torch.zeros(B * kmax, dtype=torch.int32)
        if self.on_gpu:
            self.h_mask, self.h_dev = self.h_mask.pin_memory(), self.h_dev.pin_memory()
        self.d_mask = torch.empty(B * kmax, dtype=torch.uint8, device=device)
        self.d_dev = torch.empty(B * kmax, dtype=torch.int32, device=device)
        self.h_acc = torch.empty(B, dtype=torch.int32)
        if self.on_gpu:
            self.h_acc = self.h_acc.pin_memory()

    # ---------------------------------------------------------------- admission
    def admit(self):
        """Prefill queued requests into free slots (sv_prefill, long chunks); the prefill's next token
        is the first generated token."""
        n = 0
        while self.queue and self.free:
            r = self.queue.popleft()
            r.slot = self.free.pop()
            prompt = self.prompt_fn(r)
            self.lane.prefill(r.slot, r.rid, prompt, self.chunk)
            r.t_first = self.clock()
            r.generated = 1
            self.active[r.slot] = r
            n += 1
            if r.generated >= r.out_len:
                self._finish(r)
        return n

    def _finish(self, r):
        r.t_end = self.clock()
        self.lane.release(r.slot)
        del self.active[r.slot]
        self.free.append(r.slot)
        self.done.append(r)

    # ---------------------------------------------------------------- one verify step
    def step(self):
        if not self.active:
            return 0
        slots = sorted(self.active)[: self.cfg.max_batch]
        reqs = [self.active[s] for s in slots]
        k = max(1, min(self.depth, self.kmax))
        depths = [min(k, max(1, r.out_len - r.generated)) for r in reqs]
        rows = sum(depths)
        # planted drafter: per request, each draft deviates from the planted successor with
        # probability 1 - alpha (the dataset's acceptance profile)
        m = self.h_mask.numpy()
        t = self.h_dev.numpy()
        off = 0
        for r, d in zip(reqs, depths):
            m[off:off + d] = self.rng.random(d) >= r.alpha
            t[off:off + d] = self.rng.integers(0, self.cfg.vocab, d)
            off += d
        self.d_mask[:rows].copy_(self.h_mask[:rows], non_blocking=True)
        self.d_dev[:rows].copy_(self.h_dev[:rows], non_blocking=True)
        self.lane.draft_planted(slots, depths, self.succ_d, self.d_mask, self.d_dev, self.drafts)
        self.lane.verify(slots, depths, self.drafts, None, seed=1000 + self.steps, mode="sample",
                         out=(self.acc, self.tok))
        self.lane.commit()
        self.h_acc[: len(slots)].copy_(self.acc[: len(slots)], non_blocking=self.on_gpu)
        if self.on_gpu:
            torch.cuda.current_stream().synchronize()
        a = self.h_acc[: len(slots)].tolist()
        emitted = 0
        for r, ai in zip(reqs, a):
            e = int(ai) + 1
            r.generated += e
            emitted += e
            if r.generated >= r.out_len:
                self._finish(r)
        self.steps += 1
        return emitted

    # ---------------------------------------------------------------- 500 ms metrics window
    def maybe_publish(self, now, force=False):
        """Every METRICS_INTERVAL_S: the window's (a, t, l) -> SpecuStream depth; the FlowGuard
        snapshot (timestamp, cache hit 0, M, Q, L) is published for routing."""
        if not force and now - self.t_window < METRICS_INTERVAL_S:
            return False
        s1 = self.lane.stats_raw()
        secs = max(now - self.t_window, 1e-9)
        active = len(self.active)
        if self.ctl is not None:
            plan = self.ctl.step(self.s0, s1, secs, active, self.cfg.max_batch)
            self.depth = max(1, min(plan.depth, self.kmax))
        drafted = s1.drafted - self.s0.drafted
        win = {"t": round(now, 4), "a": (s1.accepted - self.s0.accepted) / drafted if drafted else 0.0,
               "tokens_per_s": (s1.emitted - self.s0.emitted) / secs, "active": active, "queue": len(self.queue),
               "depth": self.depth}
        self.trace.append(win)
        self.s0, self.t_window = s1, now
        act, free_pages = self.lane.occupancy()
        self.published = (int(now * 1e3), 0.0, 1.0 - free_pages / self.cfg.n_pages, float(len(self.queue)),
                          act / self.cfg.max_slots)
        return True


class ClosedLoop:
    """Closed-loop driver over the lanes of all ranks: keeps `concurrency` requests in flight
    (submitted - finished), routes each submission with FlowGuard, and runs until the trace is done."""

    def __init__(self, engine, trace, concurrency, rank=0, world=1, clock=time.perf_counter, device=None,
                 control_every=8, route_cfg=None):
        self.eng, self.trace = engine, trace
        self.C, self.rank, self.world = concurrency, rank, world
        self.clock = clock
        self.device = device
        self.control_every = control_every
        self.route_cfg = route_cfg
        self.next_q = 0
        self.finished_global = 0
        self.routed = [0] * world
        self.timed_out = False
        self.stop_all = False

    def control_tick(self, now):
        """All ranks: exchange (finished count, published snapshot), then route the same new
        submissions (deterministic), each rank queuing the ones routed to it."""
        e = self.eng
        e.maybe_publish(now)
        pub = e.published if e.published is not None else (int(now * 1e3), 0.0, 0.0, 0.0, 0.0)
        local = (float(len(e.done)),) + tuple(float(x) for x in pub) + (float(self.timed_out),)
        allv = self._gather_rows(local)
        self.finished_global = int(sum(r[0] for r in allv))
        self.stop_all = any(r[6] > 0 for r in allv)
        snaps = [(int(r[1]), r[2], r[3], r[4], r[5]) for r in allv]
        in_flight = self.next_q - self.finished_global
        n_new = max(0, min(self.C - in_flight, len(self.trace) - self.next_q))
        if n_new:
            lanes = svdist.route_requests(n_new, snaps, int(now * 1e3), self.route_cfg) if self.world > 1 \
                else [0] * n_new
            for lane_i in lanes:
                q = self.trace[self.next_q]
                self.next_q += 1
                self.routed[lane_i] += 1
                if lane_i == self.rank:
                    r = Request(q, svdist.request_id(self.rank, q["qid"]))
                    r.t_submit = now
                    r.lane = lane_i
                    e.queue.append(r)
        return n_new

    def _gather_rows(self, local):
        if self.world == 1:
            return [local]
        t = torch.tensor(local, dtype=torch.float64, device=self.device)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        torch.distributed.all_gather(out, t)
        return [tuple(float(x) for x in o.tolist()) for o in out]

    def run(self, max_seconds=600.0):
        e = self.eng
        t0 = self.clock()
        e.t_window = t0
        e.s0 = e.lane.stats_raw()
        tokens = 0
        it = 0
        while True:
            now = self.clock()
            # control ticks are collectives for world > 1: every rank ticks every control_every steps
            if it % self.control_every == 0 or (self.world == 1 and not e.active):
                self.timed_out = now - t0 > max_seconds
                self.control_tick(now)
                if self.finished_global >= len(self.trace) or self.stop_all:
                    break
            e.admit()
            tokens += e.step()
            it += 1
        e.maybe_publish(self.clock(), force=True)
        return {"seconds": self.clock() - t0, "generated_tokens_lane": sum(r.generated for r in e.done),
                "completed_lane": len(e.done), "steps": e.steps, "routed": self.routed}


def level_report(concurrency, results, seconds, world, lane_windows):
    """Per-concurrency JSON report from every lane's completed requests."""
    lat = [r["latency_s"] for r in results]
    tpot = [r["tpot_s"] for r in results]
    gen = sum(r["generated"] for r in results)
    by_ds = {}
    for r in results:
        by_ds.setdefault(r["dataset"], []).append(r)
    accs = [w["a"] for ws in lane_windows for w in ws if w.get("a")]
    return {
        "concurrency": concurrency, "lanes": world, "requests": len(results), "seconds": round(seconds, 3),
        "system_generated_tokens_per_s": round(gen / seconds, 1) if seconds > 0 else None,
        "system_processed_tokens_per_s": round((gen + sum(r["prompt_len"] for r in results)) / seconds, 1)
        if seconds > 0 else None,
        "latency_s": {"mean": round(float(np.mean(lat)), 4) if lat else None,
                      **{f"p{p}": round(nearest_rank(lat, p), 4) if lat else None for p in (50, 90, 95, 99)}},
        "tpot_s": {"mean": round(float(np.mean(tpot)), 5) if tpot else None,
                   "p50": round(nearest_rank(tpot, 50), 5) if tpot else None},
        "per_request_throughput_tps": round(float(np.mean([r["throughput_tps"] for r in results])), 1)
        if results else None,
        "by_dataset": {d: {"n": len(v), "latency_mean_s": round(float(np.mean([x["latency_s"] for x in v])), 4),
                           "tpot_mean_s": round(float(np.mean([x["tpot_s"] for x in v])), 5)}
                       for d, v in sorted(by_ds.items())},
        "acceptance_windows_mean": round(float(np.mean(accs)), 4) if accs else None,
        "depth_last": [ws[-1]["depth"] for ws in lane_windows if ws],
    }
