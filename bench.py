#!/usr/bin/env python
"""Benchmark of the speculative-verify hot path (BASELINE.json metric):
accepted tokens/s of the verify step, verify-step us, % of the HBM / tensor roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ns|ns32|ns_tree|c2|c2_filter|c3|c4|toy]
    python bench.py --impl reference ...        # the fp64 CPU oracle arm
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one planted-drafter launch (bench fixture) + sv_verify + sv_commit on one
decode lane holding `batch` requests. Weak scaling: every
rank runs its own lane (own requests, no collective on the data path). Inputs
(weights, KV) live in HBM before the timed region and exceed L2 (126 MB).
Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_09562_b200 import dist as svdist  # noqa: E402

METRIC = "accepted tokens/s (verify step)"
UNIT = "tokens/s"
HOST_DRAFTER_STEPS = 10   # e2e variant with the drafter on the host (a full round trip per step)
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _json_default(o):
    if hasattr(o, "item"):                            # numpy / torch scalars
        return o.item()
    raise TypeError(f"not JSON serializable: {type(o).__name__}")


def peaks():
    try:
        p = json.load(open(PEAKS_FILE))
        return dict(hbm=p["hbm_gbs"], bf16=p["bf16_tflops"], bf16_sus=p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


def ncu_traffic():
    """DRAM bytes (read + write) per launch of each roofline kernel from the committed
    `ncu --set full` capture (profiles/<round>_ncu_full.json, newest round), or {}."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "*_ncu_full.json")))
    if not files:
        return {}
    try:
        rows = json.load(open(files[-1]))
    except Exception:
        return {}
    names = {"gemm_sw_kernel": "lm_head", "attn_tc2_kernel": "attention"}
    return {names[r["kernel"]]: {"bytes": int(r["dram_bytes"]), "src": os.path.basename(files[-1])}
            for r in rows if r.get("kernel") in names}


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    """Samples SM clock and clock-event (throttle) reasons through NVML every 2 ms while the
    timed region runs (same fields as nvidia-smi's clocks / clocks_event_reasons)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self.reason_count = {}
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # the driver's cumulative power-policy violation time: unlike the sampled reason bits it
            # cannot miss a cap that engages between two samples
            try:
                self.v0 = pynvml.nvmlDeviceGetViolationStatus(self.h, pynvml.NVML_PERF_POLICY_POWER).violationTime
            except Exception:
                self.v0 = None
            self.w0 = time.perf_counter()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
                        self.reason_count[name] = self.reason_count.get(name, 0) + 1
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop.set()
        self.power_violation = None
        if self.nv:
            self.t.join(timeout=1)
            if self.v0 is not None:
                try:
                    v1 = self.nv.nvmlDeviceGetViolationStatus(self.h, self.nv.NVML_PERF_POLICY_POWER).violationTime
                    span_ns = (time.perf_counter() - self.w0) * 1e9
                    self.power_violation = max(0.0, min(1.0, (v1 - self.v0) / span_ns)) if span_ns > 0 else None
                    if self.power_violation:
                        self.reasons.add("sw_power_cap")
                except Exception:
                    pass

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        out = {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
               "samples": len(self.sm),
               "reason_frac": {k: round(v / len(self.sm), 3) for k, v in sorted(self.reason_count.items())}}
        if getattr(self, "power_violation", None) is not None:
            out["power_cap_violation_frac"] = round(self.power_violation, 3)   # NVML power-policy violation time
        return out

    def power_capped(self):
        """True when sw_power_cap held for most of the region: the kernels then ran at the clocks
        the sustained peak was measured at, so that is the roofline denominator; else the burst."""
        sampled = bool(self.sm) and self.reason_count.get("sw_power_cap", 0) > 0.5 * len(self.sm)
        return sampled or (getattr(self, "power_violation", None) or 0.0) > 0.5


# ------------------------------------------------------------------ workload setup
def planted_weights(wl, device="cpu"):
    w = synth.model_weights(wl.cfg, seed=0, embed_std=wl.embed_std, device=device)
    if wl.beta > 0:
        return synth.planted_successor(wl.cfg, w, seed=1, beta=wl.beta)
    return w, torch.randperm(wl.cfg.vocab, generator=torch.Generator().manual_seed(1)).to(torch.int32)


def build_lane(wl, rank, dev, stream=None):
    from paper_2604_09562_b200 import sv
    cfg = wl.cfg
    gdev = dev if wl.gen_on_device else "cpu"
    w, succ = planted_weights(wl, gdev)
    wd = {k: v.to(dev) for k, v in w.items()}
    lane = sv.Lane(cfg, wd, stream=stream)
    ctx = synth.ctx_lengths(wl, seed=100 + rank)
    reqs = []
    for i, n in enumerate(ctx):
        k, v = synth.context_kv(cfg, n, seed=10_000 * (rank + 1) + i, device=gdev)
        pend = int(synth.random_tokens(1, cfg.vocab, seed=20_000 * (rank + 1) + i)[0])
        rid = svdist.request_id(rank, i)
        lane.append_kv(i, rid, k.to(dev), v.to(dev), pend)
        reqs.append(dict(L=n, rid=rid, pending=pend, k=None if wl.gen_on_device else k,
                         v=None if wl.gen_on_device else v))
    if wl.top_k or wl.top_p < 1.0:
        lane.set_filter(wl.top_k, wl.top_p)          # R31 filtered target (SAMPLE workloads)
    torch.cuda.synchronize(dev)
    return lane, w, succ, reqs


def draft_and_verify(lane, wl, slots, ks, succ_d, mask_d, devtok_d, drafts, seed, out, parents_d=None):
    """One drafter launch + one verify through the public API (chain, or token tree for tree workloads)."""
    if wl.tree:
        lane.draft_planted_tree(slots, ks, parents_d, succ_d, mask_d, devtok_d, drafts)
        lane.verify_tree(slots, ks, parents_d, drafts, None, seed=seed, mode=wl.mode, temperature=wl.temperature,
                         out=out)
    else:
        lane.draft_planted(slots, ks, succ_d, mask_d, devtok_d, drafts)
        lane.verify(slots, ks, drafts, None, seed=seed, mode=wl.mode, temperature=wl.temperature, out=out)


def tree_parents(wl, dev):
    return torch.tensor(list(wl.tree) * wl.batch, dtype=torch.int32, device=dev) if wl.tree else None


def depths_for(wl, n_steps, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(wl.kmin, wl.kmax + 1, (n_steps, wl.batch), generator=g).tolist()


def algorithmic(wl, ctx_lens, depths):
    """Algorithmic bytes / flops per launch of the two roofline kernels."""
    cfg = wl.cfg
    T = sum(k + 1 for k in depths)
    kv_tok = 2 * cfg.n_kv_heads * cfg.head_dim * 2                       # 4096 B / token / layer
    attn_bytes = sum(L * kv_tok for L in ctx_lens) + T * kv_tok + T * 2 * cfg.n_q_heads * cfg.head_dim * 2
    lm_flops = 2.0 * T * cfg.d_model * cfg.vocab
    return dict(T=T, attn_bytes=attn_bytes, lm_flops=lm_flops)      # per launch: attention runs once per layer


class ControlledDepths:
    """Depths from the SpecuStream controller (NEXT-1, R21-R24): every WINDOW steps the
    lane's counters (sv_stats) give a = accepted / drafted, t = emitted / seconds and l = 1 (full
    batch); Alg. 4 in the library returns d*, and all requests of the lane draft min(d*, kmax) tokens
    until the next window. Per-request planted acceptance follows AR(1) around wl.alpha
    (SPEC.md:360), so the controller's gradient tracking has a signal to follow."""
    WINDOW = 8

    def __init__(self, wl, n_steps, seed):
        from paper_2604_09562_b200 import specustream as sps
        self.wl, self.B, self.K = wl, wl.batch, wl.kmax
        self.ctl = sps.Controller()
        alphas = synth.ar1_alphas(n_steps, self.B, wl.alpha, wl.alpha_sigma, 0.9, seed)
        self.mreq, self.treq = synth.planted_masks_req(n_steps, self.B, self.K, alphas, wl.cfg.vocab, seed + 1)
        self.d = min(int(self.ctl.cfg.d_base), self.K)
        self.depths = [[self.d] * self.B for _ in range(n_steps)]
        self.masks = torch.zeros(n_steps, self.B * self.K, dtype=torch.uint8).pin_memory()
        self.devtok = torch.zeros(n_steps, self.B * self.K, dtype=torch.int32).pin_memory()
        self.trace, self.s0, self.t0 = [], None, 0.0

    def prepare(self, i, masks_d=None, devtok_d=None):
        """Lay out step i's drafter inputs for the current depth (ragged, request-major)."""
        d, B = self.d, self.B
        self.depths[i] = [d] * B
        self.masks[i, :B * d] = self.mreq[i, :, :d].reshape(-1)
        self.devtok[i, :B * d] = self.treq[i, :, :d].reshape(-1)
        if masks_d is not None:
            masks_d[i].copy_(self.masks[i], non_blocking=True)
            devtok_d[i].copy_(self.devtok[i], non_blocking=True)

    def restart(self, lane):
        self.s0, self.t0 = lane.stats_raw(), time.perf_counter()

    def tick(self, lane, i):
        if (i + 1) % self.WINDOW:
            return
        s1, now = lane.stats_raw(), time.perf_counter()
        if self.s0 is not None:
            plan = self.ctl.step(self.s0, s1, max(now - self.t0, 1e-9), self.B, self.B)
            self.d = max(1, min(plan.depth, self.K))
            self.trace.append({"step": i + 1, "a": round((s1.accepted - self.s0.accepted) /
                                                         max(1, s1.drafted - self.s0.drafted), 4),
                               "depth": plan.depth, "raw": round(plan.raw_depth, 4), "mag": round(plan.mag, 5)})
        self.s0, self.t0 = s1, now


VERIFY_GRAPH_REPLAYS = 100   # verify-step µs as SURVEY.md §8(d) defines it (graph replay, drafting excluded)


def run_gpu(args, wl, rank, world, dev):
    """The lane runs on a created stream (capturable), made torch's current stream so the bench's
    events and copies order with the lane's kernels."""
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        return _run_gpu(args, wl, rank, world, dev, stream)


def verify_step_graph(lane, wl, slots, ks, drafts, seed, out, par_d, dev, n):
    """Verify-step µs per SURVEY.md §8(d): CUDA-event time of one graph replay of sv_verify +
    sv_commit with the drafting excluded (the last timed step's depths and drafts, replayed n times)."""
    lane.graph_begin()
    if wl.tree:
        lane.verify_tree(slots, ks, par_d, drafts, None, seed=seed, mode=wl.mode, temperature=wl.temperature, out=out)
    else:
        lane.verify(slots, ks, drafts, None, seed=seed, mode=wl.mode, temperature=wl.temperature, out=out)
    lane.commit()
    g = lane.graph_end()
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    lane.graph_launch(g)                              # warm replay
    for a, b in ev:
        a.record(stream)
        lane.graph_launch(g)
        b.record(stream)
    torch.cuda.synchronize(dev)
    lane.graph_destroy(g)
    us = sorted(1e3 * a.elapsed_time(b) for a, b in ev)
    return {"median": round(statistics.median(us), 1), "p10": round(us[len(us) // 10], 1),
            "p90": round(us[(9 * len(us)) // 10], 1), "replays": n,
            "what": "CUDA graph replay of sv_verify + sv_commit, drafting excluded (SURVEY.md §8(d))"}


def kernels_from(prof):
    tot = max(1e-9, sum(v[0] for v in prof.values()))
    return {name: dict(ms_per_launch=ms / n, launches=n, share=ms / tot) for name, (ms, n) in prof.items() if n}


def roofline(kern, alg, pk, capped, traffic=None):
    """Roofline of the two dominant kernels: achieved = algorithmic work per launch / measured launch
    time. The peak follows the clock record of the region: the sustained bf16 peak when sw_power_cap
    held for most of it (the regime that peak was measured in), else the burst peak; both fractions
    are printed. HBM has one measured peak (copy bandwidth)."""
    traffic = traffic or {}
    lm, at = kern.get("lm_head"), kern.get("attention")
    roof = {}
    if lm:
        ach = alg["lm_flops"] / (lm["ms_per_launch"] * 1e-3) / 1e12
        peak = pk["bf16_sus"] if capped else pk["bf16"]
        roof["lm_head"] = {"bound": "tensor", "achieved": round(ach, 2), "peak": peak, "unit": "TFLOP/s",
                           "frac": round(ach / peak, 4), "peak_kind": "sustained" if capped else "burst",
                           "frac_burst": round(ach / pk["bf16"], 4), "frac_sustained": round(ach / pk["bf16_sus"], 4),
                           "traffic": traffic.get("lm_head", {}).get("bytes"),
                           "traffic_src": traffic.get("lm_head", {}).get("src"),
                           "flops_per_launch": alg["lm_flops"], "us_per_launch": round(lm["ms_per_launch"] * 1e3, 2)}
    if at:
        ach = alg["attn_bytes"] / (at["ms_per_launch"] * 1e-3) / 1e9
        roof["attention"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm"], "unit": "GB/s",
                             "frac": round(ach / pk["hbm"], 4), "frac_of_8tbs": round(ach / 8000.0, 4),
                             "traffic": traffic.get("attention", {}).get("bytes"), "bytes_per_launch": alg["attn_bytes"],
                             "traffic_src": traffic.get("attention", {}).get("src"),
                             "us_per_launch": round(at["ms_per_launch"] * 1e3, 2)}
    return roof


STEADY_MAX_STEPS = 2000      # steady-state phase: >= --steady-s seconds of steps, at most this many


def steady_cap(wl):
    return STEADY_MAX_STEPS if wl.cfg.n_layers == 1 else 100


def steady_state(args, wl, lane, depths, ms_step, pk, dev, stream):
    """Steady-state phase right after the timed region (VERDICT r1 "make the roofline line honest"):
    >= args.steady_s seconds of steps, the timed region's depths and drafter inputs replayed in order,
    each step committing ONE token per request (n_keep = 1) so contexts grow by one token per step
    instead of a+1 (the algorithmic bytes use the measured lengths). Reports ms/step, the two
    roofline kernels' µs and fractions and the clocks of this phase."""
    if args.steady_s <= 0 or args.steps < 1:
        return None
    cfg, B = wl.cfg, wl.batch
    n = int(min(steady_cap(wl), max(10, args.steady_s * 1e3 / max(ms_step, 1e-3))))
    keep1 = torch.ones(B, dtype=torch.int32, device=dev)
    slots = list(range(B))
    masks_d, devtok_d = args._masks_d, args._devtok_d
    succ_d, drafts, out, par_d = args._succ_d, args._drafts, args._out, args._par_d
    ln0 = lane.tap("len", torch.int32, (cfg.max_slots,))[:B].cpu().tolist()
    lane.profile(["lm_head", "attention"])
    lane.profile_read(reset=True)
    lane.stats(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    with Clocks(dev.index) as clk:
        e0.record(stream)
        for i in range(n):
            j = args.warmup + i % args.steps
            draft_and_verify(lane, wl, slots, depths[j], succ_d, masks_d[j], devtok_d[j], drafts, 777 + i, out, par_d)
            lane.commit(keep1)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    prof = lane.profile_read(reset=True)
    lane.profile(False)
    st = lane.stats(reset=True)
    ln1 = lane.tap("len", torch.int32, (cfg.max_slots,))[:B].cpu().tolist()
    mid = [(x + y) / 2.0 for x, y in zip(ln0, ln1)]
    algs = [algorithmic(wl, mid, depths[args.warmup + i % args.steps]) for i in range(n)]
    alg = {k: sum(a[k] for a in algs) / len(algs) for k in algs[0]}
    kk = kernels_from(prof)
    roof = roofline(kk, alg, pk, clk.power_capped())
    return {"steps": n, "seconds": round(ms * 1e-3, 3), "ms_per_step": round(ms / n, 4),
            "verified_rows_per_s": round(st["rows"] / (ms * 1e-3), 1),
            "kernels": {k: {x: v[x] for x in ("us_per_launch", "achieved", "unit", "frac", "peak", "peak_kind",
                                              "frac_burst", "frac_sustained", "frac_of_8tbs") if x in v}
                        for k, v in roof.items()},
            "ctx_mean": [round(sum(ln0) / B, 1), round(sum(ln1) / B, 1)], "clocks": clk.summary(),
            "what": "steps right after the timed region, n_keep = 1 (context +1 token/step), same depths/drafter"}


def decision_check(wl, lane, reqs, succ, masks, devtok, depths, start, dev):
    """Teacher-forced decision parity at the bench's own configuration:
    one more verify with logits_out; the oracle's decision rule (oracle/verify.py) is run on the GPU's
    fp32 logits for EVERY request and the decisions are compared. Sampled-mode mismatches are
    counted as borderline when |u - p/q| < 1e-5 or the race's top-2 scores are within 1e-5 relative
    (north_star: "those borderline flips are counted and reported"); any other mismatch is an error."""
    from oracle import verify as ov
    from oracle.philox import uniform_accept
    if wl.tree:
        return {"skipped": "token-tree workload (tree decisions are checked in tests/test_gpu_tree*.py)"}
    cfg, B = wl.cfg, wl.batch
    ks = depths[start - 1]
    T = sum(k + 1 for k in ks)
    lg = torch.empty(T, cfg.vocab, dtype=torch.float32, device=dev)
    drafts = torch.empty(max(1, B * wl.kmax), dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
    ln = lane.tap("len", torch.int32, (cfg.max_slots,))[:B].cpu().tolist()
    slots = list(range(B))
    lane.draft_planted(slots, ks, succ.to(dev), masks[start - 1].to(dev), devtok[start - 1].to(dev), drafts)
    seed = 31337
    lane.verify(slots, ks, drafts, None, seed=seed, mode=wl.mode, temperature=wl.temperature, logits_out=lg,
                out=(acc, tok))
    torch.cuda.synchronize(dev)
    lane.commit()
    L = lg.cpu().numpy().astype(np.float64)
    a_g, t_g, d_h = acc.cpu().numpy(), tok.cpu().numpy(), drafts.cpu().numpy()
    mode = ov.GREEDY if wl.mode == "greedy" else ov.SAMPLE
    mism = border = 0
    r0 = off = 0
    t0 = time.perf_counter()
    for b in range(B):
        k = ks[b]
        rows = L[r0:r0 + k + 1]
        dr = [int(x) for x in d_h[off:off + k]]
        rid = reqs[b]["rid"]
        r = ov.verify_request(rows, dr, None, seed, rid, ln[b], mode, wl.temperature, wl.top_k, wl.top_p)
        if int(a_g[b]) != r["a"] or list(t_g[b][:r["a"] + 1]) != r["emitted"]:
            bl = False
            if mode == ov.SAMPLE:
                p = ov.filtered_probs(rows, wl.temperature, wl.top_k, wl.top_p)
                bl = any(abs(uniform_accept(seed, rid, ln[b] + j) - p[j - 1][dr[j - 1]]) < 1e-5
                         for j in range(1, k + 1))
                a = r["a"]
                sc = ov.race_scores(rows[a], None, dr[a] if a < k else -1, seed, rid, ln[b] + a + 1, wl.temperature,
                                    a < k, wl.top_k, wl.top_p)
                top2 = np.sort(sc[np.isfinite(sc)])[-2:]
                bl = bl or (len(top2) == 2 and top2[1] - top2[0] <= 1e-5 * abs(top2[1]))
            border += int(bl)
            mism += int(not bl)
        r0 += k + 1
        off += k
    return {"requests": B, "rows": T, "mismatches": mism, "borderline_flips": border,
            "oracle_seconds": round(time.perf_counter() - t0, 2),
            "what": "oracle decision rule on the GPU's fp32 logits of one extra verify, every request (S12/S13)"}


def _run_gpu(args, wl, rank, world, dev, stream):
    from paper_2604_09562_b200 import sv
    import torch.distributed as dist
    lane, w, succ, reqs = build_lane(wl, rank, dev, stream)
    cfg = wl.cfg
    B = wl.batch
    total = args.warmup + args.steps
    depths = depths_for(wl, total + args.e2e_steps + HOST_DRAFTER_STEPS, seed=7 + rank)
    kmax_rows = B * wl.kmax
    masks, devtok = synth.planted_masks(total + args.e2e_steps + HOST_DRAFTER_STEPS, kmax_rows, wl.alpha, cfg.vocab,
                                        seed=9 + rank)
    ctl = None
    if wl.controller:
        ctl = ControlledDepths(wl, total + args.e2e_steps + HOST_DRAFTER_STEPS, seed=11 + rank)
        depths, masks, devtok = ctl.depths, ctl.masks, ctl.devtok
    masks_d, devtok_d, succ_d = masks.to(dev), devtok.to(dev), succ.to(dev)
    drafts = torch.empty(kmax_rows, dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
    slots = list(range(B))
    par_d = tree_parents(wl, dev)
    args._masks_d, args._devtok_d, args._succ_d, args._drafts, args._out, args._par_d = \
        masks_d, devtok_d, succ_d, drafts, (acc, tok), par_d

    def step(i):
        if ctl:
            ctl.prepare(i, masks_d, devtok_d)
        draft_and_verify(lane, wl, slots, depths[i], succ_d, masks_d[i], devtok_d[i], drafts, 1234 + i, (acc, tok),
                         par_d)
        lane.commit()

    for i in range(args.warmup):
        step(i)
        if ctl:
            ctl.tick(lane, i)
    torch.cuda.synchronize(dev)
    lane.stats(reset=True)
    if ctl:
        ctl.restart(lane)
    # context lengths at the start of the timed region (for the algorithmic attention bytes)
    ln = lane.tap("len", torch.int32, (cfg.max_slots,))[:B].cpu().tolist()
    # only the roofline kernels are bracketed by events in the timed region (every record is a
    # host call and a stream dependency); --detail times every stage and says so in the line
    lane.profile(True if args.detail else ["lm_head", "attention"])
    lane.profile_read(reset=True)
    # The timed region replays ONE captured step (planted drafter + verify + commit) as a CUDA graph,
    # the production decode path (PipeServe-Engine lanes run the same step every iteration): the
    # profiled stages' events are nodes of the graph, re-pointed at fresh events every replay, so the
    # roofline kernels are still timed per launch inside the region. Depth vectors that change per step
    # (c2, c3's controller) go through the dynamic-depth graph's staging buffer; each step's drafter
    # inputs are copied into the buffers the graph reads. --eager times the same steps as eager calls.
    # The timed steps replay two graphs of the same step: the one whose stage events are graph nodes on
    # every --prof-every-th step (the roofline averages come from those), the one without events on the
    # others (an event node between two kernels costs the PDL overlap there: ~2 % of an ns step).
    # Depth-varying workloads use two dynamic-depth graphs (sharing the lane's staging buffers).
    dynamic = wl.controller or wl.kmin != wl.kmax
    graph = plain = None
    # depth-varying workloads: graphs only where launches bound the step (toy: 0.080 -> 0.065 ms); at
    # Llama shape their event-timed replays measured 1 % slower (c2) or even (c3) than eager calls
    launch_bound = cfg.d_model <= 1024
    if not args.eager and (not dynamic or args.graph_dynamic or launch_bound) and not (dynamic and wl.tree):
        try:
            m_stage = torch.empty_like(masks_d[0])
            t_stage = torch.empty_like(devtok_d[0])

            def capture():
                if dynamic:
                    lane.graph_begin_dynamic(B)
                else:
                    lane.graph_begin()
                draft_and_verify(lane, wl, slots, depths[args.warmup - 1], succ_d, m_stage, t_stage, drafts, 1234,
                                 (acc, tok), par_d)
                lane.commit()                         # captured, not run
                return lane.graph_end()
            graph = capture()                         # profiled stages -> event-record nodes
            lane.profile(False)
            plain = capture()                         # (dynamic graphs share the lane's staging buffers)
            lane.profile(True if args.detail else ["lm_head", "attention"])
            torch.cuda.synchronize(dev)
        except Exception as ex:                       # fall back to timing eager calls
            print(f"[bench] graph capture failed ({ex}); timing eager steps", file=sys.stderr)
            lane.profile(True if args.detail else ["lm_head", "attention"])
            graph = plain = None

    def gstep(i, j):
        if ctl:
            ctl.prepare(j, masks_d, devtok_d)
        m_stage.copy_(masks_d[j])
        t_stage.copy_(devtok_d[j])
        g = graph if i % args.prof_every == 0 else plain
        if dynamic:
            lane.graph_set_batch(g, slots, depths[j])
        lane.graph_launch(g)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    stream = torch.cuda.current_stream(dev)
    launches0 = sv.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with Clocks(dev.index) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            if graph is not None:
                gstep(i, args.warmup + i)
            else:
                step(args.warmup + i)
            ev[i + 1].record(stream)
            if ctl:                                   # the control loop reads the counters (syncs)
                ctl.tick(lane, args.warmup + i)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = sv.launch_count() - launches0
    elapsed_ms = ev[0].elapsed_time(ev[-1])
    per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    prof = lane.profile_read(reset=True)
    lane.profile(False)
    if graph is not None:
        lane.graph_destroy(graph)
        if plain is not graph:
            lane.graph_destroy(plain)
    st = lane.stats()
    tokens = st["emitted"]
    # ----- roofline of the dominant kernels (live CUDA-event durations, averaged per launch)
    pk = peaks()
    traffic = ncu_traffic() if wl.name == "ns" else {}      # the committed capture is of the ns workload
    capped = clk.power_capped()
    # per-launch algorithmic work averaged over the timed region: mean T over its steps, context
    # lengths at the region's midpoint (they grow by the emitted tokens)
    ln1 = lane.tap("len", torch.int32, (cfg.max_slots,))[:B].cpu().tolist()
    mid = [(x + y) / 2.0 for x, y in zip(ln, ln1)]
    algs = [algorithmic(wl, mid, depths[args.warmup + i]) for i in range(args.steps)]
    alg = {k: sum(a[k] for a in algs) / len(algs) for k in algs[0]}
    kern = kernels_from(prof)
    roof = roofline(kern, alg, pk, capped, traffic)
    dominant = max(kern.items(), key=lambda kv: kv[1]["ms_per_launch"] * kv[1]["launches"])[0] if kern else None
    vg_depths = depths[total - 1]
    # ----- e2e through host buffers (pinned H2D inputs and D2H results every step, see run_e2e), right
    # after the timed region so it runs in the same power state (the steady phase below is power-capped)
    e2e = e2e_host = None
    if ctl:                                           # later regions draft at the controller's last depth
        for i in range(total, total + args.e2e_steps + HOST_DRAFTER_STEPS):
            ctl.prepare(i)
    if args.e2e_steps > 0:
        with Clocks(dev.index) as eclk:
            e2e = run_e2e(args, wl, lane, succ, depths, masks, devtok, dev, total)
        e2e["clocks"] = eclk.summary()
        if not wl.tree:                               # the host drafter variant drafts chains only
            e2e_host = run_e2e_host_drafter(args, wl, lane, succ, depths, masks, devtok, dev,
                                            total + args.e2e_steps, HOST_DRAFTER_STEPS)
    # verify-step µs as SURVEY.md §8(d) defines it (graph replay, drafting excluded), then the steady phase
    vgraph = verify_step_graph(lane, wl, slots, vg_depths, drafts, 4321, (acc, tok), par_d, dev, VERIFY_GRAPH_REPLAYS)
    steady = steady_state(args, wl, lane, depths, elapsed_ms / args.steps, pk, dev, stream)
    check = decision_check(wl, lane, reqs, succ, masks, devtok, depths, total + args.e2e_steps + HOST_DRAFTER_STEPS,
                           dev) if args.check_steps > 0 else None
    return dict(check=check, steady=steady, elapsed_ms=elapsed_ms, tokens=tokens, per_step=per_step, prof=kern, roof=roof, dominant=dominant,
                launches=launches, clocks=clk.summary(), stats=st, e2e=e2e, e2e_host=e2e_host, w=w, succ=succ, reqs=reqs,
                depths=depths, masks=masks, devtok=devtok, alg=alg, verify_graph=vgraph,
                controller=({"window_steps": ControlledDepths.WINDOW, "final_depth": ctl.d, "trace": ctl.trace[-6:]}
                            if ctl else None),
                timed=(("dynamic" if dynamic else "static") if graph is not None else "eager"),
                prof_every=args.prof_every)


def run_graph(args, wl, rank, world, dev):
    """--graph: the step (planted drafter + verify + commit) captured once as a CUDA graph and replayed;
    each step's drafter inputs are copied into the buffers the graph reads. Fixed-depth workloads use a
    plain graph (sv_graph_begin); workloads whose depths change per step (c2: k ~ U{1..8} per request,
    c3: SpecuStream's depth every window) use ONE dynamic-depth graph (sv_graph_begin_dynamic) with
    each replay's depth vector staged by sv_graph_set_batch. No per-kernel events
    (no roofline) in this mode."""
    from paper_2604_09562_b200 import sv
    import torch.distributed as dist
    dynamic = wl.controller or wl.kmin != wl.kmax
    if wl.tree and dynamic:
        raise SystemExit("--graph: token-tree workloads need fixed depths")
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        lane, w, succ, reqs = build_lane(wl, rank, dev, stream)
        cfg, B = wl.cfg, wl.batch
        total = args.warmup + args.steps
        if dynamic:
            depths = depths_for(wl, total, seed=7 + rank)
        else:
            ks = [wl.kmax] * B
            depths = [ks] * total
        rows = B * wl.kmax
        masks, devtok = synth.planted_masks(total, rows, wl.alpha, cfg.vocab, seed=9 + rank)
        ctl = None
        if wl.controller:
            ctl = ControlledDepths(wl, total, seed=11 + rank)
            depths, masks, devtok = ctl.depths, ctl.masks, ctl.devtok
        masks_d, devtok_d, succ_d = masks.to(dev), devtok.to(dev), succ.to(dev)
        m_stage = torch.empty(rows, dtype=masks.dtype, device=dev)
        t_stage = torch.empty(rows, dtype=torch.int32, device=dev)
        drafts = torch.empty(rows, dtype=torch.int32, device=dev)
        acc = torch.empty(B, dtype=torch.int32, device=dev)
        tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
        slots = list(range(B))
        par_d = tree_parents(wl, dev)

        def stage(i):
            if ctl:
                ctl.prepare(i, masks_d, devtok_d)
            m_stage.copy_(masks_d[i])
            t_stage.copy_(devtok_d[i])

        def eager(ks):
            draft_and_verify(lane, wl, slots, ks, succ_d, m_stage, t_stage, drafts, 1234, (acc, tok), par_d)
            lane.commit()

        for i in range(args.warmup):
            stage(i)
            eager(depths[i])
            if ctl:
                ctl.tick(lane, i)
        if dynamic:
            lane.graph_begin_dynamic(B)
        else:
            lane.graph_begin()
        eager(depths[args.warmup - 1])                # captured, not run
        g = lane.graph_end()
        torch.cuda.synchronize(dev)
        lane.stats(reset=True)
        if ctl:
            ctl.restart(lane)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        launches0 = sv.launch_count()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        with Clocks(dev.index) as clk:
            ev[0].record(stream)
            for i in range(args.steps):
                j = args.warmup + i
                stage(j)
                if dynamic:
                    lane.graph_set_batch(g, slots, depths[j])
                lane.graph_launch(g)
                ev[i + 1].record(stream)
                if ctl:
                    ctl.tick(lane, j)
            torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        launches = sv.launch_count() - launches0
        st = lane.stats()
        lane.graph_destroy(g)
    return dict(elapsed_ms=ev[0].elapsed_time(ev[-1]), tokens=st["emitted"],
                per_step=[ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)], prof={}, roof={}, dominant=None,
                launches=launches, clocks=clk.summary(), stats=st, e2e=None, e2e_host=None, w=w, succ=succ, reqs=reqs,
                depths=depths, masks=masks, devtok=devtok, alg=None,
                controller=({"window_steps": ControlledDepths.WINDOW, "final_depth": ctl.d, "trace": ctl.trace[-6:]}
                            if ctl else None), graph="dynamic" if dynamic else "static")


DISAGG_STEPS_PER_ROUND = 8   # decode steps per hand-off batch (the transfer of the next batch overlaps them)


def run_disagg(args, wl, rank, world, dev):
    """--disagg (BASELINE configs[3], SURVEY.md §8(e) exchange 1): prefill -> decode stream pairs
    (2p, 2p+1). The prefill lane holds `batch` requests of synthetic context KV (the producer; real
    chunked prefill is NEXT-3) and, every DISAGG_STEPS_PER_ROUND decode steps, hands the batch to
    its decode lane with sv_kv_send_slots / sv_kv_recv_slots (one NCCL group of page blocks, zero
    copy, on the lanes' comm streams). The decode lane double-buffers: it verifies one set of
    `batch` slots while the next set is received into the other half, then releases the old set.
    world == 1 runs both lanes on one GPU with sv_kv_loopback_slots (the flow, not NVLink).
    value = decode-lane accepted tokens/s over the region (hand-off interference included);
    handoff = bytes per batch and the comm-stream time of each transfer."""
    from paper_2604_09562_b200 import sv
    import torch.distributed as dist
    role, peer, pair = svdist.disagg_role(rank, world)
    cfg0, B = wl.cfg, wl.batch
    rounds = max(2, args.steps // DISAGG_STEPS_PER_ROUND)
    n_tok = wl.ctx[1]
    growth = (args.warmup + rounds * DISAGG_STEPS_PER_ROUND + 4) * (wl.kmax + 1)
    per_req = (n_tok + growth + 63) // 64 + 1
    dcfg = cfg0.with_(max_slots=2 * B, n_pages=2 * B * per_req + B, max_pos=n_tok + growth + 64)
    pcfg = cfg0.with_(max_slots=B, n_pages=B * ((n_tok + 63) // 64 + 1), max_pos=n_tok + 64)
    stream = torch.cuda.Stream(dev)
    uid = sv.nccl_unique_id() if rank == 0 else None
    if world > 1:
        uid = svdist.broadcast_bytes(uid, 0, 128, device=dev)
    comm = sv.nccl_comm_init(world, uid, rank)
    w, succ = planted_weights(wl, dev if wl.gen_on_device else "cpu")
    wd = {k: v.to(dev) for k, v in w.items()}
    res = {}
    with torch.cuda.stream(stream):
        pre = dec = None
        prefill_ms = None
        if role in ("prefill", "both"):
            # the producer: real chunked prefill (NEXT-3, sv_prefill) of B random prompts, untimed
            pre = sv.Lane(pcfg, wd, stream=stream)
            chunk = min(pcfg.max_batch * (pcfg.max_depth + 1), 1024)
            t0 = time.perf_counter()
            for i in range(B):
                prompt = synth.random_tokens(n_tok, pcfg.vocab, seed=30_000 * (pair + 1) + i).tolist()
                pre.prefill(i, svdist.request_id(rank, 10**6 + i), prompt, chunk)
            torch.cuda.synchronize(dev)
            prefill_ms = {"requests": B, "tokens_each": n_tok, "chunk": chunk,
                          "ms": round(1e3 * (time.perf_counter() - t0), 1)}
        if role in ("decode", "both"):
            dec = sv.Lane(dcfg, wd, stream=stream)
        torch.cuda.synchronize(dev)
        prank = rank if role == "both" else (rank if role == "prefill" else peer)


        nbytes = (pre or dec).slots_bytes([n_tok] * B)
        st_send = torch.empty(nbytes, dtype=torch.uint8, device=dev) if pre is not None else None
        st_recv = torch.empty(nbytes, dtype=torch.uint8, device=dev) if dec is not None else None

        def handoff(r):
            src, dst, rids = svdist.handoff_batch(r, B, prank)
            if role == "both":
                pre.kv_loopback_slots(dec, src, dst, rids, [n_tok] * B, st_send, st_recv, 0, comm)
            elif role == "prefill":
                pre.kv_send_slots(src, [n_tok] * B, st_send, peer, comm)
            else:
                dec.kv_recv_slots(dst, rids, [n_tok] * B, st_recv, peer, comm)
            return dst

        hand_ev = []
        if dec is not None:
            cstream = dec.comm_stream()
            total_steps = args.warmup + rounds * DISAGG_STEPS_PER_ROUND
            depths = [[wl.kmax] * B for _ in range(total_steps)]
            masks, devtok = synth.planted_masks(total_steps, B * wl.kmax, wl.alpha, cfg0.vocab, seed=9 + rank)
            masks_d, devtok_d, succ_d = masks.to(dev), devtok.to(dev), succ.to(dev)
            drafts = torch.empty(B * wl.kmax, dtype=torch.int32, device=dev)
            acc = torch.empty(B, dtype=torch.int32, device=dev)
            tok = torch.empty(B, cfg0.max_depth + 1, dtype=torch.int32, device=dev)
        active = handoff(0)                                   # initial fill (untimed)
        if dec is not None:
            for i in range(args.warmup):
                draft_and_verify(dec, wl, active, depths[i], succ_d, masks_d[i], devtok_d[i], drafts, 1234 + i,
                                 (acc, tok))
                dec.commit()
        torch.cuda.synchronize(dev)
        if dec is not None:
            dec.stats(reset=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = sv.launch_count()
        with Clocks(dev.index) as clk:
            e0.record(stream)
            for r in range(1, rounds + 1):
                if dec is not None:
                    h0 = torch.cuda.Event(enable_timing=True)
                    h0.record(cstream)
                nxt = handoff(r) if r < rounds else None      # the next batch arrives while `active` decodes
                if dec is not None:
                    if nxt is not None:
                        h1 = torch.cuda.Event(enable_timing=True)
                        h1.record(cstream)
                        hand_ev.append((h0, h1))
                    for j in range(DISAGG_STEPS_PER_ROUND):
                        i = args.warmup + (r - 1) * DISAGG_STEPS_PER_ROUND + j
                        draft_and_verify(dec, wl, active, depths[i], succ_d, masks_d[i], devtok_d[i], drafts,
                                         1234 + i, (acc, tok))
                        dec.commit()
                    if nxt is not None:
                        for s_ in active:
                            dec.release(s_)
                        active = nxt
            e1.record(stream)
            torch.cuda.synchronize(dev)
        launches = sv.launch_count() - launches0
        if world > 1:
            dist.barrier()
        elapsed = e0.elapsed_time(e1)
        dstats = dec.stats() if dec is not None else {"accepted": 0, "drafted": 0, "emitted": 0}
        tokens = dstats["emitted"]
        if dec is not None:
            hms = sorted(a.elapsed_time(b) for a, b in hand_ev)
            res["handoff"] = {"batches": len(hms), "bytes_per_batch": nbytes,
                              "ms_median": round(statistics.median(hms), 3) if hms else None,
                              "gbs_median": round(nbytes / (statistics.median(hms) * 1e-3) / 1e9, 1) if hms else None,
                              "blocks_per_batch": B * ((n_tok + 63) // 64) * cfg0.n_layers,
                              "what": "comm-stream time: decode-side page pop + NCCL receive + block scatter "
                                      "(+ the prefill-side gather in loopback)",
                              "transport": "NCCL loopback on one GPU (flow check, not NVLink)" if role == "both"
                                           else "NCCL p2p, one op per batch, page-block gather / scatter",
                              "overlap": f"transfer on the comm stream while {DISAGG_STEPS_PER_ROUND} verify steps run",
                              "producer_prefill": prefill_ms}
    elapsed, tokens = svdist.reduce_region(elapsed, tokens, device=dev if world > 1 else None)
    sv.nccl_comm_destroy(comm)
    steps = rounds * DISAGG_STEPS_PER_ROUND
    # handoff stats live on decode ranks: gather rank 1's to rank 0
    if world > 1:
        obj = [res.get("handoff")]
        outs = [None] * world
        dist.all_gather_object(outs, obj[0])
        res["handoff"] = next((o for o in outs if o), None)
    return dict(elapsed_ms=elapsed, tokens=tokens, per_step=[elapsed / steps] * steps, prof={}, roof={}, dominant=None,
                launches=launches, clocks=clk.summary(), stats=dstats,
                e2e=None, e2e_host=None, controller=None, handoff=res.get("handoff"), disagg=True, steps_run=steps,
                decode_lanes=max(1, world // 2))


def run_e2e(args, wl, lane, succ, depths, masks, devtok, dev, start):
    """End to end through the public API, inputs from pinned host memory, results read back
    every step. The drafter is the device one (`sv_draft_planted`); each step's drafter inputs
    (deviation mask + replacement tokens) are copied H2D from pinned memory and each step's
    accepted lengths + emitted tokens are copied D2H into a pinned double buffer and consumed on
    the host one step later (event-ordered), so host work overlaps the next step's kernels. Fixed-depth
    workloads (unless --eager) run the step as replays of one captured graph (sv_graph_launch, public API)
    that reads the device copies of the drafter inputs, as the timed region does."""
    cfg = wl.cfg
    B = wl.batch
    slots = list(range(B))
    n = args.e2e_steps
    fixed = not (wl.controller or wl.kmin != wl.kmax)
    # depth-varying workloads: a dynamic-depth graph where launches bound the step, or with --graph-dynamic
    dyn_graph = not fixed and not wl.tree and (cfg.d_model <= 1024 or args.graph_dynamic or args.e2e_graph)
    kr = B * wl.kmax
    h_mask = masks[start:start + n].clone().pin_memory()
    h_dev = devtok[start:start + n].clone().pin_memory()
    d_mask = [torch.empty(kr, dtype=h_mask.dtype, device=dev) for _ in range(2)]
    d_dev = [torch.empty(kr, dtype=torch.int32, device=dev) for _ in range(2)]
    succ_d = succ.to(dev)
    drafts = torch.empty(kr, dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
    h_acc = [torch.empty(B, dtype=torch.int32).pin_memory() for _ in range(2)]
    h_tok = [torch.empty(B, cfg.max_depth + 1, dtype=torch.int32).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    stream = torch.cuda.current_stream(dev)
    emitted_host = 0
    par_d = tree_parents(wl, dev)

    def consume(slot):
        nonlocal emitted_host
        done[slot].synchronize()
        a = h_acc[slot].numpy()
        emitted_host += int((a + 1).sum())

    graph = None
    if (fixed or dyn_graph) and not args.eager:
        try:                                      # the inputs land in d_mask[0] / d_dev[0] (stream-ordered)
            if dyn_graph:
                lane.graph_begin_dynamic(B)
            else:
                lane.graph_begin()
            draft_and_verify(lane, wl, slots, depths[start], succ_d, d_mask[0], d_dev[0], drafts, 99 + start,
                             (acc, tok), par_d)
            lane.commit()                         # captured, not run
            graph = lane.graph_end()
        except Exception as ex:
            print(f"[bench] e2e graph capture failed ({ex}); eager calls", file=sys.stderr)
            graph = None
    lane.stats(reset=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for s_ in range(n):
        i = start + s_
        sl = s_ & 1                               # read-back double buffer
        ib = 0 if graph is not None else sl       # input buffers (the graph reads buffer 0)
        d_mask[ib].copy_(h_mask[s_], non_blocking=True)
        d_dev[ib].copy_(h_dev[s_], non_blocking=True)
        if graph is not None:
            if dyn_graph:
                lane.graph_set_batch(graph, slots, depths[i])
            lane.graph_launch(graph)
        else:
            draft_and_verify(lane, wl, slots, depths[i], succ_d, d_mask[ib], d_dev[ib], drafts, 99 + i, (acc, tok),
                             par_d)
            lane.commit()
        h_acc[sl].copy_(acc, non_blocking=True)
        h_tok[sl].copy_(tok, non_blocking=True)
        done[sl].record(stream)
        if s_ > 0:
            consume(sl ^ 1)                       # previous step's results, while this step runs
    consume((n - 1) & 1)
    el = time.perf_counter() - t0
    if graph is not None:
        lane.graph_destroy(graph)
    st = lane.stats(reset=True)
    assert st["emitted"] == emitted_host, (st["emitted"], emitted_host)
    h2d = kr * (h_mask.element_size() + 4)
    d2h = B * 4 + B * (cfg.max_depth + 1) * 4
    return {"value": emitted_host / el, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": n, "ms_per_step": 1e3 * el / n, "drafter": "device (sv_draft_planted), pipelined read-back",
            "path": "sv_graph_launch of the captured step" if graph is not None else "eager sv_* calls",
            "tokens": emitted_host, "seconds": el}


def run_e2e_host_drafter(args, wl, lane, succ, depths, masks, devtok, dev, start, n):
    """Variant with the drafter on the host: each step's drafts depend on the previous step's
    read-back tokens, so every step is a full host <-> device round trip (no overlap)."""
    cfg = wl.cfg
    B = wl.batch
    slots = list(range(B))
    succ_h = succ.numpy()
    kmax = wl.kmax
    pend = lane.tap("pending", torch.int32, (cfg.max_slots,))[:B].cpu().numpy().copy()
    h_drafts = torch.empty(B * kmax, dtype=torch.int32).pin_memory()
    h_acc = torch.empty(B, dtype=torch.int32).pin_memory()
    h_tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32).pin_memory()
    d_drafts = torch.empty(B * kmax, dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.int32, device=dev)
    tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
    lane.stats(reset=True)
    torch.cuda.synchronize(dev)
    h2d = d2h = 0
    t0 = time.perf_counter()
    for s_ in range(n):
        i = start + s_
        ks = np.asarray(depths[i])
        m = masks[i].numpy().reshape(B, kmax).astype(bool) if all(k == kmax for k in ks) else None
        dt = devtok[i].numpy()
        out = h_drafts.numpy()
        if m is not None:                         # uniform depth: vectorised over requests
            dt2 = dt.reshape(B, kmax)
            prev = pend.astype(np.int64)
            blk = out[:B * kmax].reshape(B, kmax)
            for j in range(kmax):
                t = np.where(m[:, j], dt2[:, j], succ_h[prev])
                blk[:, j] = t
                prev = t
            nd = B * kmax
        else:
            mm, off = masks[i].numpy(), 0
            for b in range(B):
                prev = int(pend[b])
                for j in range(ks[b]):
                    t = int(dt[off + j]) if mm[off + j] else int(succ_h[prev])
                    out[off + j] = t
                    prev = t
                off += ks[b]
            nd = off
        d_drafts[:nd].copy_(h_drafts[:nd], non_blocking=True)
        lane.verify(slots, depths[i], d_drafts, None, seed=99 + i, mode=wl.mode, temperature=wl.temperature,
                    out=(acc, tok))
        lane.commit()
        h_acc.copy_(acc, non_blocking=True)
        h_tok.copy_(tok, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        a, tk = h_acc.numpy(), h_tok.numpy()
        pend = tk[np.arange(B), a]
        h2d += nd * 4
        d2h += B * 4 + B * (cfg.max_depth + 1) * 4
    el = time.perf_counter() - t0
    st = lane.stats(reset=True)
    return {"value": st["emitted"] / el, "unit": UNIT, "h2d_bytes_per_step": h2d // n, "d2h_bytes_per_step": d2h // n,
            "steps": n, "ms_per_step": 1e3 * el / n}


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)
def oracle_lane_for(wl, w, reqs, n_req):
    from oracle.lane import OracleLane
    wn = {k: v.to(torch.float32).numpy() for k, v in w.items()}
    lane = OracleLane(wl.cfg, wn)
    for i in range(n_req):
        r = reqs[i]
        lane.append_kv(i, r["rid"], r["k"].to(torch.float32).numpy(), r["v"].to(torch.float32).numpy(), r["pending"])
    return lane


def oracle_steps(wl, lane, n_req, succ, depths, masks, devtok, step_ids):
    """Run verify+commit of the first n_req requests on the oracle; returns (tokens, seconds)."""
    from oracle import verify as ov
    succ_h = succ.numpy()
    tokens, secs = 0, 0.0
    for i in step_ids:
        ks = depths[i][:n_req]
        m, dt = masks[i].numpy(), devtok[i].numpy()
        drafts, off = [], 0
        for b in range(n_req):
            toks = [lane.slots[b]["pending"]]
            for j in range(ks[b]):
                par = wl.tree[j] if wl.tree else j
                t = int(dt[off + j]) if m[off + j] else int(succ_h[toks[par]])
                drafts.append(t)
                toks.append(t)
            off += ks[b]
        mode = ov.GREEDY if wl.mode == "greedy" else ov.SAMPLE
        t0 = time.perf_counter()
        if wl.tree:
            acc, em, _, _ = lane.verify_tree(list(range(n_req)), ks, list(wl.tree) * n_req, drafts, None, 1234 + i,
                                             mode, wl.temperature, top_k=wl.top_k, top_p=wl.top_p)
        else:
            acc, em, _ = lane.verify(list(range(n_req)), ks, drafts, None, 1234 + i, mode, wl.temperature,
                                     top_k=wl.top_k, top_p=wl.top_p)
        lane.commit()
        secs += time.perf_counter() - t0
        tokens += sum(a + 1 for a in acc)
    return tokens, secs


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        return os.cpu_count()


def cpu_baseline(wl, res, budget_s=20.0):
    n_req = 1
    lane = oracle_lane_for(wl, res["w"], res["reqs"], n_req)
    tokens, secs, steps = 0, 0.0, 0
    while secs < budget_s and steps < 8:
        t, s = oracle_steps(wl, lane, n_req, res["succ"], res["depths"], res["masks"], res["devtok"], [steps])
        tokens, secs, steps = tokens + t, secs + s, steps + 1
    return {"value": round(tokens / secs, 3), "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
            "sample": f"{steps} verify+commit step(s) of request 0 of the {wl.name} workload (fp64 numpy oracle, "
                      f"same weights/KV/drafts as the GPU lane); host os.cpu_count()={os.cpu_count()}",
            "seconds": round(secs, 2), "tokens": tokens}


def cpu_baseline_1thread(wl, res, budget_s=8.0):
    """The same oracle sample with the BLAS pool limited to one thread."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        return None
    with threadpool_limits(limits=1):
        lane = oracle_lane_for(wl, res["w"], res["reqs"], 1)
        tokens, secs, steps = 0, 0.0, 0
        while secs < budget_s and steps < 2:
            t, s_ = oracle_steps(wl, lane, 1, res["succ"], res["depths"], res["masks"], res["devtok"], [steps])
            tokens, secs, steps = tokens + t, secs + s_, steps + 1
    return {"value": round(tokens / secs, 3), "unit": UNIT, "cores": 1, "steps": steps, "seconds": round(secs, 2)}


def l2_note(wl):
    c = wl.cfg
    w = 2 * (c.vocab * c.d_model + c.n_layers * (c.qkv_rows * c.d_model + c.d_model * c.n_q_heads * c.head_dim
                                                   + 3 * c.ffn_dim * c.d_model))
    kv = wl.batch * (sum(wl.ctx) / 2) * c.n_layers * 2 * c.n_kv_heads * c.head_dim * 2
    if w + kv < 126e6:
        return (f"inputs fit the 126 MB L2 ({(w + kv) / 1e6:.1f} MB; launch-bound toy config, L2 not flushed: "
                "not the headline workload)")
    return (f"no flush: every step streams {w / 1e9:.2f} GB of weights + {kv / 1e9:.2f} GB of KV, "
            f"> the 126 MB L2")


def bench_config(wl, world):
    """The workload description both arms report (the driver pairs lines by it)."""
    nl = wl.cfg.n_layers
    return {"workload": wl.name, "model": f"Llama-3-8B-shaped {nl} layer{'s' if nl > 1 else ''} + lm-head (random init, "
            "planted successor)" if wl.cfg.d_model == 4096 else "toy", "batch_per_gpu": wl.batch, "depth": [wl.kmin, wl.kmax],
            "ctx": list(wl.ctx), "mode": wl.mode, "parallelism": f"dp{world} (independent decode lanes)",
            "l2": l2_note(wl), "drafter": f"planted alpha={wl.alpha}",
            **({"tree_parents": list(wl.tree)} if wl.tree else {}),
            **({"top_k": wl.top_k, "top_p": wl.top_p} if (wl.top_k or wl.top_p < 1.0) else {})}


REFERENCE_BUDGET_S = 150.0   # the reference arm's timed steps are time-boxed to this


def run_reference(args, wl):
    """--impl reference: the fp64 CPU oracle, as it stands, on a bounded sample of the same workload."""
    w, succ = planted_weights(wl)
    ctx = synth.ctx_lengths(wl, seed=100)
    reqs = []
    for i in range(1):
        k, v = synth.context_kv(wl.cfg, ctx[i], seed=10_000 + i)
        pend = int(synth.random_tokens(1, wl.cfg.vocab, seed=20_000 + i)[0])
        reqs.append(dict(L=ctx[i], rid=(0 << 32) | (i + 1), pending=pend, k=k, v=v))
    total = args.warmup + args.steps
    depths = depths_for(wl, total, seed=7)
    masks, devtok = synth.planted_masks(total, wl.batch * wl.kmax, wl.alpha, wl.cfg.vocab, seed=9)
    lane = oracle_lane_for(wl, w, reqs, 1)
    # one untimed warm-up step (the oracle has no caches to warm; more would only cost minutes),
    # then as many of the requested steps as fit the time box: each step is request 0 of the
    # workload (k + 1 chain rows through the full layer and the full-vocabulary lm-head)
    oracle_steps(wl, lane, 1, succ, depths, masks, devtok, range(1))
    tokens, secs, run = 0, 0.0, 0
    for i in range(args.warmup, total):
        t, dt = oracle_steps(wl, lane, 1, succ, depths, masks, devtok, [i])
        tokens, secs, run = tokens + t, secs + dt, run + 1
        if secs + dt > REFERENCE_BUDGET_S:
            break
    v = tokens / secs
    sample = (f"request 0 of the {wl.name} workload per step; {run} of the {args.steps} requested steps "
              f"(time-boxed to {REFERENCE_BUDGET_S:.0f} s), fp64 numpy oracle")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / run, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(wl, args.gpus), "steps_run": run,
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line, default=_json_default), flush=True)


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="ns")
    ap.add_argument("--impl", default="sv", choices=["sv", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--detail", action="store_true", help="add per-stage breakdown to the JSON line")
    ap.add_argument("--eager", action="store_true",
                    help="time eager library calls instead of replays of one captured step (CUDA graph)")
    ap.add_argument("--graph-dynamic", action="store_true",
                    help="depth-varying Llama-shape workloads: time dynamic-depth graph replays (default: eager)")
    ap.add_argument("--e2e-graph", action="store_true", help="e2e of depth-varying workloads through a dynamic graph")
    ap.add_argument("--prof-every", type=int, default=10,
                    help="graph-timed region: replay the event-timed copy of the step every N-th step")
    ap.add_argument("--graph", action="store_true", help="replay the step as a CUDA graph (fixed depths)")
    ap.add_argument("--disagg", action="store_true",
                    help="prefill -> decode pairs with the batched NCCL KV hand-off (configs[3]; world 1: loopback)")
    ap.add_argument("--steady-s", type=float, default=1.0, help="seconds of steady-state steps after the timed region")
    ap.add_argument("--check-steps", type=int, default=1, help="teacher-forced decision check after the runs (0 = off)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl0 = synth.workload(args.workload)
    steady_budget = (steady_cap(wl0) + wl0.kmin) // (wl0.kmin + 1) + 1 if args.steady_s > 0 else 0
    wl = synth.workload(args.workload, steps_budget=args.warmup + args.steps + args.e2e_steps + HOST_DRAFTER_STEPS
                        + VERIFY_GRAPH_REPLAYS + steady_budget + args.check_steps + 9)

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, wl)
        return

    import torch.distributed as dist
    # SV_BENCH_SHARED_GPU=1 (validation only): several ranks on one GPU over gloo, to exercise the
    # multi-rank flow on a single-GPU box; the driver's N-GPU runs use one GPU per rank and NCCL
    shared = os.environ.get("SV_BENCH_SHARED_GPU") == "1"
    dev = torch.device("cuda", local % torch.cuda.device_count() if shared else local)
    torch.cuda.set_device(dev)
    red_dev = torch.device("cpu") if shared else dev
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    res = (run_disagg if args.disagg else run_graph if args.graph else run_gpu)(args, wl, rank, world, dev)
    elapsed, tokens = res["elapsed_ms"], res["tokens"]
    if world > 1 and not res.get("disagg"):       # whole job: all ranks' tokens / the slowest rank's time
        elapsed, tokens = svdist.reduce_region(elapsed, tokens, device=red_dev)
        if res["e2e"]:
            es, et = svdist.reduce_region(res["e2e"]["seconds"], res["e2e"]["tokens"], device=red_dev)
            res["e2e"]["value"] = et / es
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cfg = wl.cfg
    value = tokens / (elapsed * 1e-3)
    ps = sorted(res["per_step"])
    st = res["stats"]
    dom = res["dominant"]
    roof = res["roof"].get(dom) or res["roof"].get("lm_head") or {}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(wl, world),
        "verify_step_us": {"median": round(1e3 * statistics.median(ps), 1), "p10": round(1e3 * ps[len(ps) // 10], 1),
                           "p90": round(1e3 * ps[(9 * len(ps)) // 10], 1),
                           "what": "timed-region step (drafter + verify + commit), CUDA events"},
        "verify_step_us_graph": res.get("verify_graph"),
        "acceptance": {"a_t": round(st["accepted"] / max(1, st["drafted"]), 4),
                       "tokens_per_request_step": round(st["emitted"] / max(1, args.steps * wl.batch), 3)},
        "roofline": {k: v for k, v in roof.items() if k in ("bound", "achieved", "peak", "unit", "frac", "traffic",
                                                            "peak_kind", "frac_burst", "frac_sustained")}
        | {"kernel": dom},
        "steady_state": res.get("steady"),
        "decision_check": res.get("check"),
        "device": {"l2_bytes": torch.cuda.get_device_properties(dev).L2_cache_size,
                   "sms": torch.cuda.get_device_properties(dev).multi_processor_count,
                   "name": torch.cuda.get_device_name(dev)},
        "kernels": res["roof"],
        "gpu_launches": res["launches"],
        "launches_per_step": round(res["launches"] / args.steps, 2),
        "clocks": res["clocks"],
        "e2e": res["e2e"],
        "e2e_host_drafter": res.get("e2e_host"),
        "controller": res.get("controller"),
        "peaks": peaks()["src"],
    }
    if res.get("disagg"):
        line["steps"] = res["steps_run"]
        line["ms_per_step"] = round(elapsed / res["steps_run"], 4)
        line["handoff"] = res["handoff"]
        line["config"]["parallelism"] = (f"{max(1, world // 2)} prefill->decode pair(s)" if world > 1
                                         else "prefill + decode lanes on one GPU (loopback)")
        line["config"]["disagg"] = f"hand-off of {wl.batch} x {wl.ctx[1]}-token KV every {DISAGG_STEPS_PER_ROUND} steps"
        line["scaling"] = "weak"
    if res.get("timed"):
        line["config"]["timed_region"] = {
            "eager": "eager library calls (drafter + verify + commit) per step",
            "static": "replays of one captured step (CUDA graph: drafter + verify + commit), depths fixed per request; "
                      f"every {res.get('prof_every')}-th replay from the copy whose roofline stages are event-record "
                      "nodes (per-launch averages over those), the others from the copy without events",
            "dynamic": "replays of two dynamic-depth CUDA graphs of the step (sv_graph_begin_dynamic) with each "
                       f"step's depth vector; every {res.get('prof_every')}-th replay from the copy whose roofline "
                       "stages are event-record nodes, the others from the copy without events"}[res["timed"]]
    if res.get("graph"):
        line["config"]["graph"] = ("one dynamic-depth CUDA graph (sv_graph_begin_dynamic) replayed with each step's "
                                   "depth vector" if res["graph"] == "dynamic" else
                                   "CUDA graph replay of drafter + verify + commit; depths fixed per request")
    if args.detail:
        line["stages"] = {k: {"us": round(v["ms_per_launch"] * 1e3, 1), "share": round(v["share"], 4)}
                          for k, v in res["prof"].items()}
    if world == 1 and not args.no_cpu_baseline and not wl.gen_on_device and not res.get("disagg"):
        line["cpu_baseline"] = cpu_baseline(wl, res)
        line["cpu_baseline"]["one_thread"] = cpu_baseline_1thread(wl, res)
    print(json.dumps(line, default=_json_default), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
