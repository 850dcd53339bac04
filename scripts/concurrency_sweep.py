"""Config 5 (BASELINE configs[4], NEXT-2): closed-loop concurrency sweep of the 320-query mixed
ALPACA / GSM8K / HUMANEVAL / SUM trace (synth.mixed_trace) over decode lanes (one per rank), with
the 500 ms metrics cadence feeding SpecuStream (depth) and FlowGuard (routing), per-request latency /
TPOT / throughput (PAPER.md eq:latency_computation .. eq:throughput_computation) and nearest-rank
percentiles. One JSON report line per concurrency level (and the whole list with --out).

    python scripts/concurrency_sweep.py [--levels 1,2,4,...,512] [--requests 320] [--out file.json]
    torchrun --nproc-per-node N scripts/concurrency_sweep.py ...     # N colocated lanes, FlowGuard-routed

Model: Llama-3-8B-shaped 1 layer + lm-head, planted-successor weights (acceptance per dataset profile),
each lane prefills its own requests (long-chunk sv_prefill) and decodes them in sampled mode."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_09562_b200 import engine, sv  # noqa: E402
from paper_2604_09562_b200 import specustream as sps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", default="1,2,4,8,16,32,64,128,256,512")
    ap.add_argument("--requests", type=int, default=320)
    ap.add_argument("--max-batch", type=int, default=256)
    ap.add_argument("--max-seconds", type=float, default=120.0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
    trace = synth.mixed_trace(n_per_dataset=max(1, args.requests // 4))[: args.requests]
    max_prompt = max(q["prompt_len"] for q in trace)
    max_out = max(q["out_len"] for q in trace)
    B = args.max_batch
    per_req_pages = (max_prompt + max_out + 16) // 64 + 2
    cfg = synth.LLAMA.with_(max_slots=B, max_batch=B, max_depth=8, n_pages=B * per_req_pages // 2 + 4 * per_req_pages,
                            max_pos=max_prompt + max_out + 64)
    wl = synth.workload("c2")
    w, succ = synth.planted_successor(cfg, synth.model_weights(cfg, seed=0, embed_std=wl.embed_std), seed=1,
                                      beta=wl.beta)
    stream = torch.cuda.Stream(dev)
    reports = []
    with torch.cuda.stream(stream):
        lane = sv.Lane(cfg, {k: v.to(dev) for k, v in w.items()}, stream=stream)
        prompt_fn = lambda r: synth.random_tokens(r.prompt_len, cfg.vocab, seed=r.prompt_seed).tolist()  # noqa: E731
        for C in [int(x) for x in args.levels.split(",")]:
            eng = engine.LaneEngine(lane, cfg, succ, 8, prompt_fn, controller=sps.Controller(), device=dev,
                                    seed=1000 * rank + C)
            loop = engine.ClosedLoop(eng, trace, C, rank=rank, world=world, device=dev)
            torch.cuda.synchronize(dev)
            run = loop.run(max_seconds=args.max_seconds)
            torch.cuda.synchronize(dev)
            res = [r.report() for r in eng.done]
            windows = [eng.trace]
            if world > 1:
                allres = [None] * world
                torch.distributed.all_gather_object(allres, (res, eng.trace, run["seconds"]))
                res = [x for a in allres for x in a[0]]
                windows = [a[1] for a in allres]
                run["seconds"] = max(a[2] for a in allres)
            rep = engine.level_report(C, res, run["seconds"], world, windows)
            rep["steps_lane0"] = run["steps"]
            rep["routed"] = run["routed"]
            rep["metrics_windows_lane0"] = len(eng.trace)
            reports.append(rep)
            if rank == 0:
                print(json.dumps(rep), flush=True)
            for s in list(eng.active):                  # a timed-out level leaves requests: release them
                lane.release(s)
            lane.stats(reset=True)
    if rank == 0 and args.out:
        json.dump({"trace": "synth.mixed_trace (80 x ALPACA/GSM8K/HUMANEVAL/SUM)", "lanes": world,
                   "levels": reports}, open(args.out, "w"), indent=1)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
