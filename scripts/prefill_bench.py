"""Chunked prefill throughput (sv_prefill, NEXT-3 / R29) at Llama-3-8B shape (1 layer + lm-head):
prompt tokens per second for several chunk sizes (long chunks: k_attn_prefill.cu; a chunk is at most
the workspace's max_batch * (max_depth + 1) rows). Per-stage device time from the lane's events.
Usage: python scripts/prefill_bench.py [prompt_len]"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = synth.LLAMA.with_(n_pages=(n // 64 + 8) * 3, max_slots=3, max_batch=64, max_depth=15, max_pos=n + 128)
w = {k: v.cuda() for k, v in synth.model_weights(cfg, seed=0, embed_std=8.0).items()}
lane = sv.Lane(cfg, w)
prompt = synth.random_tokens(n, cfg.vocab, seed=1).tolist()
out = {}
for chunk in (16, 256, 512, 1024):
    lane.prefill(0, 11, prompt[:1024], chunk)            # warm-up (TMA maps, smem opt-in)
    lane.release(0)
    torch.cuda.synchronize()
    lane.profile(True)
    lane.profile_read(reset=True)
    t0 = time.perf_counter()
    y = lane.prefill(1, 12, prompt, chunk)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    prof = lane.profile_read(reset=True)
    lane.profile(False)
    lane.release(1)
    stages = {k: round(v[0], 3) for k, v in prof.items() if v[1]}
    out[chunk] = {"ms": round(dt * 1e3, 2), "tokens_per_s": round(n / dt), "next_token": y, "stage_ms": stages}
    print(f"chunk {chunk:5d}: {n} tokens in {dt * 1e3:.2f} ms = {n / dt:.0f} prompt tokens/s (next token {y}) "
          f"{json.dumps(stages)}", flush=True)
lane.close()
print(json.dumps({"prompt": n, "results": out}))
