"""Chunked prefill throughput (sv_prefill, NEXT-3 / R29) at Llama-3-8B shape (1 layer + lm-head):
prompt tokens per second for chunk sizes 9 and 16 (a lane's chunk limit is max_depth + 1, and
(max_depth + 1) * G <= 64 query rows per kv head). Intermediate chunks skip the lm-head. Usage: python scripts/prefill_bench.py [prompt_len]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = None
for md in (8, 15):
    cfg = synth.LLAMA.with_(n_pages=(n // 64 + 8) * 2, max_slots=2, max_batch=2, max_depth=md, max_pos=n + 128)
    if w is None:
        w = {k: v.cuda() for k, v in synth.model_weights(cfg, seed=0, embed_std=8.0).items()}
    lane = sv.Lane(cfg, w)
    prompt = synth.random_tokens(n, cfg.vocab, seed=1).tolist()
    lane.prefill(0, 11, prompt[:256], md + 1)            # warm-up
    lane.release(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    y = lane.prefill(1, 12, prompt, md + 1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"chunk {md + 1:3d}: {n} tokens in {dt * 1e3:.1f} ms = {n / dt:.0f} prompt tokens/s (next token {y})")
    lane.close()
