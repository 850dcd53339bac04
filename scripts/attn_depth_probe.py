"""Attention time vs verify depth at the north-star batch (bs 64, 4096-token contexts, Llama shape):
if the softmax warps (not the KV stream) bound the kernel, time grows with the query slots
(k+1)*G per kv head. Live CUDA-event time of the attention stage over repeated verify steps."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

B, L = 64, 4096
cfg = synth.LLAMA.with_(n_pages=B * (L // 64 + 4), max_slots=B, max_batch=B, max_depth=15, max_pos=L + 512, ffn_dim=0)
w = {k: v.cuda() for k, v in synth.model_weights(cfg, seed=0).items()}
lane = sv.Lane(cfg, w)
for i in range(B):
    k, v = synth.context_kv(cfg, L, seed=10 + i)
    lane.append_kv(i, i + 1, k.cuda(), v.cuda(), 5 + i)
for depth in (0, 3, 7, 8, 11, 15):
    d = synth.random_tokens(max(1, depth * B), cfg.vocab, seed=3).cuda()
    lane.profile(["attention"])
    for rep in range(3):                                   # warm-up
        lane.verify(list(range(B)), [depth] * B, d, mode="greedy")
        lane.commit(torch.ones(B, dtype=torch.int32, device="cuda"))   # keep 1 row: contexts grow by 1
    lane.profile_read(reset=True)
    for rep in range(30):
        lane.verify(list(range(B)), [depth] * B, d, mode="greedy")
        lane.commit(torch.ones(B, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    prof = lane.profile_read(reset=True)
    ms, n = prof["attention"]
    print(f"k={depth:2d} slots/kv-head={(depth + 1) * 4:2d}: attention {1e3 * ms / n:.1f} us", flush=True)
    lane.profile(False)
