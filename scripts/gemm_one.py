"""One GEMM launch on a verify-step shape (for ncu): python scripts/gemm_one.py <shape> <variant>."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

shapes = {"lm_head": (576, 128256, 4096), "qkv": (576, 6144, 4096), "o_proj": (576, 4096, 4096),
          "gate_up": (576, 28672, 4096), "down": (576, 4096, 14336)}
M, N, K = shapes[sys.argv[1]]
var = int(sys.argv[2])
cfg = synth.TOY.with_(max_batch=64, max_slots=8, n_pages=16)
w = synth.model_weights(cfg, seed=0)
lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
c = torch.empty(M, N, device="cuda")
for _ in range(3):
    lane.debug_gemm(a, b, c, var)
torch.cuda.synchronize()
