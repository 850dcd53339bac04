"""N-width sweep of the weight-major GEMM (variants 5 / 6 = real / MMA only) on the lm-head shape."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

cfg = synth.TOY.with_(max_batch=64, max_slots=8, n_pages=16)
w = synth.model_weights(cfg, seed=0)
lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
M, N, K = 576, 128256, 4096
if len(sys.argv) > 1:
    M, N, K = map(int, sys.argv[1:4])
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
c = torch.empty(M, N, device="cuda")
res = []
for var in (5, 6, 9):
    lane.debug_gemm(a, b, c, var)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lane.debug_gemm(a, b, c, var)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    res.append(f"v{var} {us:7.1f} us {2 * M * N * K / us / 1e6:6.0f} TF")
print(f"NT={os.environ.get('SV_SW_NT', 'auto')}: " + "  ".join(res), flush=True)
