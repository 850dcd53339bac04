"""K sweep of the 1-SM tcgen05 GEMM on the qkv shape: separates fixed per-launch cost from the
per-k-block cost (variant 4 = MMA only, operand loads skipped after the fill)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

cfg = synth.TOY.with_(max_batch=64, max_slots=8, n_pages=16)
w = synth.model_weights(cfg, seed=0)
lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for N in (6144, 256 * 148):
    for K in (64, 256, 1024, 2048, 4096):
        a = torch.randn(576, K, device="cuda").to(torch.bfloat16)
        b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        c = torch.empty(576, N, device="cuda")
        r = {v: t(lambda: lane.debug_gemm(a, b, c, v)) for v in (1, 4)}
        cu = t(lambda: torch.matmul(a, b.T))
        print(f"N {N:6d} K {K:5d}  1sm {r[1]:7.1f}  mma-only {r[4]:7.1f}  cublas {cu:7.1f} us", flush=True)
k = torch.empty(1, device="cuda")
print(f"empty torch launch {t(lambda: k.add_(1)):.1f} us")
