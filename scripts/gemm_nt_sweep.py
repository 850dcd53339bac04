"""Token-tile width sweep of the weight-major 2-SM GEMM (sv_debug_gemm variant 5) on the step's
shapes (M = 576 tokens): SV_SW_NT overrides gemm_sw_choose_nt per call. CUDA-event times, inputs
resident (weights > L2 only for the large shapes)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

cfg = synth.TOY.with_(max_batch=64, max_slots=8, n_pages=16)
w = synth.model_weights(cfg, seed=0)
lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})


def t(fn, n=30):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


M = 576
for name, N, K in (("qkv", 6144, 4096), ("o", 4096, 4096), ("down", 4096, 14336), ("gate_up", 28672, 4096)):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    c = torch.empty(M, N, device="cuda")
    row = []
    os.environ.pop("SV_SW_NT", None)
    row.append(("auto", t(lambda: lane.debug_gemm(a, b, c, 5))))
    for nt in (96, 128, 144, 160, 176, 192, 224, 256):
        os.environ["SV_SW_NT"] = str(nt)
        row.append((nt, t(lambda: lane.debug_gemm(a, b, c, 5))))
    os.environ.pop("SV_SW_NT", None)
    cu = t(lambda: torch.matmul(a, b.T))
    fl = 2.0 * M * N * K
    print(name, " ".join(f"{k}:{v:.1f}" for k, v in row), f"cublas:{cu:.1f} us", f"({fl / 1e9:.1f} GFLOP)", flush=True)
