"""Micro-benchmark of the library's tcgen05 GEMM kernels (sv_debug_gemm) vs cuBLAS on the
verify step's shapes; also checks the result against torch (fp32 accumulation)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

cfg = synth.LLAMA.with_(n_pages=16, max_slots=8, max_batch=64, max_pos=256)
w = synth.model_weights(synth.TOY, seed=0)
lane = sv.Lane(cfg.with_(vocab=512, d_model=128, n_q_heads=2, n_kv_heads=2, head_dim=64, ffn_dim=0),
               {k: v.cuda() for k, v in w.items()})
shapes = {"lm_head": (576, 128256, 4096), "qkv": (576, 6144, 4096), "o_proj": (576, 4096, 4096),
          "gate_up": (576, 28672, 4096), "down": (576, 4096, 14336)}
for name, (M, N, K) in shapes.items():
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    c = torch.empty(M, N, device="cuda")
    ref = a.float() @ b.float().T
    res = {}
    for var, label in ((1, "1sm"), (2, "2sm"), (5, "wmaj"), (4, "mma-only"), (6, "w-mma"), (7, "w-noepi"), (8, "w-both")):
        lane.debug_gemm(a, b, c, var)
        torch.cuda.synchronize()
        err = ((c - ref).abs().max() / ref.abs().max()).item()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            lane.debug_gemm(a, b, c, var)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        res[label] = (us, 2 * M * N * K / us / 1e6, err)
    torch.matmul(a, b.T)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.matmul(a, b.T)
    e1.record()
    torch.cuda.synchronize()
    cu = e0.elapsed_time(e1) / 10 * 1e3
    print(f"{name:8s} " + "  ".join(f"{k}: {v[0]:7.1f} us {v[1]:6.0f} TF err {v[2]:.1e}" for k, v in res.items())
          + f"  cublas {cu:7.1f} us", flush=True)
