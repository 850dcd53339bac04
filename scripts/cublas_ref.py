"""cuBLAS (torch.matmul) timing on the verify step's GEMM shapes — a library yardstick only."""
import torch
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
shapes = {"lm_head": (576, 128256, 4096), "qkv": (576, 6144, 4096), "o_proj": (576, 4096, 4096),
          "gate_up": (576, 28672, 4096), "down": (576, 4096, 14336), "lm_head_T352": (352, 128256, 4096)}
for name, (M, N, K) in shapes.items():
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        c = a @ b.T
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        c = a @ b.T
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(f"{name:14s} M={M} N={N} K={K}: {us:8.1f} us  {2*M*N*K/us/1e6:8.1f} TFLOP/s")
