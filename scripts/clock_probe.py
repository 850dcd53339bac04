"""SM clock / throttle reasons (NVML) while one GEMM shape runs back to back for ~2 s."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import bench
import synth
from paper_2604_09562_b200 import sv

cfg = synth.TOY.with_(max_batch=64, max_slots=8, n_pages=16)
w = synth.model_weights(cfg, seed=0)
lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
M, N, K = 576, 128256, 4096
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
c = torch.empty(M, N, device="cuda")
for var in (5, 7):
    lane.debug_gemm(a, b, c, var)
    torch.cuda.synchronize()
    with bench.Clocks(0) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4000):
            lane.debug_gemm(a, b, c, var)
        e1.record()
        torch.cuda.synchronize()
    s = sorted(clk.sm)
    print(f"variant {var}: {e0.elapsed_time(e1) / 4000 * 1e3:.1f} us/launch; sm clock p10 {s[len(s) // 10]} median "
          f"{s[len(s) // 2]} p90 {s[9 * len(s) // 10]} MHz, reasons {sorted(clk.reasons)}", flush=True)
