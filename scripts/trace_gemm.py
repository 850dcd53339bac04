"""Per-tile timeline (CTA 0, SM cycles) and per-cluster start / end spread of one GEMM kind of the ns
step (SV_TRACE=1, SV_TRACE_GEMM=kind: 1 QKV+RoPE, 2 residual (the last one of the step: down),
3 gate/up+SwiGLU, 4 lm-head). Usage: python scripts/trace_gemm.py KIND"""
import os
import sys

kind = sys.argv[1] if len(sys.argv) > 1 else "4"
os.environ["SV_TRACE"] = "1"
os.environ["SV_TRACE_GEMM"] = kind
sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench
import synth

wl = synth.workload("ns", steps_budget=40)
dev = torch.device("cuda:0")
lane, w, succ, reqs = bench.build_lane(wl, 0, dev)
B, cfg = wl.batch, wl.cfg
depths = bench.depths_for(wl, 8, seed=7)
masks, devtok = synth.planted_masks(8, B * wl.kmax, wl.alpha, cfg.vocab, seed=9)
drafts = torch.empty(B * wl.kmax, dtype=torch.int32, device=dev)
acc = torch.empty(B, dtype=torch.int32, device=dev)
tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
for i in range(4):
    lane.draft_planted(list(range(B)), depths[i], succ.to(dev), masks[i].to(dev), devtok[i].to(dev), drafts)
    lane.verify(list(range(B)), depths[i], drafts, None, seed=i, mode=wl.mode, out=(acc, tok))
    lane.commit()
torch.cuda.synchronize()
tr = lane.tap("trace", torch.int64, (16, 256)).cpu().numpy().astype(np.int64)
ms, me, es, ee = tr[12], tr[13], tr[14], tr[15]
n = int((ms > 0).sum())
t0 = ms[0]
print(f"kind {kind}: {n} tiles on CTA 0 (cycles from the first MMA issue)")
for i in range(n):
    print(f"tile {i:2d}: mma {ms[i] - t0:8d} .. {me[i] - t0:8d} ({me[i] - ms[i]:6d})   epi {es[i] - t0:8d} .. {ee[i] - t0:8d} "
          f"({ee[i] - es[i]:6d})")
st, en = tr[10], tr[11]
nc = int((st[:128] > 0).sum())
g0 = st[:nc].min()
dur = (en[:nc] - g0) / 1e3
print(f"{nc} clusters (global timer, us): start spread {(st[:nc].max() - g0) / 1e3:.1f}; end min {dur.min():.1f} "
      f"median {np.median(dur):.1f} max {dur.max():.1f}")
