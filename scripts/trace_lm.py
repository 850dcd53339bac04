"""Per-tile timeline of the lm-head GEMM on CTA 0 (SV_TRACE=1): MMA issue span per tile and the
epilogue span per tile, in SM cycles."""
import os
import sys

os.environ["SV_TRACE"] = "1"
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
print(f"{n} tiles on CTA 0; kernel start->end per cluster below")
for i in range(n):
    print(f"tile {i:2d}: mma {ms[i] - t0:8d} .. {me[i] - t0:8d} ({me[i] - ms[i]:6d})   epi {es[i] - t0:8d} .. {ee[i] - t0:8d} "
          f"({ee[i] - es[i]:6d})")

st, en = tr[10], tr[11]
nc = 74
g0 = st[:nc].min()
dur = (en[:nc] - g0) / 1e3
print(f"{nc} clusters: start spread {(st[:nc].max() - g0) / 1e3:.1f} us; end min {dur.min():.1f} median "
      f"{np.median(dur):.1f} max {dur.max():.1f} us")
print("slowest clusters:", np.argsort(-dur)[:10].tolist(), np.sort(dur)[-10:].round(1).tolist())
print("fastest clusters:", np.argsort(dur)[:10].tolist(), np.sort(dur)[:10].round(1).tolist())
