"""Phase timeline of the finalize kernel (SV_TRACE=1): per CTA (request, slice) the global-timer times of
its phases, us from the earliest start. Usage: python scripts/trace_finalize.py [workload]"""
import os
import sys

os.environ["SV_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench
import synth

wl = synth.workload(sys.argv[1] if len(sys.argv) > 1 else "c2", steps_budget=40)
dev = torch.device("cuda:0")
lane, w, succ, reqs = bench.build_lane(wl, 0, dev)
B, cfg = wl.batch, wl.cfg
masks, devtok = synth.planted_masks(8, B * wl.kmax, wl.alpha, cfg.vocab, seed=9)
drafts = torch.empty(B * wl.kmax, dtype=torch.int32, device=dev)
acc = torch.empty(B, dtype=torch.int32, device=dev)
tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
for i in range(4):
    ks = bench.depths_for(wl, 8, seed=7)[i]
    lane.draft_planted(list(range(B)), ks, succ.to(dev), masks[i].to(dev), devtok[i].to(dev), drafts)
    lane.verify(list(range(B)), ks, drafts, None, seed=i, mode=wl.mode, temperature=wl.temperature, out=(acc, tok))
    lane.commit()
torch.cuda.synchronize()
tr = lane.tap("trace", torch.int64, (16, 256)).cpu().numpy().astype(np.int64)[:10]
ok = tr[0] > 0
t0 = tr[0][ok].min()
ph = (tr[:, ok] - t0) / 1e3
names = ["start", "dep-wait", "row stats", "accept", "race", "merge"]
for i, n in enumerate(names):
    print(f"{n:10s} min {ph[i].min():7.2f} median {np.median(ph[i]):7.2f} max {ph[i].max():7.2f}")
d = np.diff(ph, axis=0)
for i in range(1, 6):
    print(f"{names[i - 1]}->{names[i]:10s} median {np.median(d[i - 1]):6.2f} max {d[i - 1].max():6.2f}")
sub = ["loads", "max+sync", "M", "sums+sync"]
prev = ph[1]
for i, n in enumerate(sub):
    print(f"row stats group 0: {n:10s} median {np.median(ph[6 + i] - prev):6.2f} max {(ph[6 + i] - prev).max():6.2f}")
    prev = ph[6 + i]
print("accepted", acc.cpu().numpy()[:16])
