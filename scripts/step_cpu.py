"""Is the verify step launch-bound?  Measures, on the bench workload: GPU time per step with the
per-stage profiling events off and on, and the host time to enqueue one step."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import bench
import synth

wl = synth.workload(os.environ.get("WL", "ns"), steps_budget=400)
dev = torch.device("cuda:0")
lane, w, succ, reqs = bench.build_lane(wl, 0, dev)
B, cfg = wl.batch, wl.cfg
n = 60
depths = bench.depths_for(wl, n * 4, seed=7)
masks, devtok = synth.planted_masks(n * 4, B * wl.kmax, wl.alpha, cfg.vocab, seed=9)
masks_d, devtok_d, succ_d = masks.to(dev), devtok.to(dev), succ.to(dev)
drafts = torch.empty(B * wl.kmax, dtype=torch.int32, device=dev)
acc = torch.empty(B, dtype=torch.int32, device=dev)
tok = torch.empty(B, cfg.max_depth + 1, dtype=torch.int32, device=dev)
slots = list(range(B))
it = [0]


def step():
    i = it[0] % (n * 4)
    it[0] += 1
    lane.draft_planted(slots, depths[i], succ_d, masks_d[i], devtok_d[i], drafts)
    lane.verify(slots, depths[i], drafts, None, seed=1234 + i, mode=wl.mode, temperature=wl.temperature,
                out=(acc, tok))
    lane.commit()


for _ in range(5):
    step()
torch.cuda.synchronize()
for prof in (False, ["lm_head", "attention"], True, False):
    lane.profile(prof)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"profile={prof}: gpu {e0.elapsed_time(e1) / n * 1e3:7.1f} us/step  host enqueue "
          f"{(t1 - t0) / n * 1e6:7.1f} us/step  wall {(t2 - t0) / n * 1e6:7.1f} us/step", flush=True)
    lane.profile_read(reset=True)
# host cost of the verify call alone while the GPU is busy
torch.cuda._sleep(int(2e9))
t0 = time.perf_counter()
for _ in range(10):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"enqueue while GPU busy: {(t1 - t0) / 10 * 1e6:.1f} us/step")
