"""Print the CTA-0 timeline of the tcgen05 attention kernel (SV_TRACE=1)."""
import os, sys
os.environ["SV_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth
from paper_2604_09562_b200 import sv
nreq, L = 64, 4096
cfg = synth.LLAMA.with_(n_pages=nreq * (L // 64 + 4), max_slots=nreq, max_batch=nreq, max_pos=L + 256, ffn_dim=0)
w = synth.model_weights(cfg, seed=0)
lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
for i in range(nreq):
    k, v = synth.context_kv(cfg, L, seed=10 + i)
    lane.append_kv(i, i + 1, k.cuda(), v.cuda(), 5 + i)
d = synth.random_tokens(8 * nreq, cfg.vocab, seed=3).cuda()
for rep in range(3):
    lane.verify(list(range(nreq)), [8] * nreq, d)
    torch.cuda.synchronize()
    tr = lane.tap("trace", torch.int64, (16, 256)).cpu().numpy().astype(np.int64)
    lane.commit()
t0 = tr[tr > 0].min()
names = ["P_slot", "P_issue", "M_kvfull", "M_QK", "M_PV", "S_sfull", "S_pdone", "item", "S_ld", "S_vote",
         "S_sfree", "S_exp"]
cols = [0, 1, 2, 3, 4, 5, 8, 9, 10, 11, 6]
print("tile " + " ".join(f"{names[c]:>9s}" for c in cols))
for t in range(8, 40):
    row = [tr[e, t] - t0 if tr[e, t] > 0 else -1 for e in cols]
    print(f"{t:4d} " + " ".join(f"{x:9d}" for x in row))
print("item ends", [int(tr[7, i] - t0) for i in range(16) if tr[7, i] > 0])
