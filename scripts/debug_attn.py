"""Attention TC vs SIMT on a multi-item-per-CTA shape (debug)."""
import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
import synth
from paper_2604_09562_b200 import sv
nreq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = synth.LLAMA.with_(n_pages=nreq * (L // 64 + 4), max_slots=nreq, max_batch=nreq, max_pos=L + 256, ffn_dim=0)
w = synth.model_weights(cfg, seed=0)
wd = {k: v.cuda() for k, v in w.items()}
outs = {}
for mode in ("simt", "tc"):
    os.environ["SV_ATTN"] = mode
    lane = sv.Lane(cfg, wd)
    for i in range(nreq):
        k, v = synth.context_kv(cfg, L, seed=10 + i)
        lane.append_kv(i, i + 1, k.cuda(), v.cuda(), 5 + i)
    d = synth.random_tokens(8 * nreq, cfg.vocab, seed=3).cuda()
    torch.cuda.synchronize()
    t0 = time.time()
    lane.verify(list(range(nreq)), [8] * nreq, d)
    torch.cuda.synchronize()
    print(mode, "verify s", time.time() - t0, flush=True)
    T = 9 * nreq
    outs[mode] = lane.tap("o", torch.bfloat16, (T, 4096)).float().cpu().clone()
    lane.close()
diff = (outs["simt"] - outs["tc"]).abs()
print("max abs diff", diff.max().item(), "rms o", outs["simt"].pow(2).mean().sqrt().item(), flush=True)
