import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import synth
from oracle import verify, model
from gpu_util import Setup, f64
V = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
cfg = synth.ModelConfig(n_layers=1, d_model=64, n_q_heads=1, n_kv_heads=1, head_dim=64, vocab=V, ffn_dim=0,
                        n_pages=16, max_slots=4, max_batch=4, max_depth=4, max_pos=256)
S = Setup(cfg, [3, 0, 5, 7], seed=1)
depths = [2, 0, 1, 3]
T = sum(depths) + 4
g = torch.Generator().manual_seed(0)
logits = torch.randn(T, V, generator=g) * 2
drafts = synth.random_tokens(sum(depths), V, seed=3)
for mode in ("greedy", "sample"):
    acc, tok = S.lane.verify_logits([0, 1, 2, 3], depths, drafts.cuda(), logits.cuda(), None, seed=5, mode=mode)
    torch.cuda.synchronize()
    nt = (V + 255) // 256
    tm = S.lane.tap("tile_max", torch.float32, (T, nt)).cpu().numpy()
    ta = S.lane.tap("tile_arg", torch.int32, (T, nt)).cpu().numpy()
    mx, se, am = model.tile_stats(f64(logits))
    print(mode, "tile max eq", np.array_equal(tm, mx.astype(np.float32)), "arg eq", np.array_equal(ta, am))
    print(" gpu acc", acc.cpu().numpy(), "tok", tok.cpu().numpy().tolist())
    r0 = off = 0
    for b, k in enumerate(depths):
        r = verify.verify_request(f64(logits[r0:r0 + k + 1]), [int(t) for t in drafts[off:off + k]], None, 5,
                                  S.ctx[b]["rid"], S.ctx[b]["L"], verify.GREEDY if mode == "greedy" else verify.SAMPLE)
        print(" oracle", b, r, "argmax rows", [int(np.argmax(f64(logits[r0 + j]))) for j in range(k + 1)])
        r0 += k + 1; off += k
