"""One small workload for compute-sanitizer (memcheck / racecheck / synccheck): toy+mlp lane,
chain verifies in greedy and sampled mode (dense q, filtered target), a token-tree verify, commits,
an append and a release; then the Llama-shaped path (tcgen05 GEMMs, keys-on-lanes attention with
split-KV) on a 2-request batch. Run as
    compute-sanitizer --tool memcheck python scripts/sanitize_toy.py
Exits non-zero on any CUDA error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_09562_b200 import sv  # noqa: E402


def lane_with(cfg, ctx, seed):
    w = synth.model_weights(cfg, seed=seed)
    lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})
    for i, n in enumerate(ctx):
        k, v = synth.context_kv(cfg, n, seed=seed * 10 + i)
        lane.append_kv(i, 100 + i, k.cuda(), v.cuda(), 3 + i)
    return lane


def main():
    cfg = synth.TOY_MLP
    lane = lane_with(cfg, [128, 5, 700, 64], 1)
    depths = [1, 2, 3, 4]
    d = synth.random_tokens(sum(depths), cfg.vocab, seed=2).cuda()
    q = synth.draft_probs_dense(sum(depths), cfg.vocab, seed=3).cuda()
    lane.verify([0, 1, 2, 3], depths, d, mode="greedy")
    lane.commit()
    lane.verify([0, 1, 2, 3], depths, d, q, seed=5, mode="sample", temperature=0.8)
    lane.commit()
    lane.set_filter(20, 0.9)
    lane.verify([0, 1, 2, 3], depths, d, q, seed=6, mode="sample")
    lane.commit()
    lane.set_filter(0, 1.0)
    par = torch.tensor([0, 0, 1, 0, 1, 1, 0, 1, 2, 2], dtype=torch.int32).cuda()
    lane.verify_tree([0, 1, 2, 3], depths, par, d, q, seed=7, mode="sample")
    lane.commit()
    lane.release(1)
    k, v = synth.context_kv(cfg, 70, seed=9)
    lane.append_kv(1, 555, k.cuda(), v.cuda(), 1)
    lane.verify([1, 3], [2, 0], d[:2], mode="greedy")
    lane.commit()
    st = lane.stats()
    torch.cuda.synchronize()
    print("toy ok", st["steps"], "steps")
    lcfg = synth.LLAMA.with_(n_pages=96, max_slots=2, max_batch=2, max_pos=3072)
    ll = lane_with(lcfg, [2100, 300], 4)
    d = synth.random_tokens(9, lcfg.vocab, seed=5).cuda()
    ll.verify([0, 1], [8, 1], d[:9], mode="greedy")
    ll.commit()
    # sampled at Llama vocabulary: the pruned race fast path (one-hot and dense drafts, split slices)
    ll.verify([0, 1], [8, 1], d[:9], mode="sample", seed=3, temperature=0.9)
    ll.commit()
    qd = synth.draft_probs_dense(9, lcfg.vocab, seed=6).cuda()
    ll.verify([0, 1], [8, 1], d[:9], qd, mode="sample", seed=4)
    ll.commit()
    torch.cuda.synchronize()
    print("llama ok", ll.stats()["steps"], "steps")


if __name__ == "__main__":
    main()
