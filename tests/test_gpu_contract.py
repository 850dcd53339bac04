"""Decision-level contract on the GPU (a6 / a7) through sv_verify_logits, against the oracle
(oracle/verify.py) on the same fp32 logits:

* the FULL lane counter struct (steps, rows, drafted, accepted, emitted, accepted_independent,
  hist_accepted, drafted_by_k, accepted_by_k) against `verify.accumulate_stats` of the oracle's
  per-request results;
* the degenerate cases of the sampler that SURVEY.md §8(c) S4/S5 (R3/R4) fix:
  q(d) = 0 -> accept, p(d) = 0 -> reject, zero residual mass -> resample from p;
* greedy argmax ties spread over several 128-wide vocab tiles -> lowest token id (S8 / R6);
* batch 128 (BASELINE configs[2]) at V = 128256, sampled, dense q."""
import numpy as np
import pytest
import torch

import synth
from oracle import verify

from gpu_util import Setup, f64
from test_gpu_parity import decisions

pytestmark = pytest.mark.gpu

V_FULL = 128256


def _lane(V, batch, depth=8, ctx_max=300, seed=11):
    cfg = synth.ModelConfig(n_layers=1, d_model=64, n_q_heads=1, n_kv_heads=1, head_dim=64, vocab=V, ffn_dim=0,
                            n_pages=8 * batch, max_slots=batch, max_batch=batch, max_depth=depth, max_pos=512)
    S = Setup(cfg, [int(x) for x in np.random.default_rng(seed).integers(0, ctx_max, size=batch)], seed=seed)
    return cfg, S


def _oracle_stats(depths, res):
    st = verify.new_stats()
    return verify.accumulate_stats(st, depths, res)


def _check_stats(gpu, ref):
    for key in ("steps", "rows", "drafted", "accepted", "emitted", "accepted_independent"):
        assert int(gpu[key]) == int(ref[key]), (key, gpu[key], ref[key])
    for key in ("hist_accepted", "drafted_by_k", "accepted_by_k"):
        g = [int(x) for x in gpu[key]]
        r = [int(x) for x in ref[key]]
        assert g[:len(r)] == r and not any(g[len(r):]), (key, g, r)


def _run(S, depths, drafts, logits, probs, seed, mode, temperature):
    B = len(depths)
    acc, tok = S.lane.verify_logits(list(range(B)), depths, drafts.cuda(), logits.cuda(),
                                    None if probs is None else probs.cuda(), seed=seed, mode=mode,
                                    temperature=temperature)
    torch.cuda.synchronize()
    acc, tok = acc.cpu().numpy(), tok.cpu().numpy()
    res = decisions(S, list(range(B)), depths, drafts, probs, f64(logits), seed, mode, temperature)
    border = []
    for b, r in enumerate(res):
        if not (acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"]):
            assert mode == "sample" and r["borderline"], (b, depths[b], acc[b], list(tok[b]), r)
            border.append(b)
        assert all(t == -1 for t in tok[b][acc[b] + 1:])
    return acc, tok, res, border


@pytest.mark.parametrize("mode,dense", [("greedy", False), ("sample", False), ("sample", True)])
def test_full_counter_struct_matches_oracle(mode, dense):
    """Two verify calls at V = 128256, k ~ U{0..8}: every field of sv_lane_stats equals the oracle's
    accumulate_stats over the oracle's decisions (including accepted_independent, the histogram of
    a_i and the per-depth sums)."""
    cfg, S = _lane(V_FULL, 64)
    B = cfg.max_batch
    ref = verify.new_stats()
    total_border = 0
    for call in range(2):
        depths = [int(x) for x in synth.depths_uniform(B, 0, 8, seed=31 + call)]
        T = sum(depths) + B
        g = torch.Generator().manual_seed(32 + call)
        logits = torch.randn(T, cfg.vocab, generator=g) * 2.0
        drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=33 + call)
        r0, off = 0, 0
        for k in depths:                       # drafts likely under the target: a spread of a_i
            for j in range(k):
                if (j + off + call) % 4:       # +16: p(d) ~ 0.9 against 128k N(0, 4) logits
                    logits[r0 + j, int(drafts[off + j])] += 16.0
            r0 += k + 1
            off += k
        probs = None
        if dense:
            probs = synth.draft_probs_dense(sum(depths), cfg.vocab, seed=34 + call)
            probs[torch.arange(sum(depths)), drafts.long()] += 0.5
            probs /= probs.sum(dim=1, keepdim=True)
        acc, tok, res, border = _run(S, depths, drafts, logits, probs, 77 + call, mode, 0.9)
        total_border += len(border)
        if border:                             # a borderline flip: fold the GPU's own decision
            for b in border:
                res[b] = dict(res[b], a=int(acc[b]))
        verify.accumulate_stats(ref, depths, res)
    st = S.lane.stats()
    assert st["device_error"] == 0
    if total_border == 0:
        _check_stats(st, ref)
    else:                                      # indep may differ on a borderline row: the rest must not
        for key in ("steps", "rows", "drafted", "accepted", "emitted", "hist_accepted", "drafted_by_k",
                    "accepted_by_k"):
            _check_stats({k: st[k] for k in st} | {x: ref[x] for x in ("accepted_independent",)}, ref)
    assert ref["hist_accepted"][0] > 0 and max(a for a, n in enumerate(ref["hist_accepted"]) if n) >= 3


def test_degenerate_sampler_cases():
    """S4 / S5 on the device (V = 512, one-row decisions, dense q):
    request 0: q(d) = 0 at an accept test -> accepted whatever u (ratio +inf);
    request 1: p(d) = 0 (logit -1e4: exp underflows to exactly 0 in fp32 and fp64) -> rejected;
    request 2: unnormalised q >= p everywhere -> the residual max(0, p - q) has zero mass, so the
               replacement is drawn from p itself (R4), i.e. one of p's two support tokens;
    request 3: the same with p concentrated on a single token -> that token, deterministically."""
    V = 512
    cfg, S = _lane(V, 4, depth=2)
    depths = [1, 1, 1, 1]
    NEG = -1.0e4
    lg = np.full((8, V), NEG, dtype=np.float32)
    q = np.zeros((4, V), dtype=np.float32)
    # request 0: p_1 spread, draft 7 with q(7) = 0
    lg[0, :16] = np.linspace(0, 2, 16)
    lg[1, :] = 0.0
    q[0, 100:110] = 0.1
    # request 1: draft 9 has p(9) = 0; q puts mass on it
    lg[2, :8] = 1.0
    lg[3, :] = 0.0
    q[1, 9] = 0.5
    q[1, :8] = 0.5 / 8
    # request 2: p = {0: .5, 1: .5}, q = {0: 1, 1: 1} (unnormalised): ratio 1/2, residual 0 -> y ~ p
    lg[4, 0] = lg[4, 1] = 0.0
    lg[5, :] = 0.0
    q[2, 0] = q[2, 1] = 1.0
    # request 3: p = {5: 1}, q = {5: 2}: ratio 1/2, residual 0 -> y = 5 whenever rejected
    lg[6, 5] = 0.0
    lg[7, :] = 0.0
    q[3, 5] = 2.0
    drafts = torch.tensor([7, 9, 0, 5], dtype=torch.int32)
    logits, probs = torch.from_numpy(lg), torch.from_numpy(q)
    seen_reject = {2: False, 3: False}
    for seed in range(40):
        acc, tok, res, border = _run(S, depths, drafts, logits, probs, 500 + seed, "sample", 1.0)
        assert not border
        assert acc[0] == 1                                 # q(d) = 0: accept
        assert acc[1] == 0 and tok[1][0] in range(8)       # p(d) = 0: reject, y from max(0, p - q)
        if acc[2] == 0:
            seen_reject[2] = True
            assert tok[2][0] in (0, 1)                      # drawn from p (zero residual)
        if acc[3] == 0:
            seen_reject[3] = True
            assert tok[3][0] == 5
    assert seen_reject[2] and seen_reject[3]               # the fallback path actually ran


def test_greedy_ties_across_vocab_tiles():
    """Equal maxima at ids in different 128-wide vocab tiles (and inside one tile): greedy takes
    the lowest id, on both the accept scan and the emitted token (S8)."""
    cfg, S = _lane(V_FULL, 8, depth=3)
    B = 8
    depths = [3] * B
    T = 4 * B
    rng = np.random.default_rng(3)
    lg = (rng.standard_normal((T, V_FULL)) * 2).astype(np.float32)
    groups = [(5, 300, 128000), (127, 128), (128255, 70000), (1000, 1001, 1002), (0, 128255), (4095, 4096, 99999)]
    drafts = []
    for b in range(B):
        for j in range(4):
            ids = groups[(b + j) % len(groups)]
            lg[4 * b + j, list(ids)] = lg[4 * b + j].max() + 3.0
            if j < 3:                      # draft the lowest tied id, except a higher tied id at j = b % 3
                drafts.append(max(ids) if (b % 4 == 3 and j == b % 3) else min(ids))
    drafts = torch.tensor(drafts, dtype=torch.int32)
    acc, tok, res, _ = _run(S, depths, drafts, torch.from_numpy(lg), None, 1, "greedy", 1.0)
    for b in range(B):
        if b % 4 == 3:
            assert acc[b] == b % 3
        else:
            assert acc[b] == 3
        ids = groups[(b + int(acc[b])) % len(groups)]
        assert tok[b][acc[b]] == min(ids)


def test_batch_128_sampled_dense_full_vocab():
    """BASELINE configs[2] batch (128 requests) at V = 128256, sampled with dense q: decisions and
    counters against the oracle (the finalize race splits fewer CTAs per request at this batch)."""
    cfg, S = _lane(V_FULL, 128, depth=8, ctx_max=400, seed=12)
    B = 128
    depths = [int(x) for x in synth.depths_uniform(B, 5, 8, seed=41)]
    T = sum(depths) + B
    logits = torch.randn(T, cfg.vocab, generator=torch.Generator().manual_seed(42)) * 2.0
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=43)
    r0, off = 0, 0
    for k in depths:
        for j in range(k):
            if (j + off) % 5:
                logits[r0 + j, int(drafts[off + j])] += 10.0
        r0 += k + 1
        off += k
    probs = synth.draft_probs_dense(sum(depths), cfg.vocab, seed=44)
    probs[torch.arange(sum(depths)), drafts.long()] += 0.6
    probs /= probs.sum(dim=1, keepdim=True)
    acc, tok, res, border = _run(S, depths, drafts, logits, probs, 91, "sample", 1.0)
    assert len(border) <= 1
    if not border:
        _check_stats(S.lane.stats(), _oracle_stats(depths, res))
