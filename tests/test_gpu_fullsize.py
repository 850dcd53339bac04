"""Parity at the north-star size, in the launch configuration bench.py times (workload `ns`:
64 requests x 4096-token contexts x depth 8 = 576 chain rows, Llama-3-8B-shaped layer +
lm-head, planted-successor weights, greedy), on outputs the oracle can compute one by one:

* verify attention of sampled requests (every split-KV item of theirs, all 32 heads), teacher-
  forced on the GPU's Q / chain K,V, within the derived tolerance;
* the residual stream h1 and lm-head logits of sampled rows (fp64 products of the GPU's inputs);
* the vocab-tile statistics of sampled rows, recomputed from the GPU's fp32 logits;
* greedy decisions of ALL 64 requests, bit-exact against the oracle's accept scan on the GPU's
  fp32 logits, plus the invariants a_i <= k_i and the emitted-token layout."""
import numpy as np
import pytest
import torch

import bench
import synth
from oracle import model, verify

from gpu_util import f64
from test_gpu_parity import ATTN_REL, LOGIT_REL, RESID_REL, attention_tolerance, survey_attention_error

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def step():
    wl = synth.workload("ns", steps_budget=4)
    dev = torch.device("cuda:0")
    lane, w, succ, reqs = bench.build_lane(wl, 0, dev)
    lane.set_taps(True)
    cfg, B = wl.cfg, wl.batch
    depths = [wl.kmax] * B
    masks, devtok = synth.planted_masks(1, B * wl.kmax, wl.alpha, cfg.vocab, seed=9)
    drafts = torch.empty(B * wl.kmax, dtype=torch.int32, device=dev)
    lane.draft_planted(list(range(B)), depths, succ.to(dev), masks[0].to(dev), devtok[0].to(dev), drafts)
    acc, tok = lane.verify(list(range(B)), depths, drafts, None, seed=1234, mode="greedy")
    torch.cuda.synchronize()
    T = B * (wl.kmax + 1)
    tap = lambda n, dt, sh: lane.tap(n, dt, sh).cpu().clone()
    Tmax = cfg.max_batch * (cfg.max_depth + 1)
    out = dict(wl=wl, cfg=cfg, w=w, reqs=reqs, depths=depths, drafts=drafts.cpu().numpy(), T=T,
               acc=acc.cpu().numpy(), tok=tok.cpu().numpy(),
               q=tap("q", torch.bfloat16, (T, cfg.n_q_heads, cfg.head_dim)),
               kc=tap("kc", torch.bfloat16, (cfg.n_layers, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T],
               vc=tap("vc", torch.bfloat16, (cfg.n_layers, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T],
               o=tap("o", torch.bfloat16, (T, cfg.n_q_heads * cfg.head_dim)),
               h0=tap("h0", torch.float32, (T, cfg.d_model)), h1=tap("h1", torch.float32, (T, cfg.d_model)),
               z=tap("z", torch.bfloat16, (T, cfg.d_model)), logits=tap("logits", torch.float32, (T, cfg.vocab)))
    nt = (cfg.vocab + 127) // 128
    for n in ("tile_max", "tile_sum"):
        out[n] = tap(n, torch.float32, (T, nt))
    out["tile_arg"] = tap("tile_arg", torch.int32, (T, nt))
    return out


def test_attention_sampled_requests(step):
    s, cfg = step, step["cfg"]
    R = s["wl"].kmax + 1
    worst, worst_survey = 0.0, 0.0
    for b in (0, 21, 42, 63):
        r0 = b * R
        q = f64(s["q"][r0:r0 + R])
        ck, cv = f64(s["reqs"][b]["k"][0]), f64(s["reqs"][b]["v"][0])
        assert ck.shape[0] == 4096                         # 4 split-KV items + the chain
        kc, vc = f64(s["kc"][r0:r0 + R]), f64(s["vc"][r0:r0 + R])
        ref = model.verify_attention(q, ck, cv, kc, vc).reshape(R, cfg.n_q_heads, cfg.head_dim)
        g = f64(s["o"][r0:r0 + R]).reshape(R, cfg.n_q_heads, cfg.head_dim)
        tol, exact = attention_tolerance(q, ck, cv, kc, vc, with_exact=True)
        worst = max(worst, float((np.abs(g - ref) / tol).max()))
        worst_survey = max(worst_survey, survey_attention_error(g, exact))
    print("ns attention: max err / derived tol", worst, "survey criterion (x rms)", worst_survey)
    assert worst <= 1.0, worst
    assert worst_survey <= ATTN_REL, worst_survey


def test_residual_and_logits_sampled_rows(step):
    s, cfg, W = step, step["cfg"], step["w"]
    rows = np.random.default_rng(0).choice(s["T"], 12, replace=False)
    h0, o, h1 = f64(s["h0"][rows]), f64(s["o"][rows]), f64(s["h1"][rows])
    ref_h1 = model.attn_out(h0, o, W["wo"][0].float().numpy())
    rms = np.sqrt((ref_h1 ** 2).mean(axis=1))
    assert (np.abs(h1 - ref_h1).max(axis=1) / rms).max() <= RESID_REL
    z = f64(s["z"][rows])
    ref_l = model.lm_head(z, W["lm_head"].float().numpy())
    lg = f64(s["logits"][rows])
    err = np.abs(lg - ref_l).max(axis=1) / np.maximum(1.0, np.abs(ref_l).max(axis=1))
    assert err.max() <= LOGIT_REL, err.max()
    # vocab-tile statistics of these rows from the GPU's own fp32 logits (greedy: inv_temp = 1)
    mx, se, am = model.tile_stats(s["logits"][rows].numpy().astype(np.float64), tile=128)
    assert np.array_equal(s["tile_max"][rows].numpy(), mx.astype(np.float32))
    assert np.array_equal(s["tile_arg"][rows].numpy(), am)
    gse = s["tile_sum"][rows].numpy()
    assert np.max(np.abs(gse - se) / se) < 1e-5


def test_greedy_decisions_all_requests_bit_exact(step):
    s = step
    K = s["wl"].kmax
    lg = s["logits"].numpy().astype(np.float64)
    for b in range(64):
        c = s["reqs"][b]
        dr = [int(t) for t in s["drafts"][b * K:(b + 1) * K]]
        r = verify.verify_request(lg[b * (K + 1):(b + 1) * (K + 1)], dr, None, 1234, c["rid"], c["L"],
                                  verify.GREEDY, 1.0)
        a = int(s["acc"][b])
        assert a == r["a"], (b, a, r["a"])
        assert list(s["tok"][b][:a + 1]) == r["emitted"]
        assert all(t == -1 for t in s["tok"][b][a + 1:])
        assert 0 <= a <= K and list(s["tok"][b][:a]) == dr[:a]
    # the planted drafter makes acceptance realistic at this size
    assert 0.2 < s["acc"].mean() / K < 0.8


def test_greedy_decisions_all_rows_on_fp64_logits_from_gpu_z(step):
    """the oracle recomputes every row's logits in fp64 from the GPU's bf16 z
    (all 576 rows x 128256), takes the lowest-index argmax and runs the accept scan. A decision
    may differ from the GPU's only on a row whose oracle top-2 gap is below 2 * max|l_gpu - l_oracle|
    of that row (the excuse rule); such rows are counted and must be rare."""
    s, cfg, W = step, step["cfg"], step["w"]
    K, T = s["wl"].kmax, s["T"]
    z = f64(s["z"])
    ref = model.lm_head(z, W["lm_head"].float().numpy())             # [576, 128256] fp64
    lg = s["logits"].numpy().astype(np.float64)
    row_err = np.abs(lg - ref).max(axis=1)
    srt = np.sort(ref, axis=1)
    gap = srt[:, -1] - srt[:, -2]
    near_tie = gap < 2.0 * row_err
    excused = 0
    for b in range(64):
        c = s["reqs"][b]
        rows = slice(b * (K + 1), (b + 1) * (K + 1))
        dr = [int(t) for t in s["drafts"][b * K:(b + 1) * K]]
        r = verify.verify_request(ref[rows], dr, None, 1234, c["rid"], c["L"], verify.GREEDY, 1.0)
        a = int(s["acc"][b])
        if a != r["a"] or list(s["tok"][b][:a + 1]) != r["emitted"]:
            # excused only if a row the two decisions depend on is a near tie
            assert near_tie[rows][:min(a, r["a"]) + 1].any(), (b, a, r["a"], gap[rows], row_err[rows])
            excused += 1
    print("ns greedy on fp64 logits: excused", excused, "near-tie rows", int(near_tie.sum()),
          "max row err", float(row_err.max()), "min gap", float(gap.min()))
    assert excused <= 1


@pytest.mark.parametrize("ctx", [(4100, 6150), (4500, 6300), (5000, 6350)])
def test_attention_ragged_long_contexts(ctx):
    """Ragged long contexts (4.1-6.4 k keys, five-six 1024-key split-KV items per request, the last one
    partial): all 8 requests' verify attention against the oracle under the same criteria as above.
    (The opt-in wide 2048-key items, SV_WIDE_SPLIT=1, measured 1.001 % on the survey criterion in one
    of these three cases, 0.79-0.83 % in the others.)"""
    import dataclasses
    base = synth.workload("ns", steps_budget=4)
    cfg8 = base.cfg.with_(n_pages=8 * 100, max_slots=8, max_batch=8, max_pos=6400)   # 6150 + chains fit
    wl = dataclasses.replace(base, cfg=cfg8, batch=8, ctx=ctx)
    dev = torch.device("cuda:0")
    lane, w, succ, reqs = bench.build_lane(wl, 0, dev)
    lane.set_taps(True)
    cfg, B = wl.cfg, wl.batch
    lens = [r["L"] for r in reqs]
    assert min(lens) >= 4096 and any(L % 1024 for L in lens)
    depths = [wl.kmax] * B
    masks, devtok = synth.planted_masks(1, B * wl.kmax, wl.alpha, cfg.vocab, seed=5)
    drafts = torch.empty(B * wl.kmax, dtype=torch.int32, device=dev)
    lane.draft_planted(list(range(B)), depths, succ.to(dev), masks[0].to(dev), devtok[0].to(dev), drafts)
    lane.verify(list(range(B)), depths, drafts, None, seed=7, mode="greedy")
    torch.cuda.synchronize()
    R, T = wl.kmax + 1, B * (wl.kmax + 1)
    Tmax = cfg.max_batch * (cfg.max_depth + 1)
    q = lane.tap("q", torch.bfloat16, (T, cfg.n_q_heads, cfg.head_dim)).cpu()
    kc = lane.tap("kc", torch.bfloat16, (cfg.n_layers, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T].cpu()
    vc = lane.tap("vc", torch.bfloat16, (cfg.n_layers, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T].cpu()
    o = lane.tap("o", torch.bfloat16, (T, cfg.n_q_heads * cfg.head_dim)).cpu()
    lane.commit()
    worst, worst_survey = 0.0, 0.0
    for b in range(B):
        r0 = b * R
        qb = f64(q[r0:r0 + R])
        ck, cv = f64(reqs[b]["k"][0]), f64(reqs[b]["v"][0])
        kb, vb = f64(kc[r0:r0 + R]), f64(vc[r0:r0 + R])
        ref = model.verify_attention(qb, ck, cv, kb, vb).reshape(R, cfg.n_q_heads, cfg.head_dim)
        g = f64(o[r0:r0 + R]).reshape(R, cfg.n_q_heads, cfg.head_dim)
        tol, exact = attention_tolerance(qb, ck, cv, kb, vb, with_exact=True)
        worst = max(worst, float((np.abs(g - ref) / tol).max()))
        worst_survey = max(worst_survey, survey_attention_error(g, exact))
    print("long-context attention: max err / derived tol", worst, "survey criterion (x rms)", worst_survey)
    assert worst <= 1.0, worst
    assert worst_survey <= ATTN_REL, worst_survey
