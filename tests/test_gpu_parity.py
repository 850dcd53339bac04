"""GPU parity of every verify-step stage against the fp64 oracle, teacher-forced
(DESIGN.md "Parity contract"): each oracle stage is fed the
GPU's own inputs to that stage (read back through sv_get_tap) and its output is
compared element by element with the GPU's, at the tolerance written below.
All calls go through the C ABI (libsv.so) via the ctypes binding."""
import numpy as np
import pytest
import torch

import synth
from oracle import model, verify
from oracle.numerics import round_bf16

from gpu_util import Setup, bf16_ulp_diff, to_bf16, f64

pytestmark = pytest.mark.gpu

# tolerances (DESIGN.md §"Parity contract")
BF16_FLIP_FRAC = 0.02          # fraction of bf16 elements allowed to differ (by <= 1 ulp)
ATTN_REL = 1e-2                # max|dO| <= 1e-2 * rms(O_ref) per (row, head)
RESID_REL = 2e-3               # max|dh| <= 2e-3 * rms(h_ref) per row
LOGIT_REL = 2e-3               # max|dl| <= 2e-3 * max(1, max|l_ref|) per row (north_star)


def _cmp_bf16(name, gpu, ref, report):
    """gpu: torch bf16; ref: fp64 numpy of bf16 values. <= 1 ulp, except near-zero elements."""
    r = to_bf16(ref).reshape(gpu.shape)
    ulp = bf16_ulp_diff(gpu, r)
    refv = torch.from_numpy(np.ascontiguousarray(ref)).reshape(gpu.shape)
    rms = float(refv.pow(2).mean().sqrt())
    tiny = refv.abs() < rms * 2.0 ** -6
    absd = (gpu.to(torch.float64) - refv).abs()
    bad = (ulp > 1) & ~(tiny & (absd <= rms * 2.0 ** -9))
    frac = float((ulp > 0).double().mean())
    report[name] = dict(max_ulp=int(ulp.max()), flip_frac=frac)
    assert int(bad.sum()) == 0, (name, int(bad.sum()), int(ulp.max()))
    assert frac <= BF16_FLIP_FRAC, (name, frac)


def run_and_check(S, slots, depths, drafts, mode, seed=1234, temperature=1.0, probs=None, check_attention=True):
    cfg = S.cfg
    lane = S.lane
    d_dev = drafts.cuda()
    p_dev = probs.cuda() if probs is not None else None
    acc, tok = lane.verify(slots, depths, d_dev, p_dev, seed=seed, mode=mode, temperature=temperature)
    torch.cuda.synchronize()
    acc, tok = acc.cpu().numpy(), tok.cpu().numpy()
    T = sum(k + 1 for k in depths)
    D, V = cfg.d_model, cfg.vocab
    Hq, Hkv, dh = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
    report = {}
    # chain tokens and positions, request-major
    toks, pos, off = [], [], 0
    for b, (s, k) in enumerate(zip(slots, depths)):
        c = S.ctx[s]
        toks += [c["pending"]] + [int(t) for t in drafts[off:off + k]]
        pos += list(range(c["L"], c["L"] + k + 1))
        off += k
    toks, pos = np.array(toks), np.array(pos)
    W = S.wnp
    # a2: embed + norm
    h0 = S.tap("h0", torch.float32, (T, D))
    assert np.array_equal(f64(h0), model.embed(W["embed"], toks))
    a = S.tap("a", torch.bfloat16, (T, D))
    _cmp_bf16("a", a, model.attn_norm(f64(h0), W["attn_norm"][0].astype(np.float64), cfg.norm_eps), report)
    # a2: QKV + RoPE (fp32 table from the lane, checked against the oracle's own table)
    cos = S.tap("rope_cos", torch.float32, (cfg.max_pos, dh // 2)).numpy()
    sin = S.tap("rope_sin", torch.float32, (cfg.max_pos, dh // 2)).numpy()
    ocos, osin = model.rope_table(cfg.max_pos, dh, cfg.rope_theta)
    assert np.mean(cos != ocos) < 1e-4 and np.max(np.abs(cos - ocos)) <= 2 ** -23
    assert np.mean(sin != osin) < 1e-4 and np.max(np.abs(sin - osin)) <= 2 ** -23
    q, k, v = model.qkv_rope(f64(a), W["wqkv"][0], pos, cos, sin, Hq, Hkv, dh)
    gq = S.tap("q", torch.bfloat16, (T, Hq, dh))
    Tmax = cfg.max_batch * (cfg.max_depth + 1)
    gk = S.tap("kc", torch.bfloat16, (cfg.n_layers, Tmax, Hkv, dh))[0, :T]
    gv = S.tap("vc", torch.bfloat16, (cfg.n_layers, Tmax, Hkv, dh))[0, :T]
    _cmp_bf16("q", gq, q, report)
    _cmp_bf16("k", gk, k, report)
    _cmp_bf16("v", gv, v, report)
    # a3: attention, fed the GPU's q and chain k/v
    go = S.tap("o", torch.bfloat16, (T, Hq * dh))
    if check_attention:
        worst, worst_sig, worst_survey = 0.0, 0.0, 0.0
        r0 = 0
        for s, kk in zip(slots, depths):
            c = S.ctx[s]
            R = kk + 1
            q_, ck, cv = f64(gq[r0:r0 + R]), f64(c["k"][0]), f64(c["v"][0])
            kc_, vc_ = f64(gk[r0:r0 + R]), f64(gv[r0:r0 + R])
            ref = model.verify_attention(q_, ck, cv, kc_, vc_).reshape(R, Hq, dh)
            g = f64(go[r0:r0 + R]).reshape(R, Hq, dh)
            err = np.abs(g - ref)
            rms = np.sqrt((ref ** 2).mean(axis=2))
            worst = max(worst, float((err.max(axis=2) / np.maximum(rms, 1e-30)).max()))
            tol, exact = attention_tolerance(q_, ck, cv, kc_, vc_, with_exact=True)
            worst_sig = max(worst_sig, float((err / tol).max()))
            worst_survey = max(worst_survey, survey_attention_error(g, exact))
            r0 += R
        report["o"] = dict(max_rel=worst, max_err_over_tol=worst_sig, survey_rel=worst_survey)
        assert worst_sig <= 1.0, (worst_sig, worst)
        assert worst_survey <= ATTN_REL, worst_survey
    # a4: O-proj + residual, MLP
    h1 = S.tap("h1", torch.float32, (T, D))
    ref_h1 = model.attn_out(f64(h0), f64(go), W["wo"][0])
    _cmp_resid("h1", f64(h1), ref_h1, report)
    if cfg.ffn_dim > 0:
        b_ = S.tap("b", torch.bfloat16, (T, D))
        _cmp_bf16("b", b_, model.ffn_norm(f64(h1), W["ffn_norm"][0].astype(np.float64), cfg.norm_eps), report)
        u = S.tap("u", torch.bfloat16, (T, cfg.ffn_dim))
        _cmp_bf16("u", u, model.swiglu(f64(b_), W["w_gate_up"][0]), report)
        h2 = S.tap("h2", torch.float32, (T, D))
        _cmp_resid("h2", f64(h2), model.down_residual(f64(h1), f64(u), W["w_down"][0]), report)
    else:
        h2 = h1
    # a5: final norm + lm-head + tile statistics
    z = S.tap("z", torch.bfloat16, (T, D))
    _cmp_bf16("z", z, model.final_norm(f64(h2), W["final_norm"].astype(np.float64), cfg.norm_eps), report)
    lg = S.tap("logits", torch.float32, (T, V))
    ref_l = model.lm_head(f64(z), W["lm_head"])
    row_err = np.abs(f64(lg) - ref_l).max(axis=1) / np.maximum(1.0, np.abs(ref_l).max(axis=1))
    report["logits"] = dict(max_rel=float(row_err.max()))
    assert row_err.max() <= LOGIT_REL, row_err.max()
    nt = (V + 127) // 128
    inv_t = 1.0 / temperature if mode == "sample" else 1.0
    lg32 = lg.numpy().astype(np.float32)
    scaled = (lg32 * np.float32(inv_t)).astype(np.float64)   # the same fp32 product the GPU forms
    mx, se, am = model.tile_stats(scaled, tile=128)
    assert np.array_equal(S.tap("tile_max", torch.float32, (T, nt)).numpy(), mx.astype(np.float32))
    assert np.array_equal(S.tap("tile_arg", torch.int32, (T, nt)).numpy(), am)
    gse = S.tap("tile_sum", torch.float32, (T, nt)).numpy()
    assert np.max(np.abs(gse - se) / se) < 1e-5
    # a6: decisions, teacher-forced on the GPU's own fp32 logits
    res = decisions(S, slots, depths, drafts, probs, f64(lg), seed, mode, temperature)
    borderline = 0
    for b, r in enumerate(res):
        ok = acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"]
        if not ok:
            assert mode == "sample" and r["borderline"], (b, acc[b], r)
            borderline += 1
        assert all(t == -1 for t in tok[b][acc[b] + 1:])
    report["borderline"] = borderline
    return report, acc, tok


def survey_attention_error(g, exact):
    """SURVEY.md §8(c) a3 criterion, max|dO| <= 1e-2 rms(O_ref) per (row, head), measured against
    the UNROUNDED fp64 output with the GPU's own final bf16 rounding (<= 1/2 ulp of its output)
    taken out (reading R32): an element of 2.5 rms sits where one bf16 ulp is 1.6e-2 rms,
    so comparing two independently rounded outputs would fail the criterion on a single rounding
    flip that neither side can avoid. Returns max over (row, head) of that error / rms."""
    half_ulp = np.ldexp(1.0, np.frexp(np.abs(g))[1] - 9)          # bf16: 8 significant bits
    e = np.maximum(np.abs(g - exact) - half_ulp, 0.0)
    rms = np.sqrt((exact ** 2).mean(axis=2))
    return float((e.max(axis=2) / np.maximum(rms, 1e-30)).max())


def attention_tolerance(q, ck, cv, kc, vc, with_exact=False):
    """Per-element tolerance of the GPU attention output (a3).

    The GPU rounds the softmax weights P to bf16 (8 significant bits) before the P.V
    tensor-core product: relative error |dw_i / w_i| <= 2^-8, ~uniform. With w the exact
    weights and O the exact output, that perturbs O_d by sum_i dw_i (v_id - O_d) / sum w, a
    zero-mean sum with std sigma_d <= 2^-8/sqrt(3) * sqrt(sum_i w_i^2 (v_id - O_d)^2). Both
    sides then round O to bf16 (<= 2^-8 |O_d| each). Tolerance = 6 sigma_d + 2^-7 |O_d|
    (+ fp32 slack)."""
    R, Hq, dh = q.shape
    Hkv = kc.shape[1]
    G = Hq // Hkv
    L = ck.shape[0]
    tol = np.zeros((R, Hq, dh))
    exact = np.zeros((R, Hq, dh))
    for j in range(R):
        keys = np.concatenate([ck[:L], kc[: j + 1]])
        vals = np.concatenate([cv[:L], vc[: j + 1]])
        for hq in range(Hq):
            w = model.softmax(keys[:, hq // G, :] @ q[j, hq] / np.sqrt(dh))
            v = vals[:, hq // G, :]
            o = w @ v
            sig = 2.0 ** -8 / np.sqrt(3.0) * np.sqrt((w[:, None] ** 2 * (v - o[None]) ** 2).sum(axis=0))
            tol[j, hq] = 6 * sig + 2.0 ** -7 * np.abs(o) + 1e-6 * np.abs(v).max()
            exact[j, hq] = o
    return (tol, exact) if with_exact else tol


def _cmp_resid(name, g, ref, report):
    rms = np.sqrt((ref ** 2).mean(axis=1))
    err = np.abs(g - ref).max(axis=1) / rms
    report[name] = dict(max_rel=float(err.max()))
    assert err.max() <= RESID_REL, (name, err.max())


def decisions(S, slots, depths, drafts, probs, logits, seed, mode, temperature):
    """Oracle decisions per request on given logits; flags borderline cases (|u - p/q| < 1e-5,
    or race top-2 within 1e-5 relative) — SURVEY.md §8(c) S12."""
    out, r0, off = [], 0, 0
    m = verify.GREEDY if mode == "greedy" else verify.SAMPLE
    for s, k in zip(slots, depths):
        c = S.ctx[s]
        lrow = logits[r0:r0 + k + 1]
        dr = [int(t) for t in drafts[off:off + k]]
        qr = None if probs is None else f64(probs[off:off + k])
        r = verify.verify_request(lrow, dr, qr, seed, c["rid"], c["L"], m, temperature)
        r["borderline"] = False
        if m == verify.SAMPLE:
            p = verify.target_probs(lrow, temperature)
            from oracle.philox import uniform_accept
            for j in range(1, k + 1):
                u = uniform_accept(seed, c["rid"], c["L"] + j)
                qd = 1.0 if qr is None else qr[j - 1][dr[j - 1]]
                if qd > 0 and abs(u - p[j - 1][dr[j - 1]] / qd) < 1e-5:
                    r["borderline"] = True
            a = r["a"]
            sc = verify.race_scores(lrow[a], None if (qr is None or a == k) else qr[a],
                                    dr[a] if a < k else -1, seed, c["rid"], c["L"] + a + 1, temperature,
                                    residual=a < k)
            top2 = np.sort(sc[np.isfinite(sc)])[-2:]
            if len(top2) == 2 and (top2[1] - top2[0]) <= 1e-5 * abs(top2[1]):
                r["borderline"] = True
        out.append(r)
        r0 += k + 1
        off += k
    return out


# ---------------------------------------------------------------------------- tests

@pytest.mark.parametrize("cfgname", ["toy", "toy_mlp"])
@pytest.mark.parametrize("mode", ["greedy", "sample"])
def test_toy_stages(cfgname, mode):
    """BASELINE configs[0]: 4 requests, k = 1..4, context 128 (+ ragged variants)."""
    cfg = synth.CONFIGS[cfgname]
    S = Setup(cfg, [128, 128, 128, 128, 5, 700], seed=3)
    slots, depths = [0, 1, 2, 3], [1, 2, 3, 4]
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=7)
    probs = synth.draft_probs_dense(sum(depths), cfg.vocab, seed=8) if mode == "sample" else None
    rep, acc, _ = run_and_check(S, slots, depths, drafts, mode, probs=probs, temperature=0.8)
    print(cfgname, mode, rep)


def test_toy_ragged_edge_cases():
    """k = 0, max depth, short (5) and long (700, spans several splits) contexts, batch order."""
    cfg = synth.TOY_MLP
    S = Setup(cfg, [128, 1, 5, 700, 64, 511], seed=4)
    slots, depths = [3, 1, 5, 0, 2, 4], [0, 8, 3, 8, 1, 5]
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=9)
    rep, _, _ = run_and_check(S, slots, depths, drafts, "sample", temperature=1.3)
    print(rep)


def test_llama_shape_stages():
    """Llama-3-8B-shaped layer + lm-head (BASELINE configs[1] shape) on a request subset."""
    cfg = synth.LLAMA.with_(n_pages=256, max_slots=8, max_batch=8, max_pos=2048)
    S = Setup(cfg, [256, 300, 511, 700, 1024, 64], seed=5)
    slots, depths = [0, 1, 2, 3, 4, 5], [8, 1, 4, 0, 6, 3]
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=10)
    rep, _, _ = run_and_check(S, slots, depths, drafts, "greedy")
    print("llama greedy", rep)


def test_llama_long_contexts_split_kv():
    """Contexts of 1..5 split-KV work items (1024 page keys each) per (request, kv head): the
    keys-on-lanes kernel merges the splits' partials in-kernel (last split to finish)."""
    cfg = synth.LLAMA.with_(n_pages=256, max_slots=4, max_batch=4, max_pos=6144)
    S = Setup(cfg, [2100, 4200, 1030, 3000], seed=11)
    slots, depths = [0, 1, 2, 3], [8, 3, 5, 0]
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=12)
    rep, _, _ = run_and_check(S, slots, depths, drafts, "greedy")
    print("llama long contexts", rep)


def test_llama_deep_chains_rows_on_lanes():
    """max_depth 20 at G = 4 (SpecuStream's d* reaches 20, Alg. 4): a verify whose deepest chain
    has (k + 1) G > 64 query rows per kv head runs the rows-on-lanes tcgen05 kernel (32 rows x 4 heads per
    item), one within 64 the keys-on-lanes kernel, on the same lane; every stage within the contract."""
    cfg = synth.LLAMA.with_(n_pages=96, max_slots=6, max_batch=6, max_depth=20, max_pos=2048)
    for slots, depths, seed in (([0, 1, 2, 3, 4, 5], [20, 9, 15, 0, 3, 17], 18), ([1, 3], [8, 2], 19)):
        S = Setup(cfg, [256, 1100, 40, 700, 2000, 1], seed=17)
        drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=seed)
        rep, _, _ = run_and_check(S, slots, depths, drafts, "greedy")
        print("deep chains", depths, rep["o"])
        S.lane.close()
