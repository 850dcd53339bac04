"""GPU tests of the lane state machine through the C ABI: device Philox vs the oracle,
commit/rollback (bitwise), append/release and the free list, decision parity on
caller logits at the full Llama vocabulary, GPU-side distribution laws, invariants
(batch permutation, incremental consistency, determinism) and error paths."""
import numpy as np
import pytest
import torch
from scipy import stats

import synth
from oracle import verify
from oracle.philox import uniform_race, uniform_accept
from paper_2604_09562_b200 import sv

from gpu_util import Setup, f64

pytestmark = pytest.mark.gpu


def _dense_cache(S, slot, layer=0):
    """Read slot's cache back through the page table (K, V [L][Hkv][dh] bf16)."""
    cfg = S.cfg
    torch.cuda.synchronize()
    ln = S.lane.tap("len", torch.int32, (cfg.max_slots,)).cpu()
    mpps = (cfg.max_pos + cfg.page_size - 1) // cfg.page_size
    pt = S.lane.tap("page_table", torch.int32, (cfg.max_slots, mpps)).cpu()
    pool = S.lane.kv_pool.view(torch.bfloat16).view(cfg.n_layers, cfg.n_pages, 2, cfg.n_kv_heads,
                                                    cfg.page_size, cfg.head_dim)
    L = int(ln[slot])
    t = torch.arange(L)
    pages = pt[slot][t // cfg.page_size].long().cuda()
    offs = (t % cfg.page_size).cuda()
    k = pool[layer, pages, 0, :, offs].cpu()        # [L, Hkv, dh]
    v = pool[layer, pages, 1, :, offs].cpu()
    return k, v, L


def test_device_philox_matches_oracle():
    S = Setup(synth.TOY, [4])
    for seed, rid, z in [(0, 0, 0), (1234, 0xDEADBEEF12345678, 4097), (2**64 - 1, 77, 2**32 - 1)]:
        u = S.lane.debug_uniforms(seed, rid, z, 1, 0, 128256).cpu().numpy().astype(np.float64)
        assert np.array_equal(u, uniform_race(seed, rid, z, 128256))
        ua = S.lane.debug_uniforms(seed, rid, z, 0, 0, 1).cpu().numpy()[0]
        assert float(ua) == uniform_accept(seed, rid, z)


def test_commit_rollback_bitwise_and_pending():
    cfg = synth.TOY_MLP
    S = Setup(cfg, [60, 64, 130, 0 + 1], seed=6)
    slots, depths = [0, 1, 2, 3], [4, 8, 3, 2]
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=12)
    acc, tok = S.lane.verify(slots, depths, drafts.cuda(), seed=5, mode="sample")
    torch.cuda.synchronize()
    acc, tok = acc.cpu().numpy().copy(), tok.cpu().numpy().copy()
    T = sum(depths) + len(depths)
    Tmax = cfg.max_batch * (cfg.max_depth + 1)
    kc = S.lane.tap("kc", torch.bfloat16, (1, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T].cpu().clone()
    vc = S.lane.tap("vc", torch.bfloat16, (1, Tmax, cfg.n_kv_heads, cfg.head_dim))[0, :T].cpu().clone()
    # verify is side-effect free on the cache
    for s in slots:
        k, v, L = _dense_cache(S, s)
        assert L == S.ctx[s]["L"]
    S.lane.commit()
    r0 = 0
    for b, s in enumerate(slots):
        k, v, L = _dense_cache(S, s)
        n = int(acc[b]) + 1
        assert L == S.ctx[s]["L"] + n
        assert torch.equal(k, torch.cat([S.ctx[s]["k"][0], kc[r0:r0 + n]]))
        assert torch.equal(v, torch.cat([S.ctx[s]["v"][0], vc[r0:r0 + n]]))
        pend = S.lane.tap("pending", torch.int32, (cfg.max_slots,)).cpu()
        assert int(pend[s]) == int(tok[b][n - 1])
        r0 += depths[b] + 1


def test_n_keep_truncation_and_release():
    cfg = synth.TOY
    S = Setup(cfg, [63, 10], seed=7)
    drafts = synth.random_tokens(6, cfg.vocab, seed=13)
    acc, tok = S.lane.verify([0, 1], [3, 3], drafts.cuda(), mode="sample", seed=9)
    torch.cuda.synchronize()
    acc, tok = acc.cpu().numpy().copy(), tok.cpu().numpy().copy()
    keep = torch.tensor([1, 2], dtype=torch.int32, device="cuda")
    S.lane.commit(keep)
    _, _, L0 = _dense_cache(S, 0)
    _, _, L1 = _dense_cache(S, 1)
    assert L0 == 63 + 1 and L1 == 10 + min(2, int(acc[1]) + 1)
    pend = S.lane.tap("pending", torch.int32, (cfg.max_slots,)).cpu()
    assert int(pend[0]) == int(tok[0][0])
    top0 = int(S.lane.tap("free_top", torch.int32, (1,)).cpu()[0])
    S.lane.release(0)
    top1 = int(S.lane.tap("free_top", torch.int32, (1,)).cpu()[0])
    assert top1 == top0 + 1                                  # 63 + 1 = 64 tokens -> one page
    S.lane.release(1)
    assert int(S.lane.tap("free_top", torch.int32, (1,)).cpu()[0]) == cfg.n_pages


def test_incremental_consistency_and_determinism():
    """verify after commit == verify on a fresh lane holding the full committed sequence (bitwise)."""
    cfg = synth.TOY_MLP
    S = Setup(cfg, [100, 37], seed=8)
    d1 = synth.random_tokens(7, cfg.vocab, seed=14)
    S.lane.verify([0, 1], [3, 4], d1.cuda(), mode="sample", seed=2)
    S.lane.commit()
    k0, v0, _ = _dense_cache(S, 0)
    k1, v1, _ = _dense_cache(S, 1)
    pend = S.lane.tap("pending", torch.int32, (cfg.max_slots,)).cpu().clone()
    d2 = synth.random_tokens(9, cfg.vocab, seed=15)
    lo1 = torch.empty(11, cfg.vocab, device="cuda")
    a1, t1 = [x.cpu().clone() for x in S.lane.verify([0, 1], [5, 4], d2.cuda(), mode="sample", seed=3,
                                                      logits_out=lo1)]
    F = sv.Lane(cfg, S.wd)
    F.append_kv(0, S.ctx[0]["rid"], k0[None].cuda(), v0[None].cuda(), int(pend[0]))
    F.append_kv(1, S.ctx[1]["rid"], k1[None].cuda(), v1[None].cuda(), int(pend[1]))
    lo2 = torch.empty(11, cfg.vocab, device="cuda")
    a2, t2 = [x.cpu().clone() for x in F.verify([0, 1], [5, 4], d2.cuda(), mode="sample", seed=3, logits_out=lo2)]
    assert torch.equal(a1, a2) and torch.equal(t1, t2) and torch.equal(lo1, lo2)


def test_batch_permutation_and_slot_invariance():
    cfg = synth.TOY_MLP
    S1 = Setup(cfg, [50, 90, 130], seed=9)
    d = synth.random_tokens(2 + 5 + 3, cfg.vocab, seed=16)
    a1, t1 = [x.cpu().clone() for x in S1.lane.verify([0, 1, 2], [2, 5, 3], d.cuda(), mode="sample", seed=4)]
    S2 = Setup(cfg, [50, 90, 130], seed=9)
    dp = torch.cat([d[7:10], d[0:2], d[2:7]])
    a2, t2 = [x.cpu().clone() for x in S2.lane.verify([2, 0, 1], [3, 2, 5], dp.cuda(), mode="sample", seed=4)]
    assert torch.equal(a1, a2[[1, 2, 0]]) and torch.equal(t1, t2[[1, 2, 0]])


def _finalize_lane(V=128256, batch=64, depth=8):
    cfg = synth.ModelConfig(n_layers=1, d_model=64, n_q_heads=1, n_kv_heads=1, head_dim=64, vocab=V, ffn_dim=0,
                            n_pages=512, max_slots=batch, max_batch=batch, max_depth=depth, max_pos=512)
    S = Setup(cfg, [int(x) for x in np.random.default_rng(0).integers(0, 300, size=batch)], seed=11)
    return cfg, S


@pytest.mark.parametrize("mode,dense", [("greedy", False), ("sample", False), ("sample", True)])
def test_decision_parity_full_vocab(mode, dense):
    """a6/a7 on caller logits (sv_verify_logits) at V = 128256, k ~ U{0..8}."""
    from test_gpu_parity import decisions
    cfg, S = _finalize_lane()
    B = cfg.max_batch
    depths = [int(x) for x in synth.depths_uniform(B, 0, 8, seed=21)]
    T = sum(depths) + B
    g = torch.Generator().manual_seed(22)
    logits = torch.randn(T, cfg.vocab, generator=g) * 2.0
    # plant the draft as a likely token so acceptance is non-trivial
    drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=23)
    r0, off = 0, 0
    for k in depths:
        for j in range(k):
            if (j + off) % 3:
                logits[r0 + j, int(drafts[off + j])] += 9.0
        r0 += k + 1
        off += k
    probs = synth.draft_probs_dense(sum(depths), cfg.vocab, seed=24) if dense else None
    if dense:       # put most draft mass on the drafted token
        probs[torch.arange(sum(depths)), drafts.long()] += 0.5
        probs /= probs.sum(dim=1, keepdim=True)
    acc, tok = S.lane.verify_logits(list(range(B)), depths, drafts.cuda(), logits.cuda(),
                                    None if probs is None else probs.cuda(), seed=77, mode=mode, temperature=0.9)
    torch.cuda.synchronize()
    acc, tok = acc.cpu().numpy(), tok.cpu().numpy()
    res = decisions(S, list(range(B)), depths, drafts, probs, f64(logits), 77, mode, 0.9)
    border = 0
    for b, r in enumerate(res):
        if not (acc[b] == r["a"] and list(tok[b][: r["a"] + 1]) == r["emitted"]):
            assert mode == "sample" and r["borderline"], (b, depths[b], acc[b], list(tok[b]), r)
            border += 1
    assert border <= 1
    st = S.lane.stats()
    assert st["device_error"] == 0
    assert st["steps"] == 1 and st["accepted"] == int(acc.sum()) and st["drafted"] == sum(depths)
    assert st["emitted"] == int(acc.sum()) + B


def test_gpu_first_token_law_chi_square():
    """P1 on the GPU: the first emitted token follows p_1 for any draft q (V = 16)."""
    V, B, calls, k = 16, 128, 40, 3
    cfg = synth.ModelConfig(n_layers=1, d_model=64, n_q_heads=1, n_kv_heads=1, head_dim=64, vocab=V, ffn_dim=0,
                            n_pages=2 * B, max_slots=B, max_batch=B, max_depth=4, max_pos=256)
    S = Setup(cfg, [3] * B, seed=12)
    rng = np.random.default_rng(5)
    p = rng.exponential(size=(k + 1, V)) ** 2
    p /= p.sum(axis=1, keepdims=True)
    q = rng.exponential(size=(k, V)) ** 2
    q /= q.sum(axis=1, keepdims=True)
    logits = torch.tensor(np.log(p), dtype=torch.float32).repeat(B, 1).cuda()
    qt = torch.tensor(q, dtype=torch.float32).repeat(B, 1).cuda()
    counts = np.zeros(V)
    for c in range(calls):
        drafts = torch.tensor(np.concatenate([[rng.choice(V, p=q[j]) for j in range(k)] for _ in range(B)]),
                              dtype=torch.int32).cuda()
        acc, tok = S.lane.verify_logits(list(range(B)), [k] * B, drafts, logits, qt, seed=1000 + c, mode="sample")
        torch.cuda.synchronize()
        for t in tok[:, 0].cpu().numpy():
            counts[t] += 1
    p1 = np.exp(np.log(p[0]).astype(np.float32).astype(np.float64))
    p1 /= p1.sum()
    assert stats.chisquare(counts, p1 * counts.sum()).pvalue > 0.001


def test_error_paths():
    cfg = synth.TOY
    S = Setup(cfg, [10, 10], seed=13)
    L = S.lane
    d = synth.random_tokens(4, cfg.vocab, seed=1).cuda()
    with pytest.raises(sv.SvError) as e:
        L.commit()
    assert e.value.status == sv.SV_ESTATE
    with pytest.raises(sv.SvError) as e:
        L.verify([0, 0], [1, 1], d)
    assert e.value.status == sv.SV_EINVAL
    with pytest.raises(sv.SvError) as e:
        L.verify([0], [cfg.max_depth + 1], d)
    assert e.value.status == sv.SV_EINVAL
    with pytest.raises(sv.SvError) as e:
        L.verify([5], [1], d)                       # EMPTY slot
    assert e.value.status == sv.SV_ESTATE
    with pytest.raises(sv.SvError) as e:
        L.verify([0], [1], d, mode="sample", temperature=0.0)
    assert e.value.status == sv.SV_EINVAL
    L.verify([0], [2], d)
    with pytest.raises(sv.SvError) as e:
        L.verify([1], [1], d)                       # one outstanding verify per lane
    assert e.value.status == sv.SV_ESTATE
    with pytest.raises(sv.SvError) as e:
        L.append_kv(0, S.ctx[0]["rid"], None, None, 3)
    assert e.value.status == sv.SV_ESTATE
    L.commit()
    # device-detected bad draft token: accepted_len = -1 and a sticky error
    bad = torch.tensor([cfg.vocab + 5], dtype=torch.int32, device="cuda")
    acc, _ = L.verify([1], [1], bad)
    torch.cuda.synchronize()
    assert int(acc[0]) == -1
    with pytest.raises(sv.SvError) as e:
        L.stats()
    assert e.value.status == sv.SV_EDEVICE


def test_free_list_exhaustion():
    cfg = synth.TOY.with_(n_pages=4)
    S = Setup(cfg, [200], seed=14)                  # 4 pages
    k, v = synth.context_kv(cfg, 100, seed=3)
    S.lane.append_kv(1, 99, k.cuda(), v.cuda(), 1)  # needs 2 more pages -> exhausted
    with pytest.raises(sv.SvError) as e:
        S.lane.stats()
    assert e.value.status == sv.SV_ENOKV


def test_chain_past_max_pos_is_refused_not_crashed():
    """A chain that would run past the position table sets SV_DERR_MAX_POS, returns
    accepted_len = -1 for that request and commits nothing for it; the others are unaffected."""
    cfg = synth.TOY.with_(max_pos=256)
    S = Setup(cfg, [253, 100], seed=15)             # chain positions 253..257 > 255
    d = synth.random_tokens(8, cfg.vocab, seed=4).cuda()
    acc, _ = S.lane.verify([0, 1], [4, 4], d)
    S.lane.commit()
    torch.cuda.synchronize()
    assert int(acc[0]) == -1 and 0 <= int(acc[1]) <= 4
    ln = S.lane.tap("len", torch.int32, (cfg.max_slots,)).cpu()
    assert int(ln[0]) == 253 and int(ln[1]) == 100 + int(acc[1]) + 1
    with pytest.raises(sv.SvError) as e:
        S.lane.stats()
    assert e.value.status == sv.SV_EDEVICE


def test_greedy_without_taps_skips_logits_but_decides_the_same():
    """A greedy verify with taps off does not store the fp32 logits (its decisions read only the
    vocab-tile statistics); decisions must equal those of a lane that keeps every tap."""
    cfg = synth.LLAMA.with_(n_layers=1, n_pages=64, max_slots=4, max_batch=4, max_pos=1024)
    d = synth.random_tokens(4 * 6, cfg.vocab, seed=21).cuda()
    d2 = synth.random_tokens(4 * 6, cfg.vocab, seed=23).cuda()
    out = []
    for taps in (True, False):
        S = Setup(cfg, [100, 300, 64, 700], seed=22)
        S.lane.set_taps(taps)
        acc, tok = S.lane.verify([0, 1, 2, 3], [6, 6, 6, 6], d)
        a1, t1 = acc.cpu().clone(), tok.cpu().clone()
        S.lane.commit()
        lg = S.lane.tap("logits", torch.float32, (4 * 7, cfg.vocab))   # device view (sized by the last T)
        lg.fill_(float("nan"))
        acc, tok = S.lane.verify([0, 1, 2, 3], [6, 6, 6, 6], d2)
        torch.cuda.synchronize()
        out.append((a1, t1, acc.cpu().clone(), tok.cpu().clone(), bool(torch.isnan(lg).all())))
    for i in range(4):
        assert torch.equal(out[0][i], out[1][i])
    assert not out[0][4] and out[1][4]          # taps on: logits stored; off: untouched


def test_lane_occupancy():
    cfg = synth.TOY.with_(n_pages=32)
    S = Setup(cfg, [100, 64, 1], seed=16)                          # 2 + 1 + 1 pages
    active, free = S.lane.occupancy()
    assert active == 3 and free == 32 - 4
    S.lane.release(1)
    assert S.lane.occupancy() == (2, 32 - 3)


@pytest.mark.parametrize("mode", ["greedy", "sample"])
def test_fused_plan_embed_equals_separate_launches(mode, monkeypatch):
    """plan_embed_kernel (a1 + a2 in one launch, each row CTA scanning the batch itself) writes the same
    row tables, work items and h0 / a as plan_kernel + embed_norm_vec_kernel (SV_SPLIT_PLAN=1): the
    verify's outputs and every tapped intermediate agree bit for bit."""
    cfg = synth.TOY_MLP
    d = synth.random_tokens(2 + 5 + 0 + 3, cfg.vocab, seed=21)
    res = []
    for split in (False, True):
        if split:
            monkeypatch.setenv("SV_SPLIT_PLAN", "1")
        else:
            monkeypatch.delenv("SV_SPLIT_PLAN", raising=False)
        S = Setup(cfg, [50, 90, 7, 130], seed=12)
        a, t = [x.cpu().clone() for x in S.lane.verify([0, 1, 2, 3], [2, 5, 0, 3], d.cuda(), mode=mode, seed=8)]
        T = 2 + 5 + 0 + 3 + 4
        taps = [S.tap("h0", torch.float32, (T, cfg.d_model)), S.tap("a", torch.bfloat16, (T, cfg.d_model)),
                S.tap("o", torch.bfloat16, (T, cfg.n_q_heads * cfg.head_dim))]
        S.lane.commit()
        res.append((a, t, taps))
    (a0, t0, x0), (a1, t1, x1) = res
    assert torch.equal(a0, a1) and torch.equal(t0, t1)
    for u, v in zip(x0, x1):
        assert torch.equal(u, v)
