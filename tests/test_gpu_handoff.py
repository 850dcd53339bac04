"""a9 prefill -> decode KV hand-off (PAPER.md:255-267 eq:kv_concatenation).

A request's context KV reaches a decode lane either through sv_append_kv (unpacked) or as a
hand-off message (sv_kv_pack wire format) appended by sv_kv_append_packed / received over NCCL.
The appended state must be indistinguishable: a verify on it gives bitwise-identical outputs.
The NCCL path runs on one GPU as a single-rank loopback (send to self + receive in one group)."""
import pytest
import torch

import synth
from paper_2604_09562_b200 import sv

pytestmark = pytest.mark.gpu


def _lane(cfg, w):
    lane = sv.Lane(cfg, w)
    lane.set_taps(True)
    return lane


def _verify(lane, slots, depths, drafts, V):
    lo = torch.empty(sum(depths) + len(depths), V, device="cuda")
    acc, tok = lane.verify(slots, depths, drafts, None, mode="sample", seed=77, logits_out=lo)
    torch.cuda.synchronize()
    return acc.cpu().clone(), tok.cpu().clone(), lo.cpu().clone()


@pytest.mark.parametrize("transport", ["packed", "nccl_loopback"])
def test_handoff_equals_direct_append(transport):
    cfg = synth.TOY_MLP.with_(n_layers=2, n_pages=64)
    w = {k: v.cuda() for k, v in synth.model_weights(cfg, seed=31).items()}
    ctx = [(300, 1001, 17), (64, 1002, 3), (1, 1003, 250)]        # (n_tokens, request id, pending token)
    direct, handed = _lane(cfg, w), _lane(cfg, w)
    comm = None
    if transport == "nccl_loopback":
        comm = sv.nccl_comm_init(1, sv.nccl_unique_id(), 0)
    try:
        for slot, (n, rid, pend) in enumerate(ctx):
            k, v = synth.context_kv(cfg, n, seed=40 + slot)
            k, v = k.cuda(), v.cuda()
            direct.append_kv(slot, rid, k, v, pend)
            nb = handed.packed_bytes(n)
            packed = torch.empty(nb, dtype=torch.uint8, device="cuda")
            sv.kv_pack(k, v, pend, packed)
            if transport == "packed":
                handed.kv_append_packed(slot, rid, n, packed)
            else:
                staging = torch.empty(nb, dtype=torch.uint8, device="cuda")
                handed.kv_loopback_append(slot, rid, n, packed, staging, 0, comm)
        torch.cuda.synchronize()
        for name in ("len", "pending"):
            assert torch.equal(direct.tap(name, torch.int32, (cfg.max_slots,)),
                               handed.tap(name, torch.int32, (cfg.max_slots,))), name
        slots, depths = [0, 1, 2], [3, 1, 4]
        drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=41).cuda()
        a = _verify(direct, slots, depths, drafts, cfg.vocab)
        b = _verify(handed, slots, depths, drafts, cfg.vocab)
        for x, y in zip(a, b):
            assert torch.equal(x, y)
    finally:
        if comm is not None:
            sv.nccl_comm_destroy(comm)


def test_pack_wire_format():
    """[n_layers][n][2][H_kv][d_h] bf16 followed by the 16-byte trailer {pending, 0, 0, 0}."""
    cfg = synth.TOY_MLP.with_(n_layers=2)
    n = 5
    k, v = synth.context_kv(cfg, n, seed=50)
    packed = torch.empty(sv.packed_bytes(cfg, n), dtype=torch.uint8, device="cuda")
    sv.kv_pack(k.cuda(), v.cuda(), 123, packed)
    torch.cuda.synchronize()
    body = packed[:-16].view(torch.bfloat16).view(cfg.n_layers, n, 2, cfg.n_kv_heads, cfg.head_dim).cpu()
    assert torch.equal(body[:, :, 0], k) and torch.equal(body[:, :, 1], v)
    assert packed[-16:].view(torch.int32).cpu().tolist()[0] == 123


def _dense(lane, cfg, slot):
    """A slot's committed K/V [n_layers][L][Hkv][dh] read back through its page table."""
    torch.cuda.synchronize()
    ln = int(lane.tap("len", torch.int32, (cfg.max_slots,))[slot])
    mpps = (cfg.max_pos + cfg.page_size - 1) // cfg.page_size
    pt = lane.tap("page_table", torch.int32, (cfg.max_slots, mpps))[slot].cpu()
    pool = lane.kv_pool.view(torch.bfloat16).view(cfg.n_layers, cfg.n_pages, 2, cfg.n_kv_heads, cfg.page_size,
                                                  cfg.head_dim)
    t = torch.arange(ln)
    pages, offs = pt[t // cfg.page_size].long().cuda(), (t % cfg.page_size).cuda()
    k = torch.stack([pool[l, pages, 0, :, offs] for l in range(cfg.n_layers)]).cpu()    # [n_layers][L][Hkv][dh]
    v = torch.stack([pool[l, pages, 1, :, offs] for l in range(cfg.n_layers)]).cpu()
    return k, v, ln


@pytest.mark.parametrize("cfgname", ["toy_mlp_2layer", "llama"])
def test_batched_handoff_loopback(cfgname):
    """sv_kv_send_slots / sv_kv_recv_slots (one NCCL op per batch: page blocks gathered from the
    prefill lane's pages, scattered into the decode lane's popped pages) on one GPU via
    sv_kv_loopback_slots:
    every transferred row bitwise equal (a9 criterion), len / pending / request id as sent, and
    verifies on the received slots bitwise equal to a lane filled by sv_append_kv. A verify of other
    slots is enqueued on the decode lane before the transfer (it overlaps on the comm stream) and is
    itself unaffected."""
    if cfgname == "llama":
        cfg = synth.LLAMA.with_(n_pages=96, max_slots=6, max_batch=6, max_pos=2048)
    else:
        cfg = synth.TOY_MLP.with_(n_layers=2, n_pages=96, max_slots=6, max_batch=6)
    w = {k: v.cuda() for k, v in synth.model_weights(cfg, seed=32).items()}
    pre, dec, ref = _lane(cfg, w), _lane(cfg, w), _lane(cfg, w)
    comm = sv.nccl_comm_init(1, sv.nccl_unique_id(), 0)
    try:
        reqs = [(700, 2001, 5), (64, 2002, 9), (1, 2003, 11), (129, 2004, 13)]   # (n, rid, pending)
        kvs = []
        for slot, (n, rid, pend) in enumerate(reqs):
            k, v = synth.context_kv(cfg, n, seed=60 + slot)
            kvs.append((k, v))
            pre.append_kv(slot + 1, rid, k.cuda(), v.cuda(), pend)       # prefill lane slots 1..4
            ref.append_kv(slot, rid, k.cuda(), v.cuda(), pend)
        # decode lane already serves one request (slot 5) and has a verify in flight
        kx, vx = synth.context_kv(cfg, 200, seed=70)
        dec.append_kv(5, 3001, kx.cuda(), vx.cuda(), 1)
        ref.append_kv(5, 3001, kx.cuda(), vx.cuda(), 1)
        dx = synth.random_tokens(3, cfg.vocab, seed=71).cuda()
        a0 = dec.verify([5], [3], dx, mode="greedy")
        ntok = [r[0] for r in reqs]
        nb = pre.slots_bytes(ntok)
        blk = 2 * cfg.n_kv_heads * cfg.page_size * cfg.head_dim * 2
        assert nb == cfg.n_layers * sum((n + 63) // 64 for n in ntok) * blk + 16
        st_src = torch.empty(nb, dtype=torch.uint8, device="cuda")
        st_dst = torch.empty(nb, dtype=torch.uint8, device="cuda")
        pre.kv_loopback_slots(dec, [1, 2, 3, 4], [0, 1, 2, 3], [r[1] for r in reqs], ntok, st_src, st_dst, 0, comm)
        dec.commit()
        a1 = ref.verify([5], [3], dx, mode="greedy")
        ref.commit()
        torch.cuda.synchronize()
        assert torch.equal(a0[0].cpu(), a1[0].cpu()) and torch.equal(a0[1].cpu(), a1[1].cpu())
        for slot, (n, rid, pend) in enumerate(reqs):
            k, v, ln = _dense(dec, cfg, slot)
            assert ln == n
            assert torch.equal(k, kvs[slot][0]) and torch.equal(v, kvs[slot][1])
        pend_d = dec.tap("pending", torch.int32, (cfg.max_slots,)).cpu()
        assert [int(pend_d[s]) for s in range(4)] == [r[2] for r in reqs]
        slots, depths = [0, 1, 2, 3], [3, 1, 4, 2]
        drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=72).cuda()
        a = _verify(dec, slots, depths, drafts, cfg.vocab)
        b = _verify(ref, slots, depths, drafts, cfg.vocab)
        for x, y in zip(a, b):
            assert torch.equal(x, y)
        dec.commit()
        ref.commit()
        # misuse is refused before anything is posted
        with pytest.raises(sv.SvError) as e:                 # destination slot not EMPTY
            pre.kv_loopback_slots(dec, [1], [0], [9], [10], st_src, st_dst, 0, comm)
        assert e.value.status == sv.SV_ESTATE
        with pytest.raises(sv.SvError) as e:                 # more rows than the source slot holds
            pre.kv_loopback_slots(dec, [2], [4], [9], [65], st_src, st_dst, 0, comm)
        assert e.value.status == sv.SV_EINVAL
        tiny = _lane(cfg.with_(n_pages=4), w)                # 700 tokens need 11 pages: refused, nothing popped
        with pytest.raises(sv.SvError) as e:
            pre.kv_loopback_slots(tiny, [1], [0], [9], [700], st_src, st_dst, 0, comm)
        assert e.value.status == sv.SV_ENOKV
        assert tiny.occupancy() == (0, 4)
        # the sender's slots can be released after the send (release waits for the transfer)
        for s in range(1, 5):
            pre.release(s)
        torch.cuda.synchronize()
    finally:
        sv.nccl_comm_destroy(comm)
