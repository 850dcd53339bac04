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
