"""Multi-lane host logic on CPU with torch.distributed gloo, world_size 2."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_09562_b200 import dist as svdist


def test_shard_partition_properties():
    for n in (0, 1, 7, 64, 65, 320):
        for world in (1, 2, 3, 4, 8):
            parts = [svdist.shard(n, r, world) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))                    # every request exactly once, in order
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1              # balanced
    ids = {svdist.request_id(r, i) for r in range(8) for i in range(1000)}
    assert len(ids) == 8000 and min(ids) > 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _route_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # lane r publishes (timestamp, C, M, Q, L); lane 1 is busier
        local = (1000, 0.0, 0.3 + 0.4 * rank, 5.0 + 20.0 * rank, 0.5 + 0.3 * rank)
        metrics = svdist.gather_metrics(local)
        assign = svdist.route_requests(12, metrics, 1200) if rank == 0 else None
        blob = svdist.broadcast_bytes(bytes(assign) if assign is not None else None, src=0, nbytes=12)
        q.put((rank, metrics, list(blob)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_flowguard_admission_routing():
    from oracle import flowguard as fg
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_route_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]        # every rank sees the same metrics / routes
    metrics = [fg.WorkerMetrics(*m) for m in res[0][1]]
    live, want = [m.queue_depth for m in metrics], []
    for _ in range(12):                                               # oracle: Alg. 2 per admission
        d = fg.select_worker(metrics, live, 1200, fg.RouteConfig())
        want.append(d.chosen)
        live[d.chosen] += 1
    assert res[0][2] == want
    assert 0 in want                                                  # the idle lane takes requests


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # per-lane timed region: lane r took (r + 1) * 10 ms and emitted 100 * (r + 1) tokens
        el, tok = svdist.reduce_region(10.0 * (rank + 1), 100 * (rank + 1))
        uid = bytes(range(128)) if rank == 0 else None
        got = svdist.broadcast_bytes(uid, src=0, nbytes=128)
        mine = svdist.shard(64, rank, world)
        q.put((rank, el, tok, got == bytes(range(128)), mine))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_reduction_and_id_broadcast():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    res.sort()
    for rank, el, tok, id_ok, mine in res:
        assert el == 20.0 and tok == 300.0                # max elapsed, total tokens: identical on all ranks
        assert id_ok
    assert res[0][4] + res[1][4] == list(range(64))


def test_reduce_region_without_process_group():
    assert svdist.reduce_region(3.5, 7) == (3.5, 7.0)


def test_disagg_roles_and_handoff_plan():
    from paper_2604_09562_b200 import dist as svdist
    assert svdist.disagg_role(0, 1) == ("both", 0, 0)
    roles = [svdist.disagg_role(r, 8) for r in range(8)]
    assert [r[0] for r in roles] == ["prefill", "decode"] * 4
    assert [r[1] for r in roles] == [1, 0, 3, 2, 5, 4, 7, 6] and [r[2] for r in roles] == [0, 0, 1, 1, 2, 2, 3, 3]
    with pytest.raises(ValueError):
        svdist.disagg_role(0, 3)
    s0, d0, r0 = svdist.handoff_batch(0, 4, 2)
    s1, d1, r1 = svdist.handoff_batch(1, 4, 2)
    assert s0 == s1 == [0, 1, 2, 3] and d0 == [0, 1, 2, 3] and d1 == [4, 5, 6, 7]
    assert len(set(r0 + r1)) == 8 and all(r >> 32 == 2 for r in r0 + r1)
