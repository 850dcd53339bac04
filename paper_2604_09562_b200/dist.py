"""Host logic of the multi-lane (multi-GPU) path.

Requests shard across decode lanes, one process per GPU, with no collective inside the verify
step (outputs are lane-count invariant: every draw is keyed by the request id). The collectives
here are all off the data path: the max-over-ranks timing / total-token reduction of a measured
region, and the broadcast of the NCCL unique id that sets up a hand-off communicator (a9).
Works with any torch.distributed backend (NCCL on the GPU box, gloo in the CPU tests).
"""
import torch
import torch.distributed as dist


def shard(n_global, rank, world):
    """Contiguous block partition of n_global requests over `world` lanes; lane `rank`'s indices."""
    base, extra = divmod(n_global, world)
    lo = rank * base + min(rank, extra)
    return list(range(lo, lo + base + (1 if rank < extra else 0)))


def request_id(rank, i):
    """Globally unique request id of the i-th request of lane `rank` (the Philox key)."""
    return (int(rank) << 32) | (int(i) + 1)


def reduce_region(elapsed, tokens, device=None, group=None):
    """(max elapsed over ranks, total tokens over ranks) of a timed region; identity when not
    initialised. elapsed in any time unit; the job's throughput is tokens / elapsed."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(elapsed), float(tokens)
    t = torch.tensor([float(elapsed)], dtype=torch.float64, device=device)
    n = torch.tensor([float(tokens)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(n, op=dist.ReduceOp.SUM, group=group)
    return float(t.item()), float(n.item())


def broadcast_bytes(payload, src, nbytes, device=None, group=None):
    """Broadcast a fixed-size byte string (e.g. the 128-byte NCCL unique id) from rank `src`."""
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == src:
        assert payload is not None and len(payload) == nbytes
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, src=src, group=group)
    return bytes(buf.cpu().numpy().tobytes())


# ---------------------------------------------------------------- FlowGuard routing across lanes
def lane_metrics(lane, cfg, queue_depth, now_ms, cache_hit=0.0):
    """A lane's published FlowGuard signals (Table 2 / eq:flowguard_score): memory
    utilisation = KV pages in use / pool, load = occupied slots / slots, the lane's queue depth,
    and the cache hit rate (0: no prefix-cache reuse in this system). Syncs the lane's stream."""
    active, free = lane.occupancy()
    return (int(now_ms), float(cache_hit), 1.0 - free / cfg.n_pages, float(queue_depth), active / cfg.max_slots)


def gather_metrics(local, device=None, group=None):
    """all_gather of every lane's 5-field metrics tuple (SURVEY.md §8(e) exchange 2, off the hot path)."""
    t = torch.tensor([float(x) for x in local], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [(int(o[0].item()), float(o[1]), float(o[2]), float(o[3]), float(o[4])) for o in out]


def route_requests(n_requests, metrics, now_ms, cfg=None):
    """Admission routing of n new requests with FlowGuard (Alg. 2, in libsv): each assignment adds
    one to the chosen lane's live queue depth before the next request is routed."""
    from . import flowguard
    live = [m[3] for m in metrics]
    out = []
    for _ in range(n_requests):
        chosen, _, _, _ = flowguard.select(metrics, live, now_ms, cfg)
        out.append(chosen)
        live[chosen] += 1
    return out


# ---------------------------------------------------------------- disaggregated prefill -> decode pairs
def disagg_role(rank, world):
    """Zero-based stream pairs (2p, 2p+1) (PAPER.md:162 vs 437; R14): even ranks prefill,
    odd ranks decode; returns (role, peer rank, pair index). world == 1: both roles on one rank
    (the one-GPU loopback used to validate the flow)."""
    if world == 1:
        return "both", 0, 0
    if world % 2:
        raise ValueError("disaggregated pairs need an even number of ranks")
    return ("prefill", rank + 1, rank // 2) if rank % 2 == 0 else ("decode", rank - 1, rank // 2)


def handoff_batch(round_i, batch, prefill_rank):
    """Slot plan of hand-off batch `round_i` of a (prefill, decode) pair: the prefill lane sends its
    slots 0..batch-1; the decode lane receives into the half of its 2*batch slots that is not being
    decoded (double buffer), with fresh request ids (the Philox keys) for the new requests."""
    base = (round_i % 2) * batch
    return (list(range(batch)), [base + i for i in range(batch)],
            [request_id(prefill_rank, round_i * batch + i) for i in range(batch)])
