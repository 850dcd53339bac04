"""CUDA-graph replay of a fixed step (sv_graph_*): a captured planted-drafter + verify + commit step
replayed N times gives exactly the outputs, lane counters and cache lengths of the same N steps run
eagerly (per-step drafter inputs refreshed in the buffers the graph reads), in greedy and sampled
mode; capture rules (created stream, committed verify) are enforced."""
import pytest
import torch

import synth
from paper_2604_09562_b200 import sv

pytestmark = pytest.mark.gpu


def _lane(cfg, w, stream):
    lane = sv.Lane(cfg, {k: v.cuda() for k, v in w.items()}, stream=stream)
    for i in range(4):
        k, v = synth.context_kv(cfg, 50 + 30 * i, seed=10 + i)
        lane.append_kv(i, 100 + i, k.cuda(), v.cuda(), 3 + i)
    return lane


@pytest.mark.parametrize("mode", ["greedy", "sample"])
def test_graph_replay_equals_eager_steps(mode):
    cfg = synth.TOY_MLP
    w = synth.model_weights(cfg, seed=0, norm_one=False)
    w, succ = synth.planted_successor(cfg, w, seed=1, beta=0.3)
    depths = [4, 2, 3, 1]
    rows = sum(depths)
    n = 6
    masks, devtok = synth.planted_masks(n, rows, 0.7, cfg.vocab, seed=2)
    outs = {}
    for kind in ("eager", "graph"):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            lane = _lane(cfg, w, stream)
            succ_d = succ.cuda()
            m_stage = torch.empty(rows, dtype=torch.uint8, device="cuda")
            t_stage = torch.empty(rows, dtype=torch.int32, device="cuda")
            drafts = torch.empty(rows, dtype=torch.int32, device="cuda")
            acc = torch.empty(4, dtype=torch.int32, device="cuda")
            tok = torch.empty(4, cfg.max_depth + 1, dtype=torch.int32, device="cuda")

            def step():
                lane.draft_planted([0, 1, 2, 3], depths, succ_d, m_stage, t_stage, drafts)
                lane.verify([0, 1, 2, 3], depths, drafts, None, seed=77, mode=mode, temperature=0.9, out=(acc, tok))
                lane.commit()

            res = []
            g = None
            for i in range(n):
                m_stage.copy_(masks[i].cuda())
                t_stage.copy_(devtok[i].cuda())
                if kind == "eager" or i == 0:
                    step()                               # (the graph lane's step 0 warms every kernel up)
                elif g is None:
                    lane.graph_begin()
                    step()                               # captured, not run
                    g = lane.graph_end()
                    lane.graph_launch(g)
                else:
                    lane.graph_launch(g)
                stream.synchronize()
                res.append((acc.cpu().clone(), tok.cpu().clone()))
            st = lane.stats()
            ln = lane.tap("len", torch.int32, (cfg.max_slots,))[:4].cpu().clone()
            if g is not None:
                lane.graph_destroy(g)
            lane.close()
        outs[kind] = (res, st, ln)
    (re, se, le), (rg, sg, lg) = outs["eager"], outs["graph"]
    for i in range(n):
        assert torch.equal(re[i][0], rg[i][0]) and torch.equal(re[i][1], rg[i][1]), i
    assert se == sg and torch.equal(le, lg)
    assert se["steps"] == n and (mode == "sample" or se["accepted"] > 0)


def test_graph_replay_of_a_filtered_sampled_tree_verify():
    """A token-tree verify with a top-k / top-p filtered target (R30 + R31), captured and replayed,
    equals the same calls run eagerly (the filter and the tree walk run inside the graph)."""
    cfg = synth.TOY_MLP
    w = synth.model_weights(cfg, seed=4, norm_one=False)
    parents = [0, 0, 1, 1, 2, 0]
    depths = [len(parents)] * 4
    par = torch.tensor(parents * 4, dtype=torch.int32)
    n = 4
    draws = [synth.random_tokens(sum(depths), cfg.vocab, seed=20 + i) for i in range(n)]
    outs = {}
    for kind in ("eager", "graph"):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            lane = _lane(cfg, w, stream)
            lane.set_filter(40, 0.9)
            par_d = par.cuda()
            d_stage = torch.empty(sum(depths), dtype=torch.int32, device="cuda")
            acc = torch.empty(4, dtype=torch.int32, device="cuda")
            tok = torch.empty(4, cfg.max_depth + 1, dtype=torch.int32, device="cuda")

            def step():
                lane.verify_tree([0, 1, 2, 3], depths, par_d, d_stage, None, seed=5, mode="sample", temperature=0.8,
                                 out=(acc, tok))
                lane.commit()

            res, g = [], None
            for i in range(n):
                d_stage.copy_(draws[i].cuda())
                if kind == "eager" or i == 0:
                    step()
                elif g is None:
                    lane.graph_begin()
                    step()
                    g = lane.graph_end()
                    lane.graph_launch(g)
                else:
                    lane.graph_launch(g)
                stream.synchronize()
                res.append((acc.cpu().clone(), tok.cpu().clone()))
            st = lane.stats()
            if g is not None:
                lane.graph_destroy(g)
            lane.close()
        outs[kind] = (res, st)
    for i in range(n):
        assert torch.equal(outs["eager"][0][i][0], outs["graph"][0][i][0])
        assert torch.equal(outs["eager"][0][i][1], outs["graph"][0][i][1])
    assert outs["eager"][1] == outs["graph"][1]


def test_graph_capture_rules():
    cfg = synth.TOY
    w = synth.model_weights(cfg, seed=0)
    lane = _lane(cfg, w, torch.cuda.current_stream())        # legacy default stream: not capturable
    with pytest.raises(sv.SvError):
        lane.graph_begin()
    lane.close()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        lane = _lane(cfg, w, stream)
        d = synth.random_tokens(4, cfg.vocab, seed=3).cuda()
        lane.verify([0], [4], d)                          # warm-up (and committed)
        lane.commit()
        lane.graph_begin()
        lane.verify([0], [4], d)                          # captured verify left uncommitted
        with pytest.raises(sv.SvError):
            lane.graph_end()
        lane.close()


@pytest.mark.parametrize("cfgname,mode", [("toy_mlp", "sample"), ("llama", "greedy"), ("llama", "sample")])
def test_dynamic_graph_any_depth_vector(cfgname, mode):
    """sv_graph_begin_dynamic: ONE captured drafter + verify + commit step replayed with a different
    depth vector (and slot order) every step (sv_graph_set_batch) gives exactly the outputs, counters
    and cache lengths of the same steps run eagerly — SURVEY.md §8(b) "one CUDA graph must serve any
    depth vector"."""
    if cfgname == "llama":
        cfg = synth.LLAMA.with_(n_pages=64, max_slots=4, max_batch=4, max_pos=1024)
    else:
        cfg = synth.TOY_MLP
    w = synth.model_weights(cfg, seed=0, norm_one=False, embed_std=4.0)
    w, succ = synth.planted_successor(cfg, w, seed=1, beta=0.3)
    n = 7
    g_ = torch.Generator().manual_seed(5)
    depths = [[int(x) for x in torch.randint(0, cfg.max_depth + 1, (4,), generator=g_)] for _ in range(n)]
    depths[2] = [cfg.max_depth] * 4
    depths[3] = [0, 0, 0, 0]
    orders = [[0, 1, 2, 3], [2, 0, 3, 1], [3, 2, 1, 0], [1, 3, 0, 2]] * 2
    rows = 4 * cfg.max_depth
    masks, devtok = synth.planted_masks(n, rows, 0.7, cfg.vocab, seed=2)
    outs = {}
    for kind in ("eager", "graph"):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            lane = _lane(cfg, w, stream)
            succ_d = succ.cuda()
            m_stage = torch.empty(rows, dtype=torch.uint8, device="cuda")
            t_stage = torch.empty(rows, dtype=torch.int32, device="cuda")
            drafts = torch.empty(rows, dtype=torch.int32, device="cuda")
            acc = torch.empty(4, dtype=torch.int32, device="cuda")
            tok = torch.empty(4, cfg.max_depth + 1, dtype=torch.int32, device="cuda")

            def step(slots, ks):
                lane.draft_planted(slots, ks, succ_d, m_stage, t_stage, drafts)
                lane.verify(slots, ks, drafts, None, seed=77, mode=mode, temperature=0.9, out=(acc, tok))
                lane.commit()

            res, g = [], None
            for i in range(n):
                m_stage.copy_(masks[i].cuda())
                t_stage.copy_(devtok[i].cuda())
                if kind == "eager":
                    step(orders[i], depths[i])
                else:
                    if g is None:
                        lane.graph_begin_dynamic(4)
                        step([0, 1, 2, 3], [1, 1, 1, 1])        # captured, not run
                        g = lane.graph_end()
                    lane.graph_set_batch(g, orders[i], depths[i])
                    lane.graph_launch(g)
                torch.cuda.synchronize()
                res.append((acc.cpu().clone(), tok.cpu().clone(),
                            lane.tap("len", torch.int32, (cfg.max_slots,)).cpu().clone()))
            st = lane.stats()
            if g is not None:
                lane.graph_destroy(g)
            outs[kind] = (res, st)
    for i, (a, b) in enumerate(zip(outs["eager"][0], outs["graph"][0])):
        for x, y in zip(a, b):
            assert torch.equal(x, y), (i, depths[i], x, y)
    assert outs["eager"][1] == outs["graph"][1]
    assert outs["eager"][1]["drafted"] == sum(sum(k) for k in depths)


def test_profiled_graph_times_every_replay():
    """Stages timed while capturing become event-record nodes that each replay re-points at fresh
    events: sv_profile_read counts one launch per replay with a positive time, while the profile stays
    on; replays after sv_profile_enable(0) add nothing. Outputs equal an unprofiled graph's."""
    cfg = synth.TOY_MLP
    w = synth.model_weights(cfg, seed=0, norm_one=False)
    w, succ = synth.planted_successor(cfg, w, seed=1, beta=0.3)
    depths = [4, 2, 3, 1]
    rows = sum(depths)
    masks, devtok = synth.planted_masks(8, rows, 0.7, cfg.vocab, seed=2)
    outs = []
    for profiled in (True, False):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            lane = _lane(cfg, w, stream)
            succ_d = succ.cuda()
            m_stage = torch.empty(rows, dtype=torch.uint8, device="cuda")
            t_stage = torch.empty(rows, dtype=torch.int32, device="cuda")
            drafts = torch.empty(rows, dtype=torch.int32, device="cuda")
            acc = torch.empty(4, dtype=torch.int32, device="cuda")
            tok = torch.empty(4, cfg.max_depth + 1, dtype=torch.int32, device="cuda")

            def step():
                lane.draft_planted([0, 1, 2, 3], depths, succ_d, m_stage, t_stage, drafts)
                lane.verify([0, 1, 2, 3], depths, drafts, None, seed=5, mode="greedy", out=(acc, tok))
                lane.commit()

            m_stage.copy_(masks[0].cuda())
            t_stage.copy_(devtok[0].cuda())
            step()
            if profiled:
                lane.profile(["lm_head", "attention"])
            lane.graph_begin()
            step()                                       # captured, not run
            g = lane.graph_end()
            lane.profile_read(reset=True)
            res = []
            for i in range(1, 6):
                m_stage.copy_(masks[i].cuda())
                t_stage.copy_(devtok[i].cuda())
                lane.graph_launch(g)
                res.append((acc.clone(), tok.clone()))
            prof = lane.profile_read(reset=True)
            if profiled:
                assert prof["lm_head"][1] == 5 and prof["attention"][1] == 5
                assert prof["lm_head"][0] > 0 and prof["attention"][0] > 0
                lane.profile(False)
                lane.graph_launch(g)
                assert lane.profile_read(reset=True)["lm_head"][1] == 0
            else:
                assert all(n == 0 for _, n in prof.values())
                lane.graph_launch(g)
            torch.cuda.synchronize()
            outs.append([(a.cpu(), t.cpu()) for a, t in res])
            lane.graph_destroy(g)
    for (a0, t0), (a1, t1) in zip(*outs):
        assert torch.equal(a0, a1) and torch.equal(t0, t1)


def test_two_dynamic_graphs_alternate():
    """Two dynamic-depth graphs of the same step (one with event-timed stages, one without) share the
    lane's two staging buffers: alternating them with per-replay depth vectors gives exactly the eager
    steps; a second staging of a graph before its launch is refused, and so is a launch without one."""
    cfg = synth.TOY_MLP
    w = synth.model_weights(cfg, seed=0, norm_one=False)
    w, succ = synth.planted_successor(cfg, w, seed=1, beta=0.3)
    n = 8
    g_ = torch.Generator().manual_seed(5)
    depths = [[int(x) for x in torch.randint(0, 5, (4,), generator=g_)] for _ in range(n)]
    orders = [[int(x) for x in torch.randperm(4, generator=g_)] for _ in range(n)]
    masks, devtok = synth.planted_masks(n, 4 * 4, 0.7, cfg.vocab, seed=2)
    outs = {}
    for kind in ("eager", "graphs"):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            lane = _lane(cfg, w, stream)
            succ_d = succ.cuda()
            m_stage = torch.empty(16, dtype=torch.uint8, device="cuda")
            t_stage = torch.empty(16, dtype=torch.int32, device="cuda")
            drafts = torch.empty(16, dtype=torch.int32, device="cuda")
            acc = torch.empty(4, dtype=torch.int32, device="cuda")
            tok = torch.empty(4, cfg.max_depth + 1, dtype=torch.int32, device="cuda")

            def step(sl, ks):
                lane.draft_planted(sl, ks, succ_d, m_stage, t_stage, drafts)
                lane.verify(sl, ks, drafts, None, seed=3, mode="greedy", out=(acc, tok))
                lane.commit()

            gs = []
            if kind == "graphs":
                lane.profile(["lm_head"])
                for _ in range(2):
                    lane.graph_begin_dynamic(4)
                    step([0, 1, 2, 3], [1, 1, 1, 1])      # captured, not run
                    gs.append(lane.graph_end())
                    lane.profile(False)
                with pytest.raises(sv.SvError):
                    lane.graph_launch(gs[0])             # nothing staged
            res = []
            for i in range(n):
                m_stage.copy_(masks[i].cuda())
                t_stage.copy_(devtok[i].cuda())
                if kind == "eager":
                    step(orders[i], depths[i])
                else:
                    g = gs[i % 2]
                    lane.graph_set_batch(g, orders[i], depths[i])
                    if i == 0:
                        with pytest.raises(sv.SvError):
                            lane.graph_set_batch(g, orders[i], depths[i])   # staged, not yet launched
                    lane.graph_launch(g)
                torch.cuda.synchronize()
                res.append((acc.cpu().clone(), tok.cpu().clone()))
            for g in gs:
                lane.graph_destroy(g)
            outs[kind] = (res, lane.stats())
    for (a0, t0), (a1, t1) in zip(outs["eager"][0], outs["graphs"][0]):
        assert torch.equal(a0, a1) and torch.equal(t0, t1)
    assert outs["eager"][1] == outs["graphs"][1]
