"""Thin ctypes binding over libsv.so (include/sv.h). Argument marshalling only:
every step of the verify path runs in the library's CUDA kernels. PyTorch
supplies device memory, the stream and process groups.

    lane = Lane(cfg, weights)                        # weights: dict of cuda bf16 tensors
    lane.append_kv(slot, request_id, k, v, pending)  # k, v: [n_layers][n][Hkv][dh] bf16 (cuda)
    acc, toks = lane.verify(slots, depths, draft_tokens, draft_probs=None, seed=0, mode="sample")
    lane.commit()
    lane.stats()

There is no CPU fallback: importing without a built libsv.so, or calling on a
machine without a CUDA device, raises.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SV_LIBSV", os.path.join(_HERE, "libsv.so"))   # override: experiments only

SV_OK, SV_EINVAL, SV_ESTATE, SV_ENOKV, SV_ECUDA, SV_ENCCL, SV_EDEVICE = range(7)
GREEDY, SAMPLE, PREFILL = 0, 1, 2
_STATUS = {0: "SV_OK", 1: "SV_EINVAL", 2: "SV_ESTATE", 3: "SV_ENOKV", 4: "SV_ECUDA", 5: "SV_ENCCL", 6: "SV_EDEVICE"}

EXPORTED = [
    "sv_version", "sv_strerror", "sv_query_sizes", "sv_create", "sv_destroy", "sv_append_kv", "sv_verify",
    "sv_verify_logits", "sv_commit", "sv_release", "sv_stats", "sv_set_taps", "sv_get_tap", "sv_debug_uniforms",
    "sv_draft_planted", "sv_nccl_unique_id", "sv_nccl_comm_init", "sv_nccl_comm_destroy", "sv_kv_send",
    "sv_kv_recv_append", "sv_kv_packed_bytes", "sv_kv_pack", "sv_profile_enable", "sv_profile_num_stages",
    "sv_profile_stage_name", "sv_profile_read", "sv_launch_count", "sv_debug_gemm", "sv_kv_append_packed",
    "sv_kv_loopback_append", "sv_kv_send_slots", "sv_kv_recv_slots", "sv_kv_loopback_slots", "sv_comm_stream", "sv_kv_slots_bytes", "sv_exact_query_sizes", "sv_exact_forward", "sv_graph_begin_dynamic", "sv_graph_set_batch", "sv_spec_default_config", "sv_spec_reset", "sv_spec_adapt", "sv_spec_step",
    "sv_route_default_config", "sv_route_select", "sv_lane_occupancy", "sv_kv_pack_slot", "sv_prefill",
    "sv_verify_tree", "sv_verify_tree_logits", "sv_set_filter", "sv_draft_planted_tree", "sv_graph_begin",
    "sv_graph_end", "sv_graph_launch", "sv_graph_destroy",
]


class SvError(RuntimeError):
    def __init__(self, status, what):
        self.status = status
        super().__init__(f"{what}: {_STATUS.get(status, status)} ({strerror(status)})")


class Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("n_layers", "d_model", "n_q_heads", "n_kv_heads", "head_dim",
                                              "vocab", "ffn_dim")] + \
               [("rope_theta", ctypes.c_float), ("norm_eps", ctypes.c_float)] + \
               [(n, ctypes.c_int32) for n in ("page_size", "n_pages", "max_slots", "max_batch", "max_depth",
                                              "max_pos")]

    @classmethod
    def from_any(cls, c):
        get = (lambda k: c[k]) if isinstance(c, dict) else (lambda k: getattr(c, k))
        return cls(**{n: get(n) for n, _ in cls._fields_})


WEIGHT_NAMES = ("embed", "attn_norm", "wqkv", "wo", "ffn_norm", "w_gate_up", "w_down", "final_norm", "lm_head")


class Weights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in WEIGHT_NAMES]


class LaneStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("steps", "rows", "drafted", "accepted", "emitted",
                                               "accepted_independent")] + \
               [("hist_accepted", ctypes.c_uint64 * 33), ("drafted_by_k", ctypes.c_uint64 * 33),
                ("accepted_by_k", ctypes.c_uint64 * 33), ("device_error", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]

    def as_dict(self):
        d = {n: int(getattr(self, n)) for n in ("steps", "rows", "drafted", "accepted", "emitted",
                                               "accepted_independent", "device_error")}
        for n in ("hist_accepted", "drafted_by_k", "accepted_by_k"):
            d[n] = [int(x) for x in getattr(self, n)]
        return d


_lib = None


def load():
    """Load libsv.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2604_09562_b200.build`")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, u64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    sig = {
        "sv_version": ([], ctypes.c_char_p),
        "sv_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "sv_query_sizes": ([P(Config), P(sz), P(sz)], ctypes.c_int),
        "sv_create": ([P(Config), P(Weights), vp, vp, vp, P(vp)], ctypes.c_int),
        "sv_destroy": ([vp], ctypes.c_int),
        "sv_append_kv": ([vp, i32, u64, vp, vp, i32, i32], ctypes.c_int),
        "sv_verify": ([vp, i32, P(i32), P(i32), vp, vp, u64, ctypes.c_int, ctypes.c_float, vp, vp, vp],
                      ctypes.c_int),
        "sv_verify_logits": ([vp, i32, P(i32), P(i32), vp, vp, vp, u64, ctypes.c_int, ctypes.c_float, vp, vp],
                             ctypes.c_int),
        "sv_verify_tree": ([vp, i32, P(i32), P(i32), vp, vp, vp, u64, ctypes.c_int, ctypes.c_float, vp, vp, vp, vp],
                           ctypes.c_int),
        "sv_verify_tree_logits": ([vp, i32, P(i32), P(i32), vp, vp, vp, vp, u64, ctypes.c_int, ctypes.c_float, vp,
                                   vp, vp], ctypes.c_int),
        "sv_set_filter": ([vp, i32, ctypes.c_float], ctypes.c_int),
        "sv_graph_begin": ([vp], ctypes.c_int),
        "sv_graph_end": ([vp, P(vp)], ctypes.c_int),
        "sv_graph_launch": ([vp, vp], ctypes.c_int),
        "sv_graph_destroy": ([vp], ctypes.c_int),
        "sv_commit": ([vp, vp], ctypes.c_int),
        "sv_release": ([vp, i32], ctypes.c_int),
        "sv_stats": ([vp, P(LaneStats), ctypes.c_int], ctypes.c_int),
        "sv_set_taps": ([vp, ctypes.c_int], ctypes.c_int),
        "sv_get_tap": ([vp, ctypes.c_char_p, P(vp), P(sz)], ctypes.c_int),
        "sv_debug_uniforms": ([vp, u64, u64, ctypes.c_uint32, i32, i32, i32, vp], ctypes.c_int),
        "sv_draft_planted": ([vp, i32, P(i32), P(i32), vp, vp, vp, vp], ctypes.c_int),
        "sv_draft_planted_tree": ([vp, i32, P(i32), P(i32), vp, vp, vp, vp, vp], ctypes.c_int),
        "sv_nccl_unique_id": ([ctypes.c_char_p], ctypes.c_int),
        "sv_nccl_comm_init": ([ctypes.c_int, ctypes.c_char_p, ctypes.c_int, P(vp)], ctypes.c_int),
        "sv_nccl_comm_destroy": ([vp], ctypes.c_int),
        "sv_kv_send": ([vp, i32, i32, i32, i32, ctypes.c_int, vp, vp], ctypes.c_int),
        "sv_kv_recv_append": ([vp, i32, u64, i32, vp, ctypes.c_int, vp], ctypes.c_int),
        "sv_kv_append_packed": ([vp, i32, u64, i32, vp], ctypes.c_int),
        "sv_lane_occupancy": ([vp, P(i32), P(i32)], ctypes.c_int),
        "sv_kv_pack_slot": ([vp, i32, i32, vp], ctypes.c_int),
        "sv_prefill": ([vp, i32, u64, P(i32), i32, i32, P(i32)], ctypes.c_int),
        "sv_kv_loopback_append": ([vp, i32, u64, i32, vp, vp, ctypes.c_int, vp], ctypes.c_int),
        "sv_kv_send_slots": ([vp, i32, vp, vp, vp, ctypes.c_int, vp], ctypes.c_int),
        "sv_comm_stream": ([vp, P(vp)], ctypes.c_int),
        "sv_kv_recv_slots": ([vp, i32, vp, vp, vp, vp, ctypes.c_int, vp], ctypes.c_int),
        "sv_kv_loopback_slots": ([vp, vp, i32, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp], ctypes.c_int),
        "sv_kv_slots_bytes": ([P(Config), i32, vp], sz),
        "sv_exact_query_sizes": ([P(Config), i32, P(sz)], ctypes.c_int),
        "sv_graph_begin_dynamic": ([vp, i32], ctypes.c_int),
        "sv_graph_set_batch": ([vp, vp, vp, vp], ctypes.c_int),
        "sv_exact_forward": ([P(Config), P(Weights), i32, vp, vp, vp, vp, vp, i32, vp, sz, vp, vp], ctypes.c_int),
        "sv_kv_packed_bytes": ([P(Config), i32], sz),
        "sv_kv_pack": ([vp, vp, i32, i32, i32, i32, i32, vp, vp], ctypes.c_int),
        "sv_profile_enable": ([vp, ctypes.c_int32], ctypes.c_int),
        "sv_profile_num_stages": ([], i32),
        "sv_profile_stage_name": ([i32], ctypes.c_char_p),
        "sv_profile_read": ([vp, P(ctypes.c_double), P(ctypes.c_int64), i32, ctypes.c_int], ctypes.c_int),
        "sv_launch_count": ([], u64),
        "sv_debug_gemm": ([vp, vp, vp, vp, i32, i32, i32, i32], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def strerror(status):
    try:
        return load().sv_strerror(status).decode()
    except ImportError:
        return "?"


def _check(status, what):
    if status != SV_OK:
        raise SvError(status, what)


def _i32_array(xs):
    xs = [int(x) for x in xs]
    return (ctypes.c_int32 * max(1, len(xs)))(*xs), len(xs)


def _ptr(t):
    """Device pointer of a tensor argument (marshalling only). The C ABI reads rows with 16-byte
    vector loads, so a non-contiguous view or an element offset is refused here instead of
    faulting on the device."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensor arguments must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _aligned_empty(nbytes, device, align=1024):
    buf = torch.empty(nbytes + align, dtype=torch.uint8, device=device)
    off = (-buf.data_ptr()) % align
    return buf, buf[off:off + nbytes]


class Lane:
    """One decode lane (one sv_ctx) on the current CUDA device and stream."""

    def __init__(self, cfg, weights, stream=None, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("sv.Lane needs a CUDA device (no CPU fallback)")
        self.lib = load()
        self.cfg = Config.from_any(cfg)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        kvb, wsb = ctypes.c_size_t(), ctypes.c_size_t()
        _check(self.lib.sv_query_sizes(ctypes.byref(self.cfg), ctypes.byref(kvb), ctypes.byref(wsb)),
               "sv_query_sizes")
        self._pool_raw, self.kv_pool = _aligned_empty(kvb.value, self.device)
        self._ws_raw, self.workspace = _aligned_empty(wsb.value, self.device)
        self.weights = {}
        w = Weights()
        for n in WEIGHT_NAMES:
            t = weights[n]
            if t.dtype != torch.bfloat16 or t.device.type != "cuda" or not t.is_contiguous():
                raise ValueError(f"weight {n} must be a contiguous cuda bf16 tensor")
            self.weights[n] = t
            setattr(w, n, t.data_ptr() if t.numel() else None)
        self._w = w
        ctx = ctypes.c_void_p()
        _check(self.lib.sv_create(ctypes.byref(self.cfg), ctypes.byref(w), _ptr(self.kv_pool), _ptr(self.workspace),
                                  ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(ctx)), "sv_create")
        self.ctx = ctx
        K1 = self.cfg.max_depth + 1
        self._acc = torch.empty(self.cfg.max_batch, dtype=torch.int32, device=self.device)
        self._tok = torch.empty(self.cfg.max_batch, K1, dtype=torch.int32, device=self.device)
        self._nodes = torch.empty(self.cfg.max_batch, K1, dtype=torch.int32, device=self.device)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.sv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ calls
    def append_kv(self, slot, request_id, k, v, pending_token):
        n = 0 if k is None else int(k.shape[1])
        _check(self.lib.sv_append_kv(self.ctx, slot, request_id, _ptr(k), _ptr(v), n, int(pending_token)),
               "sv_append_kv")

    @staticmethod
    def _mode(mode):
        return {"greedy": GREEDY, "sample": SAMPLE, "prefill": PREFILL}.get(mode, mode)

    def verify(self, slots, depths, draft_tokens, draft_probs=None, seed=0, mode="greedy", temperature=1.0,
               logits_out=None, out=None):
        """Returns (accepted_len [B] int32, out_tokens [B][max_depth+1] int32) device tensors."""
        s, B = _i32_array(slots)
        dpt, _ = _i32_array(depths)
        acc, tok = (self._acc[:B], self._tok[:B]) if out is None else out
        m = self._mode(mode)
        _check(self.lib.sv_verify(self.ctx, B, s, dpt, _ptr(draft_tokens), _ptr(draft_probs), seed, m,
                                  float(temperature), _ptr(acc), _ptr(tok), _ptr(logits_out)), "sv_verify")
        return acc, tok

    def verify_logits(self, slots, depths, draft_tokens, logits, draft_probs=None, seed=0, mode="greedy",
                      temperature=1.0):
        s, B = _i32_array(slots)
        dpt, _ = _i32_array(depths)
        acc, tok = self._acc[:B], self._tok[:B]
        m = self._mode(mode)
        _check(self.lib.sv_verify_logits(self.ctx, B, s, dpt, _ptr(draft_tokens), _ptr(draft_probs), _ptr(logits),
                                         seed, m, float(temperature), _ptr(acc), _ptr(tok)), "sv_verify_logits")
        return acc, tok

    def verify_tree(self, slots, depths, parents, draft_tokens, draft_probs=None, seed=0, mode="greedy",
                    temperature=1.0, logits_out=None, nodes_out=None, out=None):
        """Token-tree verify (R30). parents: device int32 [sum k] (node n's parent in 0..n-1).
        Returns (accepted_len [B], out_tokens [B][max_depth+1], accepted_nodes [B][max_depth+1])."""
        s, B = _i32_array(slots)
        dpt, _ = _i32_array(depths)
        acc, tok = (self._acc[:B], self._tok[:B]) if out is None else out
        nodes = self._nodes[:B] if nodes_out is None else nodes_out
        _check(self.lib.sv_verify_tree(self.ctx, B, s, dpt, _ptr(parents), _ptr(draft_tokens), _ptr(draft_probs),
                                       seed, self._mode(mode), float(temperature), _ptr(acc), _ptr(tok), _ptr(nodes),
                                       _ptr(logits_out)), "sv_verify_tree")
        return acc, tok, nodes

    def verify_tree_logits(self, slots, depths, parents, draft_tokens, logits, draft_probs=None, seed=0,
                           mode="greedy", temperature=1.0):
        s, B = _i32_array(slots)
        dpt, _ = _i32_array(depths)
        acc, tok, nodes = self._acc[:B], self._tok[:B], self._nodes[:B]
        _check(self.lib.sv_verify_tree_logits(self.ctx, B, s, dpt, _ptr(parents), _ptr(draft_tokens),
                                              _ptr(draft_probs), _ptr(logits), seed, self._mode(mode),
                                              float(temperature), _ptr(acc), _ptr(tok), _ptr(nodes)),
               "sv_verify_tree_logits")
        return acc, tok, nodes

    def prefill(self, slot, request_id, prompt, chunk):
        """Chunked prefill (sv_prefill; NEXT-3, R29) of `prompt` (host ints) into an EMPTY
        slot. Returns the model's greedy next token after the prompt (the slot's pending token)."""
        p, n = _i32_array(prompt)
        nxt = ctypes.c_int32()
        _check(self.lib.sv_prefill(self.ctx, slot, request_id, p, n, chunk, ctypes.byref(nxt)), "sv_prefill")
        return nxt.value

    def commit(self, n_keep=None):
        _check(self.lib.sv_commit(self.ctx, _ptr(n_keep)), "sv_commit")

    def release(self, slot):
        _check(self.lib.sv_release(self.ctx, slot), "sv_release")

    def stats(self, reset=False, check=True):
        st = LaneStats()
        r = self.lib.sv_stats(self.ctx, ctypes.byref(st), 1 if reset else 0)
        if check:
            _check(r, "sv_stats")
        return st.as_dict()

    def occupancy(self):
        """(active slots, free KV pages) — the router's L_w and M_w inputs."""
        a, f = ctypes.c_int32(), ctypes.c_int32()
        _check(self.lib.sv_lane_occupancy(self.ctx, ctypes.byref(a), ctypes.byref(f)), "sv_lane_occupancy")
        return a.value, f.value

    def stats_raw(self, reset=False):
        """The sv_lane_stats struct itself (for the SpecuStream controller's window deltas)."""
        st = LaneStats()
        _check(self.lib.sv_stats(self.ctx, ctypes.byref(st), 1 if reset else 0), "sv_stats")
        return st

    # ------------------------------------------------------------------ CUDA graphs
    def graph_begin(self):
        """Capture the lane's next calls into a CUDA graph (sv_graph_begin; needs a created stream)."""
        _check(self.lib.sv_graph_begin(self.ctx), "sv_graph_begin")

    def graph_begin_dynamic(self, batch):
        """Capture a step that serves any depth vector of `batch` requests (sv_graph_begin_dynamic)."""
        _check(self.lib.sv_graph_begin_dynamic(self.ctx, int(batch)), "sv_graph_begin_dynamic")

    def graph_set_batch(self, g, slots, depths):
        """Stage the next replay's slots / depths of a dynamic graph (sv_graph_set_batch)."""
        s, _ = _i32_array(slots)
        d, _ = _i32_array(depths)
        _check(self.lib.sv_graph_set_batch(self.ctx, g, s, d), "sv_graph_set_batch")

    def graph_end(self):
        g = ctypes.c_void_p()
        _check(self.lib.sv_graph_end(self.ctx, ctypes.byref(g)), "sv_graph_end")
        return g

    def graph_launch(self, g):
        _check(self.lib.sv_graph_launch(self.ctx, g), "sv_graph_launch")

    def graph_destroy(self, g):
        _check(self.lib.sv_graph_destroy(g), "sv_graph_destroy")

    def set_filter(self, top_k=0, top_p=1.0):
        """Top-k / top-p filtered target for SAMPLE verifies (R31); (0, 1.0) = off."""
        _check(self.lib.sv_set_filter(self.ctx, int(top_k), float(top_p)), "sv_set_filter")

    def set_taps(self, on=True):
        """Keep every intermediate (incl. the fp32 logits a greedy verify would skip) for tap()."""
        _check(self.lib.sv_set_taps(self.ctx, 1 if on else 0), "sv_set_taps")

    def tap(self, name, dtype, shape=None):
        """Device tensor viewing the library's buffer `name` (valid until the next verify)."""
        p, nb = ctypes.c_void_p(), ctypes.c_size_t()
        _check(self.lib.sv_get_tap(self.ctx, name.encode(), ctypes.byref(p), ctypes.byref(nb)), "sv_get_tap")
        off = p.value - self.workspace.data_ptr()
        if not (0 <= off and off + nb.value <= self.workspace.numel()):
            raise RuntimeError(f"tap {name} outside the workspace")
        t = self.workspace[off:off + nb.value].view(dtype)
        return t if shape is None else t[: _numel(shape)].view(*shape)

    def debug_uniforms(self, seed, rid, z, purpose, x0, n):
        u = torch.empty(n, dtype=torch.float32, device=self.device)
        _check(self.lib.sv_debug_uniforms(self.ctx, seed, rid, z, purpose, x0, n, _ptr(u)), "sv_debug_uniforms")
        return u

    def debug_gemm(self, A, B, C, variant=0):
        """C = A B^T through the library's GEMM kernels (test hook)."""
        M, K = A.shape
        N = B.shape[0]
        _check(self.lib.sv_debug_gemm(self.ctx, _ptr(A), _ptr(B), _ptr(C), M, N, K, variant), "sv_debug_gemm")
        return C

    def draft_planted(self, slots, depths, succ, dev_mask, dev_tok, out):
        s, B = _i32_array(slots)
        dpt, _ = _i32_array(depths)
        _check(self.lib.sv_draft_planted(self.ctx, B, s, dpt, _ptr(succ), _ptr(dev_mask), _ptr(dev_tok), _ptr(out)),
               "sv_draft_planted")
        return out

    def draft_planted_tree(self, slots, depths, parents, succ, dev_mask, dev_tok, out):
        s, B = _i32_array(slots)
        dpt, _ = _i32_array(depths)
        _check(self.lib.sv_draft_planted_tree(self.ctx, B, s, dpt, _ptr(parents), _ptr(succ), _ptr(dev_mask),
                                              _ptr(dev_tok), _ptr(out)), "sv_draft_planted_tree")
        return out

    # ------------------------------------------------------------------ measurement hooks
    def profile(self, on=True):
        """on: True (all stages), False (off) or an iterable of stage names."""
        if on is True or on is False:
            mask = -1 if on else 0
        else:
            names = [self.lib.sv_profile_stage_name(i).decode() for i in range(self.lib.sv_profile_num_stages())]
            mask = 0
            for n in on:
                mask |= 1 << names.index(n)
        _check(self.lib.sv_profile_enable(self.ctx, mask), "sv_profile_enable")

    def profile_read(self, reset=True):
        """{stage: (total_ms, launches)} since the last reset (syncs the stream)."""
        n = self.lib.sv_profile_num_stages()
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(self.lib.sv_profile_read(self.ctx, ms, cnt, n, 1 if reset else 0), "sv_profile_read")
        return {self.lib.sv_profile_stage_name(i).decode(): (ms[i], cnt[i]) for i in range(n)}

    # ------------------------------------------------------------------ hand-off
    def kv_recv_append(self, slot, request_id, n_tokens, staging, peer, comm):
        _check(self.lib.sv_kv_recv_append(self.ctx, slot, request_id, n_tokens, _ptr(staging), peer, comm),
               "sv_kv_recv_append")

    def kv_pack_slot(self, slot, n_tokens, out):
        """Prefill side: committed KV rows 0..n_tokens-1 of `slot` + its pending token, wire format."""
        _check(self.lib.sv_kv_pack_slot(self.ctx, slot, n_tokens, _ptr(out)), "sv_kv_pack_slot")
        return out

    def kv_append_packed(self, slot, request_id, n_tokens, packed):
        _check(self.lib.sv_kv_append_packed(self.ctx, slot, request_id, n_tokens, _ptr(packed)), "sv_kv_append_packed")

    def kv_loopback_append(self, slot, request_id, n_tokens, packed, staging, rank, comm):
        _check(self.lib.sv_kv_loopback_append(self.ctx, slot, request_id, n_tokens, _ptr(packed), _ptr(staging), rank,
                                              comm), "sv_kv_loopback_append")

    def slots_bytes(self, n_tokens):
        """Staging bytes of a batched hand-off of requests with these token counts (sv_kv_slots_bytes)."""
        t, n = _i32_array(n_tokens)
        return int(self.lib.sv_kv_slots_bytes(ctypes.byref(self.cfg), n, t))

    def kv_send_slots(self, slots, n_tokens, staging, peer, comm):
        """Prefill side of the batched hand-off (sv_kv_send_slots)."""
        s, n = _i32_array(slots)
        t, _ = _i32_array(n_tokens)
        _check(self.lib.sv_kv_send_slots(self.ctx, n, s, t, _ptr(staging), peer, comm), "sv_kv_send_slots")

    def kv_recv_slots(self, slots, request_ids, n_tokens, staging, peer, comm):
        """Decode side of the batched hand-off (sv_kv_recv_slots)."""
        s, n = _i32_array(slots)
        t, _ = _i32_array(n_tokens)
        r = (ctypes.c_uint64 * n)(*[int(x) for x in request_ids])
        _check(self.lib.sv_kv_recv_slots(self.ctx, n, s, r, t, _ptr(staging), peer, comm), "sv_kv_recv_slots")

    def kv_loopback_slots(self, dst, src_slots, dst_slots, request_ids, n_tokens, src_staging, dst_staging, rank, comm):
        """One-GPU transport test: this lane sends, `dst` receives, one NCCL group."""
        s, n = _i32_array(src_slots)
        d, _ = _i32_array(dst_slots)
        t, _ = _i32_array(n_tokens)
        r = (ctypes.c_uint64 * n)(*[int(x) for x in request_ids])
        _check(self.lib.sv_kv_loopback_slots(self.ctx, dst.ctx, n, s, d, r, t, _ptr(src_staging), _ptr(dst_staging),
                                             rank, comm), "sv_kv_loopback_slots")

    def comm_stream(self):
        """torch ExternalStream of the lane's comm stream (hand-off transfers run there)."""
        p = ctypes.c_void_p()
        _check(self.lib.sv_comm_stream(self.ctx, ctypes.byref(p)), "sv_comm_stream")
        return torch.cuda.ExternalStream(p.value, device=self.device)

    def packed_bytes(self, n_tokens):
        return int(self.lib.sv_kv_packed_bytes(ctypes.byref(self.cfg), n_tokens))


def _numel(shape):
    n = 1
    for s in shape:
        n *= int(s)
    return n


# ---------------------------------------------------------------------- NCCL hand-off helpers
def launch_count():
    """Kernels launched by libsv.so in this process."""
    return int(load().sv_launch_count())


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(load().sv_nccl_unique_id(buf), "sv_nccl_unique_id")
    return bytes(buf.raw)


def nccl_comm_init(nranks, uid, rank):
    comm = ctypes.c_void_p()
    _check(load().sv_nccl_comm_init(nranks, uid, rank, ctypes.byref(comm)), "sv_nccl_comm_init")
    return comm


def nccl_comm_destroy(comm):
    _check(load().sv_nccl_comm_destroy(comm), "sv_nccl_comm_destroy")


def kv_pack(k, v, pending_token, out, stream=None):
    L, n, H, dh = k.shape
    st = stream if stream is not None else torch.cuda.current_stream(k.device)
    _check(load().sv_kv_pack(_ptr(k), _ptr(v), L, H, dh, n, int(pending_token), _ptr(out),
                             ctypes.c_void_p(st.cuda_stream)), "sv_kv_pack")
    return out


def kv_send(packed, n_layers, n_kv_heads, head_dim, n_tokens, peer, comm, stream=None):
    st = stream if stream is not None else torch.cuda.current_stream(packed.device)
    _check(load().sv_kv_send(_ptr(packed), n_layers, n_kv_heads, head_dim, n_tokens, peer, comm,
                             ctypes.c_void_p(st.cuda_stream)), "sv_kv_send")


def packed_bytes(cfg, n_tokens):
    c = Config.from_any(cfg)
    return int(load().sv_kv_packed_bytes(ctypes.byref(c), n_tokens))


def exact_forward(cfg, weights_f32, row_off, chain_tok, ctx_len, cache_k=None, cache_v=None, stream=None):
    """fp32-SIMT exactness instantiation (sv_exact_forward, NEXT-4): logits [T][V] fp32 of the chain rows.
    weights_f32: dict of fp32 device tensors (sv_weights names); chain_tok: device int32 [T];
    row_off / ctx_len: host lists; cache_k / cache_v: device fp32 [n_layers][batch][max_ctx][Hkv][dh]."""
    lib = load()
    c = Config.from_any(cfg)
    T = int(row_off[-1])
    dev = chain_tok.device
    for k, v in weights_f32.items():
        assert v.dtype == torch.float32 and v.is_contiguous() and v.device == dev, k
    wts = Weights(*[ctypes.c_void_p(weights_f32[n].data_ptr()) if n in weights_f32 else None for n in WEIGHT_NAMES])
    need = ctypes.c_size_t()
    _check(lib.sv_exact_query_sizes(ctypes.byref(c), T, ctypes.byref(need)), "sv_exact_query_sizes")
    ws = torch.empty(need.value, dtype=torch.uint8, device=dev)
    logits = torch.empty(T, c.vocab, dtype=torch.float32, device=dev)
    ro, _ = _i32_array(row_off)
    cl, batch = _i32_array(ctx_len)
    max_ctx = int(cache_k.shape[2]) if cache_k is not None else 0
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    _check(lib.sv_exact_forward(ctypes.byref(c), ctypes.byref(wts), batch, ro, _ptr(chain_tok), cl,
                                None if cache_k is None else ctypes.c_void_p(cache_k.data_ptr()),
                                None if cache_v is None else ctypes.c_void_p(cache_v.data_ptr()), max_ctx,
                                ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(logits.data_ptr()),
                                ctypes.c_void_p(st.cuda_stream)), "sv_exact_forward")
    return logits, ws
