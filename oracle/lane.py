"""Free-running oracle decode lane with the sv_* call semantics (dense caches).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Mirrors the boundary of include/sv.h on a dense,
per-request, fp64 cache — no pages, no batching, no shared layout:

* append_kv  — `eq:kv_concatenation`: the prefill KV is the
  start of KV_total; activates the slot and binds request_id (the RNG key).
* verify     — SURVEY.md §8(c) steps 1-5 per request (model.forward_chain then
  verify.verify_request); side-effect free until commit.
* verify_tree — token-tree drafts (oracle/tree.py, R30); commit keeps the
  accepted root-to-node path's rows.
* commit     — step 6: append chain K/V rows 0..a_i (tokens x_i, d_1..d_a) to
  the cache, L_i += a_i + 1, pending <- y; with n_keep: rows 0..n_keep-1,
  pending = emitted[n_keep-1]. Rejected rows are dropped (rollback).
* stats      — the a7 counters (verify.accumulate_stats).

Sequence-index convention (SURVEY.md §8 "Verify rows"): a request with n
committed tokens has cache length L = n - 1; the pending token sits at index
L and has no KV yet; chain row j sits at absolute position L + j.
"""
import numpy as np

from . import model, tree, verify


class OracleLane:
    def __init__(self, cfg, weights, rope=None):
        """weights: dict of numpy arrays (bf16 values, any float dtype)."""
        self.cfg = cfg
        self.w = weights
        if rope is None:
            rope = model.rope_table(cfg.max_pos, cfg.head_dim, cfg.rope_theta)
        self.cos, self.sin = rope
        self.slots = {}
        self.stats = verify.new_stats()
        self.pending_batch = None

    # ------------------------------------------------------------ state
    def append_kv(self, slot, request_id, k, v, pending_token):
        """k, v: [n_layers][n][H_kv][d_h] (bf16 values), post-RoPE."""
        k = np.asarray(k, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        st = self.slots.get(slot)
        if st is None:
            st = dict(rid=int(request_id), K=[np.zeros((0, self.cfg.n_kv_heads, self.cfg.head_dim))
                                              for _ in range(self.cfg.n_layers)],
                      V=[np.zeros((0, self.cfg.n_kv_heads, self.cfg.head_dim))
                         for _ in range(self.cfg.n_layers)], pending=None)
            self.slots[slot] = st
        assert st["rid"] == int(request_id)
        for layer in range(self.cfg.n_layers):
            st["K"][layer] = np.concatenate([st["K"][layer], k[layer]], axis=0)
            st["V"][layer] = np.concatenate([st["V"][layer], v[layer]], axis=0)
        st["pending"] = int(pending_token)

    def length(self, slot):
        return self.slots[slot]["K"][0].shape[0]

    def release(self, slot):
        del self.slots[slot]

    # ------------------------------------------------------------ verify
    def forward(self, slot, drafts):
        """Model forward for one request's chain [pending, d_1..d_k]."""
        st = self.slots[slot]
        L = self.length(slot)
        tokens = [st["pending"]] + [int(d) for d in drafts]
        pos = L + np.arange(len(tokens))
        caches = list(zip(st["K"], st["V"]))
        return model.forward_chain(self.w, tokens, pos, caches, self.cfg, self.cos, self.sin)

    def verify(self, slots, depths, draft_tokens, draft_probs, seed, mode, temperature=1.0,
               logits_override=None, top_k=0, top_p=1.0):
        """Returns (accepted_len list, emitted token lists, per-request logits).

        draft_tokens: flat [sum k]; draft_probs: flat [sum k][V] or None.
        logits_override: optional list of per-request logits (teacher-forced decisions).
        """
        results, logits_all, chain = [], [], []
        off = 0
        for i, (slot, k) in enumerate(zip(slots, depths)):
            drafts = [int(t) for t in draft_tokens[off:off + k]]
            q_rows = None if draft_probs is None else np.asarray(draft_probs[off:off + k])
            off += k
            if logits_override is not None:
                logits = np.asarray(logits_override[i], dtype=np.float64)
                kv = None
            else:
                _, logits, kv = self.forward(slot, drafts)
            r = verify.verify_request(logits, drafts, q_rows, seed, self.slots[slot]["rid"],
                                      self.length(slot), mode, temperature, top_k, top_p)
            results.append(r)
            logits_all.append(logits)
            chain.append(kv)
        verify.accumulate_stats(self.stats, list(depths), results)
        self.pending_batch = (list(slots), list(depths), results, chain)
        return [r["a"] for r in results], [r["emitted"] for r in results], logits_all

    def verify_tree(self, slots, depths, parents, draft_tokens, draft_probs, seed, mode, temperature=1.0,
                    logits_override=None, top_k=0, top_p=1.0):
        """Token-tree verify (oracle/tree.py, R30): parents flat [sum k] (per request,
        node n's parent in 0..n-1). Returns (accepted_len, emitted, logits, paths)."""
        results, logits_all, chain = [], [], []
        off = 0
        for i, (slot, k) in enumerate(zip(slots, depths)):
            drafts = [int(t) for t in draft_tokens[off:off + k]]
            par = [int(t) for t in parents[off:off + k]]
            q_rows = None if draft_probs is None else np.asarray(draft_probs[off:off + k])
            off += k
            st = self.slots[slot]
            L = self.length(slot)
            if logits_override is not None:
                logits, kv = np.asarray(logits_override[i], dtype=np.float64), None
            else:
                _, logits, kv = tree.forward_tree(self.w, [st["pending"]] + drafts, par, L,
                                                  list(zip(st["K"], st["V"])), self.cfg, self.cos, self.sin)
            r = tree.verify_tree(logits, drafts, par, q_rows, seed, st["rid"], L, mode, temperature, top_k, top_p)
            results.append(r)
            logits_all.append(logits)
            chain.append(kv)
        verify.accumulate_stats(self.stats, list(depths), results)
        self.pending_batch = (list(slots), list(depths), results, chain)
        return ([r["a"] for r in results], [r["emitted"] for r in results], logits_all,
                [r["path"] for r in results])

    def commit(self, n_keep=None):
        slots, depths, results, chain = self.pending_batch
        for i, slot in enumerate(slots):
            r = results[i]
            n = r["a"] + 1 if n_keep is None else min(int(n_keep[i]), r["a"] + 1)
            assert n >= 1
            st = self.slots[slot]
            rows = list(r.get("path", range(r["a"] + 1)))[:n]     # tree: the accepted path's rows
            for layer in range(self.cfg.n_layers):
                k, v = chain[i][layer]
                st["K"][layer] = np.concatenate([st["K"][layer], k[rows]], axis=0)
                st["V"][layer] = np.concatenate([st["V"][layer], v[rows]], axis=0)
            st["pending"] = int(r["emitted"][n - 1])
        self.pending_batch = None
