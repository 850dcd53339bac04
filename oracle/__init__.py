"""fp64 CPU oracle for the StreamServe speculative-verify hot path.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. The product path (``paper_2604_09562_b200``) never imports it and
shares no code, tables or helpers with it; the only shared module is
``synth`` (seeded input generators, no method arithmetic).

What it computes and where the paper says so:

* the verify step — Leviathan rejection sampling with a bonus token, or a
  greedy prefix match ("preserving output distribution";
  the paper never defines the procedure), written out in the
  order of SURVEY.md §8(c) "Oracle algorithm" steps 1-7;
* the single Llama-shaped layer + lm-head that produces the target logits
  (SURVEY.md §8 "Fixed definitions", §8(c) step 1);
* KV commit / rollback = ``eq:kv_concatenation``;
* acceptance statistics a_t.

Modules: ``philox`` (counter RNG), ``numerics`` (bf16 rounding), ``model``
(stage functions), ``verify`` (decisions + lane counters), ``lane``
(free-running dense-cache lane with the sv_* call semantics), ``specustream``
(Alg. 4 host controller, NEXT-1), ``flowguard`` (Alg. 2 router, NEXT-2), ``tree``
(token-tree drafts, NEXT-4).

Parity status: see each module header. Everything pinned by the tests named
there; the exact bits of a Llama-shape verify step beyond those pins are
"parity unpinned" (defined only by these stage functions).
"""
