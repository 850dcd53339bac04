/*
 * sv.h — C ABI of the B200-native speculative-verify hot path (libsv.so).
 *
 * What this library computes: one decode lane of StreamServe (arXiv 2604.09562)
 * — the batched, variable-depth speculative VERIFY step that the paper's
 * PipeServe-Engine decode worker runs ("Adapt spec depth via SpecuStream;
 * out <- llm_D.generate(req)", Alg. 3; "D_i: decode with
 * SpecuStream, report metrics", Alg. 1), plus the KV
 * concatenation it relies on (eq:kv_concatenation) and the
 * prefill->decode KV transfer. The paper never
 * defines the verification procedure; the one implemented here
 * is Leviathan rejection sampling with a bonus token / greedy prefix match
 * (PAPER.md:37, 65), fixed step by step in DESIGN.md "Readings" and
 * SURVEY.md §8(c). The model is one (or more) Llama-shaped decoder layer(s) +
 * lm-head with bf16 operands and fp32 accumulation.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless its comment says (host).
 *  - All device memory is allocated by the caller (PyTorch) and BORROWED; it
 *    must outlive the context. The library never calls cudaMalloc.
 *  - Every call enqueues work on the context's stream (given at sv_create)
 *    and returns without synchronising, except where it says "syncs".
 *    Device outputs are valid in stream order; device inputs must stay
 *    unmodified until the stream has consumed them.
 *  - Host-checkable misuse returns an error synchronously and enqueues
 *    nothing. Device-detected problems set a sticky device error word that
 *    is reported by the next sv_stats / sv_commit (see sv_status).
 *  - A context is one decode lane on one GPU; it is not thread-safe.
 *  - fp32 row buffers (draft_probs, logits, logits_out) must be 16-byte aligned (rows are read
 *    with 16-byte vector loads when V % 4 == 0); a misaligned pointer is SV_EINVAL.
 *
 * Sequence convention (SURVEY.md §8 "Verify rows"): a request with n
 * committed tokens has cache length L = n - 1; its "pending" token (index L)
 * has no KV yet. A verify of depth k evaluates the chain
 * [pending, d_1..d_k] at absolute positions L..L+k (k + 1 query rows).
 *
 * Weight layout (all bf16, row-major [out][in], layer-stacked, BORROWED):
 *   embed      [V][D]            attn_norm [n_layers][D]
 *   wqkv       [n_layers][(Hq + 2 Hkv) d_h][D]   rows: q heads | k heads | v heads
 *   wo         [n_layers][D][Hq d_h]
 *   ffn_norm   [n_layers][D]     w_gate_up [n_layers][2F][D]  rows: gate F | up F
 *   w_down     [n_layers][D][F]  final_norm [D]   lm_head [V][D]
 * Every weight pointer must be 16-byte aligned.
 *
 * KV pool layout (bf16, BORROWED, size from sv_query_sizes):
 *   [n_layers][n_pages][2 (K,V)][H_kv][page_size][d_h], keys stored post-RoPE.
 */
#ifndef SV_H_
#define SV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sv_stream_t; /* == cudaStream_t */
typedef struct sv_ctx sv_ctx;

typedef enum {
  SV_OK = 0,
  SV_EINVAL = 1,   /* bad argument (null pointer, size out of range, duplicate slot, ...) */
  SV_ESTATE = 2,   /* call not allowed in the slot's / context's current state */
  SV_ENOKV = 3,    /* device free list ran out of KV pages (sticky, device-detected) */
  SV_ECUDA = 4,    /* a CUDA runtime / driver call failed */
  SV_ENCCL = 5,    /* an NCCL call failed */
  SV_EDEVICE = 6   /* other device-detected error (bad token id, bad n_keep; sticky) */
} sv_status;

typedef enum { SV_GREEDY = 0, SV_SAMPLE = 1, SV_PREFILL = 2 } sv_mode;

/* Device error word bits (sv_lane_stats.device_error). */
#define SV_DERR_BAD_TOKEN 1   /* a draft / pending token outside [0, V) */
#define SV_DERR_NO_PAGES 2    /* free list exhausted during append / commit */
#define SV_DERR_BAD_KEEP 4    /* n_keep < 1 */
#define SV_DERR_MAX_POS 8     /* a chain or commit would pass max_pos; that request is not committed */
#define SV_DERR_BAD_TREE 16   /* a token-tree parent outside [0, n-1]; that request is not committed */

typedef struct { /* (host) model + lane configuration */
  int32_t n_layers, d_model, n_q_heads, n_kv_heads, head_dim, vocab;
  int32_t ffn_dim;           /* 0 = no MLP (attention-only layer) */
  float rope_theta, norm_eps;
  int32_t page_size;         /* tokens per KV page: 64 */
  int32_t n_pages;           /* pages in the pool (shared by all slots) */
  int32_t max_slots;         /* request slots in this lane */
  int32_t max_batch;         /* requests per sv_verify call */
  int32_t max_depth;         /* k_i <= max_depth <= 32 */
  int32_t max_pos;           /* RoPE table length >= max context + max_depth + 1 */
} sv_config;

typedef struct { /* device pointers, bf16, layouts above; BORROWED */
  const void *embed, *attn_norm, *wqkv, *wo, *ffn_norm, *w_gate_up, *w_down, *final_norm, *lm_head;
} sv_weights;

typedef struct { /* (host) lane acceptance counters — SURVEY.md §8(a) a7; a_t = accepted / drafted */
  uint64_t steps;                 /* sv_verify calls */
  uint64_t rows;                  /* sum (k_i + 1) */
  uint64_t drafted;               /* sum k_i */
  uint64_t accepted;              /* sum a_i (prefix-stopped) */
  uint64_t emitted;               /* sum (a_i + 1) */
  uint64_t accepted_independent;  /* sum_j [u_j < r_j] over all j <= k_i (greedy: d_j == argmax) */
  uint64_t hist_accepted[33];     /* count of requests with a_i = m */
  uint64_t drafted_by_k[33];      /* sum k_i over requests with k_i = k */
  uint64_t accepted_by_k[33];     /* sum a_i over requests with k_i = k */
  int32_t device_error;           /* sticky SV_DERR_* bits */
  int32_t _pad;
} sv_lane_stats;

/* Library version string, e.g. "sv 0.1 sm_100a". */
const char* sv_version(void);
/* Static message for a status code. */
const char* sv_strerror(sv_status s);

/* Bytes the caller must allocate for the KV pool and the workspace for cfg.
 * Both buffers must be 1024-byte aligned. EINVAL on an invalid cfg
 * (non-positive sizes, n_q_heads % n_kv_heads != 0, head_dim not in {64,128},
 * d_model % 64 != 0, max_depth > 32, (max_depth + 1) * group > 64 unless group <= 4 and max_depth < 32:
 * verifies whose deepest chain has (k + 1) * group <= 64 query rows per kv head run the keys-on-lanes
 * attention kernel, deeper ones (up to k = 31 at group 4) the rows-on-lanes kernel). */
sv_status sv_query_sizes(const sv_config* cfg, size_t* kv_pool_bytes, size_t* workspace_bytes);

/* Create a lane on the current CUDA device. Builds the fp32 RoPE table
 * (fp64 angles, SURVEY.md §8(c) "Model details"), the device free list and the
 * TMA descriptors, on `stream`; the kv_pool is zero-filled (attention reads whole
 * pages; zero rows beyond a slot's length keep masked keys finite).
 * Syncs `stream` once before returning. */
sv_status sv_create(const sv_config* cfg, const sv_weights* w, void* kv_pool, void* workspace,
                    sv_stream_t stream, sv_ctx** out);
/* Destroy the context (syncs its stream). Borrowed memory is not freed. */
sv_status sv_destroy(sv_ctx* ctx);

/* Append n_tokens of context KV to `slot` (eq:kv_concatenation):
 * k, v: [n_layers][n_tokens][H_kv][d_h] bf16, post-RoPE (read in stream order).
 * An EMPTY slot becomes ACTIVE and is bound to request_id (the Philox key of
 * all its draws, so outputs never depend on slot or lane); on an ACTIVE slot
 * request_id must match. Pages are popped from the device free list
 * (SV_DERR_NO_PAGES if it runs out). pending_token becomes the chain head of
 * the next verify. ESTATE on a PENDING slot (verified, not committed).
 * n_tokens may be 0 (only sets the pending token). */
sv_status sv_append_kv(sv_ctx* ctx, int32_t slot, uint64_t request_id, const void* k, const void* v,
                       int32_t n_tokens, int32_t pending_token);

/* The verify step. For each request b < batch:
 *   slots[b]  (host) distinct ACTIVE slots;  depths[b] (host) k_b in [0, max_depth]
 *   draft_tokens [sum k] int32, request-major (the drafter's tokens)
 *   draft_probs  [sum k][V] fp32 rows q_j (the drafter's distributions) or NULL = one-hot drafts
 *   seed: Philox key; mode: SV_GREEDY (argmax prefix match; seed, temperature and
 *   draft_probs ignored) or SV_SAMPLE (Leviathan: accept iff u < p/q, residual /
 *   bonus exponential race); temperature > 0 in SAMPLE (p = softmax(l / T)); or SV_PREFILL
 *   (chunked prefill, NEXT-3 / DESIGN.md R29: the "drafts" are the next prompt tokens and every
 *   row is kept, a = k; y = argmax of the last row; lane counters untouched).
 * Outputs (device, written in stream order):
 *   accepted_len [batch] int32 a_b in [0, k_b] (-1 if the request hit a device error)
 *   out_tokens   [batch][max_depth + 1] int32: d_1..d_a, y, then -1 padding
 *   logits_out   NULL or [sum (k + 1)][V] fp32 copy of the target logits (pre-temperature)
 * Lane counters are updated on the device. The call has no effect on the KV
 * cache or slot lengths: the slots become PENDING until sv_commit.
 * EINVAL: batch < 1 or > max_batch, bad depth, duplicate/out-of-range slot,
 * null pointers, temperature <= 0 in SAMPLE. ESTATE: a slot not ACTIVE. */
sv_status sv_verify(sv_ctx* ctx, int32_t batch, const int32_t* slots, const int32_t* depths,
                    const int32_t* draft_tokens, const float* draft_probs, uint64_t seed,
                    sv_mode mode, float temperature, int32_t* accepted_len, int32_t* out_tokens,
                    float* logits_out);

/* Decision-only verify (a6 + a7) on caller-provided logits [sum (k + 1)][V] fp32
 * (rows in request-major chain order). Same RNG keying as sv_verify (the slot's
 * request_id, positions from the slot's length). Runs no model and produces no
 * chain KV: slots stay ACTIVE and the call is not committable. */
sv_status sv_verify_logits(sv_ctx* ctx, int32_t batch, const int32_t* slots, const int32_t* depths,
                           const int32_t* draft_tokens, const float* draft_probs, const float* logits,
                           uint64_t seed, sv_mode mode, float temperature, int32_t* accepted_len,
                           int32_t* out_tokens);

/* Token-tree verify (SURVEY.md §8(f) NEXT-4 "tree-structured drafts"; the paper cites draft
 * trees as related work; semantics = DESIGN.md reading R30). Request b drafts
 * k_b = depths[b] tree nodes n = 1..k_b (node 0 is the slot's pending token):
 *   parents [sum k] int32 DEVICE, request-major: parents[off_b + n - 1] = parent of node n, in
 *            [0, n - 1] (topological order); anything else sets SV_DERR_BAD_TREE and the request's
 *            accepted_len = -1 (it is then not committed)
 *   draft_tokens / draft_probs as in sv_verify, one entry / q row per node (q row n - 1 = the
 *            distribution node n's token was drawn from, i.e. conditioned on its parent)
 * Node n sits at position L + depth(n) and attends the cache and its ancestors-or-self.
 * GREEDY walks from node 0 to the first child (ascending index) whose token is the argmax;
 * SAMPLE tries a node's children in index order with recursive rejection (accept iff
 * u < r(d)/q(d), r <- norm(max(0, r - q)) on rejection; u = Philox(seed, rid, L + depth + 1,
 * ACCEPT, sibling rank)), then draws y from the final r (exponential race). Outputs as in
 * sv_verify (a_b = depth of the last accepted node, out_tokens = the path's tokens then y), plus
 *   accepted_nodes NULL or DEVICE [batch][max_depth + 1] int32: the accepted path's node indices
 *            (0, n_1, .., n_a), -1 padded.
 * sv_commit then keeps the path's K/V rows (node n_m lands at position L + m). A chain
 * (parents[n-1] = n-1) gives exactly sv_verify's results. Limits and errors as sv_verify. */
sv_status sv_verify_tree(sv_ctx* ctx, int32_t batch, const int32_t* slots, const int32_t* depths,
                         const int32_t* parents, const int32_t* draft_tokens, const float* draft_probs,
                         uint64_t seed, sv_mode mode, float temperature, int32_t* accepted_len,
                         int32_t* out_tokens, int32_t* accepted_nodes, float* logits_out);

/* Decision-only token-tree verify on caller logits [sum (k + 1)][V] fp32 (row off_b + n = node n),
 * the tree analogue of sv_verify_logits (R30). Not committable. */
sv_status sv_verify_tree_logits(sv_ctx* ctx, int32_t batch, const int32_t* slots, const int32_t* depths,
                                const int32_t* parents, const int32_t* draft_tokens, const float* draft_probs,
                                const float* logits, uint64_t seed, sv_mode mode, float temperature,
                                int32_t* accepted_len, int32_t* out_tokens, int32_t* accepted_nodes);

/* CUDA graphs of a fixed step (launch-bound small configurations): between sv_graph_begin and
 * sv_graph_end the lane's calls (e.g. sv_draft_planted + sv_verify + sv_commit) are captured from
 * its stream instead of running — the host-side checks and state changes happen once, at capture —
 * and sv_graph_launch replays the captured kernels with the same arguments (slots, depths, seed,
 * device pointers: inputs that change per step are refreshed by the caller in the buffers the
 * graph reads). The lane's stream must be a created stream (not the legacy default stream), and
 * every captured sv_verify committed inside the capture (else sv_graph_end returns SV_ESTATE).
 * Stages being timed (sv_profile_enable) while capturing become event-record nodes of the graph that
 * every replay points at fresh events while the lane still times those stages, so sv_profile_read
 * covers replays as it covers eager calls. Replays advance the device state (lengths, pages,
 * counters) exactly like the captured calls. sv_graph_destroy frees the instantiated graph. */
typedef struct sv_graph sv_graph;
sv_status sv_graph_begin(sv_ctx* ctx);
/* One graph for ANY depth vector (slots / depths go through a pinned staging buffer
 * that the captured graph's H2D node reads). Like sv_graph_begin, for a step of exactly `batch`
 * requests: the captured calls (sv_draft_planted, sv_verify in GREEDY / SAMPLE mode of chains, without
 * logits_out, and sv_commit) take their slots and depths from the device copy made by the graph's
 * first node; row-gridded kernels are launched for batch * (max_depth + 1) rows and return beyond the
 * plan's device row count, the GEMMs read their rows from it. The slots / depths given at capture only
 * need to be valid then. Before each replay, sv_graph_set_batch stages that replay's slots and
 * depths (host-checked like sv_verify's); every replay of a dynamic graph takes a freshly staged batch
 * (sv_graph_launch returns SV_ESTATE otherwise). The lane owns two pinned staging buffers that its
 * dynamic graphs share: sv_graph_set_batch takes the next one once the replay that last read it has
 * finished, and refuses (SV_ESTATE) while a staging of that buffer, or of the same graph, awaits its
 * launch — so several dynamic graphs of a lane may alternate (stage one, launch it, stage the next).
 * ESTATE if the lane's GEMM / attention configuration cannot read rows from the device (SV_GEMM /
 * SV_ATTN overrides). */
sv_status sv_graph_begin_dynamic(sv_ctx* ctx, int32_t batch);
sv_status sv_graph_set_batch(sv_ctx* ctx, const sv_graph* graph, const int32_t* slots, const int32_t* depths);
sv_status sv_graph_end(sv_ctx* ctx, sv_graph** graph);
sv_status sv_graph_launch(sv_ctx* ctx, const sv_graph* graph);
sv_status sv_graph_destroy(sv_graph* graph);

/* Top-k / top-p filtered targets for SV_SAMPLE verifies of this lane (
 * DESIGN.md reading R31; the paper fixes no sampler): p = softmax(l / T) is restricted to the first
 * min(n_k, n_p) tokens in (scaled logit desc, token id asc) order — n_k = top_k (0 = no limit),
 * n_p = the smallest n whose cumulative p reaches top_p (>= 1 = no limit) — and renormalised; the
 * filtered p' replaces p in the accept test, the residual and the bonus draw (chains and trees).
 * Kept masses are summed in 2^-40 fixed point, so the kept set does not depend on summation
 * order. Greedy and prefill verifies are unaffected. Default (0, 1.0) = off. EINVAL: top_k < 0
 * or top_p <= 0 / NaN. ESTATE while a verify is uncommitted. */
sv_status sv_set_filter(sv_ctx* ctx, int32_t top_k, float top_p);

/* Commit the last sv_verify (eq:kv_concatenation): for each
 * request copy chain K/V rows 0..n-1 (n = a_b + 1, or min(n_keep[b], a_b + 1); the first n
 * nodes of the accepted path after sv_verify_tree)
 * into pages at positions L..L+n-1, popping pages at page boundaries; then
 * L += n and pending <- the n-th emitted token. Rejected rows are dropped
 * (rollback). n_keep: NULL or DEVICE int32 [batch] (values >= 1).
 * ESTATE if there is no uncommitted verify. Returns the sticky device error
 * observed so far WITHOUT syncing (i.e. from earlier sv_stats), else SV_OK. */
sv_status sv_commit(sv_ctx* ctx, const int32_t* n_keep);

/* Return the slot's pages to the free list; the slot becomes EMPTY. ESTATE if PENDING. */
sv_status sv_release(sv_ctx* ctx, int32_t slot);

/* Lane occupancy for the router (FlowGuard's M_w and L_w): slots that are not EMPTY, and pages
 * left on the device free list. Syncs the lane's stream. */
sv_status sv_lane_occupancy(sv_ctx* ctx, int32_t* active_slots, int32_t* free_pages);

/* Copy the lane counters to *out (host). Syncs the stream. reset != 0 zeroes
 * the counters (not the error word). Returns SV_ENOKV / SV_EDEVICE if the
 * sticky device error word is set. */
sv_status sv_stats(sv_ctx* ctx, sv_lane_stats* out, int reset);

/* Test hooks (teacher-forced parity). Buffers of the
 * last sv_verify, valid in stream order until the next sv_verify. Names:
 *   "h0" [T][D] f32 embed   "a" [T][D] bf16 attn-norm   "q" [T][Hq][d_h] bf16
 *   "kc","vc" [n_layers][T][Hkv][d_h] bf16 chain K/V   "o" [T][Hq d_h] bf16
 *   "h1" [T][D] f32   "b" [T][D] bf16   "u" [T][F] bf16   "h2" [T][D] f32
 *   "z" [T][D] bf16   "logits" [T][V] f32   "tile_max","tile_sum" [T][nt] f32
 *   "tile_arg" [T][nt] i32 (nt = ceil(V / 128))   "row_off" [batch+1] i32
 *   "rope_cos","rope_sin" [max_pos][d_h/2] f32   "len","pending" [max_slots] i32
 *   "page_table" [max_slots][max_pages_per_slot] i32   "free_top" [1] i32
 * (the "last layer" values when n_layers > 1). Every buffer is retained, except
 * that a greedy sv_verify skips storing "logits" (its decisions read only the
 * vocab-tile statistics) unless sv_set_taps(ctx, 1) was called or logits_out is
 * given; sv_set_taps(ctx, 0) (the default) restores that. */
sv_status sv_set_taps(sv_ctx* ctx, int enable);
sv_status sv_get_tap(sv_ctx* ctx, const char* name, void** dev_ptr, size_t* bytes);

/* Test hook: u[i] = U(seed, rid, z, purpose, x0 + i) for i < n, computed by the
 * same device Philox the verifier uses (fp32 out; purpose 0 ACCEPT, 1 RACE). */
sv_status sv_debug_uniforms(sv_ctx* ctx, uint64_t seed, uint64_t rid, uint32_t z, int32_t purpose,
                            int32_t x0, int32_t n, float* u);

/* Test hook: C[M][N] fp32 = A[M][K] * B[N][K]^T (bf16, row-major, 16-byte aligned) with the
 * lane's GEMM path (tcgen05 unless SV_GEMM=simt). M <= max_batch * (max_depth + 1), K % 64 == 0.
 * `variant`: 0 = the lane's default kernel, 1 = 1-SM tcgen05, 2 = 2-SM tcgen05, 3 = SIMT,
 *   4 = 1-SM tcgen05 with operand loads skipped after the pipeline fill (timing diagnostic only:
 *   the result is meaningless), 5 = weight-major 2-SM tcgen05 (the default), 6 / 7 / 8 = variant 5
 *   with loads skipped / epilogue skipped / both (timing diagnostics). */
sv_status sv_debug_gemm(sv_ctx* ctx, const void* A, const void* B, float* C, int32_t M, int32_t N, int32_t K,
                        int32_t variant);

/* Bench fixture (planted-successor drafter, SURVEY.md §8(d) "Acceptance control"):
 * for each request b (slots/depths (host) as in sv_verify), d_1 = succ[pending_b],
 * d_j = succ[d_{j-1}], except where dev_mask[row] != 0 the token is dev_tok[row]
 * (rows request-major, sum k). Writes draft_tokens [sum k] int32. One launch. */
sv_status sv_draft_planted(sv_ctx* ctx, int32_t batch, const int32_t* slots, const int32_t* depths,
                           const int32_t* succ, const uint8_t* dev_mask, const int32_t* dev_tok,
                           int32_t* draft_tokens);

/* The same fixture for token trees (R30): node n's token is succ[token of parents[n-1]] (node 0 =
 * the pending token) unless dev_mask marks it, then dev_tok. parents: DEVICE [sum k] as in
 * sv_verify_tree. One launch. */
sv_status sv_draft_planted_tree(sv_ctx* ctx, int32_t batch, const int32_t* slots, const int32_t* depths,
                                const int32_t* parents, const int32_t* succ, const uint8_t* dev_mask,
                                const int32_t* dev_tok, int32_t* draft_tokens);

/* Measurement hooks (bench.py): per-stage CUDA-event timing on the lane's stream.
 * sv_profile_enable(ctx, mask) brackets stage i of sv_verify / sv_commit /
 * sv_draft_planted with cudaEventRecord when bit i of mask is set (-1 = all
 * stages, 0 = off; each record costs host time and a stream dependency, so a
 * timed run enables only the stages it reports). sv_profile_read (syncs) returns, for each
 * of sv_profile_num_stages() stages (names from sv_profile_stage_name), the summed
 * device milliseconds and launch count since the last reset. sv_launch_count()
 * is the number of CUDA kernels this library has launched in the process. */
sv_status sv_profile_enable(sv_ctx* ctx, int32_t stage_mask);
int32_t sv_profile_num_stages(void);
const char* sv_profile_stage_name(int32_t i);
sv_status sv_profile_read(sv_ctx* ctx, double* ms_total, int64_t* count, int32_t n, int reset);
uint64_t sv_launch_count(void);

/* ---------------- prefill -> decode KV hand-off ----------------
 * NCCL point-to-point over NVLink ("NIXL" replaced by
 * ncclSend/ncclRecv). Communicators are created by the library; the 128-byte
 * unique id travels through the caller's process group (torch.distributed store). */
sv_status sv_nccl_unique_id(uint8_t id[128]);
sv_status sv_nccl_comm_init(int nranks, const uint8_t id[128], int rank, void** comm);
sv_status sv_nccl_comm_destroy(void* comm);

/* Prefill side: send n_tokens of packed KV [n_layers][n_tokens][2][H_kv][d_h] bf16
 * followed by a 16-byte trailer {int32 pending_token, 3 x int32 reserved}
 * (kv_packed must be contiguous, 16-byte aligned) to `peer` on `stream`. */
sv_status sv_kv_send(const void* kv_packed, int32_t n_layers, int32_t n_kv_heads, int32_t head_dim,
                     int32_t n_tokens, int peer, void* nccl_comm, sv_stream_t stream);

/* Decode side: receive that message into the lane's staging buffer and append
 * it to `slot` (sv_append_kv semantics; the pending token comes from the
 * trailer on the device). staging: DEVICE buffer of at least
 * sv_kv_packed_bytes(cfg, n_tokens) bytes, owned by the caller. The receive runs on the lane's comm
 * stream (overlapping a verify already enqueued); the append copy waits for it on the lane stream.
 * Host-checkable misuse is refused before the receive is posted. */
sv_status sv_kv_recv_append(sv_ctx* ctx, int32_t slot, uint64_t request_id, int32_t n_tokens,
                            void* staging, int peer, void* nccl_comm);
size_t sv_kv_packed_bytes(const sv_config* cfg, int32_t n_tokens);

/* Chunked prefill (NEXT-3, eq:prefill_computation PAPER.md:248-253, R29) of a prompt of
 * n >= 1 tokens (host array) into an EMPTY slot bound to request_id, in chunks of <= `chunk` prompt
 * tokens, 1 <= chunk <= max_batch * (max_depth + 1) (the workspace's rows). Each chunk runs as C rows
 * at positions L..L+C-1 through the layer stack: its K/V rows are written to their pages first and
 * the attention reads every key from the pages with a per-row causal limit (k_attn_prefill.cu,
 * tcgen05, 128 / G rows of each of the G q heads per work item); only the last chunk runs the final
 * norm + lm-head, on its last row. (If that attention is unavailable — SV_ATTN=simt, G not in
 * {1, 2, 4} — chunks of <= max_depth + 1 run as SV_PREFILL verifies + commits instead.) After
 * the call the slot holds KV for all n prompt tokens and its pending token is the model's greedy
 * next token, also written to *next_token (host, may be NULL). Synchronous (reads the token back).
 * EINVAL: bad arguments; ESTATE: slot not EMPTY or a verify outstanding. */
sv_status sv_prefill(sv_ctx* ctx, int32_t slot, uint64_t request_id, const int32_t* prompt, int32_t n,
                     int32_t chunk, int32_t* next_token);

/* Prefill side, after a chunked prefill in this lane: pack the first n_tokens committed KV rows
 * of `slot` (all layers, gathered from its pages) plus its pending token into the wire format
 * above. kv_packed: DEVICE, >= sv_kv_packed_bytes(cfg, n_tokens), 16-byte aligned. Stream-ordered
 * on the lane's stream. EINVAL: bad slot / pointer; ESTATE: slot not ACTIVE. n_tokens beyond the
 * slot's length sets SV_DERR_MAX_POS and packs nothing. */
sv_status sv_kv_pack_slot(sv_ctx* ctx, int32_t slot, int32_t n_tokens, void* kv_packed);

/* Append a hand-off message that is already in device memory (same-GPU prefill, or a
 * caller-side transport): kv_packed in the wire format above, n_tokens entries, the
 * pending token from its trailer. sv_append_kv semantics and errors. */
sv_status sv_kv_append_packed(sv_ctx* ctx, int32_t slot, uint64_t request_id, int32_t n_tokens,
                              const void* kv_packed);

/* Transport self-test on one GPU: inside one NCCL group, send kv_packed to this rank
 * and receive it into `staging`, then append it to `slot` (sv_kv_recv_append's path
 * with peer = own rank). nccl_comm: a communicator in which this process is `rank`. */
sv_status sv_kv_loopback_append(sv_ctx* ctx, int32_t slot, uint64_t request_id, int32_t n_tokens,
                                const void* kv_packed, void* staging, int rank, void* nccl_comm);

/* ---- batched page-block hand-off (a9; PAPER.md:255-260 eq:transfer_bandwidth, Alg. 3
 * "Transfer kv via NIXL P2P" PAPER.md:281-283 -> NCCL p2p over NVLink; SURVEY.md §8(e) "grouped per
 * batch of requests" on a comm stream).
 * Wire format of a batch of n requests (ONE ncclSend / ncclRecv), derived by both sides from the
 * host-known token counts (the router knows every prompt length): for request i, for layer l, for
 * page p < ceil(n_tokens[i] / page_size): the (layer, page) block of the KV pool, [2][H_kv][page_size]
 * [d_h] bf16 = 2*H_kv*page_size*d_h*2 bytes (256 KB at Llama-3-8B shape); then the n pending tokens
 * (int32), padded to 16 bytes. Size: sv_kv_slots_bytes. The prefill side gathers the blocks from its
 * pages into `staging`, the decode side receives into its `staging` and scatters the blocks into
 * freshly popped pages (whole-block copies). Rows of a last, partial page past n_tokens carry the
 * sender's (finite) page contents and are masked by len.
 * Everything runs on the lane's own comm stream (created at sv_create), so a verify already enqueued
 * on the lane's stream overlaps the transfer; the lane's later calls that touch one of the
 * transferred slots (verify, append, release, pack) make its stream wait for the transfer (an
 * event). `staging`: caller-owned DEVICE memory, 16-byte aligned, >= sv_kv_slots_bytes, not reused
 * until the transfer is done (the next hand-off call of the lane is ordered after it). The NCCL
 * communicator must span the two lanes' ranks (sv_nccl_comm_init); a failure after the peer has
 * posted its half leaves the communicator unusable (abort it). */
size_t sv_kv_slots_bytes(const sv_config* cfg, int32_t n, const int32_t* n_tokens /*(host)[n]*/);

/* Prefill side: send rows 0..n_tokens[i]-1 of ACTIVE slots[i] (n distinct slots, host arrays) plus
 * their pending tokens to `peer`. Syncs the lane's stream once (reads the committed lengths); the
 * gather and the send then run on the comm stream. The slots stay ACTIVE (sv_release of them waits
 * for the transfer). EINVAL: n < 1, bad / duplicate slot, n_tokens[i] < 1 or > the slot's committed
 * length, bad staging; ESTATE: a slot not ACTIVE, or capturing a graph. */
sv_status sv_kv_send_slots(sv_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* n_tokens, void* staging,
                           int peer, void* nccl_comm);
/* Decode side: the matching receive into EMPTY slots[i] (host), bound to request_ids[i] (the Philox
 * key, as in sv_append_kv): on the comm stream, pops ceil(n_tokens[i] / page_size) pages per request
 * (the device free list is lock-protected, so this runs concurrently with the lane's commits), sets
 * len = n_tokens[i], receives the batch and scatters it. The host never waits for the lane stream (it
 * syncs the comm stream once to check the free-page count). A slot released before is reused after
 * its release kernel. The slots are ACTIVE on return; their first verify waits for the data.
 * EINVAL: bad / duplicate slot, n_tokens[i] < 1 or >= max_pos, bad staging; ESTATE: a slot not
 * EMPTY, or capturing; SV_ENOKV: fewer free pages than the batch needs (checked before anything is
 * popped or posted). */
sv_status sv_kv_recv_slots(sv_ctx* ctx, int32_t n, const int32_t* slots, const uint64_t* request_ids,
                           const int32_t* n_tokens, void* staging, int peer, void* nccl_comm);
/* Transport self-test on one GPU: sv_kv_send_slots from `src` and sv_kv_recv_slots into `dst`
 * (two lanes with the same n_layers / H_kv / d_h / page_size) in ONE group of a communicator in
 * which this process is `rank` (sends to itself), on dst's comm stream. */
sv_status sv_kv_loopback_slots(sv_ctx* src, sv_ctx* dst, int32_t n, const int32_t* src_slots,
                               const int32_t* dst_slots, const uint64_t* request_ids, const int32_t* n_tokens,
                               void* src_staging, void* dst_staging, int rank, void* nccl_comm);

/* Measurement hook: the lane's comm stream (hand-off transfers run there), so a caller can record
 * CUDA events around them. */
sv_status sv_comm_stream(sv_ctx* ctx, sv_stream_t* out);

/* Pack context K/V [n_layers][n][H_kv][d_h] (two tensors) + pending into the
 * hand-off wire format on `stream` (used by the prefill side). */
sv_status sv_kv_pack(const void* k, const void* v, int32_t n_layers, int32_t n_kv_heads,
                     int32_t head_dim, int32_t n_tokens, int32_t pending_token, void* kv_packed,
                     sv_stream_t stream);

/* ---------------- fp32-SIMT exactness instantiation (NEXT-4; S19) ----------------
 * The verify step's model arithmetic (a2-a5: embed, RMSNorm, QKV, RoPE, chain-causal GQA attention over
 * the cache, O-proj + residual, RMSNorm, SwiGLU MLP + residual, final RMSNorm, lm-head) with fp32
 * operands, fp32 accumulation and NO bf16 rounding anywhere: its logits sit within fp32 accumulation
 * error of the fp64 definition (the oracle with its bf16 rounding points switched off). Plain SIMT
 * kernels, stateless; decisions on the logits go through sv_verify_logits (the same finalize). */
typedef struct { /* device pointers, fp32, the layouts of sv_weights; BORROWED */
  const float *embed, *attn_norm, *wqkv, *wo, *ffn_norm, *w_gate_up, *w_down, *final_norm, *lm_head;
} sv_weights_f32;
/* Workspace bytes for T chain rows (the RoPE table covers positions < cfg->max_pos). */
sv_status sv_exact_query_sizes(const sv_config* cfg, int32_t T, size_t* workspace_bytes);
/* logits [T][V] fp32 (device) of the chain rows of `batch` requests: request b's rows
 * row_off[b]..row_off[b+1]-1 (host, row_off[0] = 0, T = row_off[batch]) hold tokens chain_tok (device
 * [T]) at positions ctx_len[b] + j (host ctx_len); its context K/V (post-RoPE) are the first ctx_len[b]
 * rows of cache_k / cache_v (device fp32 [n_layers][batch][max_ctx][H_kv][d_h], dense; NULL when every
 * ctx_len is 0). Enqueued on `stream`. EINVAL on bad sizes, positions >= max_pos or a short workspace. */
sv_status sv_exact_forward(const sv_config* cfg, const sv_weights_f32* w, int32_t batch, const int32_t* row_off,
                           const int32_t* chain_tok, const int32_t* ctx_len, const float* cache_k,
                           const float* cache_v, int32_t max_ctx, void* workspace, size_t workspace_bytes,
                           float* logits, sv_stream_t stream);

/* ---------------- SpecuStream depth controller (NEXT-1; host code, no device work) ----------------
 * PAPER.md §3.5, Alg. 4 "SpecuStream Adaptation", eq:acceptance_gradient ..
 * eq_exponential_smoothing, readings DESIGN.md R21-R24. One sv_flow_state per
 * decode lane; value-in / value-out (the input state is never modified). All structs are host. */
#define SV_SPEC_MAX_H 64
typedef struct {
  double d_base;                 /* baseline depth (5) */
  double gamma;                  /* amplification (5) */
  double d_min, d_max;           /* clip range (2, 20) */
  int32_t h;                     /* flow-vector length, 1..SV_SPEC_MAX_H (10) */
  int32_t projection_source;     /* 0: t_proj from the measured t (Alg. 4); 1: from tau_recent */
  double tau_target;             /* target throughput, tokens/s (400) */
  double micro_batch_numerator;  /* 16 * 5 = 80 (eq:microbatch_size) */
} sv_spec_config;
typedef struct {
  double f[SV_SPEC_MAX_H];       /* flow vector (first h entries used) */
  int32_t idx;                   /* next write index, 0..h-1 */
  int32_t _pad;
  double tau_recent;             /* smoothed throughput, tokens/s */
} sv_flow_state;
typedef struct {
  int32_t depth;                 /* d* = round-half-up(clip(d, d_min, d_max)) */
  int32_t micro_batch;           /* max(1, floor(numerator / d*)) */
  double projected;              /* t_proj */
  double raw_depth, delta, mag, scale, adj;   /* intermediates (audit) */
} sv_spec_plan;

/* Paper defaults (d_base 5, gamma 5, d_min 2, d_max 20, h 10, tau_target 400, numerator 80). */
void sv_spec_default_config(sv_spec_config* cfg);
/* f = 0, idx = 0, tau_recent = tau_target. EINVAL on an invalid cfg
 * (need 1 <= d_min <= d_base <= d_max, 1 <= h <= SV_SPEC_MAX_H, gamma >= 0, tau_target > 0). */
sv_status sv_spec_reset(const sv_spec_config* cfg, sv_flow_state* state);
/* One Alg. 4 step on (a, l, t): a acceptance in [0,1], l load in [0,1], t throughput >= 0.
 * Writes *plan and *out (out may alias in). EINVAL on invalid cfg / state / inputs. */
sv_status sv_spec_adapt(const sv_spec_config* cfg, const sv_flow_state* in, double a, double l, double t,
                        sv_spec_plan* plan, sv_flow_state* out);
/* The lane's control step (R24): from two sv_stats snapshots taken `seconds` apart,
 * a = (accepted1 - accepted0) / (drafted1 - drafted0) (0 when nothing was drafted),
 * t = (emitted1 - emitted0) / seconds, l = active / max_batch; then sv_spec_adapt. */
sv_status sv_spec_step(const sv_spec_config* cfg, const sv_flow_state* in, const sv_lane_stats* s0,
                       const sv_lane_stats* s1, double seconds, int32_t active, int32_t max_batch,
                       sv_spec_plan* plan, sv_flow_state* out);

/* ---------------- FlowGuard lane router (NEXT-2; host code, no device work) ----------------
 * PAPER.md §3.3: eq:flowguard_score, eq:overload_detection / eq:overload_score,
 * eq:fallback_selection and Alg. 2 "FlowGuard Worker Selection"; readings
 * DESIGN.md R25-R28. Routes an incoming request to one of n decode lanes from their published
 * metrics. Pure function of its inputs; all structs are host. */
typedef struct {
  double alpha[4];        /* weights of C, 1-M, 1-Q, 1-L (0.4, 0.1, 0.3, 0.2); >= 0, sum 1 within 1e-9 */
  double tau;             /* overload threshold (0.85), > 0 */
  double q_max;           /* queue-depth normaliser (100), >= 1 */
  int64_t staleness_ms;   /* a snapshot older than this is stale (1000) */
} sv_route_config;
typedef struct {
  int64_t timestamp_ms;   /* when the lane published it */
  double cache_hit;       /* C_w in [0, 1] */
  double mem_util;        /* M_w in [0, 1] */
  double queue_depth;     /* Q_raw >= 0 */
  double active_load;     /* L_w in [0, 1] */
} sv_lane_metrics;
#define SV_ROUTE_OVERLOADED 1
#define SV_ROUTE_STALE 2

/* Paper defaults. */
void sv_route_default_config(sv_route_config* cfg);
/* Alg. 2 over n >= 1 lanes at time now_ms. live_queue: NULL or n fresh queue depths that replace
 * the snapshots' (Alg. 2 "load_i.qd <- Q_{P_i}.size()"). Writes *chosen; optional outputs:
 * scores[n] (NaN for excluded lanes), flags[n] (SV_ROUTE_* bits), *used_fallback (1 when every
 * lane was stale or overloaded and the argmin queue depth was taken). Ties: lowest index.
 * EINVAL on invalid cfg / metrics (fractions outside [0,1], negative queue, n < 1, NULL). */
sv_status sv_route_select(const sv_route_config* cfg, int32_t n, const sv_lane_metrics* metrics,
                          const double* live_queue, int64_t now_ms, int32_t* chosen, double* scores,
                          uint8_t* flags, int32_t* used_fallback);

#ifdef __cplusplus
}
#endif
#endif /* SV_H_ */
