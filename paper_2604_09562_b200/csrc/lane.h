// Internal (non-ABI) view of one decode lane: device pointers + sizes passed
// by value to every kernel, and the launch functions each kernel file exports.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace sv {

typedef __nv_bfloat16 bf16;

constexpr int kMaxBatch = 256;     // PlanArgs capacity (requests per verify)
constexpr int kMaxDepth = 32;      // k_i <= 32 (sv_lane_stats histograms have 33 bins)
constexpr int kVocabTile = 128;    // lm-head epilogue statistics tile
constexpr int kAttnRows = 64;      // (k+1) * G query rows per (request, kv head) of the keys-on-lanes / SIMT kernels
constexpr int kPartRows = 128;     // split-KV partial rows per work item (rows-on-lanes kernel: <= 32 rows x G <= 4)
#ifndef SV_SPLIT_KEYS
#define SV_SPLIT_KEYS 1024
#endif
constexpr int kSplitKeys = SV_SPLIT_KEYS;   // page keys per split-KV work item
constexpr int kNumStats = 6 + 3 * (kMaxDepth + 1);
constexpr int kMaxRaceSplits = 16;
constexpr int kFiltCap = 2048;     // top-k / top-p filter: candidate capacity (= FLT_CAP, k_finalize.cu)
constexpr int kPrefillNoHead = 3;  // internal finalize mode: a prefill chunk whose lm-head was skipped  // finalize: CTAs per request sharing a sampled row's race

struct RacePart { float rs; int rx; float ps; int px; float sr; int pad[3]; };   // one race slice's result

// indices into the u64 stats array (mirrors sv_lane_stats)
enum { ST_STEPS = 0, ST_ROWS, ST_DRAFTED, ST_ACCEPTED, ST_EMITTED, ST_INDEP, ST_HIST,
       ST_DRAFTED_BY_K = ST_HIST + kMaxDepth + 1, ST_ACCEPTED_BY_K = ST_DRAFTED_BY_K + kMaxDepth + 1 };

struct LaneDev {
  // configuration
  int n_layers, D, Hq, Hkv, dh, V, F, page, n_pages, max_slots, max_batch, max_depth, max_pos;
  int max_pages_per_slot, nt, qkv_rows, Tmax;
  int tree;                          // this verify's drafts are a token tree (R30), set per call
  int filt_on;                       // top-k / top-p filtered target (R31), set per call
  float eps;
  // borrowed weights (bf16)
  const bf16 *embed, *attn_norm, *wqkv, *wo, *ffn_norm, *w_gate_up, *w_down, *final_norm, *lm_head;
  bf16* pool;                        // [n_layers][n_pages][2][Hkv][page][dh]
  // persistent lane state (workspace)
  int* len;                          // [max_slots]
  int* pending;                      // [max_slots]
  unsigned long long* rid;           // [max_slots]
  int* page_table;                   // [max_slots][max_pages_per_slot]
  int* free_list;                    // [n_pages]
  int* free_top;                     // [2]: stack top, free-list spin lock
  unsigned long long* stats;         // [kNumStats]
  int* err;                          // [1] sticky SV_DERR_* bits
  const float *rope_cos, *rope_sin;  // [max_pos][dh/2]
  // per-call buffers (workspace)
  int *slots, *depths, *row_off, *row_req, *row_pos, *chain_tok, *req_err;
  float *h0, *h1, *h2, *cbuf, *logits, *tile_max, *tile_sum;
  int* tile_arg;
  bf16 *a, *b, *z, *q, *kc, *vc, *o, *u;
  int4* items;                       // attention work list: (request, kv head, split, 0)
  int4* row_comb;                    // [Tmax] split-KV combine: (chain row j, splits, first item, 0)
  int *item_start, *n_items;
  float *part_o, *part_ml;           // split-KV partials
  int *acc_int, *tok_int;            // internal copies of accepted_len / out_tokens for commit
  int* path_int;                     // [max_batch][max_depth+1] accepted path's chain rows (commit)
  unsigned long long* row_anc;       // [Tmax] ancestor-or-self node mask of each chain row
  int* fin_cnt;                      // [max_batch] finished race slices (zero between verifies)
  unsigned long long* row_best;      // [Tmax] greedy argmax keys from the lm-head epilogue (zero between verifies)
  RacePart* fin_part;                // [max_batch][kMaxRaceSplits]
  unsigned* filt_key;                // [Tmax] R31 filter: threshold key of the scaled logit
  int* filt_tie;                     // [Tmax] largest kept token id among threshold ties
  float *filt_inv, *filt_m;          // [Tmax] 1 / kept mass, row max (scaled logits)
  int* filt_ids;                     // [Tmax][kFiltCap] kept token ids (filter fast path), any order
  int* filt_cnt;                     // [Tmax] their number, or -1 (slow path: no list)
  int* batch_n;                      // [1] batch of the pending verify (device copy)
  int* T_dev;                        // [1] chain rows of the current verify / prefill chunk (plan writes it);
                                     // row-gridded kernels launched for Tmax rows return beyond it
  const int* dyn_ctrl;               // dynamic-depth CUDA graph (sv_graph_begin_dynamic): device copies of
                                     // this verify's slots [batch] then depths [batch]; nullptr otherwise
  unsigned long long* trace;         // [16][256] clock64 trace of CTA 0 (SV_TRACE=1) or nullptr
};

// Split-KV work items: request b (cache length L, R = k + 1 chain rows) is split over its
// page keys [0, L) into ceil(L / kSplitKeys) items (at least one); the chain keys L..L+R-1
// always belong to the last item. Item s covers keys [split_t0, split_t1).
__host__ __device__ inline int num_splits(int L) { return L <= 0 ? 1 : (L + kSplitKeys - 1) / kSplitKeys; }
__host__ __device__ inline int split_t0(int s) { return s * kSplitKeys; }
__host__ __device__ inline int split_t1(int s, int ns, int L, int R) {
  return s == ns - 1 ? L + R : (s + 1) * kSplitKeys;
}
// Wide splits (per verify, chosen by plan_embed_kernel): items of (kSplitKeys << wide) page keys. An
// item's .w holds ns | wide << 24; the helpers below take the split size explicitly.
constexpr int kItemWideShift = 24;
__host__ __device__ inline int item_ns(int w) { return w & ((1 << kItemWideShift) - 1); }
__host__ __device__ inline int item_split_keys(int w) { return kSplitKeys << (w >> kItemWideShift); }
__host__ __device__ inline int num_splits_k(int L, int sk) { return L <= 0 ? 1 : (L + sk - 1) / sk; }
__host__ __device__ inline int split_t1_k(int s, int ns, int L, int R, int sk) {
  return s == ns - 1 ? L + R : (s + 1) * sk;
}

// kernels launched by the library so far (measurement hook, sv_launch_count)
extern unsigned long long g_launch_count;
#define SV_COUNT_LAUNCH() (++::sv::g_launch_count)

// Programmatic dependent launch (PDL) for the step's kernels: the next kernel in the stream may be
// scheduled while this one finishes; every kernel calls pdl_wait() (griddepcontrol.wait) before it
// touches anything an earlier kernel of the step writes, so only its prologue (barrier / TMEM
// setup, weight prefetch) overlaps. SV_PDL=0 launches them normally.
bool pdl_enabled();

// Opt `kernel` into `bytes` of dynamic shared memory on the CURRENT device. The attribute is per
// device and one process may create lanes on several GPUs, so the opt-in is remembered per
// (kernel, device), not once per process.
cudaError_t smem_optin(const void* kernel, int bytes);
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

struct PlanArgs {
  int batch, T;
  int slots[kMaxBatch];
  int depths[kMaxBatch];
};

// ---- launchers (stream-ordered; return cudaGetLastError()) ----
// parents: NULL (chains) or device [sum k] node parents of a token tree (R30)
cudaError_t launch_plan(const LaneDev& d, const PlanArgs& p, const int* draft_tokens, const int* parents, bool attn,
                        cudaStream_t s);
cudaError_t launch_embed_norm(const LaneDev& d, int T, cudaStream_t s);
// a1 + a2 in one launch (plan tables, work items and the embed + RMSNorm of each row; `rows` = T, or
// Tmax for a dynamic-depth graph); requires plan_embed_supported(d)
bool plan_embed_supported(const LaneDev& d);
cudaError_t launch_plan_embed(const LaneDev& d, const PlanArgs& p, const int* draft_tokens, const int* parents,
                              int rows, bool allow_wide, cudaStream_t s);
cudaError_t launch_rmsnorm(const LaneDev& d, const float* x, const bf16* g, bf16* out, int T, cudaStream_t s,
                           bool bound_by_T_dev = true);
// C[M][N] (fp32) = A[M][K] (bf16) * B[N][K]^T (bf16)
cudaError_t launch_gemm_simt(const bf16* A, const bf16* B, float* C, int M, int N, int K, cudaStream_t s);
cudaError_t launch_qkv_rope_epilogue(const LaneDev& d, int layer, int T, cudaStream_t s);
cudaError_t launch_residual_epilogue(const float* hin, const float* c, float* hout, int T, int D, cudaStream_t s);
cudaError_t launch_swiglu_epilogue(const LaneDev& d, int T, cudaStream_t s);
cudaError_t launch_tile_stats(const LaneDev& d, int T, float inv_temp, cudaStream_t s);
cudaError_t launch_attention(const LaneDev& d, int layer, int batch, cudaStream_t s);
// skip_single: rows of requests with one split-KV item were written by the attention kernel itself
cudaError_t launch_attn_combine(const LaneDev& d, int T, bool skip_single, cudaStream_t s);
// use_row_best: greedy / prefill argmaxes come from d.row_best (filled by the lm-head epilogue)
cudaError_t launch_finalize(const LaneDev& d, int batch, const int* draft_tokens, const int* parents,
                            const float* draft_probs, const float* logits, uint64_t seed, int mode, float inv_temp,
                            int* accepted_len, int* out_tokens, int* accepted_nodes, cudaStream_t s,
                            bool use_row_best = false);
cudaError_t launch_filter(const LaneDev& d, int T, float inv_temp, int top_k, float top_p, cudaStream_t s);
cudaError_t launch_commit(const LaneDev& d, const int* n_keep, int batch, cudaStream_t s);
cudaError_t launch_append(const LaneDev& d, int slot, unsigned long long rid, const bf16* k, const bf16* v,
                          int n, int pending, const int* pending_dev, int packed, cudaStream_t s);
cudaError_t launch_release(const LaneDev& d, int slot, cudaStream_t s);
cudaError_t launch_handoff_gather(const LaneDev& d, const int* slots, const int* ns, const int* bstart, int n,
                                  char* staging, cudaStream_t s);
cudaError_t launch_handoff_scatter(const LaneDev& d, const int* slots, const int* ns, const int* bstart, int n,
                                   const char* staging, cudaStream_t s);
cudaError_t launch_handoff_alloc(const LaneDev& d, const int* slots, const unsigned long long* rids, const int* ns,
                                 int n, cudaStream_t s);
cudaError_t launch_init_state(const LaneDev& d, cudaStream_t s);
cudaError_t launch_debug_uniforms(uint64_t seed, uint64_t rid, uint32_t z, int purpose, int x0, int n, float* u,
                                  cudaStream_t s);
cudaError_t launch_draft_planted(const LaneDev& d, const PlanArgs& p, const int* succ, const uint8_t* mask,
                                 const int* dev_tok, const int* parents, int* draft_tokens, cudaStream_t s);
// NEXT-3 long-chunk prefill (k_prefill.cu, k_attn_prefill.cu via attn_prefill_run)
cudaError_t launch_prefill_plan(const LaneDev& d, int slot, const int* tokens, int C, cudaStream_t s);
cudaError_t launch_prefill_kv(const LaneDev& d, int layer, int C, cudaStream_t s);
cudaError_t launch_prefill_finish(const LaneDev& d, int C, int next_token, int* y_out, cudaStream_t s);
cudaError_t launch_kv_pack_slot(const LaneDev& d, int slot, int n, void* packed, cudaStream_t s);
cudaError_t launch_kv_pack(const bf16* k, const bf16* v, int n_layers, int Hkv, int dh, int n, int pending,
                           void* packed, cudaStream_t s);

}  // namespace sv
