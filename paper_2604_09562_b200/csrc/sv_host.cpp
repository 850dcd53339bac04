// Host runtime behind include/sv.h: configuration checks, workspace layout, the per-slot
// state machine, and the stream-ordered launch sequence of the verify step.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/sv.h"
#include "lane.h"
#include "gemm.h"

using sv::bf16;

namespace {

enum SlotState { EMPTY = 0, ACTIVE = 1, PENDING = 2 };

struct Layout {
  size_t total = 0;
  size_t rope_cos, rope_sin, len, pending, rid, page_table, free_list, free_top, stats, err;
  size_t slots, depths, row_off, row_req, row_pos, chain_tok, req_err;
  size_t h0, h1, h2, cbuf, logits, tile_max, tile_sum, tile_arg;
  size_t a, b, z, q, kc, vc, o, u;
  size_t items, item_start, n_items, part_o, part_ml, acc_int, tok_int, batch_n, path_int, row_anc, row_comb, filt, fin_cnt, fin_part, row_best, filt_ids;
  size_t gemm_ws, trace, prefill, handoff, tdev, dctrl;
  size_t max_items;

  size_t take(size_t bytes) {
    total = (total + 1023) & ~size_t(1023);
    const size_t off = total;
    total += bytes;
    return off;
  }
};

size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

bool valid_cfg(const sv_config* c) {
  if (!c) return false;
  if (c->n_layers < 1 || c->d_model < 64 || c->n_q_heads < 1 || c->n_kv_heads < 1 || c->vocab < 1) return false;
  if (c->n_q_heads % c->n_kv_heads) return false;
  if (c->head_dim != 64 && c->head_dim != 128) return false;
  if (c->d_model % 64 || c->ffn_dim < 0 || c->ffn_dim % 64) return false;
  if ((c->n_q_heads * c->head_dim) % 64) return false;
  if (c->page_size < 8 || c->page_size % 8 || c->n_pages < 1 || c->max_slots < 1) return false;
  if (c->max_batch < 1 || c->max_batch > sv::kMaxBatch) return false;
  if (c->max_depth < 0 || c->max_depth > sv::kMaxDepth) return false;
  {                                           // query rows per (request, kv head): keys-on-lanes / SIMT
    const int G = c->n_q_heads / c->n_kv_heads;   // kernels take (k+1) G <= 64, the rows-on-lanes one
    if ((c->max_depth + 1) * G > sv::kAttnRows && !(G <= 4 && c->max_depth + 1 <= 32)) return false;   // k+1 <= 32, G <= 4
  }
  if (c->max_pos < c->max_depth + 2) return false;
  if (!(c->rope_theta > 0.f) || !(c->norm_eps >= 0.f)) return false;
  return true;
}

Layout make_layout(const sv_config& c) {
  Layout L;
  const size_t T = (size_t)c.max_batch * (c.max_depth + 1);
  const size_t D = c.d_model, V = c.vocab, F = c.ffn_dim;
  const size_t nq = (size_t)c.n_q_heads * c.head_dim, nkv = (size_t)c.n_kv_heads * c.head_dim;
  const size_t qkv_rows = nq + 2 * nkv;
  const size_t mpps = ceil_div(c.max_pos, c.page_size);
  const size_t nt = ceil_div(V, sv::kVocabTile);
  L.rope_cos = L.take(4 * (size_t)c.max_pos * c.head_dim / 2);
  L.rope_sin = L.take(4 * (size_t)c.max_pos * c.head_dim / 2);
  L.len = L.take(4 * c.max_slots);
  L.pending = L.take(4 * c.max_slots);
  L.rid = L.take(8 * c.max_slots);
  L.page_table = L.take(4 * c.max_slots * mpps);
  L.free_list = L.take(4 * (size_t)c.n_pages);
  L.free_top = L.take(8);                          // [0] stack top, [1] spin lock (k_kv.cu)
  L.stats = L.take(8 * sv::kNumStats);
  L.err = L.take(4);
  L.slots = L.take(4 * c.max_batch);
  L.depths = L.take(4 * c.max_batch);
  L.row_off = L.take(4 * (c.max_batch + 1));
  L.row_req = L.take(4 * T);
  L.row_pos = L.take(4 * T);
  L.chain_tok = L.take(4 * T);
  L.req_err = L.take(4 * c.max_batch);
  L.h0 = L.take(4 * T * D);
  L.h1 = L.take(4 * T * D);
  L.h2 = L.take(4 * T * D);
  size_t cmax = qkv_rows;
  if (D > cmax) cmax = D;
  if (2 * F > cmax) cmax = 2 * F;
  L.cbuf = L.take(4 * T * cmax);
  L.logits = L.take(4 * T * V);
  L.tile_max = L.take(4 * T * nt);
  L.tile_sum = L.take(4 * T * nt);
  L.tile_arg = L.take(4 * T * nt);
  L.a = L.take(2 * T * D);
  L.b = L.take(2 * T * D);
  L.z = L.take(2 * T * D);
  L.q = L.take(2 * T * nq);
  L.kc = L.take(2 * (size_t)c.n_layers * T * nkv);
  L.vc = L.take(2 * (size_t)c.n_layers * T * nkv);
  L.o = L.take(2 * T * nq);
  L.u = L.take(2 * T * (F ? F : 1));
  // attention work items: sum over requests of Hkv * ceil((L_i + R_i) / split)
  const size_t max_keys = (size_t)c.n_pages * c.page_size;
  L.max_items = (size_t)c.n_kv_heads * (ceil_div(max_keys, sv::kSplitKeys) + c.max_batch);
  L.items = L.take(16 * L.max_items);
  L.item_start = L.take(4 * (c.max_batch + 1));
  L.n_items = L.take(16);
  L.part_o = L.take(4 * L.max_items * sv::kPartRows * c.head_dim);
  L.part_ml = L.take(8 * L.max_items * sv::kPartRows);
  L.acc_int = L.take(4 * c.max_batch);
  L.tok_int = L.take(4 * c.max_batch * (c.max_depth + 1));
  L.batch_n = L.take(4);
  L.path_int = L.take(4 * c.max_batch * (c.max_depth + 1));
  L.row_anc = L.take(8 * T);
  L.row_comb = L.take(16 * T);
  L.filt = L.take(16 * T);
  L.filt_ids = L.take(4 * T * sv::kFiltCap + 4 * T);
  L.fin_cnt = L.take(4 * c.max_batch);
  L.row_best = L.take(8 * T);
  L.fin_part = L.take(sizeof(sv::RacePart) * sv::kMaxRaceSplits * c.max_batch);
  L.gemm_ws = L.take(sv::gemm_workspace_bytes((int)T, (int)cmax));
  L.trace = L.take(8 * 16 * 256);
  // sv_prefill: outputs of a chunk + the whole prompt (copied to the device once, <= max_pos tokens)
  L.prefill = L.take(4 * (2 * (size_t)(c.max_depth + 2) + (size_t)c.max_pos));
  // batched hand-off (sv_kv_send_slots / sv_kv_recv_slots): slots, token counts, block starts [max_slots + 1]
  // i32 + request ids [max_slots] u64
  L.handoff = L.take(4 * (4 * (size_t)c.max_slots + 4) + 8 * (size_t)c.max_slots);
  L.tdev = L.take(16);                                  // rows of the current verify (plan writes it)
  L.dctrl = L.take(8 * (size_t)c.max_batch);            // dynamic-depth graph: slots | depths of a replay
  L.total = (L.total + 1023) & ~size_t(1023);
  return L;
}

}  // namespace

// live per-stage timing with CUDA events on the lane's stream (sv_profile_*)
enum Stage { ST_PLAN = 0, ST_EMBED, ST_QKV, ST_ATTN, ST_COMBINE, ST_OPROJ, ST_FFN_NORM, ST_GATE_UP, ST_DOWN,
             ST_FINAL_NORM, ST_LM_HEAD, ST_FINALIZE, ST_COMMIT, ST_DRAFT, ST_ATTN_NORM, ST_FILTER, ST_NUM };
static const char* kStageNames[ST_NUM] = {"plan", "embed_norm", "qkv_rope", "attention", "attn_combine", "o_proj",
                                          "ffn_norm", "gate_up_swiglu", "down", "final_norm", "lm_head",
                                          "finalize", "commit", "draft", "attn_norm", "filter"};

struct Prof {
  uint32_t mask = 0;                          // bit i: time stage i
  std::vector<cudaEvent_t> free_ev;
  struct Rec { int stage; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<Rec> captured;                  // stage events recorded into a CUDA graph being captured
  double ms[ST_NUM] = {};
  long long n[ST_NUM] = {};
  cudaEvent_t get() {
    if (free_ev.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = free_ev.back();
    free_ev.pop_back();
    return e;
  }
};

struct sv_ctx {
  sv_config cfg;
  sv_weights w;
  char* pool;
  char* ws;
  cudaStream_t stream;
  Layout lay;
  sv::LaneDev d;
  std::vector<int> state;
  std::vector<unsigned long long> rid;
  bool pending_verify = false;
  int pending_batch = 0;
  std::vector<int> pending_slots;
  int last_T = 0, last_batch = 0;
  int sticky = 0;
  bool taps = false;                 // keep every intermediate (fp32 logits included) for sv_get_tap
  bool capturing = false;            // between sv_graph_begin and sv_graph_end
  unsigned long long capture_launches0 = 0;
  int top_k = 0;                     // R31 filtered target for SAMPLE (0 / >= 1: off), sv_set_filter
  float top_p = 1.0f;
  sv::GemmPlan* gemm = nullptr;
  Prof prof;
  // prefill -> decode hand-off (a9): NCCL transfers run on their own stream so a verify already
  // enqueued on `stream` overlaps them; the lane's next device work waits for comm_done
  cudaStream_t comm = nullptr;
  cudaEvent_t comm_done = nullptr, lane_mark = nullptr;
  bool comm_pending = false;
  std::vector<char> comm_slot;       // slots whose pages / pending token a posted transfer reads or writes
  std::vector<cudaEvent_t> rel_ev;   // per slot: recorded after its last release (a receive into it waits)
  std::vector<char> rel_pending;
  // dynamic-depth CUDA graph (sv_graph_begin_dynamic): a replay's slots | depths are staged in one of
  // two pinned host buffers [2][2 max_batch] and copied to the device by the graph's first node
  int* pin_ctrl = nullptr;
  cudaEvent_t ctrl_consumed = nullptr;
  // the two pinned staging buffers belong to the lane, so several dynamic graphs can alternate: each
  // sv_graph_set_batch takes the next buffer (once the replay that last read it has finished) and the
  // graph's next launch consumes it
  long long dyn_stage_seq = 0;
  cudaEvent_t dyn_done[2] = {nullptr, nullptr};
  bool dyn_done_set[2] = {false, false};
  bool dyn_unlaunched[2] = {false, false};
  bool dyn_capture = false;
  int dyn_batch = 0;
};

// make the lane's stream wait for the posted hand-off transfers (sends read pages, receives write
// pages and pending tokens); wait_comm_slots only when the call touches one of their slots, so a
// verify of other requests overlaps the transfer
static void wait_comm(sv_ctx* c) {
  if (c->comm_pending) {
    cudaStreamWaitEvent(c->stream, c->comm_done, 0);
    c->comm_pending = false;
    std::fill(c->comm_slot.begin(), c->comm_slot.end(), 0);
  }
}
static void wait_comm_slots(sv_ctx* c, int n, const int32_t* slots) {
  if (!c->comm_pending) return;
  for (int i = 0; i < n; ++i)
    if (c->comm_slot[slots[i]]) {
      wait_comm(c);
      return;
    }
}

// while capturing a graph the records must become event-record NODES (cudaEventRecordExternal), which
// sv_graph_launch re-points per replay; a plain record would only order the capture
static void prof_record(sv_ctx* c, cudaEvent_t e) {
  if (c->capturing) cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal);
  else cudaEventRecord(e, c->stream);
}
static cudaEvent_t prof_begin(sv_ctx* c, int stage) {
  if (!(c->prof.mask >> stage & 1u)) return nullptr;
  cudaEvent_t e = c->prof.get();
  prof_record(c, e);
  return e;
}
// fold finished records into the totals; never blocks the host (a blocking fold would drain
// the stream and put bubbles into the very region being timed)
static void prof_fold(sv_ctx* c, bool wait) {
  size_t keep = 0;
  auto& recs = c->prof.recs;
  for (size_t i = 0; i < recs.size(); ++i) {
    auto& r = recs[i];
    if (!wait && cudaEventQuery(r.b) != cudaSuccess) {
      recs[keep++] = r;
      continue;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    c->prof.ms[r.stage] += ms;
    c->prof.n[r.stage] += 1;
    c->prof.free_ev.push_back(r.a);
    c->prof.free_ev.push_back(r.b);
  }
  recs.resize(keep);
}
static void prof_end(sv_ctx* c, int stage, cudaEvent_t a) {
  if (!a) return;
  cudaEvent_t b = c->prof.get();
  prof_record(c, b);
  if (c->capturing) {                         // event-record nodes of the graph: timed per replay
    c->prof.captured.push_back({stage, a, b});
    return;
  }
  c->prof.recs.push_back({stage, a, b});
  if (c->prof.recs.size() >= 8192 && c->prof.recs.size() % 1024 == 0) prof_fold(c, false);
}
// run `expr` (returning sv_status or cudaError_t) as timed stage `id`
#define STAGE(c, id, expr)                    \
  do {                                        \
    cudaEvent_t _pe = prof_begin(c, id);      \
    auto _r = (expr);                         \
    prof_end(c, id, _pe);                     \
    if (_r) return stage_status(_r);          \
  } while (0)
static sv_status stage_status(cudaError_t e);
static sv_status stage_status(sv_status s) { return s; }

static sv_status cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) {
    fprintf(stderr, "[sv] CUDA error: %s\n", cudaGetErrorString(e));
    return SV_ECUDA;
  }
  return SV_OK;
}
static sv_status stage_status(cudaError_t e) { return cuda_ok(e); }
#define SV_CUDA(x)                                   \
  do {                                               \
    sv_status _s = cuda_ok(x);                       \
    if (_s != SV_OK) return _s;                      \
  } while (0)

extern "C" {

const char* sv_version(void) { return "sv 0.1 sm_100a"; }

const char* sv_strerror(sv_status s) {
  switch (s) {
    case SV_OK: return "ok";
    case SV_EINVAL: return "invalid argument";
    case SV_ESTATE: return "call not allowed in the current slot/context state";
    case SV_ENOKV: return "KV page free list exhausted (device)";
    case SV_ECUDA: return "CUDA error";
    case SV_ENCCL: return "NCCL error";
    case SV_EDEVICE: return "device-detected error (bad token id / bad n_keep)";
  }
  return "unknown status";
}

sv_status sv_query_sizes(const sv_config* cfg, size_t* kv_pool_bytes, size_t* workspace_bytes) {
  if (!valid_cfg(cfg) || !kv_pool_bytes || !workspace_bytes) return SV_EINVAL;
  *kv_pool_bytes = (size_t)cfg->n_layers * cfg->n_pages * 2 * cfg->n_kv_heads * cfg->page_size * cfg->head_dim * 2;
  *workspace_bytes = make_layout(*cfg).total;
  return SV_OK;
}

sv_status sv_create(const sv_config* cfg, const sv_weights* w, void* kv_pool, void* workspace,
                    sv_stream_t stream, sv_ctx** out) {
  if (!valid_cfg(cfg) || !w || !kv_pool || !workspace || !out) return SV_EINVAL;
  if (((uintptr_t)kv_pool | (uintptr_t)workspace) & 1023) return SV_EINVAL;
  const void* wp[] = {w->embed, w->attn_norm, w->wqkv, w->wo, w->final_norm, w->lm_head};
  for (const void* p : wp)
    if (!p || ((uintptr_t)p & 15)) return SV_EINVAL;
  if (cfg->ffn_dim > 0 && (!w->ffn_norm || !w->w_gate_up || !w->w_down)) return SV_EINVAL;
  sv_ctx* c = new sv_ctx();
  c->cfg = *cfg;
  c->w = *w;
  c->pool = (char*)kv_pool;
  c->ws = (char*)workspace;
  c->stream = (cudaStream_t)stream;
  c->lay = make_layout(*cfg);
  c->state.assign(cfg->max_slots, EMPTY);
  c->comm_slot.assign(cfg->max_slots, 0);
  c->rel_ev.assign(cfg->max_slots, nullptr);
  c->rel_pending.assign(cfg->max_slots, 0);
  c->rid.assign(cfg->max_slots, 0ull);
  const Layout& L = c->lay;
  char* ws = c->ws;
  sv::LaneDev& d = c->d;
  memset(&d, 0, sizeof(d));
  d.n_layers = cfg->n_layers;
  d.D = cfg->d_model;
  d.Hq = cfg->n_q_heads;
  d.Hkv = cfg->n_kv_heads;
  d.dh = cfg->head_dim;
  d.V = cfg->vocab;
  d.F = cfg->ffn_dim;
  d.page = cfg->page_size;
  d.n_pages = cfg->n_pages;
  d.max_slots = cfg->max_slots;
  d.max_batch = cfg->max_batch;
  d.max_depth = cfg->max_depth;
  d.max_pos = cfg->max_pos;
  d.max_pages_per_slot = (int)ceil_div(cfg->max_pos, cfg->page_size);
  d.nt = (int)ceil_div(cfg->vocab, sv::kVocabTile);
  d.qkv_rows = (cfg->n_q_heads + 2 * cfg->n_kv_heads) * cfg->head_dim;
  d.Tmax = cfg->max_batch * (cfg->max_depth + 1);
  d.eps = cfg->norm_eps;
  d.embed = (const bf16*)w->embed;
  d.attn_norm = (const bf16*)w->attn_norm;
  d.wqkv = (const bf16*)w->wqkv;
  d.wo = (const bf16*)w->wo;
  d.ffn_norm = (const bf16*)w->ffn_norm;
  d.w_gate_up = (const bf16*)w->w_gate_up;
  d.w_down = (const bf16*)w->w_down;
  d.final_norm = (const bf16*)w->final_norm;
  d.lm_head = (const bf16*)w->lm_head;
  d.pool = (bf16*)kv_pool;
  d.len = (int*)(ws + L.len);
  d.pending = (int*)(ws + L.pending);
  d.rid = (unsigned long long*)(ws + L.rid);
  d.page_table = (int*)(ws + L.page_table);
  d.free_list = (int*)(ws + L.free_list);
  d.free_top = (int*)(ws + L.free_top);
  d.stats = (unsigned long long*)(ws + L.stats);
  d.err = (int*)(ws + L.err);
  d.rope_cos = (const float*)(ws + L.rope_cos);
  d.rope_sin = (const float*)(ws + L.rope_sin);
  d.slots = (int*)(ws + L.slots);
  d.depths = (int*)(ws + L.depths);
  d.row_off = (int*)(ws + L.row_off);
  d.row_req = (int*)(ws + L.row_req);
  d.row_pos = (int*)(ws + L.row_pos);
  d.chain_tok = (int*)(ws + L.chain_tok);
  d.req_err = (int*)(ws + L.req_err);
  d.h0 = (float*)(ws + L.h0);
  d.h1 = (float*)(ws + L.h1);
  d.h2 = (float*)(ws + L.h2);
  d.cbuf = (float*)(ws + L.cbuf);
  d.logits = (float*)(ws + L.logits);
  d.tile_max = (float*)(ws + L.tile_max);
  d.tile_sum = (float*)(ws + L.tile_sum);
  d.tile_arg = (int*)(ws + L.tile_arg);
  d.a = (bf16*)(ws + L.a);
  d.b = (bf16*)(ws + L.b);
  d.z = (bf16*)(ws + L.z);
  d.q = (bf16*)(ws + L.q);
  d.kc = (bf16*)(ws + L.kc);
  d.vc = (bf16*)(ws + L.vc);
  d.o = (bf16*)(ws + L.o);
  d.u = (bf16*)(ws + L.u);
  d.items = (int4*)(ws + L.items);
  d.item_start = (int*)(ws + L.item_start);
  d.n_items = (int*)(ws + L.n_items);
  d.part_o = (float*)(ws + L.part_o);
  d.part_ml = (float*)(ws + L.part_ml);
  d.acc_int = (int*)(ws + L.acc_int);
  d.tok_int = (int*)(ws + L.tok_int);
  d.batch_n = (int*)(ws + L.batch_n);
  d.path_int = (int*)(ws + L.path_int);
  d.row_anc = (unsigned long long*)(ws + L.row_anc);
  d.row_comb = (int4*)(ws + L.row_comb);
  d.tree = 0;
  d.filt_on = 0;
  d.fin_cnt = (int*)(ws + L.fin_cnt);
  d.T_dev = (int*)(ws + L.tdev);
  d.dyn_ctrl = nullptr;
  d.row_best = (unsigned long long*)(ws + L.row_best);
  d.fin_part = (sv::RacePart*)(ws + L.fin_part);
  d.filt_key = (unsigned*)(ws + L.filt);
  d.filt_tie = (int*)(ws + L.filt + 4 * (size_t)d.Tmax);
  d.filt_inv = (float*)(ws + L.filt + 8 * (size_t)d.Tmax);
  d.filt_m = (float*)(ws + L.filt + 12 * (size_t)d.Tmax);
  d.filt_ids = (int*)(ws + L.filt_ids);
  d.filt_cnt = (int*)(ws + L.filt_ids + 4 * (size_t)d.Tmax * sv::kFiltCap);
  d.trace = getenv("SV_TRACE") ? (unsigned long long*)(ws + L.trace) : nullptr;

  // RoPE table: fp64 angles pos * theta^(-2m/d_h), stored fp32 (SURVEY.md §8(c) "Model details")
  const int half = cfg->head_dim / 2;
  std::vector<float> cs((size_t)cfg->max_pos * half), sn((size_t)cfg->max_pos * half);
  for (int m = 0; m < half; ++m) {
    const double inv_freq = 1.0 / pow((double)cfg->rope_theta, 2.0 * m / cfg->head_dim);
    for (int p = 0; p < cfg->max_pos; ++p) {
      const double ang = (double)p * inv_freq;
      cs[(size_t)p * half + m] = (float)cos(ang);
      sn[(size_t)p * half + m] = (float)sin(ang);
    }
  }
  sv_status st = SV_OK;
  if ((st = cuda_ok(cudaMemcpyAsync(ws + L.rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, c->stream))) ||
      (st = cuda_ok(cudaMemcpyAsync(ws + L.rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice, c->stream))) ||
      (st = cuda_ok(cudaMemsetAsync(kv_pool, 0, (size_t)cfg->n_layers * cfg->n_pages * 2 * cfg->n_kv_heads *
                                                    cfg->page_size * cfg->head_dim * 2, c->stream))) ||
      (st = cuda_ok(cudaMemsetAsync(ws + L.page_table, 0xff, 4 * (size_t)cfg->max_slots * d.max_pages_per_slot,
                                    c->stream))) ||
      (st = cuda_ok(cudaMemsetAsync(ws + L.fin_cnt, 0, 4 * (size_t)cfg->max_batch, c->stream))) ||
      (st = cuda_ok(cudaMemsetAsync(ws + L.row_best, 0, 8 * (size_t)d.Tmax, c->stream))) ||
      (st = cuda_ok(sv::launch_init_state(d, c->stream)))) {
    delete c;
    return st;
  }
  c->gemm = sv::gemm_plan_create(d, ws + L.gemm_ws, c->stream);
  if ((st = cuda_ok(cudaStreamSynchronize(c->stream))) ||
      (st = cuda_ok(cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking))) ||
      (st = cuda_ok(cudaEventCreateWithFlags(&c->comm_done, cudaEventDisableTiming))) ||
      (st = cuda_ok(cudaEventCreateWithFlags(&c->lane_mark, cudaEventDisableTiming))) ||
      (st = cuda_ok(cudaEventCreateWithFlags(&c->ctrl_consumed, cudaEventDisableTiming))) ||
      (st = cuda_ok(cudaEventCreateWithFlags(&c->dyn_done[0], cudaEventDisableTiming))) ||
      (st = cuda_ok(cudaEventCreateWithFlags(&c->dyn_done[1], cudaEventDisableTiming))) ||
      (st = cuda_ok(cudaHostAlloc((void**)&c->pin_ctrl, 16 * (size_t)cfg->max_batch, cudaHostAllocDefault)))) {
    sv::gemm_plan_destroy(c->gemm);
    if (c->comm) cudaStreamDestroy(c->comm);
    if (c->comm_done) cudaEventDestroy(c->comm_done);
    delete c;
    return st;
  }
  *out = c;
  return SV_OK;
}

sv_status sv_destroy(sv_ctx* c) {
  if (!c) return SV_EINVAL;
  if (c->comm_pending) cudaEventSynchronize(c->comm_done);   // possibly recorded on a peer lane's stream
  cudaStreamSynchronize(c->comm);
  cudaStreamSynchronize(c->stream);
  cudaStreamDestroy(c->comm);
  cudaEventDestroy(c->comm_done);
  cudaEventDestroy(c->lane_mark);
  if (c->ctrl_consumed) cudaEventDestroy(c->ctrl_consumed);
  for (cudaEvent_t e : c->dyn_done)
    if (e) cudaEventDestroy(e);
  if (c->pin_ctrl) cudaFreeHost(c->pin_ctrl);
  for (cudaEvent_t e : c->rel_ev)
    if (e) cudaEventDestroy(e);
  sv::gemm_plan_destroy(c->gemm);
  for (auto e : c->prof.free_ev) cudaEventDestroy(e);
  for (auto& r : c->prof.recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  delete c;
  return SV_OK;
}

sv_status sv_append_kv(sv_ctx* c, int32_t slot, uint64_t request_id, const void* k, const void* v,
                       int32_t n_tokens, int32_t pending_token) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || n_tokens < 0) return SV_EINVAL;
  if (n_tokens > 0 && (!k || !v || (((uintptr_t)k | (uintptr_t)v) & 15))) return SV_EINVAL;
  if (pending_token < 0 || pending_token >= c->cfg.vocab) return SV_EINVAL;
  if (c->state[slot] == PENDING) return SV_ESTATE;
  if (c->state[slot] == ACTIVE && c->rid[slot] != request_id) return SV_EINVAL;
  wait_comm_slots(c, 1, &slot);
  SV_CUDA(sv::launch_append(c->d, slot, request_id, (const bf16*)k, (const bf16*)v, n_tokens, pending_token,
                            nullptr, 0, c->stream));
  c->state[slot] = ACTIVE;
  c->rid[slot] = request_id;
  return SV_OK;
}

static sv_status check_batch(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                             sv::PlanArgs& p) {
  if (batch < 1 || batch > c->cfg.max_batch || !slots || !depths) return SV_EINVAL;
  std::vector<char> seen(c->cfg.max_slots, 0);
  p.batch = batch;
  p.T = 0;
  for (int b = 0; b < batch; ++b) {
    const int s = slots[b], k = depths[b];
    if (s < 0 || s >= c->cfg.max_slots || seen[s]) return SV_EINVAL;
    if (k < 0 || k > c->cfg.max_depth) return SV_EINVAL;
    seen[s] = 1;
    p.slots[b] = s;
    p.depths[b] = k;
    p.T += k + 1;
  }
  for (int b = 0; b < batch; ++b)
    if (c->state[slots[b]] != ACTIVE) return SV_ESTATE;
  return SV_OK;
}

static sv_status gemm(sv_ctx* c, const bf16* A, const bf16* B, float* C, int M, int N, int K, int epi,
                      const sv::GemmEpi& e) {
  return cuda_ok(sv::gemm_run(c->gemm, A, B, C, M, N, K, epi, e, c->stream));
}

static bool filter_active(const sv_ctx* c) { return (c->top_k > 0 && c->top_k < c->cfg.vocab) || c->top_p < 1.0f; }

// sv_verify and sv_verify_tree (parents != NULL: token-tree drafts, R30)
// head = false (sv_prefill's intermediate chunks only): no final norm / lm-head; the chunk's rows
// are kept and no next token is predicted
static sv_status verify_impl(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                             const int32_t* parents, const int32_t* draft_tokens, const float* draft_probs,
                             uint64_t seed, sv_mode mode, float temperature, int32_t* accepted_len,
                             int32_t* out_tokens, int32_t* accepted_nodes, float* logits_out, bool head = true) {
  if (!c || !accepted_len || !out_tokens) return SV_EINVAL;
  if (mode != SV_GREEDY && mode != SV_SAMPLE && mode != SV_PREFILL) return SV_EINVAL;
  if (parents && mode == SV_PREFILL) return SV_EINVAL;
  if (mode == SV_SAMPLE && !(temperature > 0.f)) return SV_EINVAL;
  if (((uintptr_t)draft_probs | (uintptr_t)logits_out) & 15) return SV_EINVAL;   // float4 row loads / copies
  if (c->pending_verify) return SV_ESTATE;
  sv::PlanArgs p;
  sv_status st = check_batch(c, batch, slots, depths, p);
  if (st) return st;
  if (p.T > batch && !draft_tokens) return SV_EINVAL;
  sv::LaneDev d = c->d;
  d.tree = parents != nullptr && p.T > batch;
  if (!d.tree) parents = nullptr;                   // no drafts: a tree of roots is the chain
  // dynamic-depth graph capture: every replay's slots / depths come from the device copy the graph's
  // first node makes; row-gridded launches cover Tmax = batch (max_depth + 1) rows and return beyond
  // the plan's device T, the GEMMs read their rows from it
  const bool dyn = c->dyn_capture;
  if (dyn) {
    if (batch != c->dyn_batch || parents || mode == SV_PREFILL || logits_out || !draft_tokens || !head)
      return SV_EINVAL;
    d.dyn_ctrl = (const int*)(c->ws + c->lay.dctrl);
  }
  const int* Mdev = dyn ? d.T_dev : nullptr;
  int max_rows = 1;                                 // deepest chain + 1 (a dynamic graph: any depth)
  for (int b = 0; b < batch; ++b) max_rows = std::max(max_rows, p.depths[b] + 1);
  if (dyn) max_rows = c->cfg.max_depth + 1;
  const int T = dyn ? batch * (c->cfg.max_depth + 1) : p.T;
  cudaStream_t s = c->stream;
  const float inv_temp = mode == SV_SAMPLE ? 1.0f / temperature : 1.0f;
  bool row_best = false;
  wait_comm_slots(c, batch, slots);
  if (sv::plan_embed_supported(d) && !getenv("SV_SPLIT_PLAN")) {
    // plan + embed in one launch (each row's CTA scans the batch itself)
    // wide (2048-key) splits: opt-in (SV_WIDE_SPLIT=1). ns step -0.7 %, but on ragged 4.1-6.2 k contexts
    // one of three runs put the attention at 1.001 % of the survey's 1 % criterion (1024-key items:
    // 0.77-0.82 %), DESIGN.md §6.2
    const bool wide = sv::attn_uses_tc2(c->gemm, max_rows) && getenv("SV_WIDE_SPLIT") &&
                      !strcmp(getenv("SV_WIDE_SPLIT"), "1");
    STAGE(c, ST_EMBED, sv::launch_plan_embed(d, p, draft_tokens, parents, T, wide, s));
  } else {
    STAGE(c, ST_PLAN, sv::launch_plan(d, p, draft_tokens, parents, true, s));
    STAGE(c, ST_EMBED, sv::launch_embed_norm(d, T, s));
  }
  const size_t nq = (size_t)d.Hq * d.dh;
  for (int layer = 0; layer < d.n_layers; ++layer) {
    const float* hin = layer == 0 ? d.h0 : d.h2;
    if (layer > 0) STAGE(c, ST_ATTN_NORM, sv::launch_rmsnorm(d, hin, d.attn_norm + (size_t)layer * d.D, d.a, T, s));
    sv::GemmEpi e{};
    e.layer = layer;
    e.M_dev = Mdev;
    e.M_hint = p.T;
    STAGE(c, ST_QKV, gemm(c, d.a, d.wqkv + (size_t)layer * d.qkv_rows * d.D, d.cbuf, T, d.qkv_rows, d.D,
                          sv::EPI_QKV_ROPE, e));
    bool tc2 = false;
    STAGE(c, ST_ATTN, sv::attn_run(c->gemm, layer, batch, d.tree, max_rows, s, &tc2));
    STAGE(c, ST_COMBINE, sv::launch_attn_combine(d, T, tc2, s));
    float* hattn = d.F > 0 ? d.h1 : d.h2;
    e.resid_in = hin;
    e.resid_out = hattn;
    STAGE(c, ST_OPROJ, gemm(c, d.o, d.wo + (size_t)layer * d.D * nq, d.cbuf, T, d.D, (int)nq, sv::EPI_RESIDUAL, e));
    if (d.F > 0) {
      STAGE(c, ST_FFN_NORM, sv::launch_rmsnorm(d, d.h1, d.ffn_norm + (size_t)layer * d.D, d.b, T, s));
      STAGE(c, ST_GATE_UP, gemm(c, d.b, d.w_gate_up + (size_t)layer * 2 * d.F * d.D, d.cbuf, T, 2 * d.F, d.D,
                                sv::EPI_SWIGLU, e));
      e.resid_in = d.h1;
      e.resid_out = d.h2;
      STAGE(c, ST_DOWN, gemm(c, d.u, d.w_down + (size_t)layer * d.D * d.F, d.cbuf, T, d.D, d.F, sv::EPI_RESIDUAL, e));
    }
  }
  if (head) {
    STAGE(c, ST_FINAL_NORM, sv::launch_rmsnorm(d, d.h2, d.final_norm, d.z, T, s));
    sv::GemmEpi e{};
    e.inv_temp = inv_temp;
    e.M_dev = Mdev;
    e.M_hint = p.T;
    // greedy decisions need only the vocab-tile statistics: the fp32 logits (T x V x 4 bytes)
    // are stored only when something reads them
    e.write_out = c->taps || mode == SV_SAMPLE || logits_out != nullptr;
    // greedy / prefill decisions need only each row's argmax: the lm-head epilogue folds it into
    // row_best (atomicMax of order-preserving keys, deterministic) and finalize reads 1 word per row
    row_best = mode != SV_SAMPLE && sv::gemm_fills_row_best(c->gemm);
    e.row_best = row_best ? d.row_best : nullptr;
    // greedy decisions read only row_best: the epilogue skips sum exp and the tile statistics unless
    // something inspects them (taps)
    e.argmax_only = row_best && !c->taps && mode == SV_GREEDY;
    STAGE(c, ST_LM_HEAD, gemm(c, d.z, d.lm_head, d.logits, T, d.V, d.D, sv::EPI_LOGITS, e));
  }
  d.filt_on = mode == SV_SAMPLE && filter_active(c);
  if (d.filt_on) STAGE(c, ST_FILTER, sv::launch_filter(d, T, inv_temp, c->top_k, c->top_p, s));
  if (!head) row_best = false;
  STAGE(c, ST_FINALIZE, sv::launch_finalize(d, batch, draft_tokens, parents, draft_probs, d.logits, seed,
                                            head ? (int)mode : sv::kPrefillNoHead, inv_temp, accepted_len,
                                            out_tokens, accepted_nodes, s, row_best));
  if (logits_out)
    SV_CUDA(cudaMemcpyAsync(logits_out, d.logits, (size_t)T * d.V * 4, cudaMemcpyDeviceToDevice, s));
  for (int b = 0; b < batch; ++b) c->state[slots[b]] = PENDING;
  c->pending_verify = true;
  c->pending_batch = batch;
  c->pending_slots.assign(slots, slots + batch);
  c->last_T = dyn ? T : p.T;
  c->last_batch = batch;
  return SV_OK;
}

sv_status sv_verify(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                    const int32_t* draft_tokens, const float* draft_probs, uint64_t seed, sv_mode mode,
                    float temperature, int32_t* accepted_len, int32_t* out_tokens, float* logits_out) {
  return verify_impl(c, batch, slots, depths, nullptr, draft_tokens, draft_probs, seed, mode, temperature,
                     accepted_len, out_tokens, nullptr, logits_out);
}

sv_status sv_verify_tree(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                         const int32_t* parents, const int32_t* draft_tokens, const float* draft_probs,
                         uint64_t seed, sv_mode mode, float temperature, int32_t* accepted_len,
                         int32_t* out_tokens, int32_t* accepted_nodes, float* logits_out) {
  if (!parents) return SV_EINVAL;
  return verify_impl(c, batch, slots, depths, parents, draft_tokens, draft_probs, seed, mode, temperature,
                     accepted_len, out_tokens, accepted_nodes, logits_out);
}

static sv_status verify_logits_impl(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                                    const int32_t* parents, const int32_t* draft_tokens, const float* draft_probs,
                                    const float* logits, uint64_t seed, sv_mode mode, float temperature,
                                    int32_t* accepted_len, int32_t* out_tokens, int32_t* accepted_nodes) {
  if (!c || !accepted_len || !out_tokens || !logits) return SV_EINVAL;
  if (((uintptr_t)draft_probs | (uintptr_t)logits) & 15) return SV_EINVAL;        // float4 row loads
  if (mode != SV_GREEDY && mode != SV_SAMPLE && mode != SV_PREFILL) return SV_EINVAL;
  if (parents && mode == SV_PREFILL) return SV_EINVAL;
  if (mode == SV_SAMPLE && !(temperature > 0.f)) return SV_EINVAL;
  if (c->pending_verify || c->dyn_capture) return SV_ESTATE;
  sv::PlanArgs p;
  sv_status st = check_batch(c, batch, slots, depths, p);
  if (st) return st;
  if (p.T > batch && !draft_tokens) return SV_EINVAL;
  const float inv_temp = mode == SV_SAMPLE ? 1.0f / temperature : 1.0f;
  sv::LaneDev d = c->d;
  if (p.T == batch) parents = nullptr;
  d.tree = parents != nullptr;
  wait_comm_slots(c, batch, slots);
  SV_CUDA(sv::launch_plan(d, p, draft_tokens, parents, false, c->stream));
  d.logits = const_cast<float*>(logits);
  SV_CUDA(sv::launch_tile_stats(d, p.T, inv_temp, c->stream));
  d.filt_on = mode == SV_SAMPLE && filter_active(c);
  if (d.filt_on) SV_CUDA(sv::launch_filter(d, p.T, inv_temp, c->top_k, c->top_p, c->stream));
  SV_CUDA(sv::launch_finalize(d, batch, draft_tokens, parents, draft_probs, logits, seed, mode, inv_temp,
                              accepted_len, out_tokens, accepted_nodes, c->stream));
  c->last_T = p.T;
  c->last_batch = batch;
  return SV_OK;
}

sv_status sv_verify_logits(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                           const int32_t* draft_tokens, const float* draft_probs, const float* logits,
                           uint64_t seed, sv_mode mode, float temperature, int32_t* accepted_len,
                           int32_t* out_tokens) {
  return verify_logits_impl(c, batch, slots, depths, nullptr, draft_tokens, draft_probs, logits, seed, mode,
                            temperature, accepted_len, out_tokens, nullptr);
}

sv_status sv_verify_tree_logits(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                                const int32_t* parents, const int32_t* draft_tokens, const float* draft_probs,
                                const float* logits, uint64_t seed, sv_mode mode, float temperature,
                                int32_t* accepted_len, int32_t* out_tokens, int32_t* accepted_nodes) {
  if (!parents) return SV_EINVAL;
  return verify_logits_impl(c, batch, slots, depths, parents, draft_tokens, draft_probs, logits, seed, mode,
                            temperature, accepted_len, out_tokens, accepted_nodes);
}

sv_status sv_commit(sv_ctx* c, const int32_t* n_keep) {
  if (!c) return SV_EINVAL;
  if (!c->pending_verify) return SV_ESTATE;
  STAGE(c, ST_COMMIT, sv::launch_commit(c->d, n_keep, c->pending_batch, c->stream));
  for (int s : c->pending_slots) c->state[s] = ACTIVE;
  c->pending_verify = false;
  if (c->sticky & SV_DERR_NO_PAGES) return SV_ENOKV;
  if (c->sticky) return SV_EDEVICE;
  return SV_OK;
}

sv_status sv_release(sv_ctx* c, int32_t slot) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots) return SV_EINVAL;
  if (c->state[slot] == PENDING) return SV_ESTATE;
  if (c->state[slot] == EMPTY) return SV_OK;
  wait_comm_slots(c, 1, &slot);
  SV_CUDA(sv::launch_release(c->d, slot, c->stream));
  if (!c->rel_ev[slot]) SV_CUDA(cudaEventCreateWithFlags(&c->rel_ev[slot], cudaEventDisableTiming));
  SV_CUDA(cudaEventRecord(c->rel_ev[slot], c->stream));
  c->rel_pending[slot] = 1;
  c->state[slot] = EMPTY;
  c->rid[slot] = 0;
  return SV_OK;
}

sv_status sv_lane_occupancy(sv_ctx* c, int32_t* active_slots, int32_t* free_pages) {
  if (!c || !active_slots || !free_pages) return SV_EINVAL;
  int ft = 0;
  SV_CUDA(cudaMemcpyAsync(&ft, c->d.free_top, 4, cudaMemcpyDeviceToHost, c->stream));
  SV_CUDA(cudaStreamSynchronize(c->stream));
  int n = 0;
  for (int st : c->state) n += st != EMPTY;
  *active_slots = n;
  *free_pages = ft < 0 ? 0 : ft;
  return SV_OK;
}

sv_status sv_stats(sv_ctx* c, sv_lane_stats* out, int reset) {
  if (!c || !out) return SV_EINVAL;
  unsigned long long buf[sv::kNumStats];
  int err = 0;
  SV_CUDA(cudaMemcpyAsync(buf, c->d.stats, sizeof(buf), cudaMemcpyDeviceToHost, c->stream));
  SV_CUDA(cudaMemcpyAsync(&err, c->d.err, 4, cudaMemcpyDeviceToHost, c->stream));
  SV_CUDA(cudaStreamSynchronize(c->stream));
  memset(out, 0, sizeof(*out));
  out->steps = buf[sv::ST_STEPS];
  out->rows = buf[sv::ST_ROWS];
  out->drafted = buf[sv::ST_DRAFTED];
  out->accepted = buf[sv::ST_ACCEPTED];
  out->emitted = buf[sv::ST_EMITTED];
  out->accepted_independent = buf[sv::ST_INDEP];
  for (int i = 0; i <= sv::kMaxDepth; ++i) {
    out->hist_accepted[i] = buf[sv::ST_HIST + i];
    out->drafted_by_k[i] = buf[sv::ST_DRAFTED_BY_K + i];
    out->accepted_by_k[i] = buf[sv::ST_ACCEPTED_BY_K + i];
  }
  out->device_error = err;
  c->sticky = err;
  if (reset) SV_CUDA(cudaMemsetAsync(c->d.stats, 0, sizeof(buf), c->stream));
  if (err & SV_DERR_NO_PAGES) return SV_ENOKV;
  if (err) return SV_EDEVICE;
  return SV_OK;
}

sv_status sv_set_filter(sv_ctx* c, int32_t top_k, float top_p) {
  if (!c || top_k < 0 || !(top_p > 0.0f)) return SV_EINVAL;     // rejects NaN too
  if (c->pending_verify) return SV_ESTATE;
  c->top_k = top_k;
  c->top_p = top_p;
  return SV_OK;
}

sv_status sv_set_taps(sv_ctx* c, int enable) {
  if (!c) return SV_EINVAL;
  c->taps = enable != 0;
  return SV_OK;
}

sv_status sv_get_tap(sv_ctx* c, const char* name, void** dev_ptr, size_t* bytes) {
  if (!c || !name || !dev_ptr || !bytes) return SV_EINVAL;
  const sv::LaneDev& d = c->d;
  const size_t T = c->last_T, D = d.D, B = c->last_batch;
  const size_t nq = (size_t)d.Hq * d.dh, nkv = (size_t)d.Hkv * d.dh;
  struct Tap { const char* n; const void* p; size_t b; };
  const Tap taps[] = {
      {"h0", d.h0, 4 * T * D},
      {"a", d.a, 2 * T * D},
      {"q", d.q, 2 * T * nq},
      {"kc", d.kc, 2 * (size_t)d.n_layers * d.Tmax * nkv},
      {"vc", d.vc, 2 * (size_t)d.n_layers * d.Tmax * nkv},
      {"o", d.o, 2 * T * nq},
      {"h1", d.F > 0 ? d.h1 : d.h2, 4 * T * D},
      {"b", d.b, 2 * T * D},
      {"u", d.u, 2 * T * (size_t)d.F},
      {"h2", d.h2, 4 * T * D},
      {"z", d.z, 2 * T * D},
      {"logits", d.logits, 4 * T * (size_t)d.V},
      {"tile_max", d.tile_max, 4 * T * (size_t)d.nt},
      {"tile_sum", d.tile_sum, 4 * T * (size_t)d.nt},
      {"tile_arg", d.tile_arg, 4 * T * (size_t)d.nt},
      {"row_off", d.row_off, 4 * (B + 1)},
      {"rope_cos", d.rope_cos, 4 * (size_t)d.max_pos * d.dh / 2},
      {"rope_sin", d.rope_sin, 4 * (size_t)d.max_pos * d.dh / 2},
      {"len", d.len, 4 * (size_t)d.max_slots},
      {"pending", d.pending, 4 * (size_t)d.max_slots},
      {"page_table", d.page_table, 4 * (size_t)d.max_slots * d.max_pages_per_slot},
      {"free_top", d.free_top, 4},
      {"free_list", d.free_list, 4 * (size_t)d.n_pages},
      {"trace", d.trace ? (const void*)d.trace : (const void*)(c->ws + c->lay.trace), 8 * 16 * 256},
  };
  for (const Tap& t : taps)
    if (!strcmp(t.n, name)) {
      *dev_ptr = const_cast<void*>(t.p);
      *bytes = t.b;
      return SV_OK;
    }
  return SV_EINVAL;
}

sv_status sv_debug_uniforms(sv_ctx* c, uint64_t seed, uint64_t rid, uint32_t z, int32_t purpose, int32_t x0,
                            int32_t n, float* u) {
  if (!c || !u || n < 0 || x0 < 0 || (purpose != 0 && purpose != 1)) return SV_EINVAL;
  SV_CUDA(sv::launch_debug_uniforms(seed, rid, z, purpose, x0, n, u, c->stream));
  return SV_OK;
}

sv_status sv_debug_gemm(sv_ctx* c, const void* A, const void* B, float* C, int32_t M, int32_t N, int32_t K,
                        int32_t variant) {
  if (!c || !A || !B || !C || M < 1 || N < 1 || K < 64 || K % 64 || M > c->d.Tmax) return SV_EINVAL;
  if (((uintptr_t)A | (uintptr_t)B | (uintptr_t)C) & 15) return SV_EINVAL;
  SV_CUDA(sv::gemm_debug(c->gemm, (const bf16*)A, (const bf16*)B, C, M, N, K, variant, c->stream));
  return SV_OK;
}

static sv_status draft_planted_impl(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                                    const int32_t* parents, const int32_t* succ, const uint8_t* dev_mask,
                                    const int32_t* dev_tok, int32_t* draft_tokens) {
  if (!c || !succ || !dev_mask || !dev_tok || !draft_tokens) return SV_EINVAL;
  sv::PlanArgs p;
  if (batch < 1 || batch > c->cfg.max_batch || !slots || !depths) return SV_EINVAL;
  p.batch = batch;
  p.T = 0;
  for (int b = 0; b < batch; ++b) {
    if (slots[b] < 0 || slots[b] >= c->cfg.max_slots || depths[b] < 0 || depths[b] > c->cfg.max_depth)
      return SV_EINVAL;
    p.slots[b] = slots[b];
    p.depths[b] = depths[b];
    p.T += depths[b] + 1;
  }
  sv::LaneDev d = c->d;
  if (c->dyn_capture) {                            // dynamic-depth graph: this replay's slots / depths
    if (batch != c->dyn_batch || parents) return SV_EINVAL;
    d.dyn_ctrl = (const int*)(c->ws + c->lay.dctrl);
  }
  STAGE(c, ST_DRAFT, sv::launch_draft_planted(d, p, succ, dev_mask, dev_tok, parents, draft_tokens, c->stream));
  return SV_OK;
}

sv_status sv_draft_planted(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                           const int32_t* succ, const uint8_t* dev_mask, const int32_t* dev_tok,
                           int32_t* draft_tokens) {
  return draft_planted_impl(c, batch, slots, depths, nullptr, succ, dev_mask, dev_tok, draft_tokens);
}

sv_status sv_draft_planted_tree(sv_ctx* c, int32_t batch, const int32_t* slots, const int32_t* depths,
                                const int32_t* parents, const int32_t* succ, const uint8_t* dev_mask,
                                const int32_t* dev_tok, int32_t* draft_tokens) {
  if (!parents) return SV_EINVAL;
  return draft_planted_impl(c, batch, slots, depths, parents, succ, dev_mask, dev_tok, draft_tokens);
}

// one long chunk of a prompt (k_prefill.cu): C rows at positions L..L+C-1, every key from the pages;
// last: final norm + lm-head of the last row, y -> pending / y_out; else pending = next_token
static sv_status prefill_chunk(sv_ctx* c, int32_t slot, const int32_t* dtok, int C, bool last, int next_token,
                               int32_t* y_out) {
  sv::LaneDev d = c->d;
  d.tree = 0;
  d.filt_on = 0;
  cudaStream_t s = c->stream;
  const int G = d.Hq / d.Hkv, nqb = (C + 128 / G - 1) / (128 / G);
  STAGE(c, ST_PLAN, sv::launch_prefill_plan(d, slot, dtok, C, s));
  STAGE(c, ST_EMBED, sv::launch_embed_norm(d, C, s));
  const size_t nq = (size_t)d.Hq * d.dh;
  for (int layer = 0; layer < d.n_layers; ++layer) {
    const float* hin = layer == 0 ? d.h0 : d.h2;
    if (layer > 0) STAGE(c, ST_ATTN_NORM, sv::launch_rmsnorm(d, hin, d.attn_norm + (size_t)layer * d.D, d.a, C, s));
    sv::GemmEpi e{};
    e.layer = layer;
    STAGE(c, ST_QKV, gemm(c, d.a, d.wqkv + (size_t)layer * d.qkv_rows * d.D, d.cbuf, C, d.qkv_rows, d.D,
                          sv::EPI_QKV_ROPE, e));
    STAGE(c, ST_COMMIT, sv::launch_prefill_kv(d, layer, C, s));
    STAGE(c, ST_ATTN, sv::attn_prefill_run(c->gemm, layer, d.Hkv * nqb, s));
    float* hattn = d.F > 0 ? d.h1 : d.h2;
    e.resid_in = hin;
    e.resid_out = hattn;
    STAGE(c, ST_OPROJ, gemm(c, d.o, d.wo + (size_t)layer * d.D * nq, d.cbuf, C, d.D, (int)nq, sv::EPI_RESIDUAL, e));
    if (d.F > 0) {
      STAGE(c, ST_FFN_NORM, sv::launch_rmsnorm(d, d.h1, d.ffn_norm + (size_t)layer * d.D, d.b, C, s));
      STAGE(c, ST_GATE_UP, gemm(c, d.b, d.w_gate_up + (size_t)layer * 2 * d.F * d.D, d.cbuf, C, 2 * d.F, d.D,
                                sv::EPI_SWIGLU, e));
      e.resid_in = d.h1;
      e.resid_out = d.h2;
      STAGE(c, ST_DOWN, gemm(c, d.u, d.w_down + (size_t)layer * d.D * d.F, d.cbuf, C, d.D, d.F, sv::EPI_RESIDUAL, e));
    }
  }
  if (last) {                                   // only the last row predicts the next token
    STAGE(c, ST_FINAL_NORM, sv::launch_rmsnorm(d, d.h2 + (size_t)(C - 1) * d.D, d.final_norm, d.z, 1, s));
    sv::GemmEpi e{};
    e.inv_temp = 1.0f;
    e.write_out = c->taps;
    STAGE(c, ST_LM_HEAD, gemm(c, d.z, d.lm_head, d.logits, 1, d.V, d.D, sv::EPI_LOGITS, e));
  }
  STAGE(c, ST_FINALIZE, sv::launch_prefill_finish(d, C, last ? -1 : next_token, y_out, s));
  c->last_T = C;
  c->last_batch = 1;
  return SV_OK;
}

sv_status sv_prefill(sv_ctx* c, int32_t slot, uint64_t request_id, const int32_t* prompt, int32_t n, int32_t chunk,
                     int32_t* next_token) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || !prompt || n < 1 || chunk < 1) return SV_EINVAL;
  const bool long_path = sv::attn_prefill_supported(c->gemm);
  if (chunk > (long_path ? c->d.Tmax : c->cfg.max_depth + 1)) return SV_EINVAL;
  if (c->state[slot] != EMPTY || c->pending_verify || c->capturing) return SV_ESTATE;
  for (int i = 0; i < n; ++i)
    if (prompt[i] < 0 || prompt[i] >= c->cfg.vocab) return SV_EINVAL;
  const int K1 = c->cfg.max_depth + 2;
  int32_t* dacc = (int32_t*)(c->ws + c->lay.prefill);     // accepted_len [1]
  int32_t* dout = dacc + K1;                               // out_tokens [max_depth + 1]
  int32_t* dprompt = dout + K1;                            // the prompt [n <= max_pos]
  if (n > c->cfg.max_pos) return SV_EINVAL;
  wait_comm_slots(c, 1, &slot);
  // one copy of the whole prompt (a per-chunk copy from pageable memory would block the host on
  // every chunk's previous work); the chunks then read their tokens in place
  SV_CUDA(cudaMemcpyAsync(dprompt, prompt, 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
  sv_status st = sv_append_kv(c, slot, request_id, nullptr, nullptr, 0, prompt[0]);
  if (st) return st;
  int32_t y = -1;
  if (long_path) {
    // chunks of the prompt itself: rows prompt[pos .. pos+C-1] at positions pos.. (the pending token
    // set above is prompt[0], the first row of the first chunk)
    for (int pos = 0; pos < n; pos += chunk) {
      const int C = chunk < n - pos ? chunk : n - pos;
      const bool last = pos + C >= n;
      if ((st = prefill_chunk(c, slot, dprompt + pos, C, last, last ? -1 : prompt[pos + C], dacc))) return st;
    }
    SV_CUDA(cudaMemcpyAsync(&y, dacc, 4, cudaMemcpyDeviceToHost, c->stream));
  } else {
    // short chunks through the verify machinery (SV_PREFILL verifies, R29)
    int pos = 1, k = 0;
    for (;;) {
      k = chunk - 1 < n - pos ? chunk - 1 : n - pos;
      const int32_t* dtok = dprompt + pos;
      // only the last chunk's lm-head matters (its last row predicts the next token)
      const bool last = pos + k >= n;
      if ((st = verify_impl(c, 1, &slot, &k, nullptr, dtok, nullptr, 0, SV_PREFILL, 1.0f, dacc, dout, nullptr,
                            nullptr, last)))
        return st;
      if ((st = sv_commit(c, nullptr))) return st;
      pos += k;
      if (pos >= n) break;
      if ((st = sv_append_kv(c, slot, request_id, nullptr, nullptr, 0, prompt[pos]))) return st;
      pos += 1;
    }
    SV_CUDA(cudaMemcpyAsync(&y, dout + k, 4, cudaMemcpyDeviceToHost, c->stream));
  }
  SV_CUDA(cudaStreamSynchronize(c->stream));
  if (y < 0) return SV_EDEVICE;
  int err = 0;
  SV_CUDA(cudaMemcpy(&err, c->d.err, 4, cudaMemcpyDeviceToHost));
  c->sticky = err;
  if (err & SV_DERR_NO_PAGES) return SV_ENOKV;
  if (next_token) *next_token = y;
  return SV_OK;
}

sv_status sv_kv_pack_slot(sv_ctx* c, int32_t slot, int32_t n_tokens, void* kv_packed) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || n_tokens < 0 || !kv_packed || ((uintptr_t)kv_packed & 15))
    return SV_EINVAL;
  if (c->state[slot] != ACTIVE) return SV_ESTATE;
  wait_comm_slots(c, 1, &slot);
  SV_CUDA(sv::launch_kv_pack_slot(c->d, slot, n_tokens, kv_packed, c->stream));
  return SV_OK;
}

sv_status sv_kv_pack(const void* k, const void* v, int32_t n_layers, int32_t n_kv_heads, int32_t head_dim,
                     int32_t n_tokens, int32_t pending_token, void* kv_packed, sv_stream_t stream) {
  if (!k || !v || !kv_packed || n_layers < 1 || n_kv_heads < 1 || n_tokens < 0 || head_dim % 8) return SV_EINVAL;
  if (((uintptr_t)k | (uintptr_t)v | (uintptr_t)kv_packed) & 15) return SV_EINVAL;
  SV_CUDA(sv::launch_kv_pack((const bf16*)k, (const bf16*)v, n_layers, n_kv_heads, head_dim, n_tokens,
                             pending_token, kv_packed, (cudaStream_t)stream));
  return SV_OK;
}

size_t sv_kv_packed_bytes(const sv_config* cfg, int32_t n_tokens) {
  if (!cfg || n_tokens < 0) return 0;
  return (size_t)cfg->n_layers * n_tokens * 2 * cfg->n_kv_heads * cfg->head_dim * 2 + 16;
}

sv_status sv_profile_enable(sv_ctx* c, int32_t stage_mask) {
  if (!c) return SV_EINVAL;
  c->prof.mask = (uint32_t)stage_mask;
  // create the events up front: cudaEventCreate inside a timed region costs host time
  while (stage_mask && c->prof.free_ev.size() < 4096) {
    cudaEvent_t e;
    SV_CUDA(cudaEventCreate(&e));
    c->prof.free_ev.push_back(e);
  }
  return SV_OK;
}

int32_t sv_profile_num_stages(void) { return ST_NUM; }

const char* sv_profile_stage_name(int32_t i) { return (i >= 0 && i < ST_NUM) ? kStageNames[i] : nullptr; }

sv_status sv_profile_read(sv_ctx* c, double* ms_total, int64_t* count, int32_t n, int reset) {
  if (!c || !ms_total || !count || n < ST_NUM) return SV_EINVAL;
  SV_CUDA(cudaStreamSynchronize(c->stream));
  prof_fold(c, true);
  for (int i = 0; i < ST_NUM; ++i) {
    ms_total[i] = c->prof.ms[i];
    count[i] = c->prof.n[i];
    if (reset) {
      c->prof.ms[i] = 0;
      c->prof.n[i] = 0;
    }
  }
  return SV_OK;
}

uint64_t sv_launch_count(void) { return sv::g_launch_count; }

// ---------------------------------------------------------------- CUDA graphs of a fixed step
struct sv_graph {
  cudaGraphExec_t exec;
  unsigned long long kernels;        // kernel launches captured (added to sv_launch_count per replay)
  bool dynamic;                      // sv_graph_begin_dynamic: slots / depths staged per replay
  int batch;
  cudaGraph_t tmpl = nullptr;        // dynamic: the captured graph (its H2D node is retargeted per replay)
  cudaGraphNode_t h2d = nullptr;
  mutable int staged_buf = -1;       // dynamic: the lane staging buffer its next launch consumes
  sv_ctx* ctx = nullptr;             // the lane (its staging buffers are released if the graph dies staged)
  // profiled graph (stages timed while capturing): each stage's two event-record nodes are pointed at
  // fresh pool events before every replay (cudaGraphExecEventRecordNodeSetEvent), and the pair joins the
  // lane's profile records, so per-stage CUDA-event times cover replays as they do eager calls
  struct ProfNode { int stage; cudaGraphNode_t a, b; };
  std::vector<ProfNode> prof;
  std::vector<cudaEvent_t> owned;    // the events recorded at capture (the template's nodes refer to them)
  cudaEvent_t idle[2] = {nullptr, nullptr};   // targets while the lane is not profiling the stage
};

sv_status sv_graph_begin(sv_ctx* c) {
  if (!c || !c->stream) return SV_EINVAL;                 // the legacy default stream cannot be captured
  if (c->capturing || c->pending_verify) return SV_ESTATE;
  c->prof.captured.clear();
  wait_comm(c);                                           // an outside event cannot be waited on in capture
  SV_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  c->capturing = true;
  c->capture_launches0 = sv::g_launch_count;
  return SV_OK;
}

sv_status sv_graph_begin_dynamic(sv_ctx* c, int32_t batch) {
  if (!c || !c->stream || batch < 1 || batch > c->cfg.max_batch) return SV_EINVAL;
  if (c->capturing || c->pending_verify) return SV_ESTATE;
  c->prof.captured.clear();
  if (!sv::supports_dynamic_rows(c->gemm)) return SV_ESTATE;
  wait_comm(c);
  SV_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  c->capturing = true;
  c->dyn_capture = true;
  c->dyn_batch = batch;
  c->capture_launches0 = sv::g_launch_count;
  // the graph's first node: this replay's slots | depths, pinned host -> device (its source buffer is
  // switched between two pinned buffers per replay, sv_graph_set_batch)
  cudaError_t e = cudaMemcpyAsync(c->ws + c->lay.dctrl, c->pin_ctrl, 8 * (size_t)batch, cudaMemcpyHostToDevice,
                                  c->stream);
  if (e != cudaSuccess) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    c->capturing = c->dyn_capture = false;
    return cuda_ok(e);
  }
  return SV_OK;
}

sv_status sv_graph_set_batch(sv_ctx* c, const sv_graph* g, const int32_t* slots, const int32_t* depths) {
  if (!c || !g || !slots || !depths) return SV_EINVAL;
  if (!g->dynamic) return SV_ESTATE;
  if (c->capturing || c->pending_verify) return SV_ESTATE;
  sv::PlanArgs p;
  sv_status st = check_batch(c, g->batch, slots, depths, p);   // distinct, in range, ACTIVE, depth <= max
  if (st) return st;
  const int buf = (int)(c->dyn_stage_seq & 1);
  if (c->dyn_unlaunched[buf]) return SV_ESTATE;           // staged for a launch that has not happened
  if (g->staged_buf >= 0) return SV_ESTATE;               // this graph's previous staging is unlaunched
  if (c->dyn_done_set[buf]) SV_CUDA(cudaEventSynchronize(c->dyn_done[buf]));   // its last reader finished
  int* pin = c->pin_ctrl + (size_t)buf * 2 * c->cfg.max_batch;
  memcpy(pin, slots, 4 * (size_t)g->batch);
  memcpy(pin + g->batch, depths, 4 * (size_t)g->batch);
  SV_CUDA(cudaGraphExecMemcpyNodeSetParams1D(g->exec, g->h2d, c->ws + c->lay.dctrl, pin, 8 * (size_t)g->batch,
                                             cudaMemcpyHostToDevice));
  c->dyn_unlaunched[buf] = true;
  g->staged_buf = buf;
  ++c->dyn_stage_seq;
  return SV_OK;
}

sv_status sv_graph_end(sv_ctx* c, sv_graph** out) {
  if (!c || !out) return SV_EINVAL;
  if (!c->capturing) return SV_ESTATE;
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  c->capturing = false;
  const bool dyn = c->dyn_capture;
  const int dyn_batch = c->dyn_batch;
  c->dyn_capture = false;
  if (e != cudaSuccess) return SV_ECUDA;
  if (c->pending_verify) {                                // a captured verify must be committed in it
    cudaGraphDestroy(g);
    return SV_ESTATE;
  }
  cudaGraphExec_t x = nullptr;
  const cudaError_t e2 = cudaGraphInstantiate(&x, g, 0);
  const bool profiled = !c->prof.captured.empty();
  if ((!dyn && !profiled) || e2 != cudaSuccess) cudaGraphDestroy(g);
  if (e2 != cudaSuccess) {
    for (auto& r : c->prof.captured) {
      c->prof.free_ev.push_back(r.a);
      c->prof.free_ev.push_back(r.b);
    }
    c->prof.captured.clear();
    return SV_ECUDA;
  }
  sv_graph* gr = new sv_graph{x, sv::g_launch_count - c->capture_launches0, dyn, dyn_batch};
  gr->ctx = c;
  if (profiled) {                                         // map the captured stage events to their nodes
    gr->tmpl = g;
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    if (n) cudaGraphGetNodes(g, nodes.data(), &n);
    auto node_of = [&](cudaEvent_t ev) -> cudaGraphNode_t {
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        cudaEvent_t e = nullptr;
        if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeEventRecord &&
            cudaGraphEventRecordNodeGetEvent(nd, &e) == cudaSuccess && e == ev)
          return nd;
      }
      return nullptr;
    };
    bool ok = cudaEventCreate(&gr->idle[0]) == cudaSuccess && cudaEventCreate(&gr->idle[1]) == cudaSuccess;
    for (auto& r : c->prof.captured) {
      gr->owned.push_back(r.a);
      gr->owned.push_back(r.b);
      const cudaGraphNode_t na = node_of(r.a), nb = node_of(r.b);
      if (!na || !nb) ok = false;
      gr->prof.push_back({r.stage, na, nb});
    }
    c->prof.captured.clear();
    if (!ok) {
      fprintf(stderr, "[sv] sv_graph_end: profiled stage events without event-record nodes\n");
      sv_graph_destroy(gr);
      return SV_ECUDA;
    }
  }
  if (dyn) {                                              // keep the template: its H2D root is retargeted
    gr->tmpl = g;                                         // (the same template as a profiled graph's)
    size_t nroot = 1;
    cudaGraphNode_t root = nullptr;
    cudaGraphNodeType ty;
    if (cudaGraphGetRootNodes(g, &root, &nroot) != cudaSuccess || nroot < 1 ||
        cudaGraphNodeGetType(root, &ty) != cudaSuccess || ty != cudaGraphNodeTypeMemcpy) {
      sv_graph_destroy(gr);
      return SV_ECUDA;
    }
    gr->h2d = root;
  }
  *out = gr;
  sv::g_launch_count = c->capture_launches0;              // captured launches run at replay
  return SV_OK;
}

sv_status sv_graph_launch(sv_ctx* c, const sv_graph* g) {
  if (!c || !g) return SV_EINVAL;
  if (c->capturing || c->pending_verify) return SV_ESTATE;
  if (g->dynamic && g->staged_buf < 0) return SV_ESTATE;  // every replay takes a freshly staged batch
  // profiled stages: fresh events for this replay while the lane times the stage, else the idle pair
  std::vector<Prof::Rec> fresh;
  for (const auto& pn : g->prof) {
    const bool on = (c->prof.mask >> pn.stage) & 1u;
    const cudaEvent_t a = on ? c->prof.get() : g->idle[0], b = on ? c->prof.get() : g->idle[1];
    SV_CUDA(cudaGraphExecEventRecordNodeSetEvent(g->exec, pn.a, a));
    SV_CUDA(cudaGraphExecEventRecordNodeSetEvent(g->exec, pn.b, b));
    if (on) fresh.push_back({pn.stage, a, b});
  }
  SV_CUDA(cudaGraphLaunch(g->exec, c->stream));
  for (const auto& r : fresh) c->prof.recs.push_back(r);
  if (c->prof.recs.size() >= 8192 && c->prof.recs.size() % 1024 == 0) prof_fold(c, false);
  sv::g_launch_count += g->kernels;
  if (g->dynamic) {                                       // the staged buffer is free once this replay ran
    const int buf = g->staged_buf;
    SV_CUDA(cudaEventRecord(c->dyn_done[buf], c->stream));
    c->dyn_done_set[buf] = true;
    c->dyn_unlaunched[buf] = false;
    g->staged_buf = -1;
  }
  return SV_OK;
}

sv_status sv_graph_destroy(sv_graph* g) {
  if (!g) return SV_EINVAL;
  if (g->dynamic && g->staged_buf >= 0 && g->ctx) g->ctx->dyn_unlaunched[g->staged_buf] = false;
  cudaGraphExecDestroy(g->exec);
  if (g->tmpl) cudaGraphDestroy(g->tmpl);
  for (cudaEvent_t e : g->owned) cudaEventDestroy(e);
  for (cudaEvent_t e : g->idle)
    if (e) cudaEventDestroy(e);
  delete g;
  return SV_OK;
}

}  // extern "C"

// used by comm.cpp (hand-off receive): append from a packed device buffer
// host-checkable preconditions of an append from a packed message (checked BEFORE any NCCL
// receive is posted, so a refused call consumes no message)
sv_status sv_internal_append_check(sv_ctx* c, int32_t slot, uint64_t request_id, const void* packed,
                                   int32_t n_tokens) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || n_tokens < 0 || !packed) return SV_EINVAL;
  if ((uintptr_t)packed & 15) return SV_EINVAL;
  if (c->state[slot] == PENDING) return SV_ESTATE;
  if (c->state[slot] == ACTIVE && c->rid[slot] != request_id) return SV_EINVAL;
  return SV_OK;
}

sv_status sv_internal_append_packed(sv_ctx* c, int32_t slot, uint64_t request_id, const void* packed,
                                    int32_t n_tokens) {
  const sv_status chk = sv_internal_append_check(c, slot, request_id, packed, n_tokens);
  if (chk) return chk;
  const size_t body = (size_t)c->cfg.n_layers * n_tokens * 2 * c->cfg.n_kv_heads * c->cfg.head_dim * 2;
  const int* trailer = (const int*)((const char*)packed + body);
  wait_comm(c);                                          // the packed message may come from a receive
  SV_CUDA(sv::launch_append(c->d, slot, request_id, (const bf16*)packed, nullptr, n_tokens, 0, trailer, 1,
                            c->stream));
  c->state[slot] = ACTIVE;
  c->rid[slot] = request_id;
  return SV_OK;
}

cudaStream_t sv_internal_stream(sv_ctx* c) { return c->stream; }

size_t sv_internal_packed_bytes(sv_ctx* c, int32_t n_tokens) { return sv_kv_packed_bytes(&c->cfg, n_tokens); }

// ---------------------------------------------------------------- batched page-block hand-off (a9)
// Wire format of one batch (one ncclSend / ncclRecv): for request i, for layer l, for page
// p < ceil(n_i / page_size): the (layer, page) block of the KV pool — [2][Hkv][page][d_h] bf16,
// contiguous in the pool (256 KB at Llama-3-8B shape) — then the n pending tokens (int32), padded
// to 16 bytes. The prefill side gathers the blocks from its pages into its staging buffer and the
// decode side scatters them from its staging buffer into freshly popped pages: block-granular
// copies (16-byte vectors, whole 256 KB blocks), both on the lanes' comm streams.
// (One NCCL op per block and no staging was measured first: 4096 ops for a 32 x 8192-token batch
// took 22 ms on the one-GPU loopback, ~5.4 us per op, i.e. 48 GB/s; one op per batch removes it.)
static size_t block_bytes(const sv_config& c) { return (size_t)2 * c.n_kv_heads * c.page_size * c.head_dim * 2; }

static bool distinct_slots(const sv_ctx* c, int n, const int32_t* slots) {
  std::vector<char> seen(c->cfg.max_slots, 0);
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= c->cfg.max_slots || seen[slots[i]]) return false;
    seen[slots[i]] = 1;
  }
  return true;
}

extern "C" size_t sv_kv_slots_bytes(const sv_config* cfg, int32_t n, const int32_t* n_tokens) {
  if (!cfg || n < 1 || !n_tokens || cfg->page_size < 1) return 0;
  size_t blocks = 0;
  for (int i = 0; i < n; ++i) {
    if (n_tokens[i] < 0) return 0;
    blocks += (size_t)cfg->n_layers * ((n_tokens[i] + cfg->page_size - 1) / cfg->page_size);
  }
  return blocks * block_bytes(*cfg) + (((size_t)4 * n + 15) & ~(size_t)15);
}

// control arrays of a batch in the lane's hand-off workspace area: slots, n_tokens, block starts
// [n + 1], request ids; copied on `st`
static sv_status stage_ctrl(sv_ctx* c, int n, const int32_t* slots, const int32_t* ntok, const uint64_t* rids,
                            cudaStream_t st, int** d_slots, int** d_ntok, int** d_bstart,
                            unsigned long long** d_rid) {
  const int ms = c->cfg.max_slots;
  int* base = (int*)(c->ws + c->lay.handoff);
  *d_slots = base;
  *d_ntok = base + ms;
  *d_bstart = base + 2 * ms;
  *d_rid = (unsigned long long*)(base + 4 * ms + 4);
  std::vector<int> bs(n + 1, 0);
  for (int i = 0; i < n; ++i) bs[i + 1] = bs[i] + c->cfg.n_layers * ((ntok[i] + c->cfg.page_size - 1) / c->cfg.page_size);
  SV_CUDA(cudaMemcpyAsync(*d_slots, slots, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  SV_CUDA(cudaMemcpyAsync(*d_ntok, ntok, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  SV_CUDA(cudaMemcpyAsync(*d_bstart, bs.data(), 4 * (size_t)(n + 1), cudaMemcpyHostToDevice, st));
  if (rids) SV_CUDA(cudaMemcpyAsync(*d_rid, rids, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
  return SV_OK;
}

// prefill side: checks (one sync of the lane stream reads the slots' committed lengths), then on
// the comm stream, after the lane's earlier work: the block gather into `staging`. Returns the
// message size; the caller posts the send on the comm stream.
sv_status sv_internal_send_prepare(sv_ctx* c, int32_t n, const int32_t* slots, const int32_t* ntok, void* staging,
                                   size_t* bytes) {
  if (!c || n < 1 || !slots || !ntok || !staging || ((uintptr_t)staging & 15) || !distinct_slots(c, n, slots))
    return SV_EINVAL;
  if (c->capturing) return SV_ESTATE;
  for (int i = 0; i < n; ++i) {
    if (c->state[slots[i]] != ACTIVE) return SV_ESTATE;
    if (ntok[i] < 1) return SV_EINVAL;
  }
  std::vector<int> len(c->cfg.max_slots);
  wait_comm_slots(c, n, slots);
  SV_CUDA(cudaMemcpyAsync(len.data(), c->d.len, 4 * len.size(), cudaMemcpyDeviceToHost, c->stream));
  SV_CUDA(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < n; ++i)
    if (ntok[i] > len[slots[i]]) return SV_EINVAL;              // only committed rows can be sent
  cudaStream_t cs = c->comm;
  int *ds, *dn, *db;
  unsigned long long* dr;
  sv_status st = stage_ctrl(c, n, slots, ntok, nullptr, cs, &ds, &dn, &db, &dr);
  if (st) return st;
  SV_CUDA(sv::launch_handoff_gather(c->d, ds, dn, db, n, (char*)staging, cs));
  *bytes = sv_kv_slots_bytes(&c->cfg, n, ntok);
  return SV_OK;
}

// decode side, before the receive: checks and the page pop on the comm stream (the host never
// waits for the lane stream: a verify enqueued before the call keeps running; the free list is
// lock-protected against the lane's concurrent commits / releases, k_kv.cu). A slot released earlier
// is reused only after its release kernel (per-slot event). The slots become ACTIVE with
// len = n_i and request_id bound; the scatter (sv_internal_recv_finish) writes their pages and
// pending tokens, and lane work on those slots waits for it (sv_internal_comm_posted).
sv_status sv_internal_recv_prepare(sv_ctx* c, int32_t n, const int32_t* slots, const uint64_t* rids,
                                   const int32_t* ntok, void* staging, size_t* bytes) {
  if (!c || n < 1 || !slots || !rids || !ntok || !staging || ((uintptr_t)staging & 15) ||
      !distinct_slots(c, n, slots))
    return SV_EINVAL;
  if (c->capturing) return SV_ESTATE;
  long need = 0;
  for (int i = 0; i < n; ++i) {
    if (c->state[slots[i]] != EMPTY) return SV_ESTATE;
    if (ntok[i] < 1 || ntok[i] > c->cfg.max_pos - 1) return SV_EINVAL;
    need += (ntok[i] + c->cfg.page_size - 1) / c->cfg.page_size;
  }
  cudaStream_t cs = c->comm;
  for (int i = 0; i < n; ++i)
    if (c->rel_pending[slots[i]]) {
      SV_CUDA(cudaStreamWaitEvent(cs, c->rel_ev[slots[i]], 0));
      c->rel_pending[slots[i]] = 0;
    }
  int ft = 0;
  SV_CUDA(cudaMemcpyAsync(&ft, c->d.free_top, 4, cudaMemcpyDeviceToHost, cs));
  SV_CUDA(cudaStreamSynchronize(cs));
  if (need > ft) return SV_ENOKV;                               // refused before anything is popped / posted
  int *ds, *dn, *db;
  unsigned long long* dr;
  sv_status st = stage_ctrl(c, n, slots, ntok, rids, cs, &ds, &dn, &db, &dr);
  if (st) return st;
  SV_CUDA(sv::launch_handoff_alloc(c->d, ds, dr, dn, n, cs));
  for (int i = 0; i < n; ++i) {
    c->state[slots[i]] = ACTIVE;
    c->rid[slots[i]] = rids[i];
  }
  *bytes = sv_kv_slots_bytes(&c->cfg, n, ntok);
  return SV_OK;
}

// decode side, after the receive was posted on the comm stream: the block scatter into the pages
sv_status sv_internal_recv_finish(sv_ctx* c, int32_t n, const void* staging) {
  const int ms = c->cfg.max_slots;
  int* base = (int*)(c->ws + c->lay.handoff);
  SV_CUDA(sv::launch_handoff_scatter(c->d, base, base + ms, base + 2 * ms, n, (const char*)staging, c->comm));
  return SV_OK;
}

cudaStream_t sv_internal_comm_stream(sv_ctx* c) { return c->comm; }

extern "C" sv_status sv_comm_stream(sv_ctx* c, sv_stream_t* out) {
  if (!c || !out) return SV_EINVAL;
  *out = (sv_stream_t)c->comm;
  return SV_OK;
}

sv_status sv_internal_config(sv_ctx* c, sv_config* out) {
  *out = c->cfg;
  return SV_OK;
}

// transfers touching `slots` were enqueued on `on`: lane work on those slots waits for them
sv_status sv_internal_comm_posted(sv_ctx* c, cudaStream_t on, int32_t n, const int32_t* slots) {
  SV_CUDA(cudaEventRecord(c->comm_done, on));
  c->comm_pending = true;
  for (int i = 0; i < n; ++i) c->comm_slot[slots[i]] = 1;
  return SV_OK;
}
