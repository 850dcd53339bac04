// GEMM dispatch. Default: the tcgen05 kernel with fused epilogues (k_gemm_tc.cu).
// SV_GEMM=simt selects the SIMT reference path (GEMM into fp32 scratch + separate
// epilogue kernels), kept as an in-library cross-check.
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <tuple>

#include "attn_tc.h"
#include "gemm.h"
#include "gemm_tc.h"

namespace sv {

struct GemmPlan {
  LaneDev d;
  bool use_tc = true;
  int num_sms = 148;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint32_t>, CUtensorMap> maps;
  bool use_tc_attn = true;
  bool use_tc2_attn = false;       // keys-on-lanes kernel (d_h = 128)
  bool attn_maps_ok = false;
  CUtensorMap map_q, map_q2, map_kv;
  int q_box_tokens = 16;
  int* sk_counters = nullptr;
  float* partials = nullptr;
  bool use_streamk = false;
  bool use_2sm = false;            // token-major 2-SM kernel (SV_GEMM=tc2)
  bool use_1sm = false;            // token-major 1-SM kernel (SV_GEMM=tc1)
  bool prefill_map_ok = false;     // map_qp: Q box (64, 1, 128 / G) for the long-chunk prefill attention
  CUtensorMap map_qp;
};

static size_t counter_bytes(int Tmax, int max_n) {
  const size_t n = (size_t)((Tmax + 127) / 128) * ((max_n + 255) / 256);
  return (n * 4 + 1023) & ~size_t(1023);
}

size_t gemm_workspace_bytes(int Tmax, int max_n) {
  return counter_bytes(Tmax, max_n) + gemm_tc_partial_bytes(kGemmMaxSms);
}

static bool encode_attn_maps(GemmPlan* p);

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

// bf16 row-major [rows][cols] tensor, box 64 (cols, 128 B) x box_rows, 128-byte swizzle
static const CUtensorMap* get_map(GemmPlan* p, const void* base, uint64_t rows, uint64_t cols,
                                  uint32_t box_rows = 128) {
  auto key = std::make_tuple(base, rows, cols, box_rows);
  auto it = p->maps.find(key);
  if (it != p->maps.end()) return &it->second;
  CUtensorMap m;
  memset(&m, 0, sizeof(m));
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = p->encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "[sv] cuTensorMapEncodeTiled failed (%d)\n", (int)r);
    return nullptr;
  }
  return &(p->maps[key] = m);
}

GemmPlan* gemm_plan_create(const LaneDev& d, void* ws, cudaStream_t s) {
  GemmPlan* p = new GemmPlan();
  p->d = d;
  const char* env = getenv("SV_GEMM");
  p->use_tc = !(env && !strcmp(env, "simt"));
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (p->num_sms > kGemmMaxSms) p->num_sms = kGemmMaxSms;
  // stream-K scratch: counters first (zeroed here; the kernel re-zeroes each tile it completes)
  int max_n = d.qkv_rows;
  if (d.D > max_n) max_n = d.D;
  if (2 * d.F > max_n) max_n = 2 * d.F;
  const size_t cb = counter_bytes(d.Tmax, max_n);
  p->sk_counters = reinterpret_cast<int*>(ws);
  p->partials = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + cb);
  cudaMemsetAsync(ws, 0, cb, s);
  const char* skenv = getenv("SV_STREAMK");
  p->use_streamk = skenv && !strcmp(skenv, "1");     // measured slower than whole tiles: opt-in
  p->use_2sm = env && !strcmp(env, "tc2");
  p->use_1sm = env && !strcmp(env, "tc1");
  p->encode = get_encode();
  if (!p->encode) {
    fprintf(stderr, "[sv] cuTensorMapEncodeTiled unavailable\n");
    p->use_tc = false;
  }
  const char* aenv = getenv("SV_ATTN");
  const int G = d.Hq / d.Hkv;
  p->use_tc_attn = p->encode && !(aenv && !strcmp(aenv, "simt")) && d.page == 64 && (d.dh == 64 || d.dh == 128) &&
                   G <= 4 && d.max_depth + 1 <= 32;
  // keys-on-lanes kernel: chosen per verify when its (max k + 1) G <= 64 query slots fit (attn_run)
  p->use_tc2_attn = p->use_tc_attn && d.dh == 128 && (64 % G) == 0 && !(aenv && !strcmp(aenv, "tc1"));
  if (p->use_tc_attn) p->attn_maps_ok = encode_attn_maps(p);
  return p;
}

void gemm_plan_destroy(GemmPlan* p) { delete p; }

static bool encode_attn_maps(GemmPlan* p) {
  const LaneDev& d = p->d;
  const int G = d.Hq / d.Hkv;
  // Q: 3-D (d_h, Hq, Tmax) bf16, box (64, 1, q_box_tokens) = the chain rows of one q head
  p->q_box_tokens = d.max_depth + 1 <= 8 ? 8 : (d.max_depth + 1 <= 16 ? 16 : 32);
  cuuint64_t qdims[3] = {(cuuint64_t)d.dh, (cuuint64_t)d.Hq, (cuuint64_t)d.Tmax};
  cuuint64_t qstr[2] = {(cuuint64_t)d.dh * 2, (cuuint64_t)d.Hq * d.dh * 2};
  cuuint32_t qbox[3] = {64, 1, (cuuint32_t)p->q_box_tokens};
  cuuint32_t es3[3] = {1, 1, 1};
  if (p->encode(&p->map_q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d.q, qdims, qstr, qbox, es3,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  // Q for the keys-on-lanes kernel: box (64, G, 64 / G) = slots j*G + g of one kv head
  if (p->use_tc2_attn) {
    cuuint32_t qbox2[3] = {64, (cuuint32_t)G, (cuuint32_t)(64 / G)};
    if (p->encode(&p->map_q2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d.q, qdims, qstr, qbox2, es3,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  // KV pool: 2-D (d_h, n_layers * n_pages * 2 * Hkv * page) bf16, box (64, 64) = one page of one head
  cuuint64_t kdims[2] = {(cuuint64_t)d.dh, (cuuint64_t)d.n_layers * d.n_pages * 2 * d.Hkv * d.page};
  cuuint64_t kstr[1] = {(cuuint64_t)d.dh * 2};
  cuuint32_t kbox[2] = {64, 64};
  cuuint32_t es2[2] = {1, 1};
  if (p->encode(&p->map_kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d.pool, kdims, kstr, kbox, es2,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  return true;
}

cudaError_t attn_run(GemmPlan* p, int layer, int batch, int tree, int max_rows, cudaStream_t s, bool* used_tc2) {
  LaneDev d = p->d;
  d.tree = tree;
  const int G = d.Hq / d.Hkv;
  if (used_tc2) *used_tc2 = false;
  // keys-on-lanes when this verify's deepest chain fits its 64 query slots per kv head; the rows-on-
  // lanes kernel up to 32 rows x G <= 4 (deeper chains, e.g. SpecuStream's d* up to 20); else SIMT
  if (p->use_tc2_attn && p->attn_maps_ok && max_rows * G <= kAttnRows) {
    if (used_tc2) *used_tc2 = true;
    return launch_attention_tc2(p->map_q2, p->map_kv, d, layer, p->num_sms, s);
  }
  if (p->use_tc_attn && p->attn_maps_ok && max_rows <= p->q_box_tokens)
    return launch_attention_tc(p->map_q, p->map_kv, d, layer, p->num_sms, p->q_box_tokens, s);
  if (max_rows * G > kAttnRows) return cudaErrorInvalidValue;
  return launch_attention(d, layer, batch, s);
}

bool attn_uses_tc2(GemmPlan* p, int max_rows) {
  const int G = p->d.Hq / p->d.Hkv;
  return p->use_tc2_attn && p->attn_maps_ok && max_rows * G <= kAttnRows;
}

bool gemm_fills_row_best(GemmPlan* p) { return p->use_tc && !p->use_2sm && !p->use_1sm && !p->use_streamk; }

bool supports_dynamic_rows(GemmPlan* p) { return gemm_fills_row_best(p) && p->use_tc_attn && p->attn_maps_ok; }

bool attn_prefill_supported(GemmPlan* p) {
  const LaneDev& d = p->d;
  const int G = d.Hq / d.Hkv;
  return p->use_tc_attn && p->attn_maps_ok && (G == 1 || G == 2 || G == 4);
}

cudaError_t attn_prefill_run(GemmPlan* p, int layer, int n_items, cudaStream_t s) {
  const LaneDev& d = p->d;
  const int G = d.Hq / d.Hkv;
  if (!p->prefill_map_ok) {
    cuuint64_t qdims[3] = {(cuuint64_t)d.dh, (cuuint64_t)d.Hq, (cuuint64_t)d.Tmax};
    cuuint64_t qstr[2] = {(cuuint64_t)d.dh * 2, (cuuint64_t)d.Hq * d.dh * 2};
    cuuint32_t qbox[3] = {64, 1, (cuuint32_t)(128 / G)};
    cuuint32_t es3[3] = {1, 1, 1};
    if (p->encode(&p->map_qp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d.q, qdims, qstr, qbox, es3,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    p->prefill_map_ok = true;
  }
  return launch_attention_prefill(p->map_qp, p->map_kv, d, layer, n_items, p->num_sms, s);
}

static cudaError_t gemm_simt(GemmPlan* p, const bf16* A, const bf16* B, float* C, int M, int N, int K, int epi,
                             const GemmEpi& e, cudaStream_t s) {
  cudaError_t err = launch_gemm_simt(A, B, C, M, N, K, s);
  if (err != cudaSuccess) return err;
  switch (epi) {
    case EPI_QKV_ROPE: return launch_qkv_rope_epilogue(p->d, e.layer, M, s);
    case EPI_RESIDUAL: return launch_residual_epilogue(e.resid_in, C, e.resid_out, M, N, s);
    case EPI_SWIGLU: return launch_swiglu_epilogue(p->d, M, s);
    case EPI_LOGITS: return launch_tile_stats(p->d, M, e.inv_temp, s);
    default: return cudaSuccess;
  }
}

// weight-major 2-SM kernel: weights (B) on the MMA's M side, the M tokens of A on its N side
static cudaError_t gemm_sw(GemmPlan* p, const bf16* A, const bf16* B, int M, int K, GemmTcArgs& g, cudaStream_t s,
                           int M_hint = 0) {
  const bool swiglu = g.kind == GEMM_EPI_SWIGLU;
  const int num_mp = swiglu ? g.F / 128 : (g.N + 255) / 256;
  g.nt_tok = M_hint > 0 ? gemm_sw_choose_nt(M_hint, num_mp, p->num_sms / 2, M) : gemm_sw_choose_nt(M, num_mp, p->num_sms / 2);
  if (const char* nt = getenv("SV_SW_NT")) g.nt_tok = atoi(nt);   // experiment override
  if (const char* dg = getenv("SV_SW_DIAG")) g.diag = atoi(dg);    // experiment: 1 no loads, 2 no epilogue
  {                                                                  // tile timeline (SV_TRACE): lm-head by
    const char* tk = getenv("SV_TRACE_GEMM");                        // default, or the GEMM kind named here
    if (g.kind == (tk ? atoi(tk) : (int)GEMM_EPI_LOGITS)) g.trace = p->d.trace;
  }
  const CUtensorMap* mw = get_map(p, B, (uint64_t)g.N, (uint64_t)K, swiglu ? 64 : 128);
  const CUtensorMap* mx = get_map(p, A, (uint64_t)M, (uint64_t)K, (uint32_t)(g.nt_tok / 2));  // rows >= M: zero
  if (!mw || !mx) return cudaErrorInvalidValue;
  return launch_gemm_sw(*mw, *mx, g, p->num_sms, s);
}

cudaError_t gemm_run(GemmPlan* p, const bf16* A, const bf16* B, float* C, int M, int N, int K, int epi,
                     const GemmEpi& e, cudaStream_t s) {
  if (!p->use_tc || (K % 64)) return gemm_simt(p, A, B, C, M, N, K, epi, e, s);
  const LaneDev& d = p->d;
  const CUtensorMap* ma = get_map(p, A, (uint64_t)d.Tmax, (uint64_t)K);
  const CUtensorMap* mb = get_map(p, B, (uint64_t)N, (uint64_t)K);
  if (!ma || !mb) return cudaErrorInvalidValue;
  GemmTcArgs g;
  memset(&g, 0, sizeof(g));
  g.M = M;
  g.N = N;
  g.K = K;
  g.n_tiles = (N + 255) / 256;
  g.out = C;
  g.ldo = N;
  g.M_dev = e.M_dev;
  if (p->use_streamk) {
    g.partials = p->partials;
    g.sk_counters = p->sk_counters;
  }
  switch (epi) {
    case EPI_QKV_ROPE: {
      g.kind = GEMM_EPI_QKV_ROPE;
      const size_t nkv = (size_t)d.Hkv * d.dh;
      g.q = d.q;
      g.kc = d.kc + (size_t)e.layer * d.Tmax * nkv;
      g.vc = d.vc + (size_t)e.layer * d.Tmax * nkv;
      g.row_pos = d.row_pos;
      g.rope_cos = d.rope_cos;
      g.rope_sin = d.rope_sin;
      g.Hq = d.Hq;
      g.Hkv = d.Hkv;
      g.dh = d.dh;
      break;
    }
    case EPI_RESIDUAL:
      g.kind = GEMM_EPI_RESIDUAL;
      g.resid_in = e.resid_in;
      g.resid_out = e.resid_out;
      break;
    case EPI_SWIGLU:
      if ((N / 2) % 128) return gemm_simt(p, A, B, C, M, N, K, epi, e, s);
      g.kind = GEMM_EPI_SWIGLU;
      g.u = d.u;
      g.F = N / 2;
      g.n_tiles = (N / 2) / 128;
      break;
    case EPI_LOGITS:
      g.kind = GEMM_EPI_LOGITS;
      g.tmax = d.tile_max;
      g.tsum = d.tile_sum;
      g.targ = d.tile_arg;
      g.nt = d.nt;
      g.inv_temp = e.inv_temp;
      g.row_best = e.row_best;
      g.argmax_only = e.row_best && e.argmax_only ? 1 : 0;
      if (!e.write_out) g.out = nullptr;
      break;
    default:
      g.kind = GEMM_EPI_NONE;
  }
  if (p->use_2sm && !g.partials) return launch_gemm_tc2(*ma, *mb, g, p->num_sms, s);
  if (p->use_1sm || g.partials) return launch_gemm_tc(*ma, *mb, g, p->num_sms, s);
  return gemm_sw(p, A, B, M, K, g, s, e.M_dev ? e.M_hint : 0);
}

}  // namespace sv

namespace sv {

cudaError_t gemm_debug(GemmPlan* p, const bf16* A, const bf16* B, float* C, int M, int N, int K, int variant,
                       cudaStream_t s) {
  if (variant == 3 || (variant == 0 && !p->use_tc) || !p->encode) return launch_gemm_simt(A, B, C, M, N, K, s);
  const CUtensorMap* ma = get_map(p, A, (uint64_t)M, (uint64_t)K);
  const CUtensorMap* mb = get_map(p, B, (uint64_t)N, (uint64_t)K);
  if (!ma || !mb) return cudaErrorInvalidValue;
  GemmTcArgs g;
  memset(&g, 0, sizeof(g));
  g.kind = GEMM_EPI_NONE;
  g.M = M;
  g.N = N;
  g.K = K;
  g.n_tiles = (N + 255) / 256;
  g.out = C;
  g.ldo = N;
  g.diag = variant == 4 ? 1 : 0;
  if (variant >= 6) {                                  // weight-major diagnostics (timing only)
    g.diag = variant == 6 ? 1 : variant == 7 ? 2 : variant == 8 ? 3 : 5;  // 6: MMA only, 7: no epilogue,
                                                                          // 8: both, 9: MMA only with A in TMEM
  }
  if (variant >= 5 || (variant == 0 && !p->use_2sm && !p->use_1sm)) return gemm_sw(p, A, B, M, K, g, s);
  const bool two = variant == 2 || (variant == 0 && p->use_2sm);
  return two ? launch_gemm_tc2(*ma, *mb, g, p->num_sms, s) : launch_gemm_tc(*ma, *mb, g, p->num_sms, s);
}

}  // namespace sv
