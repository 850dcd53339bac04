// GEMM front-end used by the verify sequence: C = A[M][K] * B[N][K]^T with a fused
// epilogue per call site.
#pragma once
#include "lane.h"

namespace sv {

enum GemmEpiKind { EPI_NONE = 0, EPI_QKV_ROPE = 1, EPI_RESIDUAL = 2, EPI_SWIGLU = 3, EPI_LOGITS = 4 };

struct GemmEpi {
  int layer;               // QKV: which layer's chain K/V scratch to write
  const float* resid_in;   // RESIDUAL: h_in  (fp32 [M][N])
  float* resid_out;        // RESIDUAL: h_out (fp32 [M][N]); may alias resid_in
  float inv_temp;          // LOGITS: statistics are of l * inv_temp
  bool write_out;          // LOGITS: also store the fp32 logits (tensor-core paths; SIMT always does)
  unsigned long long* row_best;   // LOGITS: per-row argmax keys (only when gemm_fills_row_best)
  bool argmax_only;                // LOGITS with row_best: only the argmax keys (no tile statistics)
  const int* M_dev;        // rows from the device (dynamic-depth graph; M = the upper bound), or nullptr
  int M_hint;              // with M_dev: typical rows, for the token-tile width (0: use M)
};

struct GemmPlan;
// stream-K scratch: per-tile counters for ceil(Tmax/128) x ceil(max_n/256) tiles + partial tiles
size_t gemm_workspace_bytes(int Tmax, int max_n);
GemmPlan* gemm_plan_create(const LaneDev& d, void* ws, cudaStream_t s);
void gemm_plan_destroy(GemmPlan* p);
// a3 verify attention: tcgen05 kernel when the shape allows (page 64, d_h 64/128), else SIMT
// max_rows: the deepest chain of this verify + 1 (picks the kernel); used_tc2 (optional): the keys-on-lanes
// kernel ran (it writes O itself for single-split requests)
cudaError_t attn_run(GemmPlan* p, int layer, int batch, int tree, int max_rows, cudaStream_t s, bool* used_tc2);
// true when the lm-head GEMM (EPI_LOGITS) also fills GemmEpi::row_best (the weight-major kernel)
bool gemm_fills_row_best(GemmPlan* p);
// true when attn_run will pick the keys-on-lanes kernel for this verify's deepest chain (the only
// attention kernel that plan_embed's wide 2048-key splits are enabled for)
bool attn_uses_tc2(GemmPlan* p, int max_rows);
// true when every GEMM of the step honours GemmEpi::M_dev and the attention reads its work list from
// the device (the dynamic-depth CUDA graph's requirements)
bool supports_dynamic_rows(GemmPlan* p);
// NEXT-3 long-chunk prefill attention (tcgen05 rows-on-lanes, G in {1, 2, 4})
bool attn_prefill_supported(GemmPlan* p);
cudaError_t attn_prefill_run(GemmPlan* p, int layer, int n_items, cudaStream_t s);
// test hook: plain C = A B^T with a chosen kernel (0 default, 1 1-SM, 2 2-SM, 3 SIMT)
cudaError_t gemm_debug(GemmPlan* p, const bf16* A, const bf16* B, float* C, int M, int N, int K, int variant,
                       cudaStream_t s);
cudaError_t gemm_run(GemmPlan* p, const bf16* A, const bf16* B, float* C, int M, int N, int K, int epi,
                     const GemmEpi& e, cudaStream_t s);

}  // namespace sv
