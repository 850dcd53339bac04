// GEMM dispatch: the SIMT path (GEMM into fp32 scratch, then a separate epilogue
// kernel). The tcgen05 path with fused epilogues plugs in here.
#include <stdlib.h>
#include <string.h>

#include "gemm.h"

namespace sv {

struct GemmPlan {
  LaneDev d;
};

size_t gemm_workspace_bytes() { return 4096; }

GemmPlan* gemm_plan_create(const LaneDev& d, void* ws, cudaStream_t s) {
  (void)ws;
  (void)s;
  GemmPlan* p = new GemmPlan();
  p->d = d;
  return p;
}

void gemm_plan_destroy(GemmPlan* p) { delete p; }

cudaError_t gemm_run(GemmPlan* p, const bf16* A, const bf16* B, float* C, int M, int N, int K, int epi,
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

}  // namespace sv
