// Arguments of the tcgen05 GEMM kernel (k_gemm_tc.cu) and its fused epilogues.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace sv {

enum GemmTcEpi { GEMM_EPI_NONE = 0, GEMM_EPI_QKV_ROPE = 1, GEMM_EPI_RESIDUAL = 2, GEMM_EPI_SWIGLU = 3,
                 GEMM_EPI_LOGITS = 4 };

struct GemmTcArgs {
  int kind;
  int M, N, K;            // logical problem (N = 2F for SWIGLU)
  int n_tiles;            // output tiles along N
  float* out;             // NONE / LOGITS: fp32 [M][ldo]
  int ldo;
  const float* resid_in;  // RESIDUAL: out = resid_in + acc, fp32 [M][ldo]
  float* resid_out;
  // QKV_ROPE
  __nv_bfloat16 *q, *kc, *vc;
  const int* row_pos;
  const float *rope_cos, *rope_sin;
  int Hq, Hkv, dh;
  // SWIGLU
  __nv_bfloat16* u;
  int F;
  // LOGITS statistics [M][nt]
  float *tmax, *tsum;
  int* targ;
  int nt;
  float inv_temp;
  // LOGITS (weight-major kernel, greedy): per token row, atomicMax of (order-preserving max bits << 32 |
  // ~argmax) over the vocab tiles = the row's lowest-index argmax (finalize reads it; zero between steps)
  unsigned long long* row_best;
  int argmax_only;        // LOGITS with row_best: skip sum exp and the per-tile statistics (greedy, no taps)
  // weight-major kernel: when set, the rows M are read from the device after the dependency wait (the
  // grid is sized for the g.M given, an upper bound; dynamic-depth CUDA graphs)
  const int* M_dev;
  // stream-K (decided at launch): partial-tile buffers [grid][2][128 x 256] fp32 and per-tile
  // arrival counters (zero between launches)
  int streamk, sk_w;
  int nt_tok;  // weight-major kernel: token tile width (N of the MMA), multiple of 16, <= 256
  unsigned long long* trace;  // weight-major kernel: per-tile clock64 trace of CTA 0 (SV_TRACE)
  int diag;  // 1: skip TMA after the first STAGES k-blocks (measures the MMA/epilogue-only time)
  float* partials;
  int* sk_counters;
};

constexpr int kGemmMaxSms = 160;
int gemm_tc_smem_bytes();
size_t gemm_tc_partial_bytes(int num_sms);
// 2-SM (cta_group::2) variant: 256 x 256 tiles per CTA pair (see k_gemm_tc.cu)
cudaError_t launch_gemm_tc2(const CUtensorMap& map_a, const CUtensorMap& map_b, const GemmTcArgs& g, int num_sms,
                            cudaStream_t s);
// weight-major 2-SM variant (k_gemm_sw.cu): map_w = weights [N][K] box (64, 128) (box rows 64 for
// SWIGLU), map_x = tokens [>= M][K] box (64, nt_tok / 2)
int gemm_sw_choose_nt(int T, int num_mp, int n_pairs, int T2 = 0);
int gemm_sw_smem_bytes();
cudaError_t launch_gemm_sw(const CUtensorMap& map_w, const CUtensorMap& map_x, const GemmTcArgs& g, int num_sms,
                           cudaStream_t s);
cudaError_t launch_gemm_tc(const CUtensorMap& map_a, const CUtensorMap& map_b, const GemmTcArgs& g, int num_sms,
                           cudaStream_t s);

}  // namespace sv
