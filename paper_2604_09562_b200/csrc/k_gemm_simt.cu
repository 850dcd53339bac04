// Reference-grade SIMT GEMM (fp32 FMA): C[M][N] = A[M][K] * B[N][K]^T, bf16 operands,
// fp32 accumulation. Used (1) as the first correct path for every projection and the
// lm-head and (2) as the in-library cross-check of the tcgen05 GEMM. Not the hot path
// once the tensor-core kernels are enabled.
#include "common.cuh"
#include "lane.h"

namespace sv {

constexpr int SG_BM = 128, SG_BN = 128, SG_BK = 32;

__global__ void __launch_bounds__(256) gemm_simt_kernel(const bf16* __restrict__ A, const bf16* __restrict__ B,
                                                        float* __restrict__ C, int M, int N, int K) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += SG_BK) {
    // 128 rows x 32 k = 512 chunks of 8 bf16 per operand; 2 per thread
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int idx = threadIdx.x + c * 256;
      const int row = idx >> 2, kc = (idx & 3) * 8;
      uint4 va = make_uint4(0, 0, 0, 0), vb = make_uint4(0, 0, 0, 0);
      if (m0 + row < M) va = *reinterpret_cast<const uint4*>(A + (size_t)(m0 + row) * K + k0 + kc);
      if (n0 + row < N) vb = *reinterpret_cast<const uint4*>(B + (size_t)(n0 + row) * K + k0 + kc);
      const bf16* pa = reinterpret_cast<const bf16*>(&va);
      const bf16* pb = reinterpret_cast<const bf16*>(&vb);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        As[kc + e][row] = bf2f(pa[e]);
        Bs[kc + e][row] = bf2f(pb[e]);
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty * 8 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx * 8 + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + ty * 8 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + tx * 8 + j;
      if (n < N) C[(size_t)m * N + n] = acc[i][j];
    }
  }
}

cudaError_t launch_gemm_simt(const bf16* A, const bf16* B, float* C, int M, int N, int K, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K % SG_BK) return cudaErrorInvalidValue;
  dim3 grid((N + SG_BN - 1) / SG_BN, (M + SG_BM - 1) / SG_BM);
  SV_COUNT_LAUNCH();
  gemm_simt_kernel<<<grid, 256, 0, s>>>(A, B, C, M, N, K);
  return cudaGetLastError();
}

}  // namespace sv
