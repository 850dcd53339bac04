// Microbenchmark: tcgen05.mma issue rate vs N (cta_group::1, M = 128; cta_group::2, M = 256),
// operands = garbage smem (SW128 K-major descriptors). One thread issues R back-to-back MMAs
// into one TMEM accumulator, commits, waits; clock64 around it. Grid = 148 CTAs (74 pairs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_09562_b200/csrc/tc.cuh"
using namespace sv;

template <int CG>
__global__ void __launch_bounds__(128, 1) mma_rate(int N, int R, int init, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (init) {   // 1: zeros, 2: pseudo-random bf16 in [-1, 1)
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
      uint32_t h = (uint32_t)i * 2654435761u ^ blockIdx.x * 40503u;
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      const uint32_t lo = 0x3f80u | (h & 0x807fu), hi = 0x3f80u | ((h >> 16) & 0x807fu);
      w[i] = init == 1 ? 0u : (lo | (hi << 16));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    if (CG == 2) tc::tmem_alloc_2sm(&holder, 512);
    else { tc::tmem_alloc(&holder, 512); tc::tmem_relinquish(); }
  }
  tc::fence_before();
  __syncthreads();
  if (CG == 2) tc::cluster_sync_all();
  tc::fence_after();
  const uint32_t tm = holder;
  const bool leader = CG == 1 || tc::cluster_rank() == 0;
  if (threadIdx.x == 0 && leader) {
    const uint32_t idesc = tc::idesc_bf16(CG == 2 ? 256 : 128, N);
    const uint64_t da = tc::sdesc_sw128(tc::smem_u32(smem), 16, 1024);
    const uint64_t db = tc::sdesc_sw128(tc::smem_u32(smem + 32768), 16, 1024);
    // warm-up
    for (int i = 0; i < 16; ++i) {
      if (CG == 2) tc::umma_bf16_2sm(tm, da + 2 * (i & 3), db + 2 * (i & 3), idesc, i > 0);
      else tc::umma_bf16(tm, da + 2 * (i & 3), db + 2 * (i & 3), idesc, i > 0);
    }
    if (CG == 2) tc::umma_commit_2sm(&bar, 0x1); else tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      if (CG == 2) tc::umma_bf16_2sm(tm, da + 2 * (i & 3), db + 2 * (i & 3), idesc, 1);
      else tc::umma_bf16(tm, da + 2 * (i & 3), db + 2 * (i & 3), idesc, 1);
    }
    if (CG == 2) tc::umma_commit_2sm(&bar, 0x1); else tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 1);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (CG == 2) tc::cluster_sync_all();
  if (warp == 0) {
    tc::fence_after();
    if (CG == 2) tc::tmem_dealloc_2sm(tm, 512); else tc::tmem_dealloc(tm, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int R = 4096;
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(mma_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_rate<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int init = 0; init < 3; ++init)
  for (int cg = 1; cg <= 2; ++cg) {
    for (int N : {64, 128, 192, 256}) {
      if (cg == 1) mma_rate<1><<<148, 128, smem>>>(N, R, init, d);
      else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, mma_rate<2>, N, R, init, d);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; i += cg) mx = h[i] > mx ? h[i] : mx;
      const int M = cg == 2 ? 256 : 128;
      printf("init %d cta_group::%d M=%d N=%3d: %6.1f cycles/MMA (floor %d)\n", init, cg, M, N, (double)mx / R,
             (M > 128 ? M : 128) * N / (256 * cg));
    }
  }
  return 0;
}
