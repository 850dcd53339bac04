// Which part of the GEMM main loop costs time? cta_group::2, M = 256, N = NT, 4 MMAs per K block:
//  mode 0: MMAs only;  1: + tcgen05.commit (multicast) to empty[stage] per K block;
//  2: + full/empty ring handshake with a producer thread that only arrives (STAGES = 6);
//  3: as 2 but the MMA thread advances the smem descriptors per stage (6 x 32 KB ring).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_09562_b200/csrc/tc.cuh"
using namespace sv;
constexpr int STAGES = 6;

__global__ void __launch_bounds__(128, 1) mma_loop(int N, int KB, int mode, int boff, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool leader = tc::cluster_rank() == 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1); }
    tc::mbar_init(&done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc_2sm(&holder, 512);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();
  tc::fence_after();
  const uint32_t tm = holder;
  const uint32_t idesc = tc::idesc_bf16(256, N);
  if (warp == 1 && lane == 0 && ((mode >= 2 && mode <= 3) || mode == 7)) {
    int stage = 0; uint32_t phase = 0;
    for (int kb = 0; kb < KB; ++kb) {
      tc::mbar_wait(&empty[stage], phase ^ 1);
      if (leader) tc::mbar_arrive(&full[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }
  if (warp == 0 && leader && mode >= 6) {
    // whole warp runs the loop (converged, uniform values); one elected lane issues
    const long long t0 = clock64();
    int stage = 0; uint32_t phase = 0;
    for (int kb = 0; kb < KB; ++kb) {
      if (mode == 7) { tc::mbar_wait(&full[stage], phase); tc::fence_after(); }
      const int off = mode == 7 ? stage * 32768 : 0;
      const uint64_t da = tc::sdesc_sw128(tc::smem_u32(smem + off), 16, 1024);
      const uint64_t db = tc::sdesc_sw128(tc::smem_u32(smem + off + boff), 16, 1024);
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::umma_bf16_2sm(tm, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
        if (mode == 7) tc::umma_commit_2sm(&empty[stage], 0x3);
      }
      __syncwarp();
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if (tc::elect_one()) tc::umma_commit_2sm(&done, 0x1);
    __syncwarp();
    tc::mbar_wait(&done, 0);
    if (lane == 0) out[blockIdx.x] = clock64() - t0;
  }
  if (warp == 0 && lane == 0 && leader && mode < 6) {
    const long long t0 = clock64();
    int stage = 0; uint32_t phase = 0;
    for (int kb = 0; kb < KB; ++kb) {
      if (mode >= 2 && mode <= 3) { tc::mbar_wait(&full[stage], phase); tc::fence_after(); }
      const int off = mode == 3 ? stage * 32768 : 0;
      const uint64_t da = tc::sdesc_sw128(tc::smem_u32(smem + off), 16, 1024);
      const uint64_t db = tc::sdesc_sw128(tc::smem_u32(smem + off + boff), 16, 1024);
      if (mode == 5) {
        for (int kk = 0; kk < 4; ++kk) tc::umma_bf16_2sm(tm, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
      } else if (mode == 4) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::umma_bf16_2sm(tm, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::umma_bf16_2sm(tm, da + 2 * kk, db + 2 * kk, idesc, 1);
      }
      if (mode >= 1 && mode <= 3) tc::umma_commit_2sm(&empty[stage], 0x3);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    tc::umma_commit_2sm(&done, 0x1);
    tc::mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();
  if (warp == 0) { tc::fence_after(); tc::tmem_dealloc_2sm(tm, 512); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int KB = 1024;
  cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * 32768 + 1024);
  for (int smem : {STAGES * 32768 + 1024})
  for (int boff : {16384})
  for (int N : {128, 192, 256}) {
    for (int mode = 0; mode < 8; ++mode) {
      if ((mode == 3 || mode == 7) && smem < STAGES * 32768) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, mma_loop, N, KB, mode, boff, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; i += 2) mx = h[i] > mx ? h[i] : mx;
      printf("smem %3d KB boff %5d N=%3d mode %d: %6.1f cycles per K block (MMA floor %d)\n", smem / 1024, boff, N, mode,
             (double)mx / KB, 4 * N / 2);
    }
  }
  return 0;
}
