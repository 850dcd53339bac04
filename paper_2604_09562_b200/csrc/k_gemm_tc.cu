// tcgen05 GEMM with fused epilogues: C[M][N] = A[M][K] * B[N][K]^T, bf16 operands (both
// K-major), fp32 accumulation in TMEM. Used for the lm-head (a5: fused softmax-statistics
// epilogue + fp32 logits) and the projections (a2 QKV + RoPE + chain-KV write, a4 O-proj /
// down-proj + residual, gate/up + SwiGLU).
//
// Design (sm_100a): persistent grid (one CTA per SM), 128x256 output tile per CTA
// (UMMA_M = 128, UMMA_N = 256, K step 16), 64-wide K blocks staged by TMA with 128-byte
// swizzle into a 4-stage smem ring, one elected thread issuing tcgen05.mma into a
// double-buffered TMEM accumulator (2 x 256 columns), and 4 epilogue warps draining TMEM
// with tcgen05.ld while the next tile's MMAs run. Warp roles:
//   warp 0: TMA producer   warp 1: MMA issuer   warp 2: TMEM allocator   warps 4-7: epilogue
// Tiles are ordered M-fastest so the CTAs working on one 256-row weight tile run together
// and the weight tile is read from HBM once (L2 reuse).
#include <cuda.h>

#include "common.cuh"
#include "gemm_tc.h"
#include "lane.h"
#include "tc.cuh"

namespace sv {

namespace {
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;             // 16 KB
constexpr int B_BYTES = BN * BK * 2;             // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // 48 KB
constexpr int THREADS = 256;
constexpr uint32_t IDESC = tc::idesc_bf16(BM, BN);
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
}  // namespace

struct TileCoord {
  int m_blk, n_blk;
};

__device__ __forceinline__ TileCoord tile_of(int t, int num_m) { return TileCoord{t % num_m, t / num_m}; }

__device__ __forceinline__ float u2f(uint32_t v) { return __uint_as_float(v); }

// ------------------------------------------------------------------ epilogues
// Each epilogue thread owns one accumulator row (TMEM lane) and walks its 256 columns
// in 8 chunks of 32 (tcgen05.ld 32x32b.x32).
__device__ __forceinline__ void epi_store_f32(const GemmTcArgs& g, int row, int n0, uint32_t tbase) {
  uint32_t r[32];
  for (int c = 0; c < BN / 32; ++c) {
    __syncwarp();
    tc::tmem_ld32(tbase + c * 32, r);
    tc::tmem_ld_wait();
    if (row >= g.M) continue;
    const int n = n0 + c * 32;
    float* dst = g.out + (size_t)row * g.ldo + n;
    if (g.kind == GEMM_EPI_RESIDUAL) {
      const float* src = g.resid_in + (size_t)row * g.ldo + n;
      float* o = g.resid_out + (size_t)row * g.ldo + n;
      if (n + 32 <= g.N) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 h = *reinterpret_cast<const float4*>(src + i);
          *reinterpret_cast<float4*>(o + i) =
              make_float4(h.x + u2f(r[i]), h.y + u2f(r[i + 1]), h.z + u2f(r[i + 2]), h.w + u2f(r[i + 3]));
        }
      } else {
        for (int i = 0; i < 32 && n + i < g.N; ++i) o[i] = src[i] + u2f(r[i]);
      }
    } else {
      if (n + 32 <= g.N) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(u2f(r[i]), u2f(r[i + 1]), u2f(r[i + 2]), u2f(r[i + 3]));
      } else {
        for (int i = 0; i < 32 && n + i < g.N; ++i) dst[i] = u2f(r[i]);
      }
    }
  }
}

// a5: fp32 logits + per-(row, 256-col tile) max / sum exp / lowest argmax of l * inv_temp
__device__ __forceinline__ void epi_logits(const GemmTcArgs& g, int row, int n0, int n_blk, uint32_t tbase) {
  uint32_t r[32];
  float m = -INFINITY, s = 0.f;
  int am = 0x7fffffff;
  for (int c = 0; c < BN / 32; ++c) {
    __syncwarp();
    tc::tmem_ld32(tbase + c * 32, r);
    tc::tmem_ld_wait();
    const int n = n0 + c * 32;
    float cm = -INFINITY;
    int ca = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float x = (n + i < g.N) ? u2f(r[i]) * g.inv_temp : -INFINITY;
      if (x > cm) { cm = x; ca = n + i; }
    }
    const float mn = fmaxf(m, cm);
    float cs = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float x = (n + i < g.N) ? u2f(r[i]) * g.inv_temp : -INFINITY;
      cs += expf(x - mn);
    }
    s = (m == -INFINITY ? 0.f : s * expf(m - mn)) + cs;
    if (cm > m) am = ca;
    m = mn;
    if (row < g.M) {
      float* dst = g.out + (size_t)row * g.ldo + n;
      if (n + 32 <= g.N) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(u2f(r[i]), u2f(r[i + 1]), u2f(r[i + 2]), u2f(r[i + 3]));
      } else {
        for (int i = 0; i < 32 && n + i < g.N; ++i) dst[i] = u2f(r[i]);
      }
    }
  }
  if (row < g.M) {
    const size_t o = (size_t)row * g.nt + n_blk;
    g.tmax[o] = m;
    g.tsum[o] = s;
    g.targ[o] = am;
  }
}

// a2: q/k RoPE (rotate_half, fp32 table) + bf16 store to Q / chain K; v plain bf16 store
__device__ __forceinline__ void epi_qkv(const GemmTcArgs& g, int row, int n0, uint32_t tbase) {
  const int dh = g.dh, half = dh / 2;
  const int heads_per_tile = BN / dh;
  const int nkv = g.Hkv * dh;
  const int pos = row < g.M ? g.row_pos[row] : 0;
  uint32_t x1[32], x2[32];
  for (int hh = 0; hh < heads_per_tile; ++hh) {
    const int head = n0 / dh + hh;
    const int cbase = hh * dh;                       // column of this head inside the tile
    for (int c = 0; c < half / 32; ++c) {
      __syncwarp();
      tc::tmem_ld32(tbase + cbase + c * 32, x1);
      tc::tmem_ld32(tbase + cbase + half + c * 32, x2);
      tc::tmem_ld_wait();
      if (row >= g.M || head >= g.Hq + 2 * g.Hkv) continue;
      __nv_bfloat16 o1[32], o2[32];
      if (head < g.Hq + g.Hkv) {
        const float* cs = g.rope_cos + (size_t)pos * half + c * 32;
        const float* sn = g.rope_sin + (size_t)pos * half + c * 32;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float a = u2f(x1[i]), b = u2f(x2[i]);
          o1[i] = f2bf(a * cs[i] - b * sn[i]);
          o2[i] = f2bf(b * cs[i] + a * sn[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          o1[i] = f2bf(u2f(x1[i]));
          o2[i] = f2bf(u2f(x2[i]));
        }
      }
      __nv_bfloat16* dst;
      if (head < g.Hq) dst = g.q + (size_t)row * g.Hq * dh + (size_t)head * dh;
      else if (head < g.Hq + g.Hkv) dst = g.kc + (size_t)row * nkv + (size_t)(head - g.Hq) * dh;
      else dst = g.vc + (size_t)row * nkv + (size_t)(head - g.Hq - g.Hkv) * dh;
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        *reinterpret_cast<uint4*>(dst + c * 32 + i) = *reinterpret_cast<const uint4*>(&o1[i]);
        *reinterpret_cast<uint4*>(dst + half + c * 32 + i) = *reinterpret_cast<const uint4*>(&o2[i]);
      }
    }
  }
}

// a4: u = bf16(silu(gate) * up); tile columns 0..127 are gate rows, 128..255 the matching up rows
__device__ __forceinline__ void epi_swiglu(const GemmTcArgs& g, int row, int n_blk, uint32_t tbase) {
  uint32_t gt[32], up[32];
  for (int c = 0; c < 4; ++c) {
    __syncwarp();
    tc::tmem_ld32(tbase + c * 32, gt);
    tc::tmem_ld32(tbase + 128 + c * 32, up);
    tc::tmem_ld_wait();
    if (row >= g.M) continue;
    __nv_bfloat16 o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float x = u2f(gt[i]);
      o[i] = f2bf(x / (1.0f + expf(-x)) * u2f(up[i]));
    }
    __nv_bfloat16* dst = g.u + (size_t)row * g.F + n_blk * 128 + c * 32;
#pragma unroll
    for (int i = 0; i < 32; i += 8) *reinterpret_cast<uint4*>(dst + i) = *reinterpret_cast<const uint4*>(&o[i]);
  }
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const GemmTcArgs g) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_s & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (g.M + BM - 1) / BM;
  const int num_tiles = num_m * g.n_tiles;
  const int nk = g.K / BK;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&map_a);
    tc::prefetch_tmap(&map_b);
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 128);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) {
    tc::tmem_alloc(tmem_holder, 512);
    tc::tmem_relinquish();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      const uint64_t pol_b = tc::policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const TileCoord tcd = tile_of(t, num_m);
        const int arow = tcd.m_blk * BM;
        int brow0, brow1;
        if (g.kind == GEMM_EPI_SWIGLU) {
          brow0 = tcd.n_blk * 128;
          brow1 = g.F + tcd.n_blk * 128;
        } else {
          brow0 = tcd.n_blk * BN;
          brow1 = brow0 + 128;
        }
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          tc::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tc::tma_load_2d(sA + stage * A_BYTES, &map_a, &full[stage], kb * BK, arow);
          uint8_t* b = sB + stage * B_BYTES;
          tc::tma_load_2d_hint(b, &map_b, &full[stage], kb * BK, brow0, pol_b);
          tc::tma_load_2d_hint(b + B_BYTES / 2, &map_b, &full[stage], kb * BK, brow1, pol_b);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint64_t da = tc::sdesc_sw128(tc::smem_u32(sA + stage * A_BYTES), 16, 1024);
          const uint64_t db = tc::sdesc_sw128(tc::smem_u32(sB + stage * B_BYTES), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)       // +32 B per K=16 step inside the 128-B swizzle atom
            tc::umma_bf16(d, da + 2 * kk, db + 2 * kk, IDESC, (kb | kk) != 0);
          tc::umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue warps (TMEM lanes 32*(warp%4) ..)
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const TileCoord tcd = tile_of(t, num_m);
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
      const int row = tcd.m_blk * BM + q * 32 + lane;
      switch (g.kind) {
        case GEMM_EPI_LOGITS: epi_logits(g, row, tcd.n_blk * BN, tcd.n_blk, tbase); break;
        case GEMM_EPI_QKV_ROPE: epi_qkv(g, row, tcd.n_blk * BN, tbase); break;
        case GEMM_EPI_SWIGLU: epi_swiglu(g, row, tcd.n_blk, tbase); break;
        default: epi_store_f32(g, row, tcd.n_blk * BN, tbase); break;
      }
      tc::fence_before();
      tc::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, 512);
  }
}

int gemm_tc_smem_bytes() { return SMEM_BYTES; }

cudaError_t launch_gemm_tc(const CUtensorMap& map_a, const CUtensorMap& map_b, const GemmTcArgs& g, int num_sms,
                           cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (g.M <= 0) return cudaSuccess;
  const int num_tiles = ((g.M + BM - 1) / BM) * g.n_tiles;
  const int grid = num_tiles < num_sms ? num_tiles : num_sms;
  SV_COUNT_LAUNCH();
  gemm_tc_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(map_a, map_b, g);
  return cudaGetLastError();
}

}  // namespace sv
