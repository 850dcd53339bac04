// Weight-major 2-SM GEMM (cta_group::2) for the verify step's projections and lm-head:
//   D^T[f][t] = sum_k W[f][k] X[t][k]      (W = weight rows, X = the step's T token rows)
// i.e. C = X W^T computed with the weights on the MMA's M side and the tokens on its N side.
//
// Why this orientation (measured on B200, see DESIGN.md §"GEMM"): the step has T = 576 token
// rows at the north-star shape, which is 4.5 tiles of 128 (or 2.25 pair tiles of 256) — the
// token-major kernels pad 11-33 % of their MMA work. With tokens on N the tile width is free in
// steps of 16 (N = 192 gives 3 exact tiles), weight rows come in 256-row pair tiles (every
// projection and the vocabulary are multiples of 256), so no MMA work is padding. The 1-SM
// 128 x 256 kernel is bound by shared-memory bandwidth (TMA writes + MMA reads = 192 B/clk per SM
// for 512 MMA cycles per K block; ncu: tensor pipe 75 %); the pair form halves the token
// operand each SM stages and reads (16 KB weights + NT/2 x 128 B tokens per K block).
//
// Roles (8 warps, both CTAs of the pair): warp 0 TMA producer (each CTA loads its own 128
// weight rows and its half of the token tile; both land on the leader's barrier), warp 1 MMA
// issuer (leader CTA only, one thread), warp 2 TMEM allocator, warps 4-7 epilogue (TMEM lane
// = weight row; each warp owns 32 rows, a column = a token).
//
// Epilogues (fused):
//   NONE      out[t][f] = acc                         (test hook)
//   RESIDUAL  out[t][f] = in[t][f] + acc              (a4 o-proj / down-proj; in may alias out)
//   LOGITS    out[t][f] = acc, plus per (t, 128-row vocab tile) max / sum exp / lowest argmax
//             of acc * inv_temp                       (a5)
//   QKV_ROPE  rotate_half RoPE on q and k rows, bf16 q / chain K / chain V          (a2)
//   SWIGLU    u[t][j] = bf16(silu(gate_j) * up_j); each CTA stages 64 gate rows + the 64
//             matching up rows                       (a4)
// For a fixed token column the 32 lanes of a warp hold 32 consecutive features, so every
// global store is a contiguous 128-byte (fp32) or 64-byte (bf16) warp segment.
#include <cuda.h>

#include "common.cuh"
#include "gemm_tc.h"
#include "lane.h"
#include "tc.cuh"

namespace sv {

namespace {
constexpr int BK = 64, STAGES = 6, THREADS = 384;   // 4 role warps + 8 epilogue warps
constexpr int A_BYTES = 128 * BK * 2;             // 16 KB: this CTA's 128 weight rows
constexpr int BX_BYTES = 128 * BK * 2;            // 16 KB: room for NT/2 <= 128 token rows
constexpr int STAGE_BYTES = A_BYTES + BX_BYTES;
constexpr int XCH_BYTES = 2 * 4 * 16 * 32 * 4;      // 16 KB: partner-row exchange / output staging [half][quadrant]
constexpr int RED_BYTES = 3 * 4 * 256 * 4;        // 12 KB: per-warp column statistics
constexpr int AUX_BYTES = XCH_BYTES > RED_BYTES ? XCH_BYTES : RED_BYTES;
constexpr int POS_BYTES = 256 * 4;                 // QKV: positions of the tile's tokens
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + AUX_BYTES + POS_BYTES;
constexpr int XCH_BAR = 1;                        // named barriers 1, 2: the 4 epilogue warps of a column half
constexpr int EPI_BAR = 3;                        // named barrier of all 8 epilogue warps
constexpr int EPI_THREADS = 256;
static_assert(SMEM_BYTES <= 227 * 1024, "smem");
}  // namespace

__device__ __forceinline__ float sw_u2f(uint32_t v) { return __uint_as_float(v); }

// per-tile timeline of CTA 0 (events 12-15 of the lane trace buffer, SV_TRACE=1)
#define SW_TR(g, e, i)                                                                \
  do {                                                                                \
    if ((g).trace && blockIdx.x == 0 && (i) < 256) (g).trace[(e)*256 + (i)] = clock64(); \
  } while (0)
__device__ __forceinline__ unsigned long long sw_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SwTile {
  int m_pair, n_blk;
};

struct SwEpi {
  const GemmTcArgs* g;
  int rank, q, h, lane, tid;   // quadrant (TMEM lanes 32q..), column half, lane, epilogue thread id
  float* aux;        // XCH or RED region
  int* pos;          // POS region
  uint32_t tbase;    // TMEM address of this warp's lanes, current accumulator
  int NT;
  int M;             // token rows (the launch's, or the device value of a dynamic-depth graph)
};

// 16 accumulator columns of this warp's 32 rows
__device__ __forceinline__ void sw_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  __syncwarp();
  tc::tmem_ld16(taddr, r);
  tc::tmem_ld_wait();
}

// ---------------------------------------------------------------- fp32 stores (+ residual)
// The warp's own 2 KB slot of the AUX region (output staging)
__device__ __forceinline__ float* sw_slot(const SwEpi& e) { return e.aux + (e.h * 4 + e.q) * (16 * 32); }

// fp32 outputs (+ residual): the chunk's accumulators are transposed through the warp's slot so
// every load / store is a 16-byte access of a 128-byte row segment (4 tokens per instruction);
// the residual rows of the next chunk are loaded one chunk ahead. The residual input may alias
// the output: each element is read before it is written, by the same lane.
__device__ __forceinline__ void sw_epi_f32(const SwEpi& e, const SwTile& tl) {
  const GemmTcArgs& g = *e.g;
  const int f0 = tl.m_pair * 256 + e.rank * 128 + e.q * 32;   // first feature of this warp
  const bool resid = g.kind == GEMM_EPI_RESIDUAL;
  float* out = resid ? g.resid_out : g.out;
  const int t0 = tl.n_blk * e.NT;
  float* st = sw_slot(e);                                     // [16 tokens][32 features] fp32
  // lane -> (token tok = it * 4 + lane / 8, 4 features at part * 4): whole 128-byte row segments
  const int part = e.lane & 7, fcol = f0 + part * 4;
  const bool vec = (g.ldo & 3) == 0 && fcol + 4 <= g.N;
  auto load_in = [&](float4 (&h)[4], int c) {                 // residual rows of chunk c
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int t = t0 + c + it * 4 + (e.lane >> 3);
      h[it] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (resid && vec && c < e.NT && t < e.M) h[it] = __ldcg(reinterpret_cast<const float4*>(g.resid_in + (size_t)t * g.ldo + fcol));
    }
  };
  float4 hn[4];
  load_in(hn, e.h * 16);
  for (int c = e.h * 16; c < e.NT; c += 32) {
    float4 h[4];
#pragma unroll
    for (int it = 0; it < 4; ++it) h[it] = hn[it];
    load_in(hn, c + 32);                                      // next chunk's rows in flight
    uint32_t r[16];
    sw_ld16(e.tbase + c, r);
#pragma unroll
    for (int i = 0; i < 16; ++i) st[i * 32 + e.lane] = sw_u2f(r[i]);
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int tok = it * 4 + (e.lane >> 3), t = t0 + c + tok;
      if (t >= e.M) continue;
      const float4 v = *reinterpret_cast<const float4*>(st + tok * 32 + part * 4);
      const size_t o = (size_t)t * g.ldo + fcol;
      if (vec) {
        *reinterpret_cast<float4*>(out + o) = make_float4(v.x + h[it].x, v.y + h[it].y, v.z + h[it].z, v.w + h[it].w);
      } else {                                                // ragged feature tail / unaligned rows
        const float vv[4] = {v.x, v.y, v.z, v.w};
        for (int k = 0; k < 4 && fcol + k < g.N; ++k) out[o + k] = resid ? g.resid_in[o + k] + vv[k] : vv[k];
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- lm-head logits + tile stats
// Column statistics over the warp's 32 rows (= 32 consecutive vocabulary entries), 16 columns
// per chunk: max by redux.sync (one instruction per column), argmax by ballot, and the 16 sums
// of exp by a transposing butterfly that halves the list of columns a lane carries at each
// xor-shuffle step (16 -> 8 -> 4 -> 2 -> 1), leaving column j in lanes 2j, 2j + 1.
template <int N, int OFF>
__device__ __forceinline__ void bfly_sum(float (&s)[16], int lane) {
  const bool up = lane & OFF;
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const float send = up ? s[i] : s[i + N / 2];
    const float keep = up ? s[i + N / 2] : s[i];
    s[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
  }
}

// greedy decisions (argmax_only): per column the max and lowest argmax over this warp's 32 rows, the
// 4 warps combined through shared memory, one atomicMax key per (token, 128-row tile) into row_best
__device__ __forceinline__ void sw_epi_argmax(const SwEpi& e, const SwTile& tl) {
  const GemmTcArgs& g = *e.g;
  const int fb = tl.m_pair * 256 + e.rank * 128;          // first vocab row of this CTA
  const int f = fb + e.q * 32 + e.lane;
  const bool valid = f < g.N;
  const int t0 = tl.n_blk * e.NT;
  float* rmax = e.aux;                                    // [4][256]
  int* rarg = reinterpret_cast<int*>(e.aux + 8 * 256);
  for (int c = e.h * 16; c < e.NT; c += 32) {
    uint32_t r[16];
    sw_ld16(e.tbase + c, r);
    float M[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) M[i] = tc::redux_max(valid ? sw_u2f(r[i]) : -INFINITY);
    unsigned hit[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) hit[i] = __ballot_sync(0xffffffffu, valid && sw_u2f(r[i]) == M[i]);
    if (e.lane < 16) {                                    // lane i publishes column c + i
      float mi = M[0];
      unsigned hi = hit[0];
#pragma unroll
      for (int i = 1; i < 16; ++i) {
        mi = e.lane == i ? M[i] : mi;
        hi = e.lane == i ? hit[i] : hi;
      }
      rmax[e.q * 256 + c + e.lane] = mi;
      rarg[e.q * 256 + c + e.lane] = hi ? fb + e.q * 32 + (__ffs(hi) - 1) : 0x7fffffff;
    }
  }
  tc::named_bar(EPI_BAR, EPI_THREADS);
  for (int col = e.tid; col < e.NT; col += EPI_THREADS) {
    const int t = t0 + col;
    float m = -INFINITY;
    int am = 0x7fffffff;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float v = rmax[w * 256 + col];
      if (v > m) { m = v; am = rarg[w * 256 + col]; }    // warps in feature order: first = lowest
    }
    if (t < e.M && m != -INFINITY) {
      const uint32_t u = __float_as_uint(m);
      const uint32_t ou = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
      atomicMax(g.row_best + t, ((unsigned long long)ou << 32) | (0xFFFFFFFFu - (uint32_t)am));
    }
  }
  tc::named_bar(EPI_BAR, EPI_THREADS);                    // RED is reused by the next tile
}

__device__ __forceinline__ void sw_epi_logits(const SwEpi& e, const SwTile& tl) {
  const GemmTcArgs& g = *e.g;
  const int fb = tl.m_pair * 256 + e.rank * 128;          // first vocab row of this CTA
  const int f = fb + e.q * 32 + e.lane;
  const bool valid = f < g.N;
  const int t0 = tl.n_blk * e.NT;
  float* rmax = e.aux;                                    // [4][256]
  float* rsum = e.aux + 4 * 256;
  int* rarg = reinterpret_cast<int*>(e.aux + 8 * 256);
  constexpr float kLog2e = 1.4426950408889634f;
  for (int c = e.h * 16; c < e.NT; c += 32) {
    uint32_t r[16];
    sw_ld16(e.tbase + c, r);
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int t = t0 + c + i;
      const float l = sw_u2f(r[i]);
      if (g.out && valid && t < e.M) g.out[(size_t)t * g.ldo + f] = l;
      x[i] = valid ? l * g.inv_temp : -INFINITY;
    }
    // column max over the warp's 32 rows: one redux per column, result in every lane;
    // argmax = lowest lane attaining it (lanes are in vocabulary order)
    float M[16];
    unsigned hit[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) M[i] = tc::redux_max(x[i]);
#pragma unroll
    for (int i = 0; i < 16; ++i) hit[i] = __ballot_sync(0xffffffffu, x[i] == M[i]);
    float sum[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) sum[i] = (M[i] == -INFINITY) ? 0.f : tc::ex2((x[i] - M[i]) * kLog2e);
    bfly_sum<16, 16>(sum, e.lane);
    bfly_sum<8, 8>(sum, e.lane);
    bfly_sum<4, 4>(sum, e.lane);
    bfly_sum<2, 2>(sum, e.lane);
    sum[0] += __shfl_xor_sync(0xffffffffu, sum[0], 1);   // lanes 2j, 2j+1: column j
    if ((e.lane & 1) == 0) rsum[e.q * 256 + c + (e.lane >> 1)] = sum[0];
    if (e.lane == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        rmax[e.q * 256 + c + i] = M[i];
        rarg[e.q * 256 + c + i] = fb + e.q * 32 + (__ffs(hit[i]) - 1);
      }
    }
  }
  tc::named_bar(EPI_BAR, EPI_THREADS);
  const int tile = fb / 128;
  for (int col = e.tid; col < e.NT; col += EPI_THREADS) {
    const int t = t0 + col;
    float m = -INFINITY;
    int am = 0x7fffffff;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float v = rmax[w * 256 + col];
      if (v > m) { m = v; am = rarg[w * 256 + col]; }    // warps in feature order: first = lowest
    }
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float v = rmax[w * 256 + col];
      if (v != -INFINITY) s += rsum[w * 256 + col] * tc::ex2((v - m) * kLog2e);
    }
    if (t < e.M && tile < g.nt) {
      const size_t o = (size_t)t * g.nt + tile;
      g.tmax[o] = m;
      g.tsum[o] = s;
      g.targ[o] = am;
      if (g.row_best && m != -INFINITY) {
        // order-preserving bits of m (larger m -> larger key), ties -> the lower token id wins
        const uint32_t u = __float_as_uint(m);
        const uint32_t ou = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        atomicMax(g.row_best + t, ((unsigned long long)ou << 32) | (0xFFFFFFFFu - (uint32_t)am));
      }
    }
  }
  tc::named_bar(EPI_BAR, EPI_THREADS);                    // RED is reused by the next tile
}

// ---------------------------------------------------------------- partner-row exchange
// Publishes this warp's 16 values and returns the values of row (own row ^ pmask) for the
// same columns. pmask = 32 or 64 (a partner in another warp of this CTA).
__device__ __forceinline__ void sw_exchange(const SwEpi& e, int pmask, const uint32_t (&r)[16], float (&p)[16]) {
  float* buf = e.aux + e.h * (4 * 16 * 32);
#pragma unroll
  for (int i = 0; i < 16; ++i) buf[(e.q * 16 + i) * 32 + e.lane] = sw_u2f(r[i]);
  tc::named_bar(XCH_BAR + e.h, 128);
  const int pq = e.q ^ (pmask >> 5);
#pragma unroll
  for (int i = 0; i < 16; ++i) p[i] = buf[(pq * 16 + i) * 32 + e.lane];
  tc::named_bar(XCH_BAR + e.h, 128);                    // partner reads done: own slot reusable
}


// Store a 32-feature x 16-token bf16 block (lane = feature, y[i] = token i) with 16-byte stores:
// transposed through the warp's slot, 4 lanes per token row, 8 tokens per instruction. out0 =
// address of (first token, feature of lane 0); ld = row stride in elements; ntok = valid tokens.
__device__ __forceinline__ void sw_store_bf16(const SwEpi& e, const __nv_bfloat16 (&y)[16], __nv_bfloat16* out0,
                                              size_t ld, int ntok) {
  __nv_bfloat16* st = reinterpret_cast<__nv_bfloat16*>(sw_slot(e));
#pragma unroll
  for (int i = 0; i < 16; ++i) st[i * 32 + e.lane] = y[i];
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int tok = it * 8 + (e.lane >> 2), part = e.lane & 3;
    if (tok < ntok)
      *reinterpret_cast<uint4*>(out0 + (size_t)tok * ld + part * 8) = *reinterpret_cast<const uint4*>(st + tok * 32 + part * 8);
  }
  __syncwarp();
}

// ---------------------------------------------------------------- a2 QKV + RoPE
__device__ __forceinline__ void sw_epi_qkv(const SwEpi& e, const SwTile& tl) {
  const GemmTcArgs& g = *e.g;
  const int dh = g.dh, half = dh / 2;
  const int rho = e.q * 32 + e.lane;                      // row inside the CTA's 128
  const int f = tl.m_pair * 256 + e.rank * 128 + rho;
  const int head = f / dh, d = f % dh;
  const int nheads = g.Hq + 2 * g.Hkv;
  const bool rope = head < g.Hq + g.Hkv;
  const bool lo = d < half;
  const int dd = lo ? d : d - half;
  const int d0 = d - e.lane;                              // first feature of this warp (32-aligned)
  __nv_bfloat16* dst;
  size_t ld;
  if (head < g.Hq) {
    ld = (size_t)g.Hq * dh;
    dst = g.q + (size_t)head * dh + d0;
  } else if (head < g.Hq + g.Hkv) {
    ld = (size_t)g.Hkv * dh;
    dst = g.kc + (size_t)(head - g.Hq) * dh + d0;
  } else {
    ld = (size_t)g.Hkv * dh;
    dst = g.vc + (size_t)(head - g.Hq - g.Hkv) * dh + d0;
  }
  const int t0 = tl.n_blk * e.NT;
  for (int col = e.tid; col < e.NT; col += EPI_THREADS) {     // the tile's token positions
    const int t = t0 + col;
    e.pos[col] = t < e.M ? g.row_pos[t] : 0;
  }
  tc::named_bar(EPI_BAR, EPI_THREADS);
  // RoPE table values of the next chunk are loaded while this chunk's accumulators come out of
  // TMEM and cross the partner exchange (software pipeline: a single-tile launch exposes the epilogue)
  auto load_tab = [&](float (&cs)[16], float (&sn)[16], int c) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const bool ok = rope && head < nheads && c < e.NT;
      const size_t o = ok ? (size_t)e.pos[c + i] * half + dd : 0;
      cs[i] = ok ? __ldg(g.rope_cos + o) : 1.f;
      sn[i] = ok ? __ldg(g.rope_sin + o) : 0.f;
    }
  };
  float csn[16], snn[16];
  load_tab(csn, snn, e.h * 16);
  for (int c = e.h * 16; c < e.NT; c += 32) {
    float cs[16], sn[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      cs[i] = csn[i];
      sn[i] = snn[i];
    }
    load_tab(csn, snn, c + 32);
    uint32_t r[16];
    float p[16];
    sw_ld16(e.tbase + c, r);
    sw_exchange(e, half, r, p);                           // partner = d +- half, same head
    if (head >= nheads) continue;                         // warp-uniform
    __nv_bfloat16 y[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float x = sw_u2f(r[i]);
      y[i] = f2bf(!rope ? x : lo ? x * cs[i] - p[i] * sn[i] : x * cs[i] + p[i] * sn[i]);
    }
    sw_store_bf16(e, y, dst + (size_t)(t0 + c) * ld, ld, min(16, e.M - (t0 + c)));
  }
  tc::named_bar(EPI_BAR, EPI_THREADS);                    // XCH / POS are reused by the next tile
}

// ---------------------------------------------------------------- a4 gate/up + SwiGLU
__device__ __forceinline__ void sw_epi_swiglu(const SwEpi& e, const SwTile& tl) {
  const GemmTcArgs& g = *e.g;
  const int rho = e.q * 32 + e.lane;                      // < 64: gate row, >= 64: up row
  const int j = tl.m_pair * 128 + e.rank * 64 + (rho & 63);
  const int t0 = tl.n_blk * e.NT;
  const int j0 = j - e.lane;                              // first feature of this warp (32-aligned)
  for (int c = e.h * 16; c < e.NT; c += 32) {
    uint32_t r[16];
    float p[16];
    sw_ld16(e.tbase + c, r);
    sw_exchange(e, 64, r, p);
    if (rho >= 64 || j0 >= g.F) continue;                 // warp-uniform (F % 128 == 0)
    __nv_bfloat16 y[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float x = sw_u2f(r[i]);
      y[i] = f2bf(__fdividef(x, 1.0f + __expf(-x)) * p[i]);
    }
    const int ntok = min(16, e.M - (t0 + c));
    sw_store_bf16(e, y, g.u + (size_t)(t0 + c) * g.F + j0, g.F, ntok);
  }
  tc::named_bar(EPI_BAR, EPI_THREADS);                    // XCH / POS are reused by the next tile
}

// ---------------------------------------------------------------- kernel
__global__ void __launch_bounds__(THREADS, 1)
    gemm_sw_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
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
  float* aux = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);
  int* pos_s = reinterpret_cast<int*>(smem + STAGES * STAGE_BYTES + 256 + AUX_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  const bool swiglu = g.kind == GEMM_EPI_SWIGLU;
  const int NT = g.nt_tok;
  const int num_mp = swiglu ? g.F / 128 : (g.N + 255) / 256;
  int M = g.M;                                            // g.M_dev: read after the dependency wait
  int n_tok = (M + NT - 1) / NT;
  int num_tiles = num_mp * n_tok;
  const int nk = g.K / BK;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&map_w);
    tc::prefetch_tmap(&map_x);
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 2 * EPI_THREADS);         // both CTAs' epilogue threads (leader's copy)
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc_2sm(tmem_holder, 512);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // PDL: everything above overlaps the previous kernel's tail. Weights are never written by the
  // step, so the producer also prefetches the first tile's weight stages before waiting; every other
  // global access (tokens, residuals, outputs) comes after pdl_wait.
  pdl_trigger();
  // (no pre-wait prefetch with a device M: the tile -> weight-tile map depends on it)
  const int npre = (g.diag & 1) || g.M_dev || cluster >= num_tiles ? 0 : (nk < STAGES ? nk : STAGES);
  if (warp != 0) pdl_wait();
  if (g.M_dev && warp != 0) {
    M = *g.M_dev;
    n_tok = (M + NT - 1) / NT;
    num_tiles = num_mp * n_tok;
  }
  if (g.trace && threadIdx.x == 0 && blockIdx.x < 512) g.trace[10 * 256 + blockIdx.x / 2 + (rank ? 128 : 0)] = sw_gtimer();

  // Producer and MMA roles run as whole, converged warps with one elected lane issuing: the
  // loop state is then warp-uniform and ptxas keeps the TMA / tcgen05 operands in uniform
  // registers (a lane-0-only loop costs ~120 cycles per issued instruction).
  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; bytes land on the leader's full barrier)
    const uint64_t pol_w = n_tok > 1 ? tc::policy_evict_last() : tc::policy_evict_first();
    const uint64_t pol_x = tc::policy_evict_last();
    const uint32_t tx = 2u * (A_BYTES + (NT / 2) * BK * 2);
    int stage = 0;
    uint32_t phase = 0;
    auto load_w = [&](int st, int m_pair, int kb) {
      const uint32_t fb = tc::smem_u32(&full[st]) & tc::kPeerBitMask;
      uint8_t* a = sA + st * A_BYTES;
      if (swiglu) {
        const int j0 = m_pair * 128 + (int)rank * 64;
        tc::tma_load_2d_2sm(a, &map_w, fb, kb * BK, j0, pol_w);
        tc::tma_load_2d_2sm(a + A_BYTES / 2, &map_w, fb, kb * BK, g.F + j0, pol_w);
      } else {
        tc::tma_load_2d_2sm(a, &map_w, fb, kb * BK, m_pair * 256 + (int)rank * 128, pol_w);
      }
    };
    // weight stages of the first tile, before the dependency wait (the ring starts empty)
    if (tc::elect_one()) {
      for (int kb = 0; kb < npre; ++kb) {
        if (leader) tc::mbar_arrive_expect_tx(&full[kb], tx);
        load_w(kb, cluster / n_tok, kb);
      }
    }
    __syncwarp();
    pdl_wait();
    if (g.M_dev) {
      M = *g.M_dev;
      n_tok = (M + NT - 1) / NT;
      num_tiles = num_mp * n_tok;
    }
    for (int t = cluster; t < num_tiles; t += n_clusters) {
      const int n_blk = t % n_tok, m_pair = t / n_tok;    // token tiles of one weight tile run together
      const int xrow = n_blk * NT + (int)rank * (NT / 2);
      for (int kb = 0; kb < nk; ++kb) {
        tc::mbar_wait(&empty[stage], phase ^ 1);
        const bool skip = (g.diag & 1) && (kb >= STAGES || t != cluster);   // diagnostic: stale smem
        const bool pre = t == cluster && kb < npre;       // weights already in flight
        if (tc::elect_one()) {
          if (skip) {
            if (leader) tc::mbar_arrive(&full[stage]);
          } else {
            if (!pre) {
              if (leader) tc::mbar_arrive_expect_tx(&full[stage], tx);
              load_w(stage, m_pair, kb);
            }
            const uint32_t fb = tc::smem_u32(&full[stage]) & tc::kPeerBitMask;
            tc::tma_load_2d_2sm(sB + stage * BX_BYTES, &map_x, fb, kb * BK, xrow, pol_x);
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (leader CTA): M = 256 weight rows, N = NT tokens
      const uint32_t idesc = tc::idesc_bf16(256, NT);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < num_tiles; t += n_clusters) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::fence_after();
        if (lane == 0) SW_TR(g, 12, (t - cluster) / n_clusters);
        const uint32_t d = tmem_base + acc * 256;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint64_t da = tc::sdesc_sw128(tc::smem_u32(sA + stage * A_BYTES), 16, 1024);
          const uint64_t db = tc::sdesc_sw128(tc::smem_u32(sB + stage * BX_BYTES), 16, 1024);
          if (tc::elect_one()) {
            if (g.diag & 4) {                               // diagnostic: A from (garbage) TMEM columns
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                tc::umma_bf16_ts_2sm(d, tmem_base + 448 + kk * 8, db + 2 * kk, idesc, (kb | kk) != 0);
            } else {
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                tc::umma_bf16_2sm(d, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
            }
            tc::umma_commit_2sm(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (tc::elect_one()) tc::umma_commit_2sm(&tfull[acc], 0x3);
        __syncwarp();
        if (lane == 0) SW_TR(g, 13, (t - cluster) / n_clusters);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue warps of both CTAs (TMEM lane = weight row)
    const int q = warp & 3, h = (warp - 4) >> 2;         // warps 4-7: even chunks, 8-11: odd chunks
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cluster; t < num_tiles; t += n_clusters) {
      const SwTile tl{t / n_tok, t % n_tok};
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      if (warp == 4 && lane == 0) SW_TR(g, 14, (t - cluster) / n_clusters);
      const SwEpi e{&g, (int)rank, q, h, lane, h * 128 + q * 32 + lane, aux, pos_s, tmem_base + (uint32_t(q * 32) << 16) + acc * 256, NT, M};
      switch ((g.diag & 2) ? -1 : g.kind) {
        case -1: break;                                   // diagnostic: no epilogue
        case GEMM_EPI_LOGITS:
          if (g.argmax_only && !g.out) sw_epi_argmax(e, tl);
          else sw_epi_logits(e, tl);
          break;
        case GEMM_EPI_QKV_ROPE: sw_epi_qkv(e, tl); break;
        case GEMM_EPI_SWIGLU: sw_epi_swiglu(e, tl); break;
        default: sw_epi_f32(e, tl); break;
      }
      if (warp == 4 && lane == 0) SW_TR(g, 15, (t - cluster) / n_clusters);
      tc::fence_before();
      if (leader) tc::mbar_arrive(&tempty[acc]);
      else tc::mbar_arrive_cta0(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (g.trace && threadIdx.x == 0 && blockIdx.x < 512) g.trace[11 * 256 + blockIdx.x / 2 + (rank ? 128 : 0)] = sw_gtimer();
  tc::cluster_sync_all();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc_2sm(tmem_base, 512);
  }
}

// Token tile width: the N = 16k <= 256 that splits T into equal tiles with the fewest
// pair-waves x (width + a fixed per-tile cost); T = 576 -> 192 (3 tiles) for 24+ weight tiles.
static int sw_nt_cost(int T, int nt, int num_mp, int n_pairs) {
  const int tiles = num_mp * ((T + nt - 1) / nt);
  const int waves = (tiles + n_pairs - 1) / n_pairs;
  return waves * (nt + 48);
}

// T2 > 0 (dynamic-depth graphs: the rows vary per replay around the capture's T, up to the bound T2):
// the width minimising 2 cost(T) + cost(T2)
int gemm_sw_choose_nt(int T, int num_mp, int n_pairs, int T2) {
  int best = 256, best_cost = 0x7fffffff;
  for (int k = 1; k <= 64; ++k) {
    int nt = (T + k - 1) / k;
    nt = (nt + 15) / 16 * 16;
    if (nt > 256) continue;
    if (nt < 16) nt = 16;
    const int cost = (T2 > 0 ? 2 : 1) * sw_nt_cost(T, nt, num_mp, n_pairs) + (T2 > 0 ? sw_nt_cost(T2, nt, num_mp, n_pairs) : 0);
    if (cost < best_cost) {
      best_cost = cost;
      best = nt;
    }
    if (nt == 16) break;
  }
  if (T2 > 0) {                                           // the widths chosen for T2 alone are candidates too
    for (int k = 1; k <= 64; ++k) {
      int nt = ((T2 + k - 1) / k + 15) / 16 * 16;
      if (nt > 256) continue;
      if (nt < 16) nt = 16;
      const int cost = 2 * sw_nt_cost(T, nt, num_mp, n_pairs) + sw_nt_cost(T2, nt, num_mp, n_pairs);
      if (cost < best_cost) {
        best_cost = cost;
        best = nt;
      }
      if (nt == 16) break;
    }
  }
  return best;
}

int gemm_sw_smem_bytes() { return SMEM_BYTES; }

cudaError_t launch_gemm_sw(const CUtensorMap& map_w, const CUtensorMap& map_x, const GemmTcArgs& g, int num_sms,
                           cudaStream_t s) {
  {
    const cudaError_t e = smem_optin((const void*)gemm_sw_kernel, (int)(SMEM_BYTES));
    if (e != cudaSuccess) return e;
  }
  if (g.M <= 0) return cudaSuccess;
  const int num_mp = g.kind == GEMM_EPI_SWIGLU ? g.F / 128 : (g.N + 255) / 256;
  const int num_tiles = num_mp * ((g.M + g.nt_tok - 1) / g.nt_tok);
  const int clusters = num_tiles < num_sms / 2 ? num_tiles : num_sms / 2;
  SV_COUNT_LAUNCH();
  return launch_pdl(gemm_sw_kernel, dim3(2 * clusters), dim3(THREADS), SMEM_BYTES, s, 2, map_w, map_x, g);
}

}  // namespace sv
