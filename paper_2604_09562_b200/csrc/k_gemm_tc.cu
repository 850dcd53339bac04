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
//
// Stream-K (g.streamk): when the output has too few tiles to fill the SMs (the N = 4096 / 6144
// projections at a few hundred rows), CTA c takes the global K-block range [c W, (c+1) W) of
// the tile-major K-block sequence. Whole tiles are finished in place; a tile split across CTAs
// is written as fp32 partials (one head / tail slot per CTA), and the CTA that completes the
// tile's last piece (atomic counter) sums the pieces in CTA order — a fixed order, so results
// are deterministic — and runs the epilogue.
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
constexpr int STG_BYTES = 4 * 4096;              // epilogue staging, 4 KB per epilogue warp
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + STG_BYTES;
constexpr int EPI_BAR = 1;                       // named barrier of the 4 epilogue warps
}  // namespace

struct TileCoord {
  int m_blk, n_blk;
};

__device__ __forceinline__ TileCoord tile_of(int t, int num_m) { return TileCoord{t % num_m, t / num_m}; }

__device__ __forceinline__ float u2f(uint32_t v) { return __uint_as_float(v); }

// ------------------------------------------------------------------ work pieces
// A piece = K blocks [kb0, kb1) of output tile `tile`. Without stream-K every piece is a
// whole tile (tiles blockIdx.x, blockIdx.x + grid, ...).
struct Piece {
  int tile, kb0, kb1;
};

struct PieceIter {
  int nk, num_tiles, grid, c, W;
  bool streamk;
  long long pos, end;   // stream-K: global K-block cursor; else: tile cursor
  __device__ PieceIter(const GemmTcArgs& g, int num_tiles_, int nk_)
      : nk(nk_), num_tiles(num_tiles_), grid(gridDim.x), c(blockIdx.x), W(g.sk_w), streamk(g.streamk != 0) {
    if (streamk) {
      pos = (long long)c * W;
      end = min((long long)(c + 1) * W, (long long)num_tiles * nk);
    } else {
      pos = c;
      end = num_tiles;
    }
  }
  __device__ bool next(Piece& p) {
    if (pos >= end) return false;
    if (!streamk) {
      p = Piece{(int)pos, 0, nk};
      pos += grid;
      return true;
    }
    const int tile = (int)(pos / nk), kb0 = (int)(pos % nk);
    const int kb1 = (int)min((long long)nk, kb0 + (end - pos));
    p = Piece{tile, kb0, kb1};
    pos += kb1 - kb0;
    return true;
  }
};

// ------------------------------------------------------------------ accumulator sources
// The epilogues read the accumulator tile in 32-column chunks through a Source: TMEM
// (tcgen05.ld, warp-collective) or, for a stream-K tile, the ordered sum of its fp32 partials.
struct TmemSrc {
  uint32_t tbase;
  __device__ __forceinline__ void get(int col, uint32_t (&r)[32]) const {
    __syncwarp();
    tc::tmem_ld32(tbase + col, r);
    tc::tmem_ld_wait();
  }
};

// partial slot layout: [slot][BN / 4][BM] float4 (column-chunk major: a warp's 32 rows
// touch 32 consecutive float4 -> coalesced)
__device__ __forceinline__ float4* partial_slot(const GemmTcArgs& g, int cta, int slot) {
  return reinterpret_cast<float4*>(g.partials) + (size_t)(cta * 2 + slot) * (BN / 4) * BM;
}

struct PartialSrc {
  const GemmTcArgs* g;
  int rl, c_lo, n, tile, nk;
  __device__ __forceinline__ void get(int col, uint32_t (&r)[32]) const {
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    for (int i = 0; i < n; ++i) {                 // CTA order = K order: deterministic
      const int cta = c_lo + i;
      const int slot = ((long long)cta * g->sk_w < (long long)tile * nk) ? 1 : 0;
      const float4* p = partial_slot(*g, cta, slot) + (size_t)(col / 4) * BM + rl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = __ldcg(p + (size_t)j * BM);
        acc[4 * j] += v.x;
        acc[4 * j + 1] += v.y;
        acc[4 * j + 2] += v.z;
        acc[4 * j + 3] += v.w;
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(acc[i]);
  }
};

// ------------------------------------------------------------------ coalesced stores
// An epilogue thread holds 32 consecutive values of ITS row (TMEM lane = row). Stored
// directly, every warp instruction would touch 32 rows = 32 partial sectors. Instead the warp
// transposes its 32 x 32 block through a 4 KB staging buffer (16-byte chunks XOR-swizzled by
// row, so both phases are bank-conflict free) and writes whole row segments: 8 lanes x 16 B
// per fp32 row (4 rows per instruction), 4 lanes x 16 B per bf16 row (8 rows per instruction).
struct Stage32 {
  uint4* s;     // this warp's staging buffer (256 x 16 B)
  int lane;
  int row0;     // global row of lane 0
};

__device__ __forceinline__ void stage_put_f32(const Stage32& st, const uint32_t (&r)[32]) {
  uint4* p = st.s + st.lane * 8;
#pragma unroll
  for (int j = 0; j < 8; ++j) p[j ^ (st.lane & 7)] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
  __syncwarp();
}

// out[row][n + i] = staged (+ in[row][n + i] when in != nullptr) for rows < M, columns < N.
// in may alias out (each element is read and written by the same lane).
__device__ __forceinline__ void stage_write_f32(const Stage32& st, float* out, const float* in, size_t ld, int M,
                                                int n, int N) {
  const int rs = st.lane >> 3, ch = st.lane & 7;
  const int col = n + ch * 4;
  const bool vec = col + 4 <= N && (ld & 3) == 0;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int r = it * 4 + rs, row = st.row0 + r;
    const uint4 u = st.s[r * 8 + (ch ^ (r & 7))];
    float v[4] = {u2f(u.x), u2f(u.y), u2f(u.z), u2f(u.w)};
    if (row < M) {
      const size_t o = (size_t)row * ld + col;
      if (vec) {
        if (in) {
          const float4 h = *reinterpret_cast<const float4*>(in + o);
          v[0] += h.x;
          v[1] += h.y;
          v[2] += h.z;
          v[3] += h.w;
        }
        *reinterpret_cast<float4*>(out + o) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
        for (int i = 0; i < 4 && col + i < N; ++i) out[o + i] = in ? in[o + i] + v[i] : v[i];
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void stage_put_bf16(const Stage32& st, const __nv_bfloat16 (&o)[32]) {
  uint4* p = st.s + st.lane * 4;
  const int f = (st.lane >> 1) & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j ^ f] = *reinterpret_cast<const uint4*>(&o[8 * j]);
  __syncwarp();
}

// out0 = address of (row0, first column); rows r < rows_valid get their 32 staged values
__device__ __forceinline__ void stage_write_bf16(const Stage32& st, __nv_bfloat16* out0, size_t ld, int rows_valid) {
  const int rs = st.lane >> 2, ch = st.lane & 3;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + rs;
    const uint4 v = st.s[r * 4 + (ch ^ ((r >> 1) & 3))];
    if (r < rows_valid) *reinterpret_cast<uint4*>(out0 + (size_t)r * ld + ch * 8) = v;
  }
  __syncwarp();
}

// ------------------------------------------------------------------ epilogues
// Each epilogue thread owns one accumulator row (TMEM lane) and walks its 256 columns
// in 8 chunks of 32; all lanes of the warp take part in every chunk (warp-collective
// tcgen05.ld and staging), rows >= M are masked at the global store.
template <class Src>
__device__ __forceinline__ void epi_store_f32(const GemmTcArgs& g, const Stage32& st, int n0, const Src& src) {
  uint32_t r[32];
  const bool resid = g.kind == GEMM_EPI_RESIDUAL;
  for (int c = 0; c < BN / 32; ++c) {
    src.get(c * 32, r);
    stage_put_f32(st, r);
    stage_write_f32(st, resid ? g.resid_out : g.out, resid ? g.resid_in : nullptr, g.ldo, g.M, n0 + c * 32, g.N);
  }
}

// a5: fp32 logits + per-(row, 128-col vocab tile) max / sum exp / lowest argmax of l * inv_temp
template <class Src>
__device__ __forceinline__ void epi_logits(const GemmTcArgs& g, const Stage32& st, int n0, int n_blk,
                                           const Src& src) {
  const int row = st.row0 + st.lane;
  uint32_t r[32];
  float m = -INFINITY, s = 0.f;
  int am = 0x7fffffff;
  for (int c = 0; c < BN / 32; ++c) {
    src.get(c * 32, r);
    const int n = n0 + c * 32;
    stage_put_f32(st, r);
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
    if (g.out) stage_write_f32(st, g.out, nullptr, g.ldo, g.M, n, g.N);
    if ((c & 3) == 3) {                            // statistics per 128-column vocab tile
      const int tile = n_blk * 2 + (c >> 2);
      if (row < g.M && tile < g.nt) {
        const size_t o = (size_t)row * g.nt + tile;
        g.tmax[o] = m;
        g.tsum[o] = s;
        g.targ[o] = am;
      }
      m = -INFINITY;
      s = 0.f;
      am = 0x7fffffff;
    }
  }
}

// a2: q/k RoPE (rotate_half, fp32 table) + bf16 store to Q / chain K; v plain bf16 store
template <class Src>
__device__ __forceinline__ void epi_qkv(const GemmTcArgs& g, const Stage32& st, int n0, const Src& src) {
  const int row = st.row0 + st.lane;
  const int dh = g.dh, half = dh / 2;
  const int heads_per_tile = BN / dh;
  const int nkv = g.Hkv * dh;
  const int pos = row < g.M ? g.row_pos[row] : 0;
  const int rows_valid = g.M - st.row0;
  uint32_t x1[32], x2[32];
  for (int hh = 0; hh < heads_per_tile; ++hh) {
    const int head = n0 / dh + hh;
    const int cbase = hh * dh;                       // column of this head inside the tile
    for (int c = 0; c < half / 32; ++c) {
      src.get(cbase + c * 32, x1);
      src.get(cbase + half + c * 32, x2);
      if (head >= g.Hq + 2 * g.Hkv) continue;        // warp-uniform
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
      size_t ld;
      if (head < g.Hq) {
        dst = g.q + (size_t)st.row0 * g.Hq * dh + (size_t)head * dh;
        ld = (size_t)g.Hq * dh;
      } else if (head < g.Hq + g.Hkv) {
        dst = g.kc + (size_t)st.row0 * nkv + (size_t)(head - g.Hq) * dh;
        ld = nkv;
      } else {
        dst = g.vc + (size_t)st.row0 * nkv + (size_t)(head - g.Hq - g.Hkv) * dh;
        ld = nkv;
      }
      stage_put_bf16(st, o1);
      stage_write_bf16(st, dst + c * 32, ld, rows_valid);
      stage_put_bf16(st, o2);
      stage_write_bf16(st, dst + half + c * 32, ld, rows_valid);
    }
  }
}

// a4: u = bf16(silu(gate) * up); tile columns 0..127 are gate rows, 128..255 the matching up rows
template <class Src>
__device__ __forceinline__ void epi_swiglu(const GemmTcArgs& g, const Stage32& st, int n_blk, const Src& src) {
  uint32_t gt[32], up[32];
  for (int c = 0; c < 4; ++c) {
    src.get(c * 32, gt);
    src.get(128 + c * 32, up);
    __nv_bfloat16 o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float x = u2f(gt[i]);
      o[i] = f2bf(x / (1.0f + expf(-x)) * u2f(up[i]));
    }
    stage_put_bf16(st, o);
    stage_write_bf16(st, g.u + (size_t)st.row0 * g.F + n_blk * 128 + c * 32, g.F, g.M - st.row0);
  }
}

template <class Src>
__device__ __forceinline__ void run_epilogue(const GemmTcArgs& g, const TileCoord& tcd, const Stage32& st,
                                             const Src& src) {
  switch (g.kind) {
    case GEMM_EPI_LOGITS: epi_logits(g, st, tcd.n_blk * BN, tcd.n_blk, src); break;
    case GEMM_EPI_QKV_ROPE: epi_qkv(g, st, tcd.n_blk * BN, src); break;
    case GEMM_EPI_SWIGLU: epi_swiglu(g, st, tcd.n_blk, src); break;
    default: epi_store_f32(g, st, tcd.n_blk * BN, src); break;
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
  int* sk_flag = reinterpret_cast<int*>(tmem_holder + 1);

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
      // weights: evict-first only when no other M tile will re-read this B tile
      const uint64_t pol_b = num_m > 1 ? tc::policy_evict_last() : tc::policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      PieceIter pi(g, num_tiles, nk);
      Piece p;
      while (pi.next(p)) {
        const TileCoord tcd = tile_of(p.tile, num_m);
        const int arow = tcd.m_blk * BM;
        int brow0, brow1;
        if (g.kind == GEMM_EPI_SWIGLU) {
          brow0 = tcd.n_blk * 128;
          brow1 = g.F + tcd.n_blk * 128;
        } else {
          brow0 = tcd.n_blk * BN;
          brow1 = brow0 + 128;
        }
        for (int kb = p.kb0; kb < p.kb1; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          if (g.diag == 1 && (kb >= STAGES || p.tile != blockIdx.x)) {  // diagnostic: MMA on stale smem
            tc::mbar_arrive(&full[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
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
      PieceIter pi(g, num_tiles, nk);
      Piece p;
      while (pi.next(p)) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = p.kb0; kb < p.kb1; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint64_t da = tc::sdesc_sw128(tc::smem_u32(sA + stage * A_BYTES), 16, 1024);
          const uint64_t db = tc::sdesc_sw128(tc::smem_u32(sB + stage * B_BYTES), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)       // +32 B per K=16 step inside the 128-B swizzle atom
            tc::umma_bf16(d, da + 2 * kk, db + 2 * kk, IDESC, (kb > p.kb0) || (kk > 0));
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
    const int rl = q * 32 + lane;                   // row inside the tile
    uint4* stg = reinterpret_cast<uint4*>(smem + STAGES * STAGE_BYTES + 256) + q * 256;
    int acc = 0;
    uint32_t acc_phase = 0;
    PieceIter pi(g, num_tiles, nk);
    Piece p;
    while (pi.next(p)) {
      const TileCoord tcd = tile_of(p.tile, num_m);
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const TmemSrc tsrc{tmem_base + (uint32_t(q * 32) << 16) + acc * BN};
      const Stage32 st{stg, lane, tcd.m_blk * BM + q * 32};
      if (p.kb0 == 0 && p.kb1 == nk) {
        run_epilogue(g, tcd, st, tsrc);
        tc::fence_before();
        tc::mbar_arrive(&tempty[acc]);
      } else {
        // stream-K piece: spill the partial tile, then whoever completes the tile reduces it
        const int c = blockIdx.x;
        const int slot = ((long long)c * g.sk_w < (long long)p.tile * nk) ? 1 : 0;
        float4* dst = partial_slot(g, c, slot) + rl;
        uint32_t r[32];
        for (int cc = 0; cc < BN / 32; ++cc) {
          tsrc.get(cc * 32, r);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(dst + (size_t)(cc * 8 + j) * BM,
                   make_float4(u2f(r[4 * j]), u2f(r[4 * j + 1]), u2f(r[4 * j + 2]), u2f(r[4 * j + 3])));
        }
        tc::fence_before();
        tc::mbar_arrive(&tempty[acc]);                // accumulator consumed
        __threadfence();
        tc::named_bar(EPI_BAR, 128);
        const long long t0 = (long long)p.tile * nk, t1 = t0 + nk;
        const int c_lo = (int)(t0 / g.sk_w), c_hi = (int)((t1 - 1) / g.sk_w);
        const int n = c_hi - c_lo + 1;
        if (threadIdx.x == 128) {
          const int old = atomicAdd(&g.sk_counters[p.tile], 1);
          *sk_flag = old == n - 1;
          if (old == n - 1) g.sk_counters[p.tile] = 0;   // ready for the next launch
        }
        tc::named_bar(EPI_BAR, 128);
        if (*sk_flag) {
          __threadfence();
          const PartialSrc psrc{&g, rl, c_lo, n, p.tile, nk};
          run_epilogue(g, tcd, st, psrc);
        }
        tc::named_bar(EPI_BAR, 128);                  // sk_flag reused by the next piece
      }
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

size_t gemm_tc_partial_bytes(int num_sms) { return (size_t)num_sms * 2 * BM * BN * sizeof(float); }

cudaError_t launch_gemm_tc(const CUtensorMap& map_a, const CUtensorMap& map_b, const GemmTcArgs& g_in, int num_sms,
                           cudaStream_t s) {
  {
    const cudaError_t e = smem_optin((const void*)gemm_tc_kernel, (int)(SMEM_BYTES));
    if (e != cudaSuccess) return e;
  }
  if (g_in.M <= 0) return cudaSuccess;
  GemmTcArgs g = g_in;
  const int num_tiles = ((g.M + BM - 1) / BM) * g.n_tiles;
  const int nk = g.K / BK;
  int grid = num_tiles < num_sms ? num_tiles : num_sms;
  g.streamk = 0;
  if (g.partials && g.sk_counters && g.kind != GEMM_EPI_LOGITS && g.kind != GEMM_EPI_SWIGLU) {
    // stream-K when the whole-tile schedule leaves enough of the machine idle
    const long long total = (long long)num_tiles * nk;
    const long long W = (total + num_sms - 1) / num_sms;
    const long long waves_tiles = (long long)((num_tiles + num_sms - 1) / num_sms) * nk;
    if (W * 115 < waves_tiles * 100 && W >= 8) {
      g.streamk = 1;
      g.sk_w = (int)W;
      grid = (int)((total + W - 1) / W);
    }
  }
  SV_COUNT_LAUNCH();
  gemm_tc_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(map_a, map_b, g);
  return cudaGetLastError();
}

// =====================================================================================
// 2-SM variant (cta_group::2): a cluster of two CTAs computes a 256 x 256 output tile with
// one tcgen05.mma.cta_group::2 stream issued by the leader CTA. Each CTA stages its own 128
// A rows and half of the B tile (128 N rows) per K block (32 KB per stage instead of 48 KB),
// so a 6-stage ring fits and each SM needs a third fewer bytes per MMA cycle; both CTAs
// keep their 128 x 256 half of the accumulator in their own TMEM (double-buffered) and run
// the same fused epilogues on their rows.
// =====================================================================================
namespace {
constexpr int PAIR_M = 256;
constexpr int B2_BYTES = 128 * BK * 2;              // 16 KB: this CTA's half of the B tile
constexpr int STAGE2_BYTES = A_BYTES + B2_BYTES;    // 32 KB
constexpr int STAGES2 = 6;
constexpr uint32_t IDESC2 = tc::idesc_bf16(PAIR_M, BN);
constexpr int SMEM2_BYTES = STAGES2 * STAGE2_BYTES + 1024 + 256 + STG_BYTES;
}  // namespace

__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    const GemmTcArgs g) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_s & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  const int num_pm = (g.M + PAIR_M - 1) / PAIR_M;
  const int num_tiles = num_pm * g.n_tiles;
  const int nk = g.K / BK;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&map_a);
    tc::prefetch_tmap(&map_b);
    for (int i = 0; i < STAGES2; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 256);                 // both CTAs' epilogue threads (leader's copy used)
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs; bytes land on the leader's full barrier)
      const uint64_t pol_b = num_pm > 1 ? tc::policy_evict_last() : tc::policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < num_tiles; t += n_clusters) {
        const int m_pair = t % num_pm, n_blk = t / num_pm;
        const int arow = m_pair * PAIR_M + (int)rank * 128;
        const int brow = g.kind == GEMM_EPI_SWIGLU ? (rank ? g.F : 0) + n_blk * 128 : n_blk * BN + (int)rank * 128;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * STAGE2_BYTES);
          const uint32_t fb = tc::smem_u32(&full[stage]) & tc::kPeerBitMask;
          tc::tma_load_2d_2sm(sA + stage * A_BYTES, &map_a, fb, kb * BK, arow, tc::policy_evict_last());
          tc::tma_load_2d_2sm(sB + stage * B2_BYTES, &map_b, fb, kb * BK, brow, pol_b);
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader CTA, one thread, cta_group::2)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < num_tiles; t += n_clusters) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint64_t da = tc::sdesc_sw128(tc::smem_u32(sA + stage * A_BYTES), 16, 1024);
          const uint64_t db = tc::sdesc_sw128(tc::smem_u32(sB + stage * B2_BYTES), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            tc::umma_bf16_2sm(d, da + 2 * kk, db + 2 * kk, IDESC2, (kb | kk) != 0);
          tc::umma_commit_2sm(&empty[stage], 0x3);
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
        tc::umma_commit_2sm(&tfull[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue warps of both CTAs (own 128 rows of the pair tile)
    const int q = warp & 3;
    uint4* stg = reinterpret_cast<uint4*>(smem + STAGES2 * STAGE2_BYTES + 256) + q * 256;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cluster; t < num_tiles; t += n_clusters) {
      const int m_pair = t % num_pm, n_blk = t / num_pm;
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const TmemSrc tsrc{tmem_base + (uint32_t(q * 32) << 16) + acc * BN};
      const Stage32 st{stg, lane, m_pair * PAIR_M + (int)rank * 128 + q * 32};
      run_epilogue(g, TileCoord{0, n_blk}, st, tsrc);
      tc::fence_before();
      if (leader) tc::mbar_arrive(&tempty[acc]);
      else tc::mbar_arrive_cta0(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();
  if (warp == 2) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

cudaError_t launch_gemm_tc2(const CUtensorMap& map_a, const CUtensorMap& map_b, const GemmTcArgs& g, int num_sms,
                            cudaStream_t s) {
  {
    const cudaError_t e = smem_optin((const void*)gemm_tc2_kernel, (int)(SMEM2_BYTES));
    if (e != cudaSuccess) return e;
  }
  if (g.M <= 0) return cudaSuccess;
  const int num_tiles = ((g.M + PAIR_M - 1) / PAIR_M) * g.n_tiles;
  const int clusters = num_tiles < num_sms / 2 ? num_tiles : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM2_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  SV_COUNT_LAUNCH();
  return cudaLaunchKernelEx(&cfg, gemm_tc2_kernel, map_a, map_b, g);
}

}  // namespace sv
