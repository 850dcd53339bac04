// a3: paged, GQA, chain-causal verify attention on the 5th-generation tensor cores.
//
// One work item = (request b, kv head h, split s) of the device work list built by the
// plan kernel (lane.h: num_splits / split_t1). Its queries are the chain rows j = 0..k of
// the G q heads of kv head h; its keys the split's KV pages (64 keys each, streamed by
// TMA) and, for the last split, the chain keys of this verify (scratch kc/vc, loaded by
// the producer warp). Per 64-key tile:
//   S  = Q K^T                tcgen05.mma M=128 N=64 K=d_h, A = Q (smem), B = K (smem)
//   P  = 2^(S*scale*log2e - m) softmax threads, online max with lazy rescale (only when the
//                             row max grows by > 2^8), P -> bf16 -> TMEM (over S)
//   O += P V                  tcgen05.mma M=128 N=d_h K=64, A = P (TMEM), B = V (smem, MN-major)
// The item's unnormalised O, max and sum go to the split-KV partials merged by
// attn_combine_kernel (same format as the SIMT kernel).
//
// Query-row placement: TMEM lane (= MMA row) 32*g + j holds (q head h*G + g, chain row j),
// so the G heads of a group occupy G different 32-lane quadrants and every quadrant is
// served by two softmax warps, each owning half of the tile's 64 key columns (the two
// halves exchange their row max through shared memory once per tile).
//
// Warp roles (persistent grid, one CTA per SM, 12 warps):
//   warp 0  producer: Q (3-D TMA over q, one box per head), K/V pages (2-D TMA over the
//           pool), chain tile (cooperative ld.global -> swizzled st.shared)
//   warp 1  MMA issuer (one thread)      warp 2  TMEM allocator      warp 3  idle
//   warps 4-11 softmax + item epilogue: warp w serves quadrant w % 4, key half (w - 4) / 4
// Smem: Q double buffer 2 x 128 rows x d_h + 4-stage K/V ring (4 x 2 x 64 x d_h) = 192 KB (d_h 128).
// TMEM: S/P double buffer 2 x 64 columns, O double buffer 2 x d_h columns.
#include <cuda.h>

#include "attn_tc.h"
#include "common.cuh"
#include "lane.h"
#include "tc.cuh"

namespace sv {

// debug timeline of CTA 0 (LaneDev::trace, enabled by SV_TRACE=1): event e, tile / item i
#define SV_TR(e, i)                                                          \
  do {                                                                       \
    if (d.trace && blockIdx.x == 0 && (i) < 256) d.trace[(e)*256 + (i)] = clock64(); \
  } while (0)

namespace {
constexpr int KT = 64;                     // keys per tile (= page size)
constexpr int ST = 4;                      // K/V ring stages
constexpr int THREADS = 384;
constexpr int SOFTMAX_THREADS = 256;
constexpr float kRescaleLog2 = 8.0f;       // rescale O only when the running max grows by > 2^8
}  // namespace

template <int DH>
struct AttnCfg {
  static constexpr int HALVES = DH / 64;                 // 64-element (128-B) swizzle atoms along d_h
  static constexpr int Q_BYTES = 128 * DH * 2;           // 128 MMA rows x d_h
  static constexpr int KV_BYTES = KT * DH * 2;           // one K or V tile
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int SMEM = 2 * Q_BYTES + ST * STAGE_BYTES + 1024 + 8192;
  static constexpr uint32_t IDESC_QK = tc::idesc_bf16(128, KT);          // A, B K-major
  static constexpr uint32_t IDESC_PV = tc::idesc_bf16(128, DH, 0, 1);    // B (V) MN-major
  static constexpr int S_COL = 0;                        // S/P buffers at columns 0, 64
  static constexpr int O_COL = 128;                      // O buffers at 128, 128 + DH
};

struct ItemInfo {
  int b, h, s, ns, slot, L, R, row0, t0, t1, n_page_tiles, n_tiles, page0;
};

__device__ __forceinline__ ItemInfo item_info(const LaneDev& d, int it) {
  const int4 w = d.items[it];
  ItemInfo I;
  I.b = w.x;
  I.h = w.y;
  I.s = w.z;
  I.ns = item_ns(w.w);
  const int sk = item_split_keys(w.w);
  I.slot = d.slots[I.b];
  I.L = d.len[I.slot];
  I.R = d.depths[I.b] + 1;
  I.row0 = d.row_off[I.b];
  I.t0 = I.s * sk;
  I.t1 = split_t1_k(I.s, I.ns, I.L, I.R, sk);
  const int page_end = min(I.t1, I.L);
  I.n_page_tiles = page_end > I.t0 ? (page_end - I.t0 + KT - 1) / KT : 0;
  I.n_tiles = I.n_page_tiles + (I.s == I.ns - 1 ? 1 : 0);
  I.page0 = I.t0 / KT;
  return I;
}

template <int DH>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                   const LaneDev d, const int layer, const int q_box_tokens) {
  using C = AttnCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_s & 1023)) & 1023);
  uint8_t* sQ = smem;                                   // [2][HALVES][128 rows][128 B]
  uint8_t* sKV = smem + 2 * C::Q_BYTES;                 // [ST][K: HALVES][64][128 B | V: HALVES][64][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + ST * C::STAGE_BYTES);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = kv_full + ST;
  uint64_t* q_full = kv_empty + ST;
  uint64_t* q_empty = q_full + 2;
  uint64_t* s_full = q_empty + 2;
  uint64_t* p_full = s_full + 2;
  uint64_t* s_free = p_full + 2;
  uint64_t* o_full = s_free + 2;
  uint64_t* o_empty = o_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_empty + 2);
  float* xmax = reinterpret_cast<float*>(bars + 64);    // [2 tile parity][2 halves][128 lanes]
  float* xl = xmax + 2 * 2 * 128;                       // [2][128] item sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = *d.n_items;
  const int G = d.Hq / d.Hkv;
  const size_t nkv = (size_t)d.Hkv * DH;

  for (int i = threadIdx.x; i < 2 * C::Q_BYTES / 16; i += THREADS)
    reinterpret_cast<uint4*>(sQ)[i] = make_uint4(0, 0, 0, 0);   // quadrants >= G stay zero
  tc::fence_proxy_async();
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&map_q);
    tc::prefetch_tmap(&map_kv);
    for (int i = 0; i < ST; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 1);
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], SOFTMAX_THREADS);
      tc::mbar_init(&s_free[i], 1);
      tc::mbar_init(&o_full[i], 1);
      tc::mbar_init(&o_empty[i], SOFTMAX_THREADS);
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
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ======================= producer (all 32 lanes; lane 0 issues TMA / barrier ops)
    const uint64_t pol = tc::policy_evict_first();
    const uint32_t q_tx = G * C::HALVES * q_box_tokens * 128;
    int stage = 0;
    uint32_t phase = 0;
    int iter = 0;
    uint32_t ptile = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      const ItemInfo I = item_info(d, it);
      const int qb = iter & 1;
      if (lane == 0) {
        tc::mbar_wait(&q_empty[qb], ((iter >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qb], q_tx);
        for (int g = 0; g < G; ++g)
          for (int hf = 0; hf < C::HALVES; ++hf)
            tc::tma_load_3d(sQ + qb * C::Q_BYTES + hf * (128 * 128) + g * (32 * 128), &map_q, &q_full[qb], hf * 64,
                            I.h * G + g, I.row0);
      }
      for (int t = 0; t < I.n_tiles; ++t) {
        if (lane == 0) tc::mbar_wait(&kv_empty[stage], phase ^ 1);
        if (lane == 0) SV_TR(0, ptile);
        __syncwarp();
        uint8_t* sk = sKV + stage * C::STAGE_BYTES;
        uint8_t* sv_ = sk + C::KV_BYTES;
        if (t < I.n_page_tiles) {
          if (lane == 0) {
            const int page = d.page_table[I.slot * d.max_pages_per_slot + I.page0 + t];
            const int rk = ((((layer * d.n_pages + page) * 2 + 0) * d.Hkv) + I.h) * KT;
            const int rv = ((((layer * d.n_pages + page) * 2 + 1) * d.Hkv) + I.h) * KT;
            tc::mbar_arrive_expect_tx(&kv_full[stage], C::STAGE_BYTES);
            for (int hf = 0; hf < C::HALVES; ++hf) {
              tc::tma_load_2d_hint(sk + hf * (KT * 128), &map_kv, &kv_full[stage], hf * 64, rk, pol);
              tc::tma_load_2d_hint(sv_ + hf * (KT * 128), &map_kv, &kv_full[stage], hf * 64, rv, pol);
            }
            SV_TR(1, ptile);
          }
        } else {
          // chain tile: keys L + c, c < R, from the chain scratch; zero rows beyond R
          const bf16* kc = d.kc + (size_t)layer * d.Tmax * nkv;
          const bf16* vc = d.vc + (size_t)layer * d.Tmax * nkv;
          constexpr int CH = DH / 8;                       // 16-B chunks per row
          for (int i = lane; i < KT * CH; i += 32) {
            const int c = i / CH, ch = i % CH;
            uint4 kvk = make_uint4(0, 0, 0, 0), kvv = make_uint4(0, 0, 0, 0);
            if (c < I.R) {
              const size_t off = (size_t)(I.row0 + c) * nkv + (size_t)I.h * DH + ch * 8;
              kvk = *reinterpret_cast<const uint4*>(kc + off);
              kvv = *reinterpret_cast<const uint4*>(vc + off);
            }
            const int hf = ch / 8, cc = ch % 8;
            const int boff = hf * (KT * 128) + c * 128 + ((cc ^ (c & 7)) * 16);
            *reinterpret_cast<uint4*>(sk + boff) = kvk;
            *reinterpret_cast<uint4*>(sv_ + boff) = kvv;
          }
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&kv_full[stage]);
          if (lane == 0) SV_TR(1, ptile);
        }
        if (++stage == ST) { stage = 0; phase ^= 1; }
        ++ptile;
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t g = 0;                      // global tile counter (S/P buffer = g & 1)
      int iter = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
        const ItemInfo I = item_info(d, it);
        const int qb = iter & 1, ob = iter & 1;
        tc::mbar_wait(&q_full[qb], (iter >> 1) & 1);
        tc::mbar_wait(&o_empty[ob], ((iter >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t sq = tc::smem_u32(sQ + qb * C::Q_BYTES);
        const uint32_t o_tm = tmem + C::O_COL + ob * DH;
        int prev_stage = -1;
        uint32_t prev_g = 0;
        for (int t = 0; t <= I.n_tiles; ++t) {
          if (t < I.n_tiles) {
            // ---- S(t) = Q K^T into S[g & 1]
            const int sb = g & 1;
            tc::mbar_wait(&kv_full[stage], phase);
            SV_TR(2, g);
            tc::mbar_wait(&s_free[sb], ((g >> 1) & 1) ^ 1);
            SV_TR(3, g);
            tc::fence_after();
            const uint32_t sk = tc::smem_u32(sKV + stage * C::STAGE_BYTES);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint32_t koff = (kk % 4) * 32;
              const uint64_t da = tc::sdesc_sw128(sq + (kk / 4) * (128 * 128) + koff, 16, 1024);
              const uint64_t db = tc::sdesc_sw128(sk + (kk / 4) * (KT * 128) + koff, 16, 1024);
              tc::umma_bf16(tmem + C::S_COL + sb * KT, da, db, C::IDESC_QK, kk > 0);
            }
            tc::umma_commit(&s_full[sb]);
          }
          if (t > 0) {
            // ---- O += P(t-1) V(t-1)
            const int pb = prev_g & 1;
            tc::mbar_wait(&p_full[pb], (prev_g >> 1) & 1);
            SV_TR(4, prev_g);
            tc::fence_after();
            const uint32_t sv_ = tc::smem_u32(sKV + prev_stage * C::STAGE_BYTES + C::KV_BYTES);
#pragma unroll
            for (int kk = 0; kk < KT / 16; ++kk) {
              // V tile [key][d_h] is the MN-major B operand: LBO = next 64-wide d_h atom, SBO = next 8 keys
              const uint64_t db = tc::sdesc_sw128(sv_ + kk * 2048, KT * 128, 1024);
              tc::umma_bf16_ts(o_tm, tmem + C::S_COL + pb * KT + kk * 8, db, C::IDESC_PV, (t > 1) || (kk > 0));
            }
            tc::umma_commit(&kv_empty[prev_stage]);
            tc::umma_commit(&s_free[pb]);
          }
          if (t < I.n_tiles) {
            prev_stage = stage;
            prev_g = g;
            ++g;
            if (++stage == ST) { stage = 0; phase ^= 1; }
          }
        }
        tc::umma_commit(&o_full[ob]);
        tc::umma_commit(&q_empty[qb]);
      }
    }
  } else if (warp >= 4) {
    // ======================= softmax + item epilogue
    const int q = warp & 3;                           // quadrant = head within the GQA group
    const int hf = (warp - 4) >> 2;                   // key half of the tile served by this warp
    const int tl = q * 32 + lane;                     // TMEM lane = MMA row
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const float sl2e = 1.4426950408889634f / sqrtf((float)DH);
    const bool quad_active = q < G;                   // warp-uniform
    const int bar_id = 1 + q;                         // named barrier of the two warps of this quadrant
    uint32_t g = 0;
    int iter = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      const ItemInfo I = item_info(d, it);
      const int j = lane;                             // chain row
      const bool row_valid = quad_active && j < I.R;
      const int vis_end = I.L + j + 1;                // keys t < vis_end are visible (causal chain)
      float m = -INFINITY, l = 0.f;
      for (int t = 0; t < I.n_tiles; ++t, ++g) {
        const int sb = g & 1;
        tc::mbar_wait(&s_full[sb], (g >> 1) & 1);
        if (warp == 4 && lane == 0) SV_TR(5, g);
        tc::fence_after();
        if (quad_active) {
          uint32_t sv[32];
          __syncwarp();
          tc::tmem_ld32(tmem + lane_off + C::S_COL + sb * KT + hf * 32, sv);
          tc::tmem_ld_wait();
          const bool chain_tile = t >= I.n_page_tiles;
          const int kbase = (chain_tile ? I.L : I.t0 + t * KT) + hf * 32;
          const int kend = chain_tile ? I.L + I.R : min(I.t1, I.L);
          const int lim = row_valid ? min(kend, vis_end) - kbase : 0;   // columns c < lim are visible
          float s[32];
          float hm = -INFINITY;
          if (chain_tile && d.tree) {
            // token tree (R30): chain key c' = kbase - L + c is visible to node j iff it is
            // an ancestor-or-self of j
            const unsigned long long anc = row_valid ? d.row_anc[I.row0 + j] : 0ull;
            const int c0 = kbase - I.L;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              s[c] = (c0 + c < I.R && ((anc >> (c0 + c)) & 1ull)) ? __uint_as_float(sv[c]) : -INFINITY;
              hm = fmaxf(hm, s[c]);
            }
          } else if (lim >= 32) {
#pragma unroll
            for (int c = 0; c < 32; ++c) s[c] = __uint_as_float(sv[c]);
#pragma unroll
            for (int c = 0; c < 32; c += 2) hm = fmaxf(hm, fmaxf(s[c], s[c + 1]));
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              s[c] = c < lim ? __uint_as_float(sv[c]) : -INFINITY;
              hm = fmaxf(hm, s[c]);
            }
          }
          float* xm = xmax + sb * 256;
          xm[hf * 128 + tl] = hm;
          tc::fence_before();
          tc::named_bar(bar_id, 64);
          tc::fence_after();
          const float mt_raw = fmaxf(hm, xm[(hf ^ 1) * 128 + tl]);
          const float mt = mt_raw * sl2e;
          const bool raise = mt > m + kRescaleLog2 || (m == -INFINITY && mt > -INFINITY);
          const bool rescale_o = raise && t > 0 && m > -INFINITY;
          if (__any_sync(0xffffffffu, rescale_o)) {
            // rows whose max grew: O(row, this warp's half of d_h) *= 2^(m - mt) once PV(t-1) landed
            const uint32_t pg = g - 1;
            tc::mbar_wait(&s_free[pg & 1], (pg >> 1) & 1);
            tc::fence_after();
            const float f = rescale_o ? tc::ex2(m - mt) : 1.0f;
            const uint32_t o_tm = tmem + lane_off + C::O_COL + (iter & 1) * DH + hf * (DH / 2);
            for (int c = 0; c < DH / 2; c += 32) {
              uint32_t ov[32];
              __syncwarp();
              tc::tmem_ld32(o_tm + c, ov);
              tc::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * f);
              tc::tmem_st32(o_tm + c, ov);
            }
            tc::tmem_st_wait();
          }
          if (raise) {
            l *= (m == -INFINITY) ? 0.f : tc::ex2(m - mt);
            m = mt;
          }
          const float mm = m == -INFINITY ? 0.f : m;     // all s = -inf then: 2^-inf = 0
          uint32_t pk[16];
          float ls = 0.f;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float p0 = tc::ex2(fmaf(s[2 * c], sl2e, -mm));
            const float p1 = tc::ex2(fmaf(s[2 * c + 1], sl2e, -mm));
            ls += p0 + p1;
            const __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);   // .x = key 2c (low half)
            pk[c] = *reinterpret_cast<const uint32_t*>(&pp);
          }
          l += ls;
          tc::tmem_st16(tmem + lane_off + C::S_COL + sb * KT + hf * 16, pk);
          tc::tmem_st_wait();
        }
        tc::fence_before();
        if (warp == 4 && lane == 0) SV_TR(6, g);
        tc::mbar_arrive(&p_full[sb]);
      }
      // ---- item epilogue: unnormalised O, m (natural-log units), l -> split-KV partials
      const int ob = iter & 1;
      tc::mbar_wait(&o_full[ob], (iter >> 1) & 1);
      tc::fence_after();
      if (quad_active) {
        xl[ob * 256 + hf * 128 + tl] = l;
        tc::named_bar(bar_id, 64);
        const float l_tot = l + xl[ob * 256 + (hf ^ 1) * 128 + tl];
        const int rl = j * G + q;                     // partial-buffer row (combine's layout)
        float* po = d.part_o + ((size_t)it * kPartRows + rl) * DH + hf * (DH / 2);
        for (int c = 0; c < DH / 2; c += 32) {
          uint32_t ov[32];
          __syncwarp();
          tc::tmem_ld32(tmem + lane_off + C::O_COL + ob * DH + hf * (DH / 2) + c, ov);
          tc::tmem_ld_wait();
          if (row_valid) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(po + c + i) =
                  make_float4(__uint_as_float(ov[i]), __uint_as_float(ov[i + 1]), __uint_as_float(ov[i + 2]),
                              __uint_as_float(ov[i + 3]));
          }
        }
        if (row_valid && hf == 0) {
          d.part_ml[((size_t)it * kPartRows + rl) * 2 + 0] = m == -INFINITY ? -INFINITY : m * 0.69314718055994531f;
          d.part_ml[((size_t)it * kPartRows + rl) * 2 + 1] = l_tot;
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&o_empty[ob]);
      if (warp == 4 && lane == 0) SV_TR(7, iter);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

int attn_tc_smem_bytes(int dh) { return dh == 128 ? AttnCfg<128>::SMEM : AttnCfg<64>::SMEM; }

template <int DH>
static cudaError_t launch_dh(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                             int num_sms, int q_box_tokens, cudaStream_t s) {
  {
    const cudaError_t e = smem_optin((const void*)attn_tc_kernel<DH>, (int)(AttnCfg<DH>::SMEM));
    if (e != cudaSuccess) return e;
  }
  SV_COUNT_LAUNCH();
  attn_tc_kernel<DH><<<num_sms, THREADS, AttnCfg<DH>::SMEM, s>>>(map_q, map_kv, d, layer, q_box_tokens);
  return cudaGetLastError();
}

cudaError_t launch_attention_tc(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                int num_sms, int q_box_tokens, cudaStream_t s) {
  return d.dh == 128 ? launch_dh<128>(map_q, map_kv, d, layer, num_sms, q_box_tokens, s)
                     : launch_dh<64>(map_q, map_kv, d, layer, num_sms, q_box_tokens, s);
}

}  // namespace sv
