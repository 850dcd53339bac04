// NEXT-3 (eq:prefill_computation): causal attention of a LONG prefill chunk —
// hundreds of query rows per kv head, which the verify kernels (<= 64 query slots per kv head)
// do not take. The chunk's own K/V rows are committed to their pages before this kernel runs
// (sv_prefill, k_kv.cu prefill_kv_kernel), so every key — the prompt prefix and the chunk — is a
// page key streamed by TMA, and causality is a per-row key limit: query row j of the chunk (at
// position L + j) sees keys 0 .. L + j.
//
// Rows on lanes: one work item = (kv head h, query block qb) with RB = 128 / G chunk rows of each
// of the G q heads of h on the 128 MMA rows (TMEM lane g * RB + j = head h*G + g, chunk row
// qb * RB + j). Per 64-key tile:
//   S  = Q K^T       tcgen05.mma M=128 N=64 K=d_h, A = Q (smem), B = K (smem)
//   P  = 2^(S*scale*log2e - m)   online max with lazy rescale (row max grows by > 2^8), P -> bf16 -> TMEM
//   O += P V         tcgen05.mma M=128 N=d_h K=64, A = P (TMEM), B = V (smem, MN-major)
// The item's keys end at L + (last row of the block) + 1, so items run whole (no split-KV) and
// write the normalised O (bf16) straight to the step's O buffer. Items are issued longest first.
// Warp roles as in the verify kernels (k_attn_tc.cu): 0 TMA producer, 1 MMA issuer, 2 TMEM
// allocator, 4-11 softmax (warp w: TMEM lane quadrant w % 4, key half (w - 4) / 4) + epilogue.
#include <cuda.h>

#include "attn_tc.h"
#include "common.cuh"
#include "lane.h"
#include "tc.cuh"

namespace sv {

namespace {
constexpr int PKT = 64;                    // keys per tile (= page size)
constexpr int PST = 4;                     // K/V ring stages
constexpr int PTHREADS = 384;
constexpr int PSOFT = 256;
constexpr float kPRescaleLog2 = 8.0f;
}  // namespace

template <int DH>
struct PrefCfg {
  static constexpr int HALVES = DH / 64;
  static constexpr int Q_BYTES = 128 * DH * 2;
  static constexpr int KV_BYTES = PKT * DH * 2;
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int SMEM = 2 * Q_BYTES + PST * STAGE_BYTES + 1024 + 8192;
  static constexpr uint32_t IDESC_QK = tc::idesc_bf16(128, PKT);
  static constexpr uint32_t IDESC_PV = tc::idesc_bf16(128, DH, 0, 1);
  static constexpr int S_COL = 0;
  static constexpr int O_COL = 128;
};

struct PrefItem {
  int h, qb, nrows, kend, n_tiles;
};

// items: d.items[i] = (0, h, qb, 0), longest first; the chunk: slot d.slots[0], R = d.depths[0] + 1
// rows at row offset 0, cache length L = d.len[slot] (not yet advanced)
__device__ __forceinline__ PrefItem pref_item(const LaneDev& d, int it, int L, int R, int RB) {
  const int4 w = d.items[it];
  PrefItem I;
  I.h = w.y;
  I.qb = w.z;
  I.nrows = min(RB, R - I.qb * RB);
  I.kend = L + I.qb * RB + I.nrows;
  I.n_tiles = (I.kend + PKT - 1) / PKT;
  return I;
}

template <int DH>
__global__ void __launch_bounds__(PTHREADS, 1)
    attn_prefill_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                        const LaneDev d, const int layer) {
  using C = PrefCfg<DH>;
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_s & 1023)) & 1023);
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + 2 * C::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + PST * C::STAGE_BYTES);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = kv_full + PST;
  uint64_t* q_full = kv_empty + PST;
  uint64_t* q_empty = q_full + 2;
  uint64_t* s_full = q_empty + 2;
  uint64_t* p_full = s_full + 2;
  uint64_t* s_free = p_full + 2;
  uint64_t* o_full = s_free + 2;
  uint64_t* o_empty = o_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_empty + 2);
  float* xmax = reinterpret_cast<float*>(bars + 64);    // [2 tile parity][2 halves][128 lanes]
  float* xl = xmax + 2 * 2 * 128;                       // [2][2][128] item sums

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = d.Hq / d.Hkv, RB = 128 / G;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&map_q);
    tc::prefetch_tmap(&map_kv);
    for (int i = 0; i < PST; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 1);
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], PSOFT);
      tc::mbar_init(&s_free[i], 1);
      tc::mbar_init(&o_full[i], 1);
      tc::mbar_init(&o_empty[i], PSOFT);
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
  pdl_wait();                                           // Q, the chunk's pages and the plan come from earlier kernels
  const int n_items = *d.n_items;
  const int slot = d.slots[0], R = d.depths[0] + 1, L = d.len[slot];

  if (warp == 0) {
    // ======================= producer
    const uint64_t pol = tc::policy_evict_first();
    const uint32_t q_tx = C::Q_BYTES;
    int stage = 0;
    uint32_t phase = 0;
    int iter = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      const PrefItem I = pref_item(d, it, L, R, RB);
      const int qbuf = iter & 1;
      if (lane == 0) {
        tc::mbar_wait(&q_empty[qbuf], ((iter >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qbuf], q_tx);
        for (int g = 0; g < G; ++g)
          for (int hf = 0; hf < C::HALVES; ++hf)
            tc::tma_load_3d(sQ + qbuf * C::Q_BYTES + hf * (128 * 128) + g * (RB * 128), &map_q, &q_full[qbuf],
                            hf * 64, I.h * G + g, I.qb * RB);
        for (int t = 0; t < I.n_tiles; ++t) {
          tc::mbar_wait(&kv_empty[stage], phase ^ 1);
          uint8_t* sk = sKV + stage * C::STAGE_BYTES;
          uint8_t* sv_ = sk + C::KV_BYTES;
          const int page = d.page_table[slot * d.max_pages_per_slot + t];
          const int rk = ((((layer * d.n_pages + page) * 2 + 0) * d.Hkv) + I.h) * PKT;
          const int rv = ((((layer * d.n_pages + page) * 2 + 1) * d.Hkv) + I.h) * PKT;
          tc::mbar_arrive_expect_tx(&kv_full[stage], C::STAGE_BYTES);
          for (int hf = 0; hf < C::HALVES; ++hf) {
            tc::tma_load_2d_hint(sk + hf * (PKT * 128), &map_kv, &kv_full[stage], hf * 64, rk, pol);
            tc::tma_load_2d_hint(sv_ + hf * (PKT * 128), &map_kv, &kv_full[stage], hf * 64, rv, pol);
          }
          if (++stage == PST) { stage = 0; phase ^= 1; }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ======================= MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t g = 0;
      int iter = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
        const PrefItem I = pref_item(d, it, L, R, RB);
        const int qbuf = iter & 1, ob = iter & 1;
        tc::mbar_wait(&q_full[qbuf], (iter >> 1) & 1);
        tc::mbar_wait(&o_empty[ob], ((iter >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t sq = tc::smem_u32(sQ + qbuf * C::Q_BYTES);
        const uint32_t o_tm = tmem + C::O_COL + ob * DH;
        int prev_stage = -1;
        uint32_t prev_g = 0;
        for (int t = 0; t <= I.n_tiles; ++t) {
          if (t < I.n_tiles) {
            const int sb = g & 1;
            tc::mbar_wait(&kv_full[stage], phase);
            tc::mbar_wait(&s_free[sb], ((g >> 1) & 1) ^ 1);
            tc::fence_after();
            const uint32_t sk = tc::smem_u32(sKV + stage * C::STAGE_BYTES);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint32_t koff = (kk % 4) * 32;
              const uint64_t da = tc::sdesc_sw128(sq + (kk / 4) * (128 * 128) + koff, 16, 1024);
              const uint64_t db = tc::sdesc_sw128(sk + (kk / 4) * (PKT * 128) + koff, 16, 1024);
              tc::umma_bf16(tmem + C::S_COL + sb * PKT, da, db, C::IDESC_QK, kk > 0);
            }
            tc::umma_commit(&s_full[sb]);
          }
          if (t > 0) {
            const int pb = prev_g & 1;
            tc::mbar_wait(&p_full[pb], (prev_g >> 1) & 1);
            tc::fence_after();
            const uint32_t sv_ = tc::smem_u32(sKV + prev_stage * C::STAGE_BYTES + C::KV_BYTES);
#pragma unroll
            for (int kk = 0; kk < PKT / 16; ++kk) {
              const uint64_t db = tc::sdesc_sw128(sv_ + kk * 2048, PKT * 128, 1024);
              tc::umma_bf16_ts(o_tm, tmem + C::S_COL + pb * PKT + kk * 8, db, C::IDESC_PV, (t > 1) || (kk > 0));
            }
            tc::umma_commit(&kv_empty[prev_stage]);
            tc::umma_commit(&s_free[pb]);
          }
          if (t < I.n_tiles) {
            prev_stage = stage;
            prev_g = g;
            ++g;
            if (++stage == PST) { stage = 0; phase ^= 1; }
          }
        }
        tc::umma_commit(&o_full[ob]);
        tc::umma_commit(&q_empty[qbuf]);
      }
    }
  } else if (warp >= 4) {
    // ======================= softmax + epilogue
    const int q = warp & 3;
    const int hf = (warp - 4) >> 2;
    const int tl = q * 32 + lane;                     // TMEM lane = MMA row
    const int gh = tl / RB, j = tl % RB;              // head within the group, row within the block
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const float sl2e = 1.4426950408889634f / sqrtf((float)DH);
    const int bar_id = 1 + q;
    const size_t ldo = (size_t)d.Hq * DH;
    uint32_t g = 0;
    int iter = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      const PrefItem I = pref_item(d, it, L, R, RB);
      const int jg = I.qb * RB + j;
      const bool row_valid = j < I.nrows;
      const int vis_end = L + jg + 1;                 // causal: keys < L + jg + 1
      float m = -INFINITY, l = 0.f;
      for (int t = 0; t < I.n_tiles; ++t, ++g) {
        const int sb = g & 1;
        tc::mbar_wait(&s_full[sb], (g >> 1) & 1);
        tc::fence_after();
        uint32_t sv[32];
        __syncwarp();
        tc::tmem_ld32(tmem + lane_off + C::S_COL + sb * PKT + hf * 32, sv);
        tc::tmem_ld_wait();
        const int kbase = t * PKT + hf * 32;
        const int lim = row_valid ? min(I.kend, vis_end) - kbase : 0;
        float s[32];
        float hm = -INFINITY;
        if (lim >= 32) {
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
        const float mt = fmaxf(hm, xm[(hf ^ 1) * 128 + tl]) * sl2e;
        const bool raise = mt > m + kPRescaleLog2 || (m == -INFINITY && mt > -INFINITY);
        const bool rescale_o = raise && t > 0 && m > -INFINITY;
        if (__any_sync(0xffffffffu, rescale_o)) {
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
        const float mm = m == -INFINITY ? 0.f : m;
        uint32_t pk[16];
        float ls = 0.f;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float p0 = tc::ex2(fmaf(s[2 * c], sl2e, -mm));
          const float p1 = tc::ex2(fmaf(s[2 * c + 1], sl2e, -mm));
          ls += p0 + p1;
          const __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);
          pk[c] = *reinterpret_cast<const uint32_t*>(&pp);
        }
        l += ls;
        tc::tmem_st16(tmem + lane_off + C::S_COL + sb * PKT + hf * 16, pk);
        tc::tmem_st_wait();
        tc::fence_before();
        tc::mbar_arrive(&p_full[sb]);
      }
      // ---- epilogue: O / l -> bf16 rows of the step's O buffer
      const int ob = iter & 1;
      tc::mbar_wait(&o_full[ob], (iter >> 1) & 1);
      tc::fence_after();
      xl[ob * 256 + hf * 128 + tl] = l;
      tc::named_bar(bar_id, 64);
      const float l_tot = l + xl[ob * 256 + (hf ^ 1) * 128 + tl];
      const float inv = l_tot > 0.f ? 1.0f / l_tot : 0.f;
      bf16* orow = d.o + (size_t)jg * ldo + (size_t)(I.h * G + gh) * DH + hf * (DH / 2);
      for (int c = 0; c < DH / 2; c += 32) {
        uint32_t ov[32];
        __syncwarp();
        tc::tmem_ld32(tmem + lane_off + C::O_COL + ob * DH + hf * (DH / 2) + c, ov);
        tc::tmem_ld_wait();
        if (row_valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 u;
            __nv_bfloat162 b0 = __floats2bfloat162_rn(__uint_as_float(ov[i]) * inv, __uint_as_float(ov[i + 1]) * inv);
            __nv_bfloat162 b1 = __floats2bfloat162_rn(__uint_as_float(ov[i + 2]) * inv, __uint_as_float(ov[i + 3]) * inv);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(ov[i + 4]) * inv, __uint_as_float(ov[i + 5]) * inv);
            __nv_bfloat162 b3 = __floats2bfloat162_rn(__uint_as_float(ov[i + 6]) * inv, __uint_as_float(ov[i + 7]) * inv);
            u.x = *reinterpret_cast<uint32_t*>(&b0);
            u.y = *reinterpret_cast<uint32_t*>(&b1);
            u.z = *reinterpret_cast<uint32_t*>(&b2);
            u.w = *reinterpret_cast<uint32_t*>(&b3);
            *reinterpret_cast<uint4*>(orow + c + i) = u;
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&o_empty[ob]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

template <int DH>
static cudaError_t launch_pref_dh(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                  int grid, cudaStream_t s) {
  {
    const cudaError_t e = smem_optin((const void*)attn_prefill_kernel<DH>, (int)(PrefCfg<DH>::SMEM));
    if (e != cudaSuccess) return e;
  }
  SV_COUNT_LAUNCH();
  return launch_pdl(attn_prefill_kernel<DH>, dim3(grid), dim3(PTHREADS), PrefCfg<DH>::SMEM, s, 1, map_q, map_kv, d,
                    layer);
}

cudaError_t launch_attention_prefill(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                     int n_items, int num_sms, cudaStream_t s) {
  const int grid = n_items < num_sms ? (n_items > 0 ? n_items : 1) : num_sms;
  return d.dh == 128 ? launch_pref_dh<128>(map_q, map_kv, d, layer, grid, s)
                     : launch_pref_dh<64>(map_q, map_kv, d, layer, grid, s);
}

}  // namespace sv
