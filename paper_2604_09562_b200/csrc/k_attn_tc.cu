// a3: paged, GQA, chain-causal verify attention on the 5th-generation tensor cores.
//
// One work item = (request b, kv head h, split s) of the device work list built by the
// plan kernel (see lane.h: num_splits / split_t1). Its query rows are the (k+1)*G rows
// (chain row j, q head h*G+g) -> row r = j*G + g (<= 64), its keys the split's KV pages
// (64 keys each, streamed by TMA) and, for the last split, the chain keys of this verify
// (scratch kc/vc, loaded by the producer warp). Per 64-key tile:
//   S  = Q K^T          tcgen05.mma M=128 (rows) N=64 (keys) K=d_h, A=Q smem, B=K smem
//   P  = exp2(S*scale*log2e - m)   one softmax thread per row (TMEM lane), online max with
//                       lazy rescale (only when the max grows by > 2^8), P -> bf16 -> TMEM
//   O += P V            tcgen05.mma M=128 N=d_h K=64, A=P from TMEM, B=V smem (MN-major)
// and the item's unnormalised O, max and sum go to the split-KV partial buffers that
// attn_combine_kernel merges (exactly the SIMT kernel's partial format).
//
// Warp roles (persistent grid, one CTA per SM, 8 warps):
//   warp 0  producer: Q tile (3-D TMA over q), K/V page tiles (2-D TMA over the pool),
//           chain tile (cooperative ld.global -> swizzled st.shared)
//   warp 1  MMA issuer (one thread)      warp 2  TMEM allocator
//   warps 4-7 softmax + item epilogue (TMEM lanes 32*(warp%4)..)
// Smem: Q double buffer 2 x 32 KB + 4-stage K/V ring 4 x 2 x 16 KB = 192 KB.
// TMEM: S/P double buffer 2 x 64 columns, O double buffer 2 x 128 columns.
#include <cuda.h>

#include "attn_tc.h"
#include "common.cuh"
#include "lane.h"
#include "tc.cuh"

namespace sv {

namespace {
constexpr int KT = 64;                     // keys per tile (= page size)
constexpr int ST = 4;                      // K/V ring stages
constexpr int THREADS = 256;
constexpr float kRescaleLog2 = 8.0f;       // rescale O only when the running max grows by > 2^8
}  // namespace

template <int DH>
struct AttnCfg {
  static constexpr int HALVES = DH / 64;                 // 64-element (128-B) swizzle atoms along d_h
  static constexpr int Q_BYTES = 128 * DH * 2;           // 128 rows (only <= 64 used) x d_h
  static constexpr int KV_BYTES = KT * DH * 2;           // one K or V tile
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int SMEM = 2 * Q_BYTES + ST * STAGE_BYTES + 1024 + 512;
  static constexpr uint32_t IDESC_QK = tc::idesc_bf16(128, KT);          // A, B K-major
  static constexpr uint32_t IDESC_PV = tc::idesc_bf16(128, DH, 0, 1);    // B (V) MN-major
  static constexpr int S_COL = 0;                        // S/P buffers at columns 0, 64
  static constexpr int O_COL = 128;                      // O buffers at 128, 128 + DH
};

struct ItemInfo {
  int b, h, s, ns, slot, L, R, row0, nr, t0, t1, n_page_tiles, n_tiles, page0;
  bool chain;
};

__device__ __forceinline__ ItemInfo item_info(const LaneDev& d, int it) {
  const int4 w = d.items[it];
  ItemInfo I;
  I.b = w.x;
  I.h = w.y;
  I.s = w.z;
  I.ns = w.w;
  I.slot = d.slots[I.b];
  I.L = d.len[I.slot];
  I.R = d.depths[I.b] + 1;
  I.row0 = d.row_off[I.b];
  I.nr = I.R * (d.Hq / d.Hkv);
  I.t0 = split_t0(I.s);
  I.t1 = split_t1(I.s, I.ns, I.L, I.R);
  I.chain = I.s == I.ns - 1;
  const int page_end = min(I.t1, I.L);
  I.n_page_tiles = page_end > I.t0 ? (page_end - I.t0 + KT - 1) / KT : 0;
  I.n_tiles = I.n_page_tiles + (I.chain ? 1 : 0);
  I.page0 = I.t0 / KT;
  return I;
}

template <int DH>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                   const LaneDev d, const int layer) {
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

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = *d.n_items;
  const int G = d.Hq / d.Hkv;
  const size_t nkv = (size_t)d.Hkv * DH;

  // zero the Q buffers once (rows 64..127 are never loaded)
  for (int i = threadIdx.x; i < 2 * C::Q_BYTES / 16; i += THREADS)
    reinterpret_cast<uint4*>(sQ)[i] = make_uint4(0, 0, 0, 0);
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
      tc::mbar_init(&p_full[i], 128);
      tc::mbar_init(&s_free[i], 1);
      tc::mbar_init(&o_full[i], 1);
      tc::mbar_init(&o_empty[i], 128);
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
    int stage = 0;
    uint32_t phase = 0;
    int iter = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      const ItemInfo I = item_info(d, it);
      const int qb = iter & 1;
      if (lane == 0) {
        tc::mbar_wait(&q_empty[qb], ((iter >> 1) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qb], C::HALVES * 64 * 128);
        for (int hf = 0; hf < C::HALVES; ++hf)
          tc::tma_load_3d(sQ + qb * C::Q_BYTES + hf * (128 * 128), &map_q, &q_full[qb], hf * 64, I.h * G, I.row0);
      }
      for (int t = 0; t < I.n_tiles; ++t) {
        if (lane == 0) tc::mbar_wait(&kv_empty[stage], phase ^ 1);
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
        }
        if (++stage == ST) { stage = 0; phase ^= 1; }
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
            tc::mbar_wait(&s_free[sb], ((g >> 1) & 1) ^ 1);
            tc::fence_after();
            const uint32_t sk = tc::smem_u32(sKV + stage * C::STAGE_BYTES);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint32_t hoff = (kk / 4) * (128 * 128), koff = (kk % 4) * 32;
              const uint64_t da = tc::sdesc_sw128(sq + hoff + koff, 16, 1024);
              const uint64_t db = tc::sdesc_sw128(sk + (kk / 4) * (KT * 128) + koff, 16, 1024);
              tc::umma_bf16(tmem + C::S_COL + sb * KT, da, db, C::IDESC_QK, kk > 0);
            }
            tc::umma_commit(&s_full[sb]);
          }
          if (t > 0) {
            // ---- O += P(t-1) V(t-1)
            const int pb = prev_g & 1;
            tc::mbar_wait(&p_full[pb], (prev_g >> 1) & 1);
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
    const int q = warp & 3;
    const int r = q * 32 + lane;                      // query row == TMEM lane
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const float sl2e = 1.4426950408889634f / sqrtf((float)DH);
    uint32_t g = 0;
    int iter = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      const ItemInfo I = item_info(d, it);
      const bool warp_active = q * 32 < I.nr;
      const bool row_valid = r < I.nr;
      const int j = r / G;                            // chain row of this query row
      const int vis_end = I.L + j + 1;                // keys t < vis_end are visible (causal chain)
      float m = -INFINITY, l = 0.f;
      for (int t = 0; t < I.n_tiles; ++t, ++g) {
        const int sb = g & 1;
        tc::mbar_wait(&s_full[sb], (g >> 1) & 1);
        tc::fence_after();
        if (warp_active) {
          uint32_t sa[32], sb2[32];
          __syncwarp();
          tc::tmem_ld32(tmem + lane_off + C::S_COL + sb * KT, sa);
          tc::tmem_ld32(tmem + lane_off + C::S_COL + sb * KT + 32, sb2);
          tc::tmem_ld_wait();
          // key index of column c: page tiles t0 + 64 t + c (valid < min(t1, L)); chain tile L + c
          const bool chain_tile = t >= I.n_page_tiles;
          const int kbase = chain_tile ? I.L : I.t0 + t * KT;
          const int kend = chain_tile ? I.L + I.R : min(I.t1, I.L);
          const int lim = min(kend, vis_end) - kbase;     // columns c < lim are visible
          float x[64];
          float mt = -INFINITY;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            x[c] = (row_valid && c < lim) ? __uint_as_float(sa[c]) * sl2e : -INFINITY;
            x[c + 32] = (row_valid && c + 32 < lim) ? __uint_as_float(sb2[c]) * sl2e : -INFINITY;
            mt = fmaxf(mt, fmaxf(x[c], x[c + 32]));
          }
          const bool raise = mt > m + kRescaleLog2 || (m == -INFINITY && mt > -INFINITY);
          const bool rescale_o = raise && t > 0 && m > -INFINITY;
          if (__any_sync(0xffffffffu, rescale_o)) {
            // O(row) *= 2^(m - mt) for the rows whose max grew: wait until PV(t-1) has landed
            // in O, then rescale in TMEM (warp-uniform path; other lanes scale by 1)
            const uint32_t pg = g - 1;
            tc::mbar_wait(&s_free[pg & 1], (pg >> 1) & 1);
            tc::fence_after();
            const float f = rescale_o ? exp2f(m - mt) : 1.0f;
            const uint32_t o_tm = tmem + lane_off + C::O_COL + (iter & 1) * DH;
            for (int c = 0; c < DH; c += 32) {
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
            l *= (m == -INFINITY) ? 0.f : exp2f(m - mt);
            m = mt;
          }
          uint32_t pk[32];
          float ls = 0.f;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float p0 = m == -INFINITY ? 0.f : exp2f(x[2 * c] - m);
            const float p1 = m == -INFINITY ? 0.f : exp2f(x[2 * c + 1] - m);
            const __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);   // .x = key 2c (low half)
            ls += __low2float(pp) + __high2float(pp);
            pk[c] = *reinterpret_cast<const uint32_t*>(&pp);
          }
          l += ls;
          tc::tmem_st32(tmem + lane_off + C::S_COL + sb * KT, pk);
          tc::tmem_st_wait();
        }
        tc::fence_before();
        tc::mbar_arrive(&p_full[sb]);
      }
      // ---- item epilogue: unnormalised O, m (natural log units), l -> split-KV partials
      const int ob = iter & 1;
      tc::mbar_wait(&o_full[ob], (iter >> 1) & 1);
      tc::fence_after();
      if (warp_active) {
        float* po = d.part_o + ((size_t)it * kAttnRows + r) * DH;
        for (int c = 0; c < DH; c += 32) {
          uint32_t ov[32];
          __syncwarp();
          tc::tmem_ld32(tmem + lane_off + C::O_COL + ob * DH + c, ov);
          tc::tmem_ld_wait();
          if (row_valid) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(po + c + i) =
                  make_float4(__uint_as_float(ov[i]), __uint_as_float(ov[i + 1]), __uint_as_float(ov[i + 2]),
                              __uint_as_float(ov[i + 3]));
          }
        }
        if (row_valid) {
          d.part_ml[((size_t)it * kAttnRows + r) * 2 + 0] = m == -INFINITY ? -INFINITY : m * 0.69314718055994531f;
          d.part_ml[((size_t)it * kAttnRows + r) * 2 + 1] = l;
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

int attn_tc_smem_bytes(int dh) { return dh == 128 ? AttnCfg<128>::SMEM : AttnCfg<64>::SMEM; }

cudaError_t launch_attention_tc(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                int num_sms, cudaStream_t s) {
  static bool attr128 = false, attr64 = false;
  if (d.dh == 128) {
    if (!attr128) {
      cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           AttnCfg<128>::SMEM);
      if (e != cudaSuccess) return e;
      attr128 = true;
    }
    SV_COUNT_LAUNCH();
    attn_tc_kernel<128><<<num_sms, THREADS, AttnCfg<128>::SMEM, s>>>(map_q, map_kv, d, layer);
  } else {
    if (!attr64) {
      cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           AttnCfg<64>::SMEM);
      if (e != cudaSuccess) return e;
      attr64 = true;
    }
    SV_COUNT_LAUNCH();
    attn_tc_kernel<64><<<num_sms, THREADS, AttnCfg<64>::SMEM, s>>>(map_q, map_kv, d, layer);
  }
  return cudaGetLastError();
}

}  // namespace sv
