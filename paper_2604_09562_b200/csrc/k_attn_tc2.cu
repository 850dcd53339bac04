// a3: paged, GQA, chain-causal verify attention, "keys-on-lanes" tcgen05 formulation (d_h = 128).
//
// Verify attention has few query rows per kv head ((k+1) * G <= 64) and long key streams, so
// this kernel puts KEYS on the 128 MMA rows / TMEM lanes and query slots on the N dimension:
//   S^T = K Q^T         tcgen05.mma M=128 keys, N=64 query slots, K=d_h; A = K tile, B = Q (smem)
//   P^T = 2^(S^T*scale*log2e - m_col)  softmax threads: one TMEM lane (= key) per thread, the
//                       per-slot column max via redux.sync.max.f32 + a 4-warp exchange, lazy
//                       per-column rescale (only when a column max grows by > 2^8), P^T -> bf16 ->
//                       smem (MN-major, 128-byte swizzle)
//   O^T += V^T P^T      tcgen05.mma M=128 (d_h), N=64 slots, K=128 keys; A = V tile read MN-major,
//                       B = P^T (smem, MN-major); accumulator in TMEM (lane = d_h)
// Every TMEM lane of every softmax warp does useful work (keys), instead of the (k+1)*G of 128
// lanes a rows-on-lanes layout would keep busy.
//
// One work item = (request b, kv head h, split s) of the plan kernel's work list (lane.h);
// 128-key tiles = two KV pages (2-D TMA over the pool) or the chain tile (this verify's chain
// keys from the kc/vc scratch). Query slot r = j*G + g (chain row j, q head h*G + g); the item's
// unnormalised O, column max and column sum go to the split-KV partials (attn_combine_kernel).
//
// Warp roles (persistent grid, one CTA per SM, 12 warps):
//   warp 0 producer (Q 3-D TMA, K/V 2-D TMA, chain tile by ld.global + swizzled st.shared)
//   warp 1 MMA issuer (one thread)   warp 2 TMEM allocator   warp 3 idle
//   warps 4-11 softmax + epilogue: key quadrant q = warp % 4 (TMEM lanes 32q..32q+31),
//              slot half ch = (warp - 4) / 4 (query slots 32ch..32ch+31)
// Smem: 3-stage K/V ring (3 x 64 KB) + Q (16 KB) + P^T (16 KB) + exchange buffers.
// TMEM: S^T double buffer 2 x 64 columns, O^T double buffer 2 x 64 columns.
#include <cuda.h>

#include "attn_tc.h"
#include "common.cuh"
#include "lane.h"
#include "tc.cuh"

namespace sv {

#define SV_TR2(e, i)                                                                 \
  do {                                                                               \
    if (d.trace && blockIdx.x == 0 && (i) < 256) d.trace[(e)*256 + (i)] = clock64(); \
  } while (0)

namespace {
constexpr int DH = 128;
constexpr int HALVES = DH / 64;
constexpr int KT = 128;                    // keys per tile (two 64-key pages)
constexpr int NQ = 64;                     // query slots (MMA N)
constexpr int KST = 2;                     // K ring stages (a K tile is released right after S = K Q^T)
constexpr int VST = 3;                     // V ring stages (released after O += V^T P^T)
constexpr int THREADS = 352;              // 11 warps: producer, MMA, TMEM alloc, 8 softmax (3..10)
constexpr int SOFTMAX_THREADS = 256;
constexpr float kRescaleLog2 = 8.0f;
constexpr int KV_BYTES = KT * DH * 2;      // 32 KB (K or V of one tile)
constexpr int Q_BYTES = NQ * DH * 2;       // 16 KB
constexpr int P_BYTES = KT * NQ * 2;       // 16 KB per P^T buffer (two buffers)
constexpr int XCOL_FLOATS = 2 * 2 * 4 * 32;  // [tile parity][slot half][quadrant][32]
constexpr int SMEM = (KST + VST) * KV_BYTES + Q_BYTES + 2 * P_BYTES + 4 * XCOL_FLOATS + 512 + 512;
static_assert(SMEM <= 232448, "attention smem exceeds the 227 KB per-CTA limit");
static_assert(2 * kSplitKeys / 64 <= 32, "an item's pages (wide splits too) are held one per producer lane");
constexpr uint32_t IDESC_QK = tc::idesc_bf16(128, NQ);          // A = K (K-major), B = Q (K-major)
constexpr uint32_t IDESC_PV = tc::idesc_bf16(128, NQ, 1, 1);    // A = V^T (MN-major), B = P^T (MN-major)
constexpr uint32_t IDESC_L = tc::idesc_bf16(128, NQ, 0, 1);     // A = ones (TMEM), B = P^T (MN-major)
constexpr int S_COL = 0;                   // S^T buffers at columns 0, 64
constexpr int O_COL = 128;                 // O^T buffers at 128, 192
constexpr int L_COL = 256;                 // column-sum buffers at 256, 320 (every lane holds the sums)
constexpr int ONE_COL = 384;               // A operand of ones (128 lanes x 128 bf16 keys) at 384..447
constexpr uint32_t BF16_ONE_PAIR = 0x3F803F80u;
}  // namespace

struct Item2 {
  int b, h, s, ns, slot, L, R, row0, t0, kend, n_page_tiles, n_pages, n_tiles, page0;
};

__device__ __forceinline__ Item2 item2(const LaneDev& d, int it) {
  const int4 w = d.items[it];
  Item2 I;
  I.b = w.x;
  I.h = w.y;
  I.s = w.z;
  I.ns = item_ns(w.w);
  const int sk = item_split_keys(w.w);                        // 1024, or 2048 for a wide-split verify
  I.slot = d.slots[I.b];
  I.L = d.len[I.slot];
  I.R = d.depths[I.b] + 1;
  I.row0 = d.row_off[I.b];
  I.t0 = I.s * sk;
  I.kend = min(split_t1_k(I.s, I.ns, I.L, I.R, sk), I.L);   // page keys of this item: [t0, kend)
  I.n_pages = I.kend > I.t0 ? (I.kend - I.t0 + 63) / 64 : 0;
  I.n_page_tiles = (I.n_pages + 1) / 2;
  I.n_tiles = I.n_page_tiles + (I.s == I.ns - 1 ? 1 : 0);
  I.page0 = I.t0 / 64;
  return I;
}

__device__ __forceinline__ float redux_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

__global__ void __launch_bounds__(THREADS, 1)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                    const LaneDev d, const int layer) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_s & 1023)) & 1023);
  uint8_t* sK = smem;                                   // [KST][HALVES][128 keys][128 B]
  uint8_t* sV = sK + KST * KV_BYTES;                    // [VST][HALVES][128 keys][128 B]
  uint8_t* sQ = sV + VST * KV_BYTES;                    // [HALVES][64 slots][128 B]
  uint8_t* sP = sQ + Q_BYTES;                           // [2][128 keys][64 slots bf16 = 128 B]
  float* xcol = reinterpret_cast<float*>(sP + 2 * P_BYTES);
  float* mref_s = xcol + XCOL_FLOATS;                   // [2 slot halves][32] column reference max
  float* fs = mref_s + 64;                              // [2][32] rescale factors of the last raise
  uint64_t* bars = reinterpret_cast<uint64_t*>(fs + 64);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + VST;
  uint64_t* q_full = v_empty + VST;
  uint64_t* q_empty = q_full + 1;
  uint64_t* s_full = q_empty + 1;
  uint64_t* p_full = s_full + 2;
  uint64_t* s_free = p_full + 2;
  uint64_t* o_full = s_free + 2;
  uint64_t* o_empty = o_full + 2;
  uint64_t* s_read = o_empty + 2;                       // softmax has read S^T buffer: MMA may refill it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_read + 2);
  float* thr_s = reinterpret_cast<float*>(bars + 32);   // [2][32] raise thresholds (mref + 8, or -inf)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0 && ((raw_s & 1023) != 0)) __trap();   // SMEM budget has no alignment slack
  pdl_trigger();
  pdl_wait();                                           // n_items, Q, pages: written by earlier kernels
  const int n_items = *d.n_items;
  const int G = d.Hq / d.Hkv;
  const size_t nkv = (size_t)d.Hkv * DH;

  // zero the K/V ring, Q and P^T once: skipped second pages / unloaded slots / the P^T columns a
  // narrow slot half does not write must hold finite values
  for (int i = threadIdx.x; i < ((KST + VST) * KV_BYTES + Q_BYTES + 2 * P_BYTES) / 16; i += THREADS)
    reinterpret_cast<uint4*>(sK)[i] = make_uint4(0, 0, 0, 0);
  tc::fence_proxy_async();
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&map_q);
    tc::prefetch_tmap(&map_kv);
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VST; ++i) {
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&v_empty[i], 1);
    }
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], SOFTMAX_THREADS);
      tc::mbar_init(&s_free[i], 1);
      tc::mbar_init(&o_full[i], 1);
      tc::mbar_init(&o_empty[i], SOFTMAX_THREADS);
      tc::mbar_init(&s_read[i], SOFTMAX_THREADS);
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
  if (warp >= 3 && warp < 7) {                        // fill the ones operand (all 128 lanes)
    uint32_t ones[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) ones[i] = BF16_ONE_PAIR;
    const uint32_t a = tmem + (uint32_t((warp & 3) * 32) << 16) + ONE_COL;
    tc::tmem_st32(a, ones);
    tc::tmem_st32(a + 32, ones);
    tc::tmem_st_wait();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  if (warp == 0 || warp == 2) {
    // ======================= producers: warp 0 streams Q and K tiles, warp 2 streams V tiles
    // (two independent rings, so V prefetch never waits behind K and vice versa)
    const bool is_k = warp == 0;
    const uint64_t pol = tc::policy_evict_first();
    const int nst = is_k ? KST : VST;
    uint8_t* ring = is_k ? sK : sV;
    uint64_t* full = is_k ? k_full : v_full;
    uint64_t* empty = is_k ? k_empty : v_empty;
    const int kv = is_k ? 0 : 1;
    int st = 0;
    uint32_t ph = 0;
    int iter = 0;
    uint32_t ptile = 0;
    // Each item's page rows are looked up once (lane p holds page p of the item, <= 16 pages), and
    // the next item's descriptor and page rows are fetched while this item streams, so neither
    // dependent-load chain sits between a free ring slot and its TMA issue.
    auto page_rows = [&](const Item2& J) {
      int row = 0;
      if (lane < J.n_pages) {
        const int page = d.page_table[J.slot * d.max_pages_per_slot + J.page0 + lane];
        row = ((((layer * d.n_pages + page) * 2 + kv) * d.Hkv) + J.h) * 64;
      }
      return row;
    };
    Item2 I;
    int prow = 0;
    if ((int)blockIdx.x < n_items) {
      I = item2(d, blockIdx.x);
      prow = page_rows(I);
    }
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      Item2 In = I;
      int prown = 0;
      if (it + (int)gridDim.x < n_items) {            // prefetch: used by the next iteration
        In = item2(d, it + gridDim.x);
        prown = page_rows(In);
      }
      if (is_k && lane == 0) {
        tc::mbar_wait(q_empty, (iter & 1) ^ 1);
        tc::mbar_arrive_expect_tx(q_full, HALVES * NQ * 128);
        for (int hf = 0; hf < HALVES; ++hf)
          tc::tma_load_3d(sQ + hf * (NQ * 128), &map_q, q_full, hf * 64, I.h * G, I.row0);
      }
      for (int t = 0; t < I.n_tiles; ++t) {
        uint8_t* dst = ring + st * KV_BYTES;
        if (t < I.n_page_tiles) {
          // converged warp: lanes 0 / 1 look up the tile's two pages, the rows are broadcast, one
          // elected lane issues (keeps the TMA issue out of a lane-0 waterfall loop)
          const int np = min(2, I.n_pages - 2 * t);
          const int row0 = __shfl_sync(0xffffffffu, prow, 2 * t), row1 = __shfl_sync(0xffffffffu, prow, 2 * t + 1);
          tc::mbar_wait(&empty[st], ph ^ 1);
          if (is_k && lane == 0) SV_TR2(0, ptile);
          if (tc::elect_one()) {
            tc::mbar_arrive_expect_tx(&full[st], np * (KV_BYTES / 2));
#pragma unroll
            for (int hf = 0; hf < HALVES; ++hf)
              tc::tma_load_2d_hint(dst + hf * (KT * 128), &map_kv, &full[st], hf * 64, row0, pol);
            if (np > 1) {
#pragma unroll
              for (int hf = 0; hf < HALVES; ++hf)
                tc::tma_load_2d_hint(dst + hf * (KT * 128) + 64 * 128, &map_kv, &full[st], hf * 64, row1, pol);
            }
          }
          if (is_k && lane == 0) SV_TR2(1, ptile);
          __syncwarp();
        } else {
          if (lane == 0) tc::mbar_wait(&empty[st], ph ^ 1);
          __syncwarp();
          // chain tile: keys L + c (c < R) from the chain scratch. Only the R real rows are written:
          // rows beyond R keep the slot's earlier contents — finite (the ring is zeroed at kernel
          // start and only ever holds KV data), so their masked scores and zero P^T columns add
          // nothing (the same invariant as a tile's skipped second page)
          const bf16* src = (is_k ? d.kc : d.vc) + (size_t)layer * d.Tmax * nkv;
          constexpr int CH = DH / 8;
          // R <= 64 / G <= 64 rows x 16 chunks: up to 32 per lane; all loads issued before the stores
          // (one memory round trip per chain tile instead of one per row group)
          constexpr int CU = 8;
          for (int i0 = lane; i0 < I.R * CH; i0 += 32 * CU) {
            uint4 v[CU];
#pragma unroll
            for (int u = 0; u < CU; ++u) {
              const int i = i0 + 32 * u, c = i / CH, cq = i % CH;
              if (i < I.R * CH)
                v[u] = *reinterpret_cast<const uint4*>(src + (size_t)(I.row0 + c) * nkv + (size_t)I.h * DH + cq * 8);
            }
#pragma unroll
            for (int u = 0; u < CU; ++u) {
              const int i = i0 + 32 * u, c = i / CH, cq = i % CH;
              const int hf = cq / 8, cc = cq % 8;
              if (i < I.R * CH) *reinterpret_cast<uint4*>(dst + hf * (KT * 128) + c * 128 + ((cc ^ (c & 7)) * 16)) = v[u];
            }
          }
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&full[st]);
        }
        if (++st == nst) { st = 0; ph ^= 1; }
        ++ptile;
      }
      I = In;
      prow = prown;
    }
  } else if (warp == 1) {
    // ======================= MMA issuer: the whole warp runs the loop (warp-uniform state, so
    // ptxas keeps descriptors in uniform registers); one elected lane issues
    {
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      uint32_t g = 0;
      int iter = 0;
      const uint32_t sq = tc::smem_u32(sQ), sp0 = tc::smem_u32(sP);
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
        const Item2 I = item2(d, it);
        const int ob = iter & 1;
        tc::mbar_wait(q_full, iter & 1);
        tc::mbar_wait(&o_empty[ob], ((iter >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t o_tm = tmem + O_COL + ob * NQ;
        const uint32_t l_tm = tmem + L_COL + ob * NQ;
        int prev_vs = -1;
        uint32_t prev_vph = 0;
        uint32_t prev_g = 0;
        for (int t = 0; t <= I.n_tiles; ++t) {
          if (t < I.n_tiles) {
            const int sb = g & 1;
            tc::mbar_wait(&k_full[ks], kph);
            if (lane == 0) SV_TR2(2, g);
            tc::mbar_wait(&s_read[sb], ((g >> 1) & 1) ^ 1);   // S^T(g-2) read out: refill now
            if (lane == 0) SV_TR2(3, g);
            tc::fence_after();
            const uint32_t sk = tc::smem_u32(sK + ks * KV_BYTES);
            if (tc::elect_one()) {
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk) {
                const uint32_t koff = (kk % 4) * 32;
                const uint64_t da = tc::sdesc_sw128(sk + (kk / 4) * (KT * 128) + koff, 16, 1024);
                const uint64_t db = tc::sdesc_sw128(sq + (kk / 4) * (NQ * 128) + koff, 16, 1024);
                tc::umma_bf16(tmem + S_COL + sb * NQ, da, db, IDESC_QK, kk > 0);
              }
              tc::umma_commit(&s_full[sb]);
              tc::umma_commit(&k_empty[ks]);                      // K tile no longer needed
              if (t == I.n_tiles - 1) tc::umma_commit(q_empty);   // last read of Q for this item
            }
            __syncwarp();
          }
          if (t > 0) {
            const int pb = prev_g & 1;
            tc::mbar_wait(&p_full[pb], (prev_g >> 1) & 1);
            tc::mbar_wait(&v_full[prev_vs], prev_vph);
            if (lane == 0) SV_TR2(4, prev_g);
            tc::fence_after();
            const uint32_t sv_ = tc::smem_u32(sV + prev_vs * KV_BYTES);
            const uint32_t sp = sp0 + pb * P_BYTES;
            if (tc::elect_one()) {
#pragma unroll
              for (int kk = 0; kk < KT / 16; ++kk) {
                // A = V^T: d_h contiguous (MN-major), LBO = next 64-wide d_h atom (128 keys * 128 B),
                // SBO = next 8 keys; B = P^T: slots contiguous (MN-major), SBO = next 8 keys
                const uint64_t da = tc::sdesc_sw128(sv_ + kk * 2048, KT * 128, 1024);
                const uint64_t db = tc::sdesc_sw128(sp + kk * 2048, 8192, 1024);
                tc::umma_bf16(o_tm, da, db, IDESC_PV, (t > 1) || (kk > 0));
              }
              // column sums of the bf16 P^T actually used: L^T += ones(128 x keys) . P^T
#pragma unroll
              for (int kk = 0; kk < KT / 16; ++kk) {
                const uint64_t db = tc::sdesc_sw128(sp + kk * 2048, 8192, 1024);
                tc::umma_bf16_ts(l_tm, tmem + ONE_COL + kk * 8, db, IDESC_L, (t > 1) || (kk > 0));
              }
              tc::umma_commit(&v_empty[prev_vs]);
              tc::umma_commit(&s_free[pb]);
            }
            __syncwarp();
          }
          if (t < I.n_tiles) {
            prev_vs = vs;
            prev_vph = vph;
            prev_g = g;
            ++g;
            if (++ks == KST) { ks = 0; kph ^= 1; }
            if (++vs == VST) { vs = 0; vph ^= 1; }
          }
        }
        if (tc::elect_one()) tc::umma_commit(&o_full[ob]);
        __syncwarp();
      }
    }
  } else if (warp >= 3) {
    // ======================= softmax + item epilogue
    const int q = warp & 3;                           // key quadrant (TMEM lanes 32q..)
    const int ch = (warp - 3) >> 2;                   // query-slot half (slots 32ch..32ch+31)
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const float sl2e = 1.4426950408889634f / sqrtf((float)DH);
    const int bar_id = 1 + ch;                        // the 4 quadrant warps of this slot half
    const int lg = __ffs(G) - 1;                      // G is a power of two (dispatch checks)
    const int kidx = q * 32 + lane;                   // key index inside a tile (= TMEM lane)
    uint32_t g = 0;
    int iter = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++iter) {
      const Item2 I = item2(d, it);
      const int RG = I.R * G;
      // columns (query slots) of this half that exist: r = 32ch + c < (k+1) G
      const uint32_t colok = RG >= ch * 32 + 32 ? 0xffffffffu : (RG <= ch * 32 ? 0u : ((1u << (RG - ch * 32)) - 1u));
      // column reference max (log2 units) of this slot half lives in mref_s[ch][32] (same for the
      // 4 quadrant warps); minit bit c: column c has a finite reference (uniform register)
      float* mref = mref_s + ch * 32;
      float* fac = fs + ch * 32;
      float* thr = thr_s + ch * 32;
      uint32_t minit = 0;
      const bool narrow = RG - ch * 32 <= 8;          // warp-uniform for the whole item (empty halves too)
      if (q == 0) {
        mref[lane] = 0.f;
        thr[lane] = -INFINITY;                        // no reference yet: any finite score raises
      }
      tc::named_bar(bar_id, 128);
      for (int t = 0; t < I.n_tiles; ++t, ++g) {
        const int sb = g & 1;
        tc::mbar_wait(&s_full[sb], (g >> 1) & 1);
        if (warp == 4 && lane == 0) SV_TR2(5, g);
        tc::fence_after();
        // The columns this warp computes: all 32, or only the first 8 when this slot half holds at most
        // 8 real slots (k = 8 at G = 4: 36 slots, 4 in the second half; k <= 7: an empty half). The
        // other columns of a narrow half are masked slots whose P^T entries stay finite stale values and
        // whose O^T / L^T columns are never read. Two textual copies (a shared generic lambda made the
        // 32-column path ~25 % slower at k = 11 / 15).
        if (narrow) {
          uint32_t sv[8];
          __syncwarp();
          tc::tmem_ld8(tmem + lane_off + S_COL + sb * NQ + ch * 32, sv);
          tc::tmem_ld_wait();
          tc::fence_before();
          tc::mbar_arrive(&s_read[sb]);               // the MMA may write S^T(g+2) into this buffer
          if (warp == 4 && lane == 0) SV_TR2(8, g);
          const bool chain_tile = t >= I.n_page_tiles;
          const int key = (chain_tile ? I.L : I.t0 + t * KT) + kidx;
          const bool kvalid = key < (chain_tile ? I.L + I.R : I.kend);
          // visibility mask over this lane's 32 slots: key valid, slot exists, and (chain tile) causal:
          // chain key kidx is visible to slot r iff kidx <= r / G  <=>  r >= kidx * G
          uint32_t vm = kvalid ? colok : 0u;
          if (chain_tile) {
            if (d.tree) {
              // token tree (R30): chain key kidx is visible to row j iff kidx is an
              // ancestor-or-self of node j (row_anc bit); rows j of this half hold slots jG..jG+G-1
              uint32_t tm = 0;
              if (kvalid) {
                const int j0 = (ch * 32) >> lg, j1 = min(I.R, (ch * 32 + 32) >> lg);
                for (int j = j0; j < j1; ++j)
                  if ((d.row_anc[I.row0 + j] >> kidx) & 1ull) tm |= uint32_t((1ull << G) - 1ull) << ((j << lg) - ch * 32);
              }
              vm &= tm;
            } else {
              const int first = (kidx << lg) - ch * 32;
              vm &= first <= 0 ? 0xffffffffu : (first >= 32 ? 0u : (0xffffffffu << first));
            }
          }
          float x[8];
          bool need = false;
#pragma unroll
          for (int c = 0; c < 8; c += 4) {
            const float4 t4 = *reinterpret_cast<const float4*>(thr + c);
            const float th[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float sc = __uint_as_float(sv[c + e]) * sl2e;
              x[c + e] = ((vm >> (c + e)) & 1u) ? sc : -INFINITY;
              need |= x[c + e] > th[e];
            }
          }
          // does any of the 128 keys push a column beyond its reference (+2^8)? (4-warp vote)
          float* xc = xcol + ((sb * 2 + ch) * 4) * 32;
          const bool wneed = __any_sync(0xffffffffu, need);
          if (lane == 0) xc[q * 32] = wneed ? 1.f : 0.f;
          tc::named_bar(bar_id, 128);
          const bool raise_any = xc[0] + xc[32] + xc[64] + xc[96] > 0.f;   // uniform in the 4 warps
          if (warp == 4 && lane == 0) SV_TR2(9, g);
          if (g > 1) {                                 // PV(g-2) has released this P^T buffer
            const uint32_t pg = g - 2;
            tc::mbar_wait(&s_free[pg & 1], (pg >> 1) & 1);
            tc::fence_after();
          }
          if (warp == 4 && lane == 0) SV_TR2(10, g);
          if (raise_any) {
            // exact column max over the 128 keys inside the warp (lane c ends with column c), then
            // across the 4 quadrant warps through shared memory
            float cmw;
            {                                          // 8 columns: one redux per column
              cmw = -INFINITY;
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const float m = redux_max(x[c]);
                cmw = lane == c ? m : cmw;
              }
            }
            float* xm = xcol + (((sb ^ 1) * 2 + ch) * 4) * 32;   // other parity: free this tile
            xm[q * 32 + lane] = cmw;
            tc::named_bar(bar_id, 128);
            // lane c decides column c (identically in the 4 warps)
            const float cm = fmaxf(fmaxf(xm[lane], xm[32 + lane]), fmaxf(xm[64 + lane], xm[96 + lane]));
            const float old = mref[lane];
            const bool init = (minit >> lane) & 1u;
            const bool raise = init ? cm > old + kRescaleLog2 : cm > -INFINITY;
            const float f = (raise && init) ? tc::ex2(old - cm) : 1.0f;
            const bool any_resc = __any_sync(0xffffffffu, raise && init);
            minit |= __ballot_sync(0xffffffffu, raise);
            tc::named_bar(bar_id, 128);               // all reads of the old references are done
            if (q == 0) {
              if (raise) {
                mref[lane] = cm;
                thr[lane] = cm + kRescaleLog2;
              }
              fac[lane] = f;
            }
            tc::named_bar(bar_id, 128);               // new references / factors visible
            if (any_resc) {                           // uniform: every warp sees the same factors
              // O^T and the column sums L^T (this warp's 32 lanes x 32 slots) *= f(slot), once
              // PV(g-1) has landed in them
              const uint32_t pg = g - 1;
              tc::mbar_wait(&s_free[pg & 1], (pg >> 1) & 1);
              tc::fence_after();
              for (int buf = 0; buf < 2; ++buf) {
                const uint32_t a = tmem + lane_off + (buf ? L_COL : O_COL) + (iter & 1) * NQ + ch * 32;
                uint32_t ov[32];
                tc::tmem_ld32(a, ov);
                tc::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * fac[c]);
                tc::tmem_st32(a, ov);
              }
              tc::tmem_st_wait();
            }
          }
          // P^T row (this key) for the NC slots -> bf16 -> swizzled st.shared
          uint32_t pk[4];
#pragma unroll
          for (int c = 0; c < 8; c += 2) {
            const float2 m2 = *reinterpret_cast<const float2*>(mref + c);
            const float p0 = tc::ex2(x[c] - m2.x);         // x = -inf -> 0 (mref finite: 0 if unset)
            const float p1 = tc::ex2(x[c + 1] - m2.y);
            const __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);
            pk[c / 2] = *reinterpret_cast<const uint32_t*>(&pp);
          }
          if (warp == 4 && lane == 0) SV_TR2(11, g);
          uint8_t* prow = sP + sb * P_BYTES + kidx * 128;
#pragma unroll
          for (int i = 0; i < 1; ++i)
            *reinterpret_cast<uint4*>(prow + (((ch * 4 + i) ^ (kidx & 7)) * 16)) =
                make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        } else {
          uint32_t sv[32];
          __syncwarp();
          tc::tmem_ld32(tmem + lane_off + S_COL + sb * NQ + ch * 32, sv);
          tc::tmem_ld_wait();
          tc::fence_before();
          tc::mbar_arrive(&s_read[sb]);               // the MMA may write S^T(g+2) into this buffer
          if (warp == 4 && lane == 0) SV_TR2(8, g);
          const bool chain_tile = t >= I.n_page_tiles;
          const int key = (chain_tile ? I.L : I.t0 + t * KT) + kidx;
          const bool kvalid = key < (chain_tile ? I.L + I.R : I.kend);
          // visibility mask over this lane's 32 slots: key valid, slot exists, and (chain tile) causal:
          // chain key kidx is visible to slot r iff kidx <= r / G  <=>  r >= kidx * G
          uint32_t vm = kvalid ? colok : 0u;
          if (chain_tile) {
            if (d.tree) {
              // token tree (R30): chain key kidx is visible to row j iff kidx is an
              // ancestor-or-self of node j (row_anc bit); rows j of this half hold slots jG..jG+G-1
              uint32_t tm = 0;
              if (kvalid) {
                const int j0 = (ch * 32) >> lg, j1 = min(I.R, (ch * 32 + 32) >> lg);
                for (int j = j0; j < j1; ++j)
                  if ((d.row_anc[I.row0 + j] >> kidx) & 1ull) tm |= uint32_t((1ull << G) - 1ull) << ((j << lg) - ch * 32);
              }
              vm &= tm;
            } else {
              const int first = (kidx << lg) - ch * 32;
              vm &= first <= 0 ? 0xffffffffu : (first >= 32 ? 0u : (0xffffffffu << first));
            }
          }
          float x[32];
          bool need = false;
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const float4 t4 = *reinterpret_cast<const float4*>(thr + c);
            const float th[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float sc = __uint_as_float(sv[c + e]) * sl2e;
              x[c + e] = ((vm >> (c + e)) & 1u) ? sc : -INFINITY;
              need |= x[c + e] > th[e];
            }
          }
          // does any of the 128 keys push a column beyond its reference (+2^8)? (4-warp vote)
          float* xc = xcol + ((sb * 2 + ch) * 4) * 32;
          const bool wneed = __any_sync(0xffffffffu, need);
          if (lane == 0) xc[q * 32] = wneed ? 1.f : 0.f;
          tc::named_bar(bar_id, 128);
          const bool raise_any = xc[0] + xc[32] + xc[64] + xc[96] > 0.f;   // uniform in the 4 warps
          if (warp == 4 && lane == 0) SV_TR2(9, g);
          if (g > 1) {                                 // PV(g-2) has released this P^T buffer
            const uint32_t pg = g - 2;
            tc::mbar_wait(&s_free[pg & 1], (pg >> 1) & 1);
            tc::fence_after();
          }
          if (warp == 4 && lane == 0) SV_TR2(10, g);
          if (raise_any) {
            // exact column max over the 128 keys inside the warp (lane c ends with column c), then
            // across the 4 quadrant warps through shared memory
            float cmw;
            {                                          // transpose-reduce
              float v[32];
#pragma unroll
              for (int c = 0; c < 32; ++c) v[c] = x[c];
#pragma unroll
              for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                const bool up = lane & s2;
#pragma unroll
                for (int i = 0; i < s2; ++i) {
                  const float send = up ? v[i] : v[i + s2];
                  const float keep = up ? v[i + s2] : v[i];
                  v[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, s2));
                }
              }
              cmw = v[0];
            }
            float* xm = xcol + (((sb ^ 1) * 2 + ch) * 4) * 32;   // other parity: free this tile
            xm[q * 32 + lane] = cmw;
            tc::named_bar(bar_id, 128);
            // lane c decides column c (identically in the 4 warps)
            const float cm = fmaxf(fmaxf(xm[lane], xm[32 + lane]), fmaxf(xm[64 + lane], xm[96 + lane]));
            const float old = mref[lane];
            const bool init = (minit >> lane) & 1u;
            const bool raise = init ? cm > old + kRescaleLog2 : cm > -INFINITY;
            const float f = (raise && init) ? tc::ex2(old - cm) : 1.0f;
            const bool any_resc = __any_sync(0xffffffffu, raise && init);
            minit |= __ballot_sync(0xffffffffu, raise);
            tc::named_bar(bar_id, 128);               // all reads of the old references are done
            if (q == 0) {
              if (raise) {
                mref[lane] = cm;
                thr[lane] = cm + kRescaleLog2;
              }
              fac[lane] = f;
            }
            tc::named_bar(bar_id, 128);               // new references / factors visible
            if (any_resc) {                           // uniform: every warp sees the same factors
              // O^T and the column sums L^T (this warp's 32 lanes x 32 slots) *= f(slot), once
              // PV(g-1) has landed in them
              const uint32_t pg = g - 1;
              tc::mbar_wait(&s_free[pg & 1], (pg >> 1) & 1);
              tc::fence_after();
              for (int buf = 0; buf < 2; ++buf) {
                const uint32_t a = tmem + lane_off + (buf ? L_COL : O_COL) + (iter & 1) * NQ + ch * 32;
                uint32_t ov[32];
                tc::tmem_ld32(a, ov);
                tc::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * fac[c]);
                tc::tmem_st32(a, ov);
              }
              tc::tmem_st_wait();
            }
          }
          // P^T row (this key) for the NC slots -> bf16 -> swizzled st.shared
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 m2 = *reinterpret_cast<const float2*>(mref + c);
            const float p0 = tc::ex2(x[c] - m2.x);         // x = -inf -> 0 (mref finite: 0 if unset)
            const float p1 = tc::ex2(x[c + 1] - m2.y);
            const __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);
            pk[c / 2] = *reinterpret_cast<const uint32_t*>(&pp);
          }
          if (warp == 4 && lane == 0) SV_TR2(11, g);
          uint8_t* prow = sP + sb * P_BYTES + kidx * 128;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(prow + (((ch * 4 + i) ^ (kidx & 7)) * 16)) =
                make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
        tc::fence_proxy_async();
        tc::fence_before();
        if (warp == 4 && lane == 0) SV_TR2(6, g);
        tc::mbar_arrive(&p_full[sb]);
      }
      // ---- item epilogue: unnormalised O, column max, column sum -> split-KV partials
      const float my_m = mref[lane];
      const bool my_init = (minit >> lane) & 1u;
      const int ob = iter & 1;
      tc::mbar_wait(&o_full[ob], (iter >> 1) & 1);
      tc::fence_after();
      uint32_t ov[32], lv[32];
      __syncwarp();
      tc::tmem_ld32(tmem + lane_off + O_COL + ob * NQ + ch * 32, ov);
      tc::tmem_ld32(tmem + lane_off + L_COL + ob * NQ + ch * 32, lv);   // every lane: all 32 column sums
      tc::tmem_ld_wait();
      float ltot = __uint_as_float(lv[0]);
#pragma unroll
      for (int c = 1; c < 32; ++c) ltot = lane == c ? __uint_as_float(lv[c]) : ltot;
      const size_t ldo = (size_t)d.Hq * DH;
      const int dcol = q * 32 + lane;                 // this thread's d_h index (TMEM lane of O^T)
      if (I.ns == 1) {
        // one split: the item holds every key of its rows; normalise and write O (bf16) directly
        tc::fence_before();
        tc::mbar_arrive(&o_empty[ob]);                // O^T / L^T are in registers
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int r = ch * 32 + c;
          if (r < RG) {
            const float l = __uint_as_float(lv[c]);
            d.o[(size_t)(I.row0 + (r >> lg)) * ldo + (size_t)(I.h * G + (r & (G - 1))) * DH + dcol] =
                __float2bfloat16_rn(__uint_as_float(ov[c]) / l);
          }
        }
        tc::named_bar(bar_id, 128);                   // exchange slots are reused by the next item
      } else {
        float* po = d.part_o + (size_t)it * kPartRows * DH + dcol;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int r = ch * 32 + c;
          if (r < RG) po[(size_t)r * DH] = __uint_as_float(ov[c]);
        }
        const int my_slot = ch * 32 + lane;
        if (q == 0 && my_slot < RG) {
          d.part_ml[((size_t)it * kPartRows + my_slot) * 2 + 0] = my_init ? my_m * 0.69314718055994531f : -INFINITY;
          d.part_ml[((size_t)it * kPartRows + my_slot) * 2 + 1] = ltot;
        }
        tc::named_bar(bar_id, 128);                   // exchange slots are reused by the next item
        tc::fence_before();
        tc::mbar_arrive(&o_empty[ob]);
      }
      // Items of a split request leave partials for attn_combine_kernel. A fused merge in the last
      // item of each (request, kv head) to finish was measured (scripts/ab_live.sh, ns, serial ncu):
      // 337 us against 198 + 16 us for this kernel + the combine — the per-thread release fence alone
      // cost 36 us and the merge's L2 round trips stalled the softmax pipeline — so it is not used.
      if (warp == 4 && lane == 0) SV_TR2(7, iter);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

int attn_tc2_smem_bytes() { return SMEM; }

cudaError_t launch_attention_tc2(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                 int num_sms, cudaStream_t s) {
  {
    const cudaError_t e = smem_optin((const void*)attn_tc2_kernel, (int)(SMEM));
    if (e != cudaSuccess) return e;
  }
  SV_COUNT_LAUNCH();
  return launch_pdl(attn_tc2_kernel, dim3(num_sms), dim3(THREADS), SMEM, s, 1, map_q, map_kv, d, layer);
}

}  // namespace sv
