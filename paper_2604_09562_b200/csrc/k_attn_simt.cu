// a3: paged, GQA, chain-causal verify attention — first (SIMT, fp32 FMA) implementation
// with split-KV partials and a combine pass. The tensor-core version replaces the main
// kernel; the work list, partial layout and combine are shared.
//
// Semantics: for request b with cache length L and chain
// rows j = 0..k, query (j, q head hq) attends cache keys 0..L-1 (pages) and chain keys
// 0..j (scratch kc/vc), kv head hq / G, scale 1/sqrt(d_h), softmax.
#include "common.cuh"
#include "lane.h"

namespace sv {

constexpr int AS_KC = 32;   // keys per chunk

__global__ void __launch_bounds__(128) attn_simt_kernel(LaneDev d, int layer) {
  extern __shared__ float smem[];
  const int dh = d.dh, G = d.Hq / d.Hkv;
  float* Qs = smem;                              // [64][dh]
  float* Ks = Qs + kAttnRows * dh;               // [dh][AS_KC + 1] (transposed)
  float* Vs = Ks + dh * (AS_KC + 1);             // [AS_KC][dh]
  float* Ps = Vs + AS_KC * dh;                   // [64][AS_KC]
  float* Ms = Ps + kAttnRows * AS_KC;            // [64] running max
  float* Ls = Ms + kAttnRows;                    // [64] running sum
  float* Cs = Ls + kAttnRows;                    // [64] correction
  const float scale = 1.0f / sqrtf(float(dh));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_items = *d.n_items;
  const size_t nkv = (size_t)d.Hkv * dh;

  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int4 item = d.items[it];
    const int b = item.x, h = item.y, split = item.z;
    const int slot = d.slots[b], R = d.depths[b] + 1, L = d.len[slot];
    const int row0 = d.row_off[b];
    const int nr = R * G;
    const int sk = item_split_keys(item.w);
    const int t0 = split * sk;
    const int t1 = split_t1_k(split, item_ns(item.w), L, R, sk);
    __syncthreads();
    for (int i = tid; i < nr * dh; i += 128) {
      const int rl = i / dh, dd = i % dh, j = rl / G, g = rl % G;
      Qs[i] = bf2f(d.q[((size_t)(row0 + j) * d.Hq + h * G + g) * dh + dd]);
    }
    for (int r = tid; r < kAttnRows; r += 128) { Ms[r] = -INFINITY; Ls[r] = 0.f; }
    const int groups = 128 / dh;                 // 1 (dh=128) or 2 (dh=64)
    const int dd_own = tid % dh, rg = tid / dh;
    float acc[kAttnRows];
#pragma unroll
    for (int i = 0; i < kAttnRows; ++i) acc[i] = 0.f;

    for (int c0 = t0; c0 < t1; c0 += AS_KC) {
      __syncthreads();
      // load K (transposed) and V for keys c0 .. c0+31
      for (int i = tid; i < AS_KC * dh; i += 128) {
        const int kt = i / dh, dd = i % dh, t = c0 + kt;
        float kv = 0.f, vv = 0.f;
        if (t < t1) {
          if (t < L) {
            const int page = d.page_table[slot * d.max_pages_per_slot + t / d.page];
            const size_t base = (((size_t)layer * d.n_pages + page) * 2) * d.Hkv;
            const size_t off = (size_t)(t % d.page) * dh + dd;
            kv = bf2f(d.pool[((base + h) * d.page) * dh + off]);
            vv = bf2f(d.pool[((base + d.Hkv + h) * d.page) * dh + off]);
          } else {
            const size_t crow = (size_t)layer * d.Tmax + row0 + (t - L);
            kv = bf2f(d.kc[crow * nkv + (size_t)h * dh + dd]);
            vv = bf2f(d.vc[crow * nkv + (size_t)h * dh + dd]);
          }
        }
        Ks[dd * (AS_KC + 1) + kt] = kv;
        Vs[kt * dh + dd] = vv;
      }
      __syncthreads();
      // scores S[rl][kt]
      for (int p = tid; p < nr * AS_KC; p += 128) {
        const int rl = p / AS_KC, kt = p % AS_KC, t = c0 + kt, j = rl / G;
        float s = -INFINITY;
        // chain keys: causal (t - L <= j), or the node's ancestors-or-self for a token tree (R30)
        if (t < t1 && (t < L || (d.tree ? ((d.row_anc[row0 + j] >> (t - L)) & 1ull) != 0 : t <= L + j))) {
          float dot = 0.f;
          const float* qr = Qs + rl * dh;
          for (int dd = 0; dd < dh; ++dd) dot = fmaf(qr[dd], Ks[dd * (AS_KC + 1) + kt], dot);
          s = dot * scale;
        }
        Ps[rl * AS_KC + kt] = s;
      }
      __syncthreads();
      // online softmax, one warp per row
      for (int rl = warp; rl < nr; rl += 4) {
        const float s = Ps[rl * AS_KC + lane];
        const float m_old = Ms[rl];
        const float m_new = fmaxf(m_old, warp_max(s));
        const float p = m_new == -INFINITY ? 0.f : expf(s - m_new);
        const float corr = m_new == -INFINITY ? 1.f : expf(m_old - m_new);
        const float ps = warp_sum(p);
        Ps[rl * AS_KC + lane] = p;
        if (lane == 0) { Ms[rl] = m_new; Ls[rl] = Ls[rl] * corr + ps; Cs[rl] = corr; }
      }
      __syncthreads();
      // O[rl][dd] = O * corr + sum_t P V
#pragma unroll
      for (int i = 0; i < kAttnRows; ++i) {
        const int rl = rg + i * groups;
        if (i * groups < kAttnRows && rl < nr) {
          float o = acc[i] * Cs[rl];
#pragma unroll 8
          for (int kt = 0; kt < AS_KC; ++kt) o = fmaf(Ps[rl * AS_KC + kt], Vs[kt * dh + dd_own], o);
          acc[i] = o;
        }
      }
    }
    __syncthreads();
    float* po = d.part_o + (size_t)it * kPartRows * dh;
#pragma unroll
    for (int i = 0; i < kAttnRows; ++i) {
      const int rl = rg + i * groups;
      if (i * groups < kAttnRows && rl < nr) po[rl * dh + dd_own] = acc[i];
    }
    for (int rl = tid; rl < nr; rl += 128) {
      d.part_ml[((size_t)it * kPartRows + rl) * 2 + 0] = Ms[rl];
      d.part_ml[((size_t)it * kPartRows + rl) * 2 + 1] = Ls[rl];
    }
  }
}

cudaError_t launch_attention(const LaneDev& d, int layer, int batch, cudaStream_t s) {
  const size_t smem = sizeof(float) * ((size_t)kAttnRows * d.dh + (size_t)d.dh * (AS_KC + 1) +
                                       (size_t)AS_KC * d.dh + kAttnRows * AS_KC + 3 * kAttnRows);
  {
    const cudaError_t e = smem_optin((const void*)attn_simt_kernel, (int)(100 * 1024));
    if (e != cudaSuccess) return e;
  }
  SV_COUNT_LAUNCH();
  attn_simt_kernel<<<148 * 4, 128, smem, s>>>(d, layer);
  return cudaGetLastError();
}

// combine split-KV partials. One CTA per (chain row, 8 q heads) (the row's chain index, split count
// and first item come from the plan's row table), one warp per q head: lanes over d_h (float4 each
// for d_h = 128, float2 for 64); the loads of up to 4 splits are issued together, with an online
// rescale between chunks of 4 splits. (One CTA per row with two heads per warp iteration ran 1.3
// waves at 3 CTAs per SM: 18.4 us for 48 MB of partials, 29 % occupancy, loads exposed.) O = sum_s e^(m_s - M) O_s / sum_s e^(m_s - M) l_s, M = max m_s.
template <int DH>
__global__ void __launch_bounds__(256, 5) attn_combine_kernel(LaneDev d, int T, int skip_single) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = DH / 32;                       // floats per lane
  constexpr int MS = 4;
  const int r = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the row's (chain row, splits, first item) from the plan's table: one load, issued with the T bound
  const int Tn = *d.T_dev;
  const int4 rc = d.row_comb[r];
  if (r >= Tn) return;                             // launched for Tmax rows (dynamic-depth graph)
  const int j = rc.x, ns = rc.y, s_base = rc.z;
  if (skip_single && ns == 1) return;              // the attention kernel wrote this row's O
  const int G = d.Hq / d.Hkv;
  // HB q heads per warp iteration (w + 8 i), their split loads issued together: a row's loads are
  // then in flight at once instead of one head's after another
  constexpr int HB = 1;
  for (int hq0 = blockIdx.y * 8 + warp; hq0 < d.Hq; hq0 += gridDim.y * 8 * HB) {
    float M[HB], l[HB], o[HB][V];
    const float* po[HB];                           // split s of head hb: po[hb] + s * kPartRows * DH
    const float* pm[HB];
    bool hok[HB];
#pragma unroll
    for (int hb = 0; hb < HB; ++hb) {
      const int hq = hq0 + 8 * hb, h = hq / G, g = hq % G;
      hok[hb] = hq < d.Hq;
      const size_t it0 = (size_t)(s_base + h * ns) * kPartRows + j * G + g;
      po[hb] = d.part_o + it0 * DH + lane * V;
      pm[hb] = d.part_ml + it0 * 2;
      M[hb] = -INFINITY;
      l[hb] = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) o[hb][i] = 0.f;
    }
    for (int s0 = 0; s0 < ns; s0 += MS) {
      float2 ml[HB][MS];
      float v[HB][MS][V];
#pragma unroll
      for (int hb = 0; hb < HB; ++hb) {
#pragma unroll
        for (int k = 0; k < MS; ++k) {
          const int s = s0 + k;
          const bool ok = hok[hb] && s < ns;
          ml[hb][k] = ok ? *reinterpret_cast<const float2*>(pm[hb] + (size_t)s * kPartRows * 2) : make_float2(-INFINITY, 0.f);
          const float* src = po[hb] + (size_t)s * kPartRows * DH;
          if constexpr (V == 4) {
            const float4 x = ok ? *reinterpret_cast<const float4*>(src) : make_float4(0.f, 0.f, 0.f, 0.f);
            v[hb][k][0] = x.x; v[hb][k][1] = x.y; v[hb][k][2] = x.z; v[hb][k][3] = x.w;
          } else {
            const float2 x = ok ? *reinterpret_cast<const float2*>(src) : make_float2(0.f, 0.f);
            v[hb][k][0] = x.x; v[hb][k][1] = x.y;
          }
        }
      }
#pragma unroll
      for (int hb = 0; hb < HB; ++hb) {
        float Mn = M[hb];
#pragma unroll
        for (int k = 0; k < MS; ++k) Mn = fmaxf(Mn, ml[hb][k].x);
        if (Mn == -INFINITY) continue;
        const float sc = M[hb] == -INFINITY ? 0.f : expf(M[hb] - Mn);
        l[hb] *= sc;
#pragma unroll
        for (int i = 0; i < V; ++i) o[hb][i] *= sc;
#pragma unroll
        for (int k = 0; k < MS; ++k) {
          const float w = ml[hb][k].x == -INFINITY ? 0.f : expf(ml[hb][k].x - Mn);
          l[hb] += ml[hb][k].y * w;
#pragma unroll
          for (int i = 0; i < V; ++i) o[hb][i] += v[hb][k][i] * w;
        }
        M[hb] = Mn;
      }
    }
#pragma unroll
    for (int hb = 0; hb < HB; ++hb) {
      const int hq = hq0 + 8 * hb;
      if (hq >= d.Hq) break;
      const float inv = 1.0f / l[hb];
      bf16* dst = d.o + (size_t)r * d.Hq * DH + (size_t)hq * DH + lane * V;
#pragma unroll
      for (int i = 0; i < V; i += 2)
        *reinterpret_cast<__nv_bfloat162*>(dst + i) = __floats2bfloat162_rn(o[hb][i] * inv, o[hb][i + 1] * inv);
    }
  }
}

cudaError_t launch_attn_combine(const LaneDev& d, int T, bool skip_single, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  const dim3 grid(T, (d.Hq + 7) / 8);
  if (d.dh == 128) return launch_pdl(attn_combine_kernel<128>, grid, dim3(256), 0, s, 1, d, T, (int)skip_single);
  return launch_pdl(attn_combine_kernel<64>, grid, dim3(256), 0, s, 1, d, T, (int)skip_single);
}

}  // namespace sv
