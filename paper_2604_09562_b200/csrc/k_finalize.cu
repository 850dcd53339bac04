// a6 + a7: finalize — combine vocab-tile statistics, accept scan (greedy prefix match or
// Leviathan u < p/q), residual / bonus exponential race with counter-based Philox, outputs,
// and the lane acceptance counters. One CTA per request.
//
// Semantics: SURVEY.md §8(c) steps 2-5 (R1-R9):
//   p_{j+1} = softmax(l_j / T);  accept d_j iff u_j < p_j(d_j) / q_j(d_j) (q = 0 -> accept),
//   u_j = U(seed, rid, L + j, ACCEPT);  a = first failure - 1;
//   y = argmax_{x: R(x) > 0} R(x) / (-ln U(seed, rid, L + a + 1, RACE, x)), ties -> lowest x,
//   R = max(0, p_{a+1} - q_{a+1}) (p_{a+1} if that sums to 0) when a < k, else p_{k+1}.
//   Greedy: a = longest prefix with d_j == argmax l_{j-1} (lowest id), y = argmax l_a.
#include <algorithm>

#include <type_traits>

#include "common.cuh"
#include "lane.h"
#include "../../include/sv.h"

namespace sv {

constexpr int FIN_THREADS = 512;
// phase timeline of every CTA (SV_TRACE=1; global timer, rows e of the lane trace buffer, index
// request * 4 + slice < 256): 0 start, 1 after the dependency wait, 2 row statistics, 3 accept scan,
// 4 race loop, 5 slice merge
#define FIN_TR(e)                                                                                 \
  do {                                                                                            \
    if (d.trace && threadIdx.x == 0 && blockIdx.x * 4 + blockIdx.y < 256) {                       \
      unsigned long long t_;                                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                      \
      d.trace[(e)*256 + blockIdx.x * 4 + blockIdx.y] = t_;                                        \
    }                                                                                             \
  } while (0)

SV_DEV float tc_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
SV_DEV float __frcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// -ln U for a race uniform U = ((w >> 9) + 0.5) 2^-23 (normal, in (0, 1)): U = 2^e m with m reduced to
// [sqrt(2)/2, sqrt(2)), ln m = 2 atanh(f / (2 + f)) with f = m - 1 exact (odd series to s^9, |s| <= 0.172,
// truncation < 4e-9 relative) — no special-case handling (U is never 0, denormal, inf or NaN), about half
// the instructions of logf; ~2e-7 relative error, inside the race's borderline band
SV_DEV float neg_log_uniform(uint32_t w) {
  const float u = word_to_uniform(w);
  const int iu = __float_as_int(u);
  int e = (iu >> 23) - 127;
  float m = __int_as_float((iu & 0x007fffff) | 0x3f800000);
  if (m > 1.41421356f) {
    m *= 0.5f;
    e += 1;
  }
  const float f = m - 1.0f;
  const float s = __fdividef(f, 2.0f + f);
  const float s2 = s * s;
  float pl = fmaf(s2, 0.11111111f, 0.14285715f);
  pl = fmaf(s2, pl, 0.2f);
  pl = fmaf(s2, pl, 0.33333334f);
  pl = fmaf(s2, pl, 1.0f);
  const float lnm = 2.0f * s * pl;
  return -fmaf((float)e, 0.69314718f, lnm);
}

struct Best { float s; int x; };
SV_DEV Best better(Best a, Best b) { return (b.s > a.s || (b.s == a.s && b.x < a.x)) ? b : a; }

SV_DEV Best warp_best(Best v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Best w{__shfl_xor_sync(0xffffffffu, v.s, o), __shfl_xor_sync(0xffffffffu, v.x, o)};
    v = better(v, w);
  }
  return v;
}

// ---------------------------------------------------------------- top-k / top-p filter (R31)
// One CTA per chain row: radix select (4 passes of 8 bits, most significant first) of the
// threshold element in (scaled logit desc, id asc) order — the first element at which the kept
// count reaches top_k or the kept mass reaches top_p of the row's mass. Masses are sums of
// e(x) = exp(l_x / T - m) in 2^-40 fixed point (u64), so every decision and S_keep are
// independent of summation order (deterministic). Ties at the threshold key are kept in id
// order up to the count / mass limit. Output per row: threshold key, the largest kept id among
// the ties, 1 / S_keep and the row max m.
constexpr int FLT_THREADS = 512;                 // 4 CTAs (rows) per SM
constexpr int SORT_N = 1024;                     // tile maxima sorted in shared memory (nt <= 1024)
constexpr double kFx = 1099511627776.0;            // 2^40

// e in (0, 1] -> round(e * 2^40): the float product is exact (power-of-two scale), then rounded
SV_DEV unsigned long long fx_mass(float e) { return __float2ull_rn(e * 1099511627776.0f); }

SV_DEV uint32_t flt_key(float v) {
  const uint32_t u = v == 0.0f ? 0u : __float_as_uint(v);     // -0 and +0 are the same value (a tie)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
SV_DEV float key_flt(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); }

constexpr int FLT_CAP = kFiltCap;                 // fast path: candidate capacity (shared memory)
constexpr size_t FLT_SMEM = (FLT_THREADS / 32) * 256 * (8 + 4);   // 48 KB: private histograms / candidates
static_assert(FLT_CAP * 16 + SORT_N * 4 <= FLT_SMEM, "filter candidate buffers exceed the smem budget");

__global__ void __launch_bounds__(FLT_THREADS) filter_kernel(LaneDev d, float inv_temp, int top_k, float top_p) {
  extern __shared__ unsigned long long flt_smem[];
  // slow path: per-warp private histograms [NW][256] (mass u64, count u32)
  unsigned long long* w_mass = flt_smem;
  unsigned int* w_cnt = reinterpret_cast<unsigned int*>(flt_smem + (FLT_THREADS / 32) * 256);
  // fast path (same memory): candidate masses / keys / ids, and the sorted tile maxima
  unsigned long long* c_mass = flt_smem;
  uint32_t* c_key = reinterpret_cast<uint32_t*>(c_mass + FLT_CAP);
  int* c_id = reinterpret_cast<int*>(c_key + FLT_CAP);
  float* srt = reinterpret_cast<float*>(c_id + FLT_CAP);          // [SORT_N]
  __shared__ unsigned int h_cnt[256];
  __shared__ unsigned long long h_mass[256];
  __shared__ float s_redf[FLT_THREADS / 32];
  __shared__ unsigned long long s_redu[FLT_THREADS / 32];
  __shared__ uint32_t s_prefix, s_D;
  __shared__ unsigned int s_cnt_above, s_nc;
  __shared__ unsigned long long s_mass_above, s_target, s_cmass;
  __shared__ int s_tie_lim, s_nkeep, s_fast;
  __shared__ float s_tau, s_S;
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = FLT_THREADS / 32;
  if (r >= *d.T_dev) return;                       // launched for Tmax rows (dynamic-depth graph)
  const int V = d.V, nt = d.nt;
  const float* row = d.logits + (size_t)r * V;
  const float* tmax = d.tile_max + (size_t)r * nt;
  const float* tsum = d.tile_sum + (size_t)r * nt;
  const bool use_k = top_k > 0 && top_k < V, use_p = top_p < 1.0f;

  // 1. tile maxima sorted descending (bitonic, in shared memory): the row max m, and a lower bound
  //    tau on the kept set — the top_k-th largest tile maximum (the k largest tile maxima are k
  //    distinct elements), and the largest tile maximum whose running mass (tile maxima only) already
  //    reaches top_p of the row's mass with a 1e-3 margin. Every kept element is >= tau.
  const bool sortable = nt <= SORT_N;
  float m;
  if (sortable) {
    for (int i = tid; i < SORT_N; i += FLT_THREADS) srt[i] = i < nt ? tmax[i] : -INFINITY;
    __syncthreads();
    for (int k2 = 2; k2 <= SORT_N; k2 <<= 1)          // bitonic: each thread one compare-exchange pair
      for (int j = k2 >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < SORT_N / 2; i += FLT_THREADS) {
          const int lo = 2 * j * (i / j) + (i % j), hi = lo + j;
          const float x = srt[lo], y = srt[hi];
          const bool desc = (lo & k2) == 0;
          if (desc ? (x < y) : (x > y)) { srt[lo] = y; srt[hi] = x; }
        }
        __syncthreads();
      }
    m = srt[0];
  } else {
    float mm = -INFINITY;
    for (int t = tid; t < nt; t += FLT_THREADS) mm = fmaxf(mm, tmax[t]);
    mm = warp_max(mm);
    if (lane == 0) s_redf[warp] = mm;
    __syncthreads();
    m = s_redf[0];
    for (int i = 1; i < nw; ++i) m = fmaxf(m, s_redf[i]);
    __syncthreads();
  }
  if (tid == 0) { s_prefix = 0; s_cnt_above = 0; s_mass_above = 0; s_nc = 0; s_cmass = 0; s_tau = -INFINITY; }
  if (sortable) {
    float tau = -INFINITY;
    if (use_k && top_k <= nt) tau = srt[top_k - 1];
    if (use_p) {
      // S from the tile statistics (fixed summation order: strided per thread, warp butterfly, warps in
      // order), and prefix sums of e(tile max) in sorted order (warp scans)
      float se = 0.f;
      for (int t = tid; t < nt; t += FLT_THREADS) se += tsum[t] * expf(tmax[t] - m);
      se = warp_sum(se);
      if (lane == 0) s_redf[warp] = se;
      __syncthreads();
      float S = 0.f;
      for (int i = 0; i < nw; ++i) S += s_redf[i];
      if (tid == 0) s_S = S;
      static_assert(SORT_N == 2 * FLT_THREADS, "the scan gives each thread two sorted maxima");
      const int i0 = 2 * tid, i1 = i0 + 1;            // a contiguous pair per thread
      const float e0 = i0 < nt ? expf(srt[i0] - m) : 0.f, e1 = i1 < nt ? expf(srt[i1] - m) : 0.f;
      float incl = e0 + e1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      __syncthreads();
      if (lane == 31) s_redf[warp] = incl;
      __syncthreads();
      float before = 0.f;
      for (int i = 0; i < warp; ++i) before += s_redf[i];
      const float c0 = before + incl - e1, c1 = c0 + e1;     // running mass through i0, i1
      __syncthreads();                                 // every warp has read s_redf
      const float need = top_p * S * 1.001f;
      const bool hit0 = i0 < nt && c0 >= need && c0 - e0 < need;   // the first index reaching it
      const bool hit1 = i1 < nt && c1 >= need && c0 < need;
      const bool hit = hit0 || hit1;
      if (hit) s_redf[0] = srt[hit0 ? i0 : i1];         // (at most one thread)
      __syncthreads();
      const bool any = __syncthreads_or(hit);
      if (any) tau = fmaxf(tau, s_redf[0]);
    }
    if (tid == 0) s_tau = tau;
  }
  __syncthreads();
  const float tau = s_tau;

  // 2. one pass over the row: candidates >= tau into shared memory. The total mass for the top-p
  //    target is the tile statistics' S (sortable rows: computed above, in a fixed order), so only
  //    candidates evaluate exp; otherwise every element's fixed-point mass is summed.
  const bool tot_from_tiles = sortable && use_p;
  unsigned long long tot = 0;
  auto visit = [&](float v, int x) {
    if (!tot_from_tiles) tot += v == -INFINITY ? 0ull : fx_mass(expf(v - m));
    if (tau > -INFINITY && v >= tau) {
      const unsigned long long e = fx_mass(expf(v - m));
      const unsigned pos = atomicAdd(&s_nc, 1u);
      if (pos < FLT_CAP) {
        c_key[pos] = flt_key(v);
        c_id[pos] = x;
        c_mass[pos] = e;
        atomicAdd(&s_cmass, e);
      }
    }
  };
  if ((V & 3) == 0) {
    // 16-byte loads (rows are 16-byte aligned when V % 4 == 0), U of them in flight per thread:
    // the pass is load-latency bound, so bytes in flight per load instruction is what counts
    constexpr int U = 4;
    const int V4 = V >> 2;
    const float4* row4 = reinterpret_cast<const float4*>(row);
    for (int x0 = tid; x0 < V4; x0 += FLT_THREADS * U) {
      float4 vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = x0 + u * FLT_THREADS;
        vv[u] = x < V4 ? row4[x] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = 4 * (x0 + u * FLT_THREADS);
        const float4 q = vv[u];
        visit(q.x == -INFINITY ? q.x : q.x * inv_temp, x);
        visit(q.y == -INFINITY ? q.y : q.y * inv_temp, x + 1);
        visit(q.z == -INFINITY ? q.z : q.z * inv_temp, x + 2);
        visit(q.w == -INFINITY ? q.w : q.w * inv_temp, x + 3);
      }
    }
  } else {
    constexpr int U = 8;                               // loads of U elements in flight per thread
    for (int x0 = tid; x0 < V; x0 += FLT_THREADS * U) {
      float vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = x0 + u * FLT_THREADS;
        vv[u] = x < V ? row[x] * inv_temp : -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) visit(vv[u], x0 + u * FLT_THREADS);
    }
  }
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0) s_redu[warp] = tot;
  __syncthreads();
  if (tid == 0) {
    unsigned long long t2 = 0;
    for (int i = 0; i < nw; ++i) t2 += s_redu[i];
    if (tot_from_tiles) t2 = (unsigned long long)((double)s_S * kFx);
    const unsigned long long target = use_p ? (unsigned long long)((double)top_p * (double)t2) : ~0ull;
    s_target = target;
    // the kept set lies inside the candidates iff a limit is reached inside them
    s_fast = tau > -INFINITY && s_nc <= (unsigned)FLT_CAP &&
             ((use_k && s_nc >= (unsigned)top_k) || (use_p && s_cmass >= target));
  }
  __syncthreads();
  const bool fast = s_fast;
  const unsigned nc = s_nc;
  const unsigned long long target = s_target;
  unsigned long long* my_mass = w_mass + warp * 256;
  unsigned int* my_cnt = w_cnt + warp * 256;

  // 3. radix select of the threshold element, 8 bits per pass, most significant first
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    const uint32_t hi_mask = pass == 0 ? 0u : (0xffffffffu << (shift + 8));
    const uint32_t prefix = s_prefix;
    if (fast) {
      for (int i = tid; i < 256; i += FLT_THREADS) { h_cnt[i] = 0; h_mass[i] = 0; }
      __syncthreads();
      for (unsigned i = tid; i < nc; i += FLT_THREADS) {
        const uint32_t k = c_key[i];
        if ((k & hi_mask) == prefix) {
          const int dg = (k >> shift) & 255;
          atomicAdd(&h_cnt[dg], 1u);
          atomicAdd(&h_mass[dg], c_mass[i]);
        }
      }
      __syncthreads();
    } else {
      for (int i = lane; i < 256; i += 32) { my_cnt[i] = 0; my_mass[i] = 0; }
      __syncwarp();
      // warp-aggregated private histograms: lanes with the same digit add count and mass with one
      // reduction (most of a warp in the early passes, where neighbouring logits share an exponent)
      for (int x0 = warp * 32; x0 < V; x0 += FLT_THREADS) {
        const int x = x0 + lane;
        float v = 0.f;
        int dg = -1;
        if (x < V) {
          v = row[x] * inv_temp;
          const uint32_t k = flt_key(v);
          if ((k & hi_mask) == prefix) dg = (k >> shift) & 255;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        if (dg >= 0) {
          const unsigned long long e = fx_mass(expf(v - m));
          const unsigned lo = (unsigned)e, hi = (unsigned)(e >> 32);
          const unsigned s0 = __reduce_add_sync(peers, lo & 0xffffu);
          const unsigned s1 = __reduce_add_sync(peers, lo >> 16);
          const unsigned s2 = __reduce_add_sync(peers, hi);
          if (lane == __ffs(peers) - 1) {
            my_cnt[dg] += (unsigned)__popc(peers);
            my_mass[dg] += (unsigned long long)s0 + ((unsigned long long)s1 << 16) + ((unsigned long long)s2 << 32);
          }
        }
      }
      __syncthreads();
      for (int bin = tid; bin < 256; bin += FLT_THREADS) {     // fixed-order merge of the warps
        unsigned int c = 0;
        unsigned long long ms = 0;
        for (int w = 0; w < nw; ++w) { c += w_cnt[w * 256 + bin]; ms += w_mass[w * 256 + bin]; }
        h_cnt[bin] = c;
        h_mass[bin] = ms;
      }
      __syncthreads();
    }
    if (warp == 0) {
      // walk the digits from the top in parallel: lane l owns digits 255 - 8l .. 248 - 8l; an exclusive
      // warp scan of the lanes' (count, mass) gives the totals above each lane's group, then the lane
      // holding the first digit at which a limit is reached (or the lowest non-empty digit) decides
      const unsigned int c0 = s_cnt_above;
      const unsigned long long ms0 = s_mass_above;
      unsigned int lc = 0;
      unsigned long long lm = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int dg = 255 - 8 * lane - i;
        lc += h_cnt[dg];
        lm += h_mass[dg];
      }
      unsigned int ec = lc;
      unsigned long long em = lm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {               // inclusive scan over lanes (top digits first)
        const unsigned int yc = __shfl_up_sync(0xffffffffu, ec, o);
        const unsigned long long ym = __shfl_up_sync(0xffffffffu, em, o);
        if (lane >= o) { ec += yc; em += ym; }
      }
      unsigned int c = c0 + ec - lc;                   // above this lane's group
      unsigned long long ms = ms0 + em - lm;
      int D = -1;                                      // the digit this lane would decide
      bool hit = false;
      int last_nz = -1;
      unsigned int c_last = 0;
      unsigned long long m_last = 0;
      for (int i = 0; i < 8 && !hit; ++i) {
        const int dg = 255 - 8 * lane - i;
        const unsigned int hc = h_cnt[dg];
        if (!hc) continue;
        const unsigned int c2 = c + hc;
        const unsigned long long m2 = ms + h_mass[dg];
        if ((use_k && c2 >= (unsigned)top_k) || (use_p && m2 >= target)) {
          hit = true;
          D = dg;
        } else {
          last_nz = dg;
          c_last = c;
          m_last = ms;
          c = c2;
          ms = m2;
        }
      }
      const unsigned hits = __ballot_sync(0xffffffffu, hit);
      const unsigned nz = __ballot_sync(0xffffffffu, last_nz >= 0);
      // the first hit in digit order, else the lowest non-empty digit (no limit reached there)
      const int src = hits ? __ffs(hits) - 1 : (nz ? 31 - __clz(nz) : 0);
      const int Dw = __shfl_sync(0xffffffffu, hit ? D : last_nz, src);
      const unsigned int cw = __shfl_sync(0xffffffffu, hit ? c : c_last, src);
      const unsigned long long mw = __shfl_sync(0xffffffffu, hit ? ms : m_last, src);
      __syncwarp();                                    // every lane has read s_cnt_above / s_mass_above
      if (lane == 0) {
        const int Dd = (hits || nz) ? Dw : 0;          // (Dd = 0 unreachable: a limit is always reached)
        s_cnt_above = (hits || nz) ? cw : c0;
        s_mass_above = (hits || nz) ? mw : ms0;
        s_prefix = prefix | (uint32_t(Dd) << shift);
        s_D = Dd;
      }
    }
    __syncthreads();
  }
  // 4. ties at the threshold key: keep them in id order up to the count / mass limit
  if (tid == 0) {
    const unsigned int n_ties = h_cnt[s_D];
    const float vstar = key_flt(s_prefix);
    const unsigned long long e = fx_mass(expf(vstar - m));
    unsigned long long n = n_ties;
    if (use_k) n = min(n, (unsigned long long)(top_k - s_cnt_above));
    if (use_p && e > 0 && target > s_mass_above) {
      const unsigned long long need = (target - s_mass_above + e - 1) / e;   // ceil
      n = min(n, max(1ull, need));
    } else if (use_p) {
      n = 1;
    }
    if (n < 1) n = 1;
    s_nkeep = (int)n;
    s_tie_lim = n >= n_ties ? V : -1;
    const unsigned long long keep = s_mass_above + n * e;
    d.filt_key[r] = s_prefix;
    d.filt_inv[r] = (float)(kFx / (double)keep);
    d.filt_m[r] = m;
  }
  __syncthreads();
  if (s_tie_lim < 0) {                                 // the n-th smallest id among the ties
    const uint32_t kstar = s_prefix;
    const int n = s_nkeep;
    if (fast) {
      for (unsigned i = tid; i < nc; i += FLT_THREADS) {
        if (c_key[i] != kstar) continue;
        int rank = 0;
        for (unsigned j = 0; j < nc; ++j) rank += c_key[j] == kstar && c_id[j] < c_id[i];
        if (rank == n - 1) s_tie_lim = c_id[i];
      }
    } else {
      unsigned int run = 0;                            // (thread 0's running count)
      for (int x0 = 0; x0 < V; x0 += FLT_THREADS) {
        const int x = x0 + tid;
        const bool tie = x < V && flt_key(row[x] * inv_temp) == kstar;
        const unsigned int bal = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) h_cnt[warp] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
          for (int w = 0; w < nw; ++w) {
            if (run + h_cnt[w] >= (unsigned)n) {       // in warp w: the (n - run)-th set lane
              s_D = w;
              s_tie_lim = -2 - (int)(n - run);         // marker: resolve below
              break;
            }
            run += h_cnt[w];
          }
        }
        __syncthreads();
        // every thread reads the marker into a register before anyone overwrites it, so all
        // warps take the same branch (and the same barriers) below
        const int mk = s_tie_lim;
        const int wd = s_D;
        __syncthreads();
        if (mk <= -2) {
          if (warp == wd) {
            const int want = -2 - mk;                  // 1-based rank inside the warp
            const unsigned int before = __popc(bal & ((1u << lane) - 1u));
            if (tie && (int)before + 1 == want) s_tie_lim = x;
          }
          __syncthreads();
          break;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) d.filt_tie[r] = s_tie_lim;
  // the kept ids (fast path: a subset of the candidates), so finalize races over them only — every
  // other token has p' = 0 and can win neither the bonus nor the residual race
  if (fast) {
    __shared__ unsigned int s_nk;
    if (tid == 0) s_nk = 0;
    __syncthreads();
    const uint32_t kstar = s_prefix;
    const int tl = s_tie_lim;
    for (unsigned i = tid; i < nc; i += FLT_THREADS) {
      const uint32_t k = c_key[i];
      const int id = c_id[i];
      if (k > kstar || (k == kstar && id <= tl)) d.filt_ids[(size_t)r * FLT_CAP + atomicAdd(&s_nk, 1u)] = id;
    }
    __syncthreads();
    if (tid == 0) d.filt_cnt[r] = (int)s_nk;
  } else if (tid == 0) {
    d.filt_cnt[r] = -1;                               // slow path: finalize scans the whole row
  }
}

cudaError_t launch_filter(const LaneDev& d, int T, float inv_temp, int top_k, float top_p, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  constexpr size_t smem = FLT_SMEM;
  {
    const cudaError_t e = smem_optin((const void*)filter_kernel, (int)((int)smem));
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(filter_kernel, dim3(T), dim3(FLT_THREADS), smem, s, 1, d, inv_temp, top_k, top_p);
}

// p'(x) of one chain row (R31): e(x) / S_keep on the kept set, else 0. The row's filter
// parameters are loaded once (FiltRow) by loops over the vocabulary.
struct FiltRow { uint32_t key; int tie; float m, inv; };
SV_DEV FiltRow filt_row(const LaneDev& d, int r) { return FiltRow{d.filt_key[r], d.filt_tie[r], d.filt_m[r], d.filt_inv[r]}; }
SV_DEV float filt_p(const FiltRow& f, int x, float lv_scaled) {
  const uint32_t k = flt_key(lv_scaled);
  if (k < f.key || (k == f.key && x > f.tie)) return 0.f;
  return expf(lv_scaled - f.m) * f.inv;
}
SV_DEV float filt_prob(const LaneDev& d, int r, int x, float lv_scaled, float m, float invS) {
  if (!d.filt_on) return expf(lv_scaled - m) * invS;
  return filt_p(filt_row(d, r), x, lv_scaled);
}

// ---------------------------------------------------------------- token trees (R30)
// r(x) at the current node after `nrej` rejected children: r_0 = p_cur, r_i = max(0, r_{i-1} - q_i) / Z_i
// (r_{i-1} when Z_i = 0); q_i = the rejected child's q row, or one-hot at its token
struct TreeResid {
  const LaneDev* d;
  int row;                    // chain row of the current node (top-k / top-p filter parameters)
  bool filt;
  FiltRow fr;
  const float* lrow;          // logits row of the current node
  float m, invS, inv_temp;
  int nrej;
  const int* rej_tok;         // [nrej] tokens of the rejected children
  const float* const* rej_q;  // [nrej] their q rows (nullptr: one-hot)
  const float* invZ;          // [nrej] (0: Z was 0, keep r)
};

SV_DEV float tree_r(const TreeResid& t, int x) {
  const float lv = t.lrow[x] * t.inv_temp;
  float r = t.filt ? filt_p(t.fr, x, lv) : expf(lv - t.m) * t.invS;
  for (int i = 0; i < t.nrej; ++i) {
    if (t.invZ[i] == 0.f) continue;
    const float q = t.rej_q[i] ? t.rej_q[i][x] : (x == t.rej_tok[i] ? 1.0f : 0.0f);
    r = fmaxf(0.f, r - q) * t.invZ[i];
  }
  return r;
}

// The tree walk of one request (called by the whole CTA). Greedy: first child (ascending index)
// whose token is the argmax. Sampled: recursive rejection over the children in index order, a
// vocabulary pass per rejection for its normaliser Z, then the exponential race over the final r.
// Writes the path (s_path[0..a]), a, indep and y.
__device__ void tree_walk(const LaneDev& d, const int* __restrict__ drafts, const int* __restrict__ parents,
                          const float* __restrict__ probs, const float* __restrict__ logits, uint64_t seed, int mode,
                          float inv_temp, int b, int k, int r0, int doff, int L, unsigned long long rid,
                          const float* s_m, const float* s_S, const int* s_top, int* s_path, int* s_a, int* s_indep,
                          int* s_y) {
  __shared__ int s_dep[kMaxDepth + 1], s_rank[kMaxDepth + 1];
  __shared__ int s_cur, s_nrej, s_scan, s_act, s_cand;
  __shared__ int s_rej_tok[kMaxDepth];
  __shared__ const float* s_rej_q[kMaxDepth];
  __shared__ float s_invZ[kMaxDepth];
  __shared__ float s_red[FIN_THREADS / 32];
  __shared__ Best s_best[FIN_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = FIN_THREADS / 32;
  const size_t V = d.V;
  const int* par = parents + doff;                 // parent of node n at par[n - 1]
  const int* tok = drafts + doff;
  if (tid == 0) {
    s_dep[0] = 0;
    s_rank[0] = 0;
    int bad = 0;
    for (int n = 1; n <= k; ++n) {
      const int p = par[n - 1];
      if (p < 0 || p >= n) { bad = 1; s_dep[n] = 0; s_rank[n] = 0; continue; }   // plan flagged it
      s_dep[n] = s_dep[p] + 1;
      int rk = 0;
      for (int c = p + 1; c < n; ++c) rk += par[c - 1] == p;
      s_rank[n] = rk;
    }
    int indep = 0;
    if (!bad) {
      for (int n = 1; n <= k; ++n) {                 // every node's own test against its parent's target
        const int p = par[n - 1], x = tok[n - 1];
        if (mode == SV_GREEDY) {
          indep += x == s_top[p];
        } else {
          const float lv = logits[(size_t)(r0 + p) * V + x] * inv_temp;
          const float pv = d.filt_on ? filt_prob(d, r0 + p, x, lv, s_m[p], 1.0f / s_S[p]) : expf(lv - s_m[p]) / s_S[p];
          const float qd = probs ? probs[(size_t)(doff + n - 1) * V + x] : 1.0f;
          const float u = uniform_accept_rank(seed, rid, uint32_t(L + s_dep[p] + 1), uint32_t(s_rank[n]));
          indep += (qd == 0.0f) || (u < pv / qd);
        }
      }
    }
    *s_indep = indep;
    s_cur = 0;
    s_nrej = 0;
    s_scan = 1;
    s_path[0] = 0;
    *s_a = 0;
    if (bad) k = 0;                                  // no walk: outputs are masked by req_err anyway
    s_cand = k;                                      // (carries the possibly-zeroed k to all threads)
  }
  __syncthreads();
  k = s_cand;
  __syncthreads();                                   // every thread has read s_cand before thread 0 reuses it
  if (mode == SV_GREEDY) {
    if (tid == 0) {
      int cur = 0, a = 0;
      for (;;) {
        const int y = s_top[cur];
        int nx = -1;
        for (int c = cur + 1; c <= k; ++c)
          if (par[c - 1] == cur && tok[c - 1] == y) { nx = c; break; }
        if (nx < 0) break;
        cur = nx;
        s_path[++a] = cur;
      }
      *s_a = a;
      *s_y = s_top[cur];
    }
    __syncthreads();
    return;
  }
  // sampled: block-uniform loop; thread 0 decides, everyone joins the vocabulary passes
  for (;;) {
    if (tid == 0) {
      const int cur = s_cur;
      int c = s_scan;
      while (c <= k && par[c - 1] != cur) ++c;       // next untried child of cur
      if (c > k) {
        s_act = 0;                                   // no child left: race over r
      } else {
        s_scan = c + 1;
        const int x = tok[c - 1];
        TreeResid t{&d, r0 + cur, d.filt_on != 0, d.filt_on ? filt_row(d, r0 + cur) : FiltRow{},
                    logits + (size_t)(r0 + cur) * V, s_m[cur], 1.0f / s_S[cur], inv_temp, s_nrej, s_rej_tok, s_rej_q,
                    s_invZ};
        const float rv = tree_r(t, x);
        const float qd = probs ? probs[(size_t)(doff + c - 1) * V + x] : 1.0f;
        const float u = uniform_accept_rank(seed, rid, uint32_t(L + s_dep[cur] + 1), uint32_t(s_nrej));
        if (qd == 0.0f || u < rv / qd) {
          s_cur = c;
          s_nrej = 0;
          s_scan = c + 1;                            // children have larger indices
          s_path[++*s_a] = c;
          s_act = 1;
        } else {
          s_cand = c;
          s_act = 2;                                 // rejected: normaliser of max(0, r - q_c)
        }
      }
    }
    __syncthreads();
    const int act = s_act;
    __syncthreads();                                 // everyone has read s_act before thread 0 rewrites it
    if (act == 1) continue;
    const int cur = s_cur, nrej = s_nrej;
    TreeResid t{&d, r0 + cur, d.filt_on != 0, d.filt_on ? filt_row(d, r0 + cur) : FiltRow{},
                logits + (size_t)(r0 + cur) * V, s_m[cur], 1.0f / s_S[cur], inv_temp, nrej, s_rej_tok, s_rej_q, s_invZ};
    if (act == 2) {
      const int c = s_cand, xc = tok[c - 1];
      const float* qc = probs ? probs + (size_t)(doff + c - 1) * V : nullptr;
      float z = 0.f;
      for (int x = tid; x < (int)V; x += FIN_THREADS)
        z += fmaxf(0.f, tree_r(t, x) - (qc ? qc[x] : (x == xc ? 1.0f : 0.0f)));
      z = warp_sum(z);
      if (lane == 0) s_red[warp] = z;
      __syncthreads();
      if (tid == 0) {
        float Z = 0.f;
        for (int i = 0; i < nw; ++i) Z += s_red[i];
        s_rej_tok[nrej] = xc;
        s_rej_q[nrej] = qc;
        s_invZ[nrej] = Z > 0.f ? 1.0f / Z : 0.f;
        s_nrej = nrej + 1;
      }
      __syncthreads();
      continue;
    }
    // race: y = argmax_{x: r(x) > 0} r(x) / E_x at z = L + depth(cur) + 1
    const uint32_t z = uint32_t(L + s_dep[cur] + 1);
    Best best{-INFINITY, 0x7fffffff};
    const int nm = (int)((V + 3) / 4);
    for (int mm = tid; mm < nm; mm += FIN_THREADS) {
      const u32x4 w = race_words(seed, rid, z, uint32_t(mm));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int x = mm * 4 + l;
        if (x >= (int)V) break;
        const float r = tree_r(t, x);
        const float invE = __frcp_rn(-logf(word_to_uniform(ws[l])));   // score r / E as r * (1/E):
        best = better(best, Best{r > 0.f ? r * invE : -INFINITY, x});  // no fp32 division slow path
      }
    }
    best = warp_best(best);
    if (lane == 0) s_best[warp] = best;
    __syncthreads();
    if (tid == 0) {
      Best B = s_best[0];
      for (int i = 1; i < nw; ++i) B = better(B, s_best[i]);
      *s_y = B.x;
    }
    __syncthreads();
    return;
  }
}

// Greedy chain decisions from the row_best keys (one warp): lane j < 32 holds chain row j (and j + 32
// for k = 32); draft j + 1 = drafts[doff + j] is accepted iff it equals row j's argmax; a = the first
// rejection (k if none), the emitted token after the accepted drafts = row a's argmax (SURVEY.md
// §8(a) a6, greedy). Outputs and counters as the generic path below writes them.
__device__ __forceinline__ void finalize_greedy_warp(const LaneDev& d, const int* __restrict__ drafts, int b,
                                                  int* __restrict__ acc_out, int* __restrict__ tok_out,
                                                  int* __restrict__ nodes_out) {
  const int lane = threadIdx.x & 31;
  const int k = d.depths[b], r0 = d.row_off[b], doff = r0 - b, err = d.req_err[b];
  const int K1 = d.max_depth + 1;
  int top[2], drf[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 32 * h;
    top[h] = -1;
    drf[h] = -1;
    if (j <= k) {
      const unsigned long long key = d.row_best[r0 + j];
      top[h] = (int)(0xFFFFFFFFu - (uint32_t)key);
    }
    if (j < k) drf[h] = drafts[doff + j];
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (lane + 32 * h <= k) d.row_best[r0 + lane + 32 * h] = 0ull;   // zero for the next verify
  const bool acc = lane < k && drf[0] == top[0];                       // k <= 32: tests j = 1..k on lanes 0..k-1
  const unsigned kmask = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
  const unsigned okm = __ballot_sync(0xffffffffu, acc) & kmask;
  const unsigned fail = ~okm & kmask;
  const int a = fail ? __ffs(fail) - 1 : k;
  const int y = a < 32 ? __shfl_sync(0xffffffffu, top[0], a & 31) : __shfl_sync(0xffffffffu, top[1], 0);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    if (i >= K1) continue;
    const int t = err ? -1 : (i < a ? drf[h] : (i == a ? y : -1));
    const int nd = (!err && i <= a) ? i : -1;
    tok_out[(size_t)b * K1 + i] = t;
    if (d.tok_int) d.tok_int[(size_t)b * K1 + i] = t;
    if (d.path_int) d.path_int[(size_t)b * K1 + i] = nd;
    if (nodes_out) nodes_out[(size_t)b * K1 + i] = nd;
  }
  if (lane == 0) {
    acc_out[b] = err ? -1 : a;
    if (d.acc_int) d.acc_int[b] = err ? -1 : a;
    if (b == 0) atomicAdd(&d.stats[ST_STEPS], 1ull);
    if (!err) {
      atomicAdd(&d.stats[ST_ROWS], (unsigned long long)(k + 1));
      atomicAdd(&d.stats[ST_DRAFTED], (unsigned long long)k);
      atomicAdd(&d.stats[ST_ACCEPTED], (unsigned long long)a);
      atomicAdd(&d.stats[ST_EMITTED], (unsigned long long)(a + 1));
      atomicAdd(&d.stats[ST_INDEP], (unsigned long long)__popc(okm));
      atomicAdd(&d.stats[ST_HIST + a], 1ull);
      atomicAdd(&d.stats[ST_DRAFTED_BY_K + k], (unsigned long long)k);
      atomicAdd(&d.stats[ST_ACCEPTED_BY_K + k], (unsigned long long)a);
    }
  }
}

__global__ void __launch_bounds__(FIN_THREADS, 2) finalize_kernel(LaneDev d, const int* __restrict__ drafts,
                                                                const int* __restrict__ parents,
                                                                const float* __restrict__ probs,
                                                                const float* __restrict__ logits, uint64_t seed,
                                                                int mode, float inv_temp, int* __restrict__ acc_out,
                                                                int* __restrict__ tok_out, int* __restrict__ nodes_out,
                                                                int use_row_best) {
  __shared__ float s_m[kMaxDepth + 1], s_S[kMaxDepth + 1];
  __shared__ int s_top[kMaxDepth + 1];
  __shared__ int s_a, s_indep, s_y, s_resid;
  __shared__ Best s_bestR[FIN_THREADS / 32], s_bestP[FIN_THREADS / 32];
  __shared__ float s_sumR[FIN_THREADS / 32];
  __shared__ int s_path[kMaxDepth + 1];             // accepted path (chain rows); identity for chains
  __shared__ int s_tb[kMaxDepth + 1];               // row statistics: tile of each row's max
  __shared__ float s_rm[FIN_THREADS / 32][8], s_rs[FIN_THREADS / 32][8];
  __shared__ int s_rt[FIN_THREADS / 32][8];

  FIN_TR(0);
  pdl_trigger();
  pdl_wait();
  FIN_TR(1);
  const int b = blockIdx.x;
  if (!parents && mode == SV_GREEDY && use_row_best) {
    // greedy chains (the lm-head epilogue left each row's argmax key): warp 0 alone, lane j holding
    // row j's argmax and draft j, the accept scan by one ballot (every load in one round trip)
    if (threadIdx.x >= 32) return;
    finalize_greedy_warp(d, drafts, b, acc_out, tok_out, nodes_out);
    return;
  }
  const int k = d.depths[b], slot = d.slots[b], r0 = d.row_off[b], doff = r0 - b;
  const int L = d.len[slot];
  const unsigned long long rid = d.rid[slot];
  const int err = d.req_err[b];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = FIN_THREADS / 32;
  const size_t V = d.V;

  // an intermediate prefill chunk (no lm-head ran): every row is kept and no token is predicted
  const bool nohead = mode == kPrefillNoHead;
  if (nohead) mode = SV_PREFILL;
  // 1. each chain row's argmax (and, for sampled decisions, max and sum of exp). Greedy / prefill
  //    with use_row_best: one word per row from the lm-head epilogue's atomicMax key (lowest-index
  //    argmax over the vocab tiles), reset here for the next verify. Otherwise combine the row's
  //    vocab-tile statistics (warp per row): one online pass, loads batched 8 deep per lane.
  if (use_row_best && !nohead && mode != SV_SAMPLE) {
    for (int j = tid; j <= k; j += FIN_THREADS) {
      const unsigned long long key = d.row_best[r0 + j];
      s_top[j] = (int)(0xFFFFFFFFu - (uint32_t)key);
      d.row_best[r0 + j] = 0ull;
    }
  }
  // Otherwise the whole CTA combines the vocab-tile statistics of up to 8 rows at a time: thread t
  // takes tiles t, t + 512, ... of every row (all loads of a group in flight together), folds them
  // online, then a warp butterfly and an in-order merge of the 16 warps; the row's argmax is the tile
  // argmax of its lowest max tile (tiles are in vocabulary order), looked up at the end.
  if (!(nohead || (use_row_best && mode != SV_SAMPLE))) {
    // per row: the block max M first (fmax trees: no exponentials), then sum_t s_t e^(m_t - M) with
    // one exponential per tile, and the lowest tile attaining M (its tile argmax is the row's argmax)
    const int nt = d.nt;
    constexpr int RG = 5;                                 // rows per group (loads of a group in flight together)
    constexpr int TPT = 2;                                // tiles per thread per sweep
    for (int j0 = 0; j0 <= k; j0 += RG) {
      float mt[RG];
#pragma unroll
      for (int jj = 0; jj < RG; ++jj) mt[jj] = -INFINITY;
      // pass 1: maxima (the loads stay in registers when nt <= TPT * FIN_THREADS)
      float vm[RG][TPT], vs[RG][TPT];
      const bool one_sweep = nt <= TPT * FIN_THREADS;
      for (int i0 = 0; i0 < nt; i0 += TPT * FIN_THREADS) {
#pragma unroll
        for (int jj = 0; jj < RG; ++jj)
#pragma unroll
          for (int i = 0; i < TPT; ++i) {
            const int j = j0 + jj, t = i0 + tid + i * FIN_THREADS;
            const bool ok = j <= k && t < nt;
            vm[jj][i] = ok ? d.tile_max[(size_t)(r0 + j) * nt + t] : -INFINITY;
            vs[jj][i] = ok ? d.tile_sum[(size_t)(r0 + j) * nt + t] : 0.f;
            mt[jj] = fmaxf(mt[jj], vm[jj][i]);
          }
      }
      if (j0 == 0) FIN_TR(6);
#pragma unroll
      for (int jj = 0; jj < RG; ++jj) {
        float m = mt[jj];
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) s_rm[warp][jj] = m;
      }
      __syncthreads();
      if (j0 == 0) FIN_TR(7);
      float M[RG];
#pragma unroll
      for (int jj = 0; jj < RG; ++jj) {                   // lanes 0..15 hold the 16 warps' maxima
        float m = s_rm[lane & 15][jj];
#pragma unroll
        for (int o = 8; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        M[jj] = m;
      }
      if (j0 == 0) FIN_TR(8);
      // pass 2: scaled sums and the lowest max tile (reloading only when the row did not fit one sweep)
      float St[RG];
      int tb[RG];
#pragma unroll
      for (int jj = 0; jj < RG; ++jj) {
        St[jj] = 0.f;
        tb[jj] = 0x7fffffff;
      }
      for (int i0 = 0; i0 < nt; i0 += TPT * FIN_THREADS) {
#pragma unroll
        for (int jj = 0; jj < RG; ++jj)
#pragma unroll
          for (int i = 0; i < TPT; ++i) {
            const int j = j0 + jj, t = i0 + tid + i * FIN_THREADS;
            const bool ok = j <= k && t < nt;
            if (!one_sweep) {
              vm[jj][i] = ok ? d.tile_max[(size_t)(r0 + j) * nt + t] : -INFINITY;
              vs[jj][i] = ok ? d.tile_sum[(size_t)(r0 + j) * nt + t] : 0.f;
            }
            if (vm[jj][i] != -INFINITY) St[jj] += vs[jj][i] * tc_ex2((vm[jj][i] - M[jj]) * 1.4426950408889634f);
            if (ok && vm[jj][i] == M[jj] && t < tb[jj]) tb[jj] = t;
          }
      }
#pragma unroll
      for (int jj = 0; jj < RG; ++jj) {
        float S = St[jj];
        int t = tb[jj];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          S += __shfl_xor_sync(0xffffffffu, S, o);
          t = min(t, __shfl_xor_sync(0xffffffffu, t, o));
        }
        if (lane == 0) {
          s_rs[warp][jj] = S;
          s_rt[warp][jj] = t;
        }
      }
      __syncthreads();
      if (warp == 0) {                                    // warps summed in a fixed tree order (deterministic)
#pragma unroll
        for (int jj = 0; jj < RG; ++jj) {
          float S = lane < nw ? s_rs[lane][jj] : 0.f;
          int t = lane < nw ? s_rt[lane][jj] : 0x7fffffff;
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            S += __shfl_xor_sync(0xffffffffu, S, o);
            t = min(t, __shfl_xor_sync(0xffffffffu, t, o));
          }
          if (lane == jj && j0 + jj <= k) {
            s_m[j0 + jj] = M[jj];
            s_S[j0 + jj] = S;
            s_tb[j0 + jj] = t;
          }
        }
      }
      __syncthreads();
      if (j0 == 0) FIN_TR(9);
    }
    if (tid <= k) s_top[tid] = s_tb[tid] < nt ? d.tile_arg[(size_t)(r0 + tid) * nt + s_tb[tid]] : 0;
  }
  __syncthreads();

  FIN_TR(2);
  // 2. accept scan (serial over k <= 32)
  if (parents) {
    tree_walk(d, drafts, parents, probs, logits, seed, mode, inv_temp, b, k, r0, doff, L, rid, s_m, s_S, s_top,
              s_path, &s_a, &s_indep, &s_y);
  } else if (tid == 0 && mode != SV_SAMPLE) {
    int a = k, indep = 0;
    if (mode == SV_PREFILL) {                      // R29: the chunk's rows are all kept
      s_y = nohead ? -1 : s_top[k];
    } else if (mode == SV_GREEDY) {
      for (int j = 1; j <= k; ++j) {
        const bool acc = drafts[doff + j - 1] == s_top[j - 1];
        indep += acc;
        if (!acc && a == k) a = j - 1;
      }
      s_y = s_top[a];
    }
    s_a = a;
    s_indep = indep;
    s_resid = 0;
    for (int i = 0; i <= a; ++i) s_path[i] = i;
  }
  if (!parents && mode == SV_SAMPLE && warp == 0) {
    // the k <= 32 accept tests are independent: lane j - 1 evaluates test j (its loads and its
    // Philox draw in parallel), a = index of the first failing lane (k if none)
    const int j = lane + 1;
    bool acc = true;
    if (j <= k) {
      const int dj = drafts[doff + j - 1];
      const float lg = logits[(size_t)(r0 + j - 1) * V + dj];
      const float qd = probs ? probs[(size_t)(doff + j - 1) * V + dj] : 1.0f;
      const float pd = d.filt_on ? filt_prob(d, r0 + j - 1, dj, lg * inv_temp, s_m[j - 1], 1.0f / s_S[j - 1])
                                 : expf(lg * inv_temp - s_m[j - 1]) / s_S[j - 1];
      const float u = uniform_accept(seed, rid, uint32_t(L + j));
      acc = (qd == 0.0f) || (u < pd / qd);
    }
    const unsigned kmask = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
    const unsigned okm = __ballot_sync(0xffffffffu, acc) & kmask;
    const unsigned fail = ~okm & kmask;
    const int a = fail ? __ffs(fail) - 1 : k;
    if (lane == 0) {
      s_a = a;
      s_indep = __popc(okm);
      s_resid = a < k;
    }
    if (lane <= a) s_path[lane] = lane;
    if (a == 32 && lane == 0) s_path[32] = 32;
  }
  __syncthreads();
  const int a = s_a;

  // 3. exponential race over the one selected row (sampled chains; trees race inside tree_walk)
  FIN_TR(3);
  if (mode == SV_SAMPLE && !parents) {

    const bool resid = s_resid;
    const float* lrow = logits + (size_t)(r0 + a) * V;
    const float m = s_m[a], invS = 1.0f / s_S[a];
    const float* qrow = (resid && probs) ? probs + (size_t)(doff + a) * V : nullptr;
    const int dnext = resid ? drafts[doff + a] : -1;
    const uint32_t z = uint32_t(L + a + 1);
    const bool filt = d.filt_on != 0;
    const FiltRow fr = filt ? filt_row(d, r0 + a) : FiltRow{};
    Best bR{-INFINITY, 0x7fffffff}, bP{-INFINITY, 0x7fffffff};
    float sumR = 0.f;
    const int nm = (int)((V + 3) / 4);
    const int RS = gridDim.y, sidx = blockIdx.y;      // vocabulary slice of this CTA (race words of 4)
    const int per = (nm + RS - 1) / RS, m_lo = sidx * per, m_hi = min(nm, m_lo + per);
    // 4 vocabulary entries per Philox word; rows are 16-byte aligned when V % 4 == 0, then the logits
    // and q of a word come in one float4 each, and two words per thread are in flight
    const bool vec = (V & 3) == 0;
    auto race4 = [&](int mm, const float4 l4, const float4 q4) {
      const u32x4 w = race_words(seed, rid, z, uint32_t(mm));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
      const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int x = mm * 4 + l;
        if (x >= (int)V) break;
        const float p = filt ? filt_p(fr, x, lv[l] * inv_temp) : expf(lv[l] * inv_temp - m) * invS;
        // score p / E as p * (1/E): one correctly rounded reciprocal per entry, and no division,
        // whose special-case path (zero numerators: filtered or zero residual mass) dominated
        const float invE = __frcp_rn(-logf(word_to_uniform(ws[l])));
        bP = better(bP, Best{p > 0.f ? p * invE : -INFINITY, x});
        if (resid) {
          const float q = qrow ? qv[l] : (x == dnext ? 1.0f : 0.0f);
          const float R = fmaxf(0.f, p - q);
          sumR += R;
          bR = better(bR, Best{R > 0.f ? R * invE : -INFINITY, x});
        }
      }
    };
    auto load4 = [&](const float* row, int mm) {
      if (vec) return *reinterpret_cast<const float4*>(row + mm * 4);
      float t[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) t[l] = mm * 4 + l < (int)V ? row[mm * 4 + l] : 0.f;
      return make_float4(t[0], t[1], t[2], t[3]);
    };
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const int nkept = filt ? d.filt_cnt[r0 + a] : -1;
    if (filt && nkept >= 0) {
      // filtered target with a kept-id list (the filter's fast path): race over those ids only; this
      // CTA takes slice sidx of the list. Ties keep the lower id (better()), so the list order is moot.
      const int* ids = d.filt_ids + (size_t)(r0 + a) * FLT_CAP;
      const int per_l = (nkept + RS - 1) / RS, lo_l = sidx * per_l, hi_l = min(nkept, lo_l + per_l);
      for (int i = lo_l + tid; i < hi_l; i += FIN_THREADS) {
        const int x = ids[i];
        const float lv = lrow[x];
        const float p = filt_p(fr, x, lv * inv_temp);
        const u32x4 w = race_words(seed, rid, z, uint32_t(x >> 2));
        const uint32_t wl = (x & 3) == 0 ? w.x : ((x & 3) == 1 ? w.y : ((x & 3) == 2 ? w.z : w.w));
        const float invE = __frcp_rn(-logf(word_to_uniform(wl)));
        bP = better(bP, Best{p > 0.f ? p * invE : -INFINITY, x});
        if (resid) {
          const float q = qrow ? qrow[x] : (x == dnext ? 1.0f : 0.0f);
          const float R = fmaxf(0.f, p - q);
          sumR += R;
          bR = better(bR, Best{R > 0.f ? R * invE : -INFINITY, x});
        }
      }
    } else if (vec && !filt) {
      // fast path (16-byte rows, no filter): p = 2^(l*it*log2e - m*log2e) / S with ex2.approx, 1 / E by
      // rcp.approx (the race is decided against the oracle's fp64 scores; both approximations are ~1e-7
      // relative, far inside the borderline band), and strict > comparisons (a thread visits x in
      // increasing order, so a tie keeps the lower id)
      const float itl = inv_temp * 1.4426950408889634f, ml = m * 1.4426950408889634f;
      // Pruning (exact, two levels):
      //  * E = -ln U >= -ln(1 - 2^-24) for every lattice uniform, so an entry's computed score p / E is at
      //    most p * 1.6777216e7 (1 + 1e-6); a Philox word (4 entries) none of whose entries can reach the
      //    lane's current bests under that cap needs no random numbers at all. Lanes push the words that
      //    do need them into a per-warp queue (ballot + prefix), and full warps drain it, so Philox runs
      //    for the needed words only instead of for every word a diverged warp touches.
      //  * E >= 1 - U: with the word's uniforms an entry whose p / (1 - U) (with a 1e-5 margin over the
      //    ~3e-7 relative error of the log / reciprocal approximations) falls below the best skips them.
      // Every lane starts from the exact scores of the row's argmax x* (tile statistics), usually the
      // winner or close to it. Pruned entries score strictly below a kept one, so the argmax (lowest id
      // on ties) is the unpruned race's; sum R is accumulated over every entry in the lane's order.
      constexpr float kPruneMargin = 1.00001f;
      constexpr float kInvEmax = 1.6777216e7f * 1.0001f;
      const int xs = s_top[a];
      auto fast = [&](auto resid_t, auto qrow_t) {
        constexpr bool RES = decltype(resid_t)::value, QR = decltype(qrow_t)::value;
        float sR = -INFINITY, sP = -INFINITY, sum = 0.f;
        int xR = 0x7fffffff, xP = 0x7fffffff;
        if (xs >= 0 && xs < (int)V) {                 // seed: x*'s exact scores (same arithmetic as below)
          const u32x4 w = race_words(seed, rid, z, uint32_t(xs >> 2));
          const uint32_t wl = (xs & 3) == 0 ? w.x : ((xs & 3) == 1 ? w.y : ((xs & 3) == 2 ? w.z : w.w));
          const float pv = tc_ex2(fmaf(lrow[xs], itl, -ml)) * invS;
          const float invE = __frcp_approx(neg_log_uniform(wl));
          sP = pv * invE;
          xP = xs;
          if constexpr (RES) {
            const float q = QR ? qrow[xs] : (xs == dnext ? 1.0f : 0.0f);
            const float R = fmaxf(0.f, pv - q);
            if (R > 0.f) {
              sR = R * invE;
              xR = xs;
            }
          }
        }
        auto word = [&](int mm, bool valid, const float4 l4, const float4 q4) {
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
          const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
          float pv[4], rv[4];
          bool any = false;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const int x = mm * 4 + l;
            pv[l] = valid ? tc_ex2(fmaf(lv[l], itl, -ml)) * invS : 0.f;
            any |= pv[l] * kInvEmax > sP;
            rv[l] = 0.f;
            if constexpr (RES) {
              const float q = QR ? qv[l] : (x == dnext ? 1.0f : 0.0f);
              rv[l] = fmaxf(0.f, pv[l] - q);
              sum += rv[l];
              any |= rv[l] > 0.f && rv[l] * kInvEmax > sR;
            }
          }
          any = any && valid;
          if (!__any_sync(0xffffffffu, any)) return;  // no lane's word can reach its bests: no Philox
          const u32x4 w = race_words(seed, rid, z, uint32_t(mm));
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const int x = mm * 4 + l;
            const float om = 1.0f - word_to_uniform(ws[l]);  // exact (U is a multiple of 2^-24)
            bool need = pv[l] * kPruneMargin > sP * om;
            if constexpr (RES) need |= rv[l] > 0.f && rv[l] * kPruneMargin > sR * om;
            if (need && valid) {
              const float invE = __frcp_approx(neg_log_uniform(ws[l]));
              const float sc = pv[l] * invE;
              if (sc > sP || (sc == sP && x < xP)) { sP = sc; xP = x; }
              if constexpr (RES) {
                const float scr = rv[l] > 0.f ? rv[l] * invE : -INFINITY;
                if (scr > sR || (scr == sR && x < xR)) { sR = scr; xR = x; }
              }
            }
          }
        };
        // warp-uniform loop (the Philox skip is a warp vote): lane l takes words mm0 + l and mm0 + 512 + l
        for (int mm0 = m_lo + warp * 32; mm0 < m_hi; mm0 += 2 * FIN_THREADS) {
          const int mm = mm0 + lane, mm2 = mm + FIN_THREADS;
          const bool one = mm < m_hi, two = mm2 < m_hi;
          const float4 l0 = one ? *reinterpret_cast<const float4*>(lrow + mm * 4) : zero4;
          const float4 l1 = two ? *reinterpret_cast<const float4*>(lrow + mm2 * 4) : zero4;
          const float4 q0 = (QR && one) ? *reinterpret_cast<const float4*>(qrow + mm * 4) : zero4;
          const float4 q1 = (QR && two) ? *reinterpret_cast<const float4*>(qrow + mm2 * 4) : zero4;
          word(mm, one, l0, q0);
          if (mm0 + FIN_THREADS < m_hi) word(mm2, two, l1, q1);    // warp-uniform condition
        }
        bP = Best{sP, xP};
        bR = Best{sR, xR};
        sumR = sum;
      };
      if (!resid) fast(std::false_type{}, std::false_type{});
      else if (qrow) fast(std::true_type{}, std::true_type{});
      else fast(std::true_type{}, std::false_type{});
    } else
    for (int mm = m_lo + tid; mm < m_hi; mm += 2 * FIN_THREADS) {
      const int mm2 = mm + FIN_THREADS;
      const bool two = mm2 < m_hi;
      const float4 l0 = load4(lrow, mm);
      const float4 l1 = two ? load4(lrow, mm2) : zero4;
      const float4 q0 = qrow ? load4(qrow, mm) : zero4;
      const float4 q1 = (qrow && two) ? load4(qrow, mm2) : zero4;
      race4(mm, l0, q0);
      if (two) race4(mm2, l1, q1);
    }
    FIN_TR(4);
    bR = warp_best(bR);
    bP = warp_best(bP);
    sumR = warp_sum(sumR);
    if (lane == 0) { s_bestR[warp] = bR; s_bestP[warp] = bP; s_sumR[warp] = sumR; }
    __syncthreads();
    __shared__ int s_last;
    if (tid == 0) {
      Best R = s_bestR[0], P = s_bestP[0];
      float sr = s_sumR[0];
      for (int i = 1; i < nw; ++i) { R = better(R, s_bestR[i]); P = better(P, s_bestP[i]); sr += s_sumR[i]; }
      s_last = 1;
      if (RS > 1) {
        // split race: publish this vocabulary slice's bests; the last CTA of the request to finish
        // merges the slices in slice order (deterministic) and writes the outputs
        RacePart* part = d.fin_part + (size_t)b * kMaxRaceSplits;
        part[sidx] = RacePart{R.s, R.x, P.s, P.x, sr};
        __threadfence();
        s_last = atomicAdd(&d.fin_cnt[b], 1) == RS - 1;
        if (s_last) {
          __threadfence();
          volatile RacePart* vp = part;
          R = Best{vp[0].rs, vp[0].rx};
          P = Best{vp[0].ps, vp[0].px};
          sr = vp[0].sr;
          for (int i = 1; i < RS; ++i) {
            R = better(R, Best{vp[i].rs, vp[i].rx});
            P = better(P, Best{vp[i].ps, vp[i].px});
            sr += vp[i].sr;
          }
          d.fin_cnt[b] = 0;                           // ready for the next verify
        }
      }
      s_y = (resid && sr > 0.f) ? R.x : P.x;
    }
    __syncthreads();
    if (!s_last) return;                              // another slice of this request finishes it
  }

  FIN_TR(5);
  // 4. outputs + lane counters (a7)
  const int K1 = d.max_depth + 1;
  for (int i = tid; i < K1; i += FIN_THREADS) {
    int t = -1;
    if (!err) t = i < a ? drafts[doff + s_path[i + 1] - 1] : (i == a ? s_y : -1);
    const int nd = (!err && i <= a) ? s_path[i] : -1;
    tok_out[(size_t)b * K1 + i] = t;
    if (d.tok_int) d.tok_int[(size_t)b * K1 + i] = t;
    if (d.path_int) d.path_int[(size_t)b * K1 + i] = nd;
    if (nodes_out) nodes_out[(size_t)b * K1 + i] = nd;
  }
  if (tid == 0) {
    acc_out[b] = err ? -1 : a;
    if (d.acc_int) d.acc_int[b] = err ? -1 : a;
    if (b == 0 && mode != SV_PREFILL) atomicAdd(&d.stats[ST_STEPS], 1ull);
    if (!err && mode != SV_PREFILL) {                 // prefill chunks are not speculation
      atomicAdd(&d.stats[ST_ROWS], (unsigned long long)(k + 1));
      atomicAdd(&d.stats[ST_DRAFTED], (unsigned long long)k);
      atomicAdd(&d.stats[ST_ACCEPTED], (unsigned long long)a);
      atomicAdd(&d.stats[ST_EMITTED], (unsigned long long)(a + 1));
      atomicAdd(&d.stats[ST_INDEP], (unsigned long long)s_indep);
      atomicAdd(&d.stats[ST_HIST + a], 1ull);
      atomicAdd(&d.stats[ST_DRAFTED_BY_K + k], (unsigned long long)k);
      atomicAdd(&d.stats[ST_ACCEPTED_BY_K + k], (unsigned long long)a);
    }
  }
}

cudaError_t launch_finalize(const LaneDev& d, int batch, const int* draft_tokens, const int* parents,
                            const float* draft_probs, const float* logits, uint64_t seed, int mode, float inv_temp,
                            int* accepted_len, int* out_tokens, int* accepted_nodes, cudaStream_t s,
                            bool use_row_best) {
  SV_COUNT_LAUNCH();
  // sampled chains: the race over the vocabulary is split across RS CTAs per request so the grid
  // fills the resident CTA slots once; the other modes need one CTA per request
  const bool race = mode == SV_SAMPLE && !parents;
  const int smem = 0;
  static int slots_dev[64] = {0};                    // resident race CTAs per device (occupancy x SMs)
  int dev = 0;
  cudaGetDevice(&dev);
  int& slots = slots_dev[dev & 63];
  if (race && !slots) {
    int sms = 148, occ = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, finalize_kernel, FIN_THREADS, 0);
    slots = std::max(1, occ) * sms;
  }
  int RS = 1;
  if (race) RS = std::min(kMaxRaceSplits, std::max(1, slots / batch));
  return launch_pdl(finalize_kernel, dim3(batch, RS), dim3(FIN_THREADS), smem, s, 1, d, draft_tokens, parents, draft_probs,
                    logits, seed, mode, inv_temp, accepted_len, out_tokens, accepted_nodes, (int)use_row_best);
}

}  // namespace sv
