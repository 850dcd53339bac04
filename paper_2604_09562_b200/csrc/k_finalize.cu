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
#include "common.cuh"
#include "lane.h"
#include "../../include/sv.h"

namespace sv {

constexpr int FIN_THREADS = 512;

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

__global__ void __launch_bounds__(FIN_THREADS) finalize_kernel(LaneDev d, const int* __restrict__ drafts,
                                                                const float* __restrict__ probs,
                                                                const float* __restrict__ logits, uint64_t seed,
                                                                int mode, float inv_temp, int* __restrict__ acc_out,
                                                                int* __restrict__ tok_out) {
  __shared__ float s_m[kMaxDepth + 1], s_S[kMaxDepth + 1];
  __shared__ int s_top[kMaxDepth + 1];
  __shared__ int s_a, s_indep, s_y, s_resid;
  __shared__ Best s_bestR[FIN_THREADS / 32], s_bestP[FIN_THREADS / 32];
  __shared__ float s_sumR[FIN_THREADS / 32];

  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  const int k = d.depths[b], slot = d.slots[b], r0 = d.row_off[b], doff = r0 - b;
  const int L = d.len[slot];
  const unsigned long long rid = d.rid[slot];
  const int err = d.req_err[b];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = FIN_THREADS / 32;
  const size_t V = d.V;

  // 1. combine the vocab-tile statistics of each chain row (warp per row): one online pass,
  //    loads batched 8 deep per lane so the memory round trips overlap
  for (int j = warp; j <= k; j += nw) {
    const float* tm = d.tile_max + (size_t)(r0 + j) * d.nt;
    const float* ts = d.tile_sum + (size_t)(r0 + j) * d.nt;
    const int* ta = d.tile_arg + (size_t)(r0 + j) * d.nt;
    float m = -INFINITY, S = 0.f;
    int am = 0x7fffffff;
    constexpr int U = 8;
    for (int t0 = lane; t0 < d.nt; t0 += 32 * U) {
      float vm[U], vs[U];
      int va[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + 32 * u;
        const bool ok = t < d.nt;
        vm[u] = ok ? tm[t] : -INFINITY;
        vs[u] = ok ? ts[t] : 0.f;
        va[u] = ok ? ta[t] : 0x7fffffff;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {                 // t increasing per lane: strict > keeps lowest
        if (vm[u] > m) {
          S = (m == -INFINITY ? 0.f : S * expf(m - vm[u])) + vs[u];
          m = vm[u];
          am = va[u];
        } else if (vm[u] != -INFINITY) {
          S += vs[u] * expf(vm[u] - m);
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o);
      const float oS = __shfl_xor_sync(0xffffffffu, S, o);
      const int oa = __shfl_xor_sync(0xffffffffu, am, o);
      const float mn = fmaxf(m, om);
      const float Sn = (m == -INFINITY ? 0.f : S * expf(m - mn)) + (om == -INFINITY ? 0.f : oS * expf(om - mn));
      if (om > m || (om == m && oa < am)) am = oa;
      m = mn;
      S = Sn;
    }
    if (lane == 0) { s_m[j] = m; s_S[j] = S; s_top[j] = am; }
  }
  __syncthreads();

  // 2. accept scan (serial over k <= 32)
  if (tid == 0) {
    int a = k, indep = 0;
    if (mode == SV_PREFILL) {                      // R29: the chunk's rows are all kept
      s_y = s_top[k];
    } else if (mode == SV_GREEDY) {
      for (int j = 1; j <= k; ++j) {
        const bool acc = drafts[doff + j - 1] == s_top[j - 1];
        indep += acc;
        if (!acc && a == k) a = j - 1;
      }
      s_y = s_top[a];
    } else {
      for (int j = 1; j <= k; ++j) {
        const int dj = drafts[doff + j - 1];
        const float lg = logits[(size_t)(r0 + j - 1) * V + dj];
        const float pd = expf(lg * inv_temp - s_m[j - 1]) / s_S[j - 1];
        const float qd = probs ? probs[(size_t)(doff + j - 1) * V + dj] : 1.0f;
        const float u = uniform_accept(seed, rid, uint32_t(L + j));
        const bool acc = (qd == 0.0f) || (u < pd / qd);
        indep += acc;
        if (!acc && a == k) a = j - 1;
      }
    }
    s_a = a;
    s_indep = indep;
    s_resid = (mode == SV_SAMPLE) && (a < k);
  }
  __syncthreads();
  const int a = s_a;

  // 3. exponential race over the one selected row (sampled mode only)
  if (mode == SV_SAMPLE) {
    const bool resid = s_resid;
    const float* lrow = logits + (size_t)(r0 + a) * V;
    const float m = s_m[a], invS = 1.0f / s_S[a];
    const float* qrow = (resid && probs) ? probs + (size_t)(doff + a) * V : nullptr;
    const int dnext = resid ? drafts[doff + a] : -1;
    const uint32_t z = uint32_t(L + a + 1);
    Best bR{-INFINITY, 0x7fffffff}, bP{-INFINITY, 0x7fffffff};
    float sumR = 0.f;
    const int nm = (int)((V + 3) / 4);
    for (int mm = tid; mm < nm; mm += FIN_THREADS) {
      const u32x4 w = race_words(seed, rid, z, uint32_t(mm));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int x = mm * 4 + l;
        if (x >= (int)V) break;
        const float p = expf(lrow[x] * inv_temp - m) * invS;
        const float E = -logf(word_to_uniform(ws[l]));
        bP = better(bP, Best{p > 0.f ? p / E : -INFINITY, x});
        if (resid) {
          const float q = qrow ? qrow[x] : (x == dnext ? 1.0f : 0.0f);
          const float R = fmaxf(0.f, p - q);
          sumR += R;
          bR = better(bR, Best{R > 0.f ? R / E : -INFINITY, x});
        }
      }
    }
    bR = warp_best(bR);
    bP = warp_best(bP);
    sumR = warp_sum(sumR);
    if (lane == 0) { s_bestR[warp] = bR; s_bestP[warp] = bP; s_sumR[warp] = sumR; }
    __syncthreads();
    if (tid == 0) {
      Best R = s_bestR[0], P = s_bestP[0];
      float sr = s_sumR[0];
      for (int i = 1; i < nw; ++i) { R = better(R, s_bestR[i]); P = better(P, s_bestP[i]); sr += s_sumR[i]; }
      s_y = (resid && sr > 0.f) ? R.x : P.x;
    }
    __syncthreads();
  }

  // 4. outputs + lane counters (a7)
  const int K1 = d.max_depth + 1;
  for (int i = tid; i < K1; i += FIN_THREADS) {
    int t = -1;
    if (!err) t = i < a ? drafts[doff + i] : (i == a ? s_y : -1);
    tok_out[(size_t)b * K1 + i] = t;
    if (d.tok_int) d.tok_int[(size_t)b * K1 + i] = t;
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

cudaError_t launch_finalize(const LaneDev& d, int batch, const int* draft_tokens, const float* draft_probs,
                            const float* logits, uint64_t seed, int mode, float inv_temp, int* accepted_len,
                            int* out_tokens, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  return launch_pdl(finalize_kernel, dim3(batch), dim3(FIN_THREADS), 0, s, 1, d, draft_tokens, draft_probs, logits,
                    seed, mode, inv_temp, accepted_len, out_tokens);
}

}  // namespace sv
