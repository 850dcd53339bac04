// NEXT-4 (S19): the fp32-SIMT exactness instantiation of the verify step's model
// arithmetic (a2-a5). The same function as the bf16 tensor-core path — embed, RMSNorm, QKV, RoPE,
// chain-causal GQA attention over the cache, O-proj + residual, RMSNorm, SwiGLU MLP + residual,
// final RMSNorm, lm-head — with fp32 operands and fp32 accumulation and NO bf16 rounding anywhere,
// so its logits sit within fp32 accumulation error of the fp64 definition. Plain SIMT kernels
// (an exactness reference, not the hot path); the decisions on its logits go through the same
// finalize kernel (sv_verify_logits). Caches are dense per request (sv.h sv_exact_forward).
#include <math.h>

#include <vector>

#include "common.cuh"
#include "lane.h"
#include "../../include/sv.h"

namespace sv {
namespace {

template <int NT>
__device__ float ex_block_sum(float v) {
  __shared__ float red[NT / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

// out[r] = RMSNorm(x[r]) * g; x = E[tok[r]] when tok != nullptr (then also h[r] = x)
__global__ void __launch_bounds__(256) ex_norm_kernel(const float* __restrict__ x, const int* __restrict__ tok,
                                                      const float* __restrict__ E, const float* __restrict__ g,
                                                      float* __restrict__ h, float* __restrict__ out, int D, float eps) {
  const int r = blockIdx.x;
  const float* xr = tok ? E + (size_t)tok[r] * D : x + (size_t)r * D;
  float ss = 0.f;
  for (int i = threadIdx.x; i < D; i += 256) ss += xr[i] * xr[i];
  const float rstd = 1.0f / sqrtf(ex_block_sum<256>(ss) / float(D) + eps);
  for (int i = threadIdx.x; i < D; i += 256) {
    if (tok) h[(size_t)r * D + i] = xr[i];
    out[(size_t)r * D + i] = xr[i] * rstd * g[i];
  }
}

// C[M][N] = A[M][K] B[N][K]^T (+ R[M][N] when R != nullptr), 64 x 64 tiles, 16-deep K slices
__global__ void __launch_bounds__(256) ex_gemm_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                      const float* R, float* C, int M, int N, int K) {
  __shared__ float sa[16][64 + 1], sb[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int r = i / 16, k = i % 16;
      sa[k][r] = (m0 + r < M && k0 + k < K) ? A[(size_t)(m0 + r) * K + k0 + k] : 0.f;
      sb[k][r] = (n0 + r < N && k0 + k < K) ? B[(size_t)(n0 + r) * K + k0 + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = sa[k][ty * 4 + i];
        b[i] = sb[k][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) C[(size_t)m * N + n] = acc[i][j] + (R ? R[(size_t)m * N + n] : 0.f);
    }
}

// qkv [T][(Hq + 2 Hkv) dh] -> q [T][Hq][dh], k, v [T][Hkv][dh]; rotate_half RoPE on q and k at pos[r]
__global__ void ex_rope_kernel(const float* __restrict__ qkv, const int* __restrict__ pos,
                               const float* __restrict__ cs, const float* __restrict__ sn, float* q, float* k,
                               float* v, int Hq, int Hkv, int dh) {
  const int r = blockIdx.x;
  const int W = (Hq + 2 * Hkv) * dh, half = dh / 2;
  const float* x = qkv + (size_t)r * W;
  for (int f = threadIdx.x; f < W; f += blockDim.x) {
    const int head = f / dh, d = f % dh;
    float y = x[f];
    if (head < Hq + Hkv) {
      const int m = d < half ? d : d - half;
      const float c = cs[(size_t)pos[r] * half + m], s = sn[(size_t)pos[r] * half + m];
      const float p = d < half ? -x[f + half] : x[f - half];
      y = x[f] * c + p * s;
    }
    if (head < Hq) q[(size_t)r * Hq * dh + f] = y;
    else if (head < Hq + Hkv) k[(size_t)r * Hkv * dh + (f - Hq * dh)] = y;
    else v[(size_t)r * Hkv * dh + (f - (Hq + Hkv) * dh)] = y;
  }
}

// one CTA per (row r, q head): softmax over the request's cache keys 0..L-1 and chain keys 0..j
__global__ void __launch_bounds__(128) ex_attn_kernel(const float* __restrict__ q, const float* __restrict__ kc,
                                                      const float* __restrict__ vc, const float* __restrict__ ck,
                                                      const float* __restrict__ cv, const int* __restrict__ row_req,
                                                      const int* __restrict__ row_j, const int* __restrict__ row0,
                                                      const int* __restrict__ ctx_len, int max_ctx, int Hq, int Hkv,
                                                      int dh, float* o) {
  extern __shared__ float sc[];                    // [L + j + 1] scores
  __shared__ float red[4];
  const int r = blockIdx.x, hq = blockIdx.y, b = row_req[r], j = row_j[r], L = ctx_len[b];
  const int hk = hq / (Hq / Hkv), n = L + j + 1;
  const float* qr = q + ((size_t)r * Hq + hq) * dh;
  const float scale = 1.0f / sqrtf((float)dh);
  float mx = -INFINITY;
  for (int t = threadIdx.x; t < n; t += 128) {
    const float* kr = t < L ? ck + (((size_t)b * max_ctx + t) * Hkv + hk) * dh
                            : kc + ((size_t)(row0[b] + t - L) * Hkv + hk) * dh;
    float s = 0.f;
    for (int d = 0; d < dh; ++d) s = fmaf(qr[d], kr[d], s);
    s *= scale;
    sc[t] = s;
    mx = fmaxf(mx, s);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float l = 0.f;
  for (int t = threadIdx.x; t < n; t += 128) {
    const float p = expf(sc[t] - mx);
    sc[t] = p;
    l += p;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = l;
  __syncthreads();
  l = red[0] + red[1] + red[2] + red[3];
  for (int d = threadIdx.x; d < dh; d += 128) {
    float acc = 0.f;
    for (int t = 0; t < n; ++t) {
      const float* vr = t < L ? cv + (((size_t)b * max_ctx + t) * Hkv + hk) * dh
                              : vc + ((size_t)(row0[b] + t - L) * Hkv + hk) * dh;
      acc = fmaf(sc[t], vr[d], acc);
    }
    o[((size_t)r * Hq + hq) * dh + d] = acc / l;
  }
}

// u = silu(gate) * up from gu [T][2F] (gate | up)
__global__ void ex_swiglu_kernel(const float* __restrict__ gu, float* __restrict__ u, int T, int F) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)T * F) return;
  const size_t r = i / F, c = i % F;
  const float g = gu[r * 2 * F + c], up = gu[r * 2 * F + F + c];
  u[i] = g / (1.0f + expf(-g)) * up;
}

void gemm(const float* A, const float* B, const float* R, float* C, int M, int N, int K, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  ex_gemm_kernel<<<dim3((N + 63) / 64, (M + 63) / 64), 256, 0, s>>>(A, B, R, C, M, N, K);
}

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct ExLayout {
  size_t h0, h1, h2, a, c, q, k, v, o, u, cs, sn, ints, total;
};

ExLayout ex_layout(const sv_config& c, int T) {
  ExLayout L{};
  const size_t D = c.d_model, nq = (size_t)c.n_q_heads * c.head_dim, nkv = (size_t)c.n_kv_heads * c.head_dim;
  size_t cw = nq + 2 * nkv;
  if (D > cw) cw = D;
  if ((size_t)2 * c.ffn_dim > cw) cw = 2 * c.ffn_dim;
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t r = o; o += al(bytes); return r; };
  L.h0 = take(4 * T * D);
  L.h1 = take(4 * T * D);
  L.h2 = take(4 * T * D);
  L.a = take(4 * T * D);
  L.c = take(4 * T * cw);
  L.q = take(4 * T * nq);
  L.k = take(4 * (size_t)c.n_layers * T * nkv);
  L.v = take(4 * (size_t)c.n_layers * T * nkv);
  L.o = take(4 * T * nq);
  L.u = take(4 * T * (c.ffn_dim ? c.ffn_dim : 1));
  L.cs = take(4 * (size_t)c.max_pos * c.head_dim / 2);
  L.sn = take(4 * (size_t)c.max_pos * c.head_dim / 2);
  L.ints = take(4 * (5 * (size_t)T + 2 * (size_t)c.max_batch + 2));
  L.total = o;
  return L;
}

}  // namespace
}  // namespace sv

extern "C" {

sv_status sv_exact_query_sizes(const sv_config* cfg, int32_t T, size_t* workspace_bytes) {
  if (!cfg || T < 1 || !workspace_bytes || cfg->d_model < 1 || cfg->n_kv_heads < 1 || cfg->head_dim < 2 ||
      cfg->n_q_heads % cfg->n_kv_heads || cfg->head_dim % 2 || cfg->max_pos < 2)
    return SV_EINVAL;
  *workspace_bytes = sv::ex_layout(*cfg, T).total;
  return SV_OK;
}

sv_status sv_exact_forward(const sv_config* cfg, const sv_weights_f32* w, int32_t batch, const int32_t* row_off,
                           const int32_t* chain_tok, const int32_t* ctx_len, const float* cache_k,
                           const float* cache_v, int32_t max_ctx, void* workspace, size_t workspace_bytes,
                           float* logits, sv_stream_t stream) {
  using namespace sv;
  if (!cfg || !w || batch < 1 || batch > cfg->max_batch || !row_off || !chain_tok || !ctx_len || !workspace ||
      !logits || max_ctx < 0 || ((cache_k == nullptr) != (cache_v == nullptr)))
    return SV_EINVAL;
  if (!w->embed || !w->attn_norm || !w->wqkv || !w->wo || !w->final_norm || !w->lm_head) return SV_EINVAL;
  if (cfg->ffn_dim > 0 && (!w->ffn_norm || !w->w_gate_up || !w->w_down)) return SV_EINVAL;
  const int T = row_off[batch];
  if (row_off[0] != 0 || T < batch) return SV_EINVAL;
  std::vector<int> rreq(T), rj(T), rpos(T);
  for (int b = 0; b < batch; ++b) {
    if (row_off[b + 1] <= row_off[b] || ctx_len[b] < 0 || ctx_len[b] > max_ctx) return SV_EINVAL;
    if (ctx_len[b] > 0 && !cache_k) return SV_EINVAL;
    for (int r = row_off[b]; r < row_off[b + 1]; ++r) {
      rreq[r] = b;
      rj[r] = r - row_off[b];
      rpos[r] = ctx_len[b] + rj[r];
      if (rpos[r] >= cfg->max_pos) return SV_EINVAL;
    }
  }
  size_t need = 0;
  if (sv_exact_query_sizes(cfg, T, &need) || need > workspace_bytes) return SV_EINVAL;
  const ExLayout Ly = ex_layout(*cfg, T);
  char* ws = (char*)workspace;
  cudaStream_t s = (cudaStream_t)stream;
  const int D = cfg->d_model, Hq = cfg->n_q_heads, Hkv = cfg->n_kv_heads, dh = cfg->head_dim, F = cfg->ffn_dim;
  const int V = cfg->vocab, qkv_rows = (Hq + 2 * Hkv) * dh, nq = Hq * dh, nkv = Hkv * dh, half = dh / 2;
  // RoPE table of the positions used: fp64 angles, stored fp32 (the same table as the bf16 path)
  int pmax = 0;
  for (int r = 0; r < T; ++r) pmax = rpos[r] > pmax ? rpos[r] : pmax;
  std::vector<float> cs((size_t)(pmax + 1) * half), sn((size_t)(pmax + 1) * half);
  for (int m = 0; m < half; ++m) {
    const double inv = 1.0 / pow((double)cfg->rope_theta, 2.0 * m / dh);
    for (int p = 0; p <= pmax; ++p) {
      cs[(size_t)p * half + m] = (float)cos((double)p * inv);
      sn[(size_t)p * half + m] = (float)sin((double)p * inv);
    }
  }
  int* ints = (int*)(ws + Ly.ints);
  int *d_req = ints, *d_j = ints + T, *d_pos = ints + 2 * T, *d_row0 = ints + 3 * T, *d_len = d_row0 + batch;
  std::vector<int> r0(row_off, row_off + batch), ln(ctx_len, ctx_len + batch);
  float *h0 = (float*)(ws + Ly.h0), *h1 = (float*)(ws + Ly.h1), *h2 = (float*)(ws + Ly.h2), *a = (float*)(ws + Ly.a);
  float *cb = (float*)(ws + Ly.c), *q = (float*)(ws + Ly.q), *kc = (float*)(ws + Ly.k), *vc = (float*)(ws + Ly.v);
  float *o = (float*)(ws + Ly.o), *u = (float*)(ws + Ly.u), *dcs = (float*)(ws + Ly.cs), *dsn = (float*)(ws + Ly.sn);
  if (cudaMemcpyAsync(dcs, cs.data(), 4 * cs.size(), cudaMemcpyHostToDevice, s) ||
      cudaMemcpyAsync(dsn, sn.data(), 4 * sn.size(), cudaMemcpyHostToDevice, s) ||
      cudaMemcpyAsync(d_req, rreq.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, s) ||
      cudaMemcpyAsync(d_j, rj.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, s) ||
      cudaMemcpyAsync(d_pos, rpos.data(), 4 * (size_t)T, cudaMemcpyHostToDevice, s) ||
      cudaMemcpyAsync(d_row0, r0.data(), 4 * (size_t)batch, cudaMemcpyHostToDevice, s) ||
      cudaMemcpyAsync(d_len, ln.data(), 4 * (size_t)batch, cudaMemcpyHostToDevice, s))
    return SV_ECUDA;
  int maxn = 0;
  for (int r = 0; r < T; ++r) maxn = rpos[r] + 1 > maxn ? rpos[r] + 1 : maxn;
  const size_t attn_smem = 4 * (size_t)maxn;
  if (attn_smem > 48 * 1024 &&
      cudaFuncSetAttribute(ex_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attn_smem))
    return SV_ECUDA;
  SV_COUNT_LAUNCH();
  ex_norm_kernel<<<T, 256, 0, s>>>(nullptr, chain_tok, w->embed, w->attn_norm, h0, a, D, cfg->norm_eps);
  for (int layer = 0; layer < cfg->n_layers; ++layer) {
    const float* hin = layer == 0 ? h0 : h2;
    if (layer > 0) {
      SV_COUNT_LAUNCH();
      ex_norm_kernel<<<T, 256, 0, s>>>(hin, nullptr, nullptr, w->attn_norm + (size_t)layer * D, nullptr, a, D,
                                       cfg->norm_eps);
    }
    gemm(a, w->wqkv + (size_t)layer * qkv_rows * D, nullptr, cb, T, qkv_rows, D, s);
    float* kl = kc + (size_t)layer * T * nkv;
    float* vl = vc + (size_t)layer * T * nkv;
    SV_COUNT_LAUNCH();
    ex_rope_kernel<<<T, 256, 0, s>>>(cb, d_pos, dcs, dsn, q, kl, vl, Hq, Hkv, dh);
    const size_t lstride = (size_t)batch * max_ctx * nkv;
    SV_COUNT_LAUNCH();
    ex_attn_kernel<<<dim3(T, Hq), 128, attn_smem, s>>>(q, kl, vl, cache_k ? cache_k + layer * lstride : nullptr,
                                                       cache_v ? cache_v + layer * lstride : nullptr, d_req, d_j,
                                                       d_row0, d_len, max_ctx, Hq, Hkv, dh, o);
    float* hattn = F > 0 ? h1 : h2;
    gemm(o, w->wo + (size_t)layer * D * nq, hin, hattn, T, D, nq, s);   // h + o Wo^T
    if (F > 0) {
      SV_COUNT_LAUNCH();
      ex_norm_kernel<<<T, 256, 0, s>>>(h1, nullptr, nullptr, w->ffn_norm + (size_t)layer * D, nullptr, a, D,
                                       cfg->norm_eps);
      gemm(a, w->w_gate_up + (size_t)layer * 2 * F * D, nullptr, cb, T, 2 * F, D, s);
      SV_COUNT_LAUNCH();
      ex_swiglu_kernel<<<(unsigned)(((size_t)T * F + 255) / 256), 256, 0, s>>>(cb, u, T, F);
      gemm(u, w->w_down + (size_t)layer * D * F, h1, h2, T, D, F, s);
    }
  }
  SV_COUNT_LAUNCH();
  ex_norm_kernel<<<T, 256, 0, s>>>(h2, nullptr, nullptr, w->final_norm, nullptr, a, D, cfg->norm_eps);
  gemm(a, w->lm_head, nullptr, logits, T, V, D, s);
  return cudaGetLastError() == cudaSuccess ? SV_OK : SV_ECUDA;
}

}  // extern "C"
