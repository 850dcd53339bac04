// Row-wise kernels of the verify step:
//   a1  plan: ragged batch assembly (row offsets, chain tokens, positions, attention work list)
//   a2  embed + attn RMSNorm; generic RMSNorm; QKV RoPE epilogue
//   a4  residual and SwiGLU epilogues
//   a5  lm-head vocab-tile statistics (max, sum exp, lowest argmax)
// plus test / fixture kernels (device Philox uniforms, planted drafter) and
// lane-state initialisation.
#include <stdlib.h>

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "lane.h"
#include "../../include/sv.h"

namespace sv {

unsigned long long g_launch_count = 0;

cudaError_t smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({kernel, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kernel, dev});
  return e;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ------------------------------------------------------------------ a1: plan
// One CTA. Serial prefix over <= 256 requests in thread 0, then parallel fills.
__global__ void plan_kernel(LaneDev d, PlanArgs p, const int* __restrict__ draft_tokens,
                            const int* __restrict__ parents, int attn) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_off[kMaxBatch + 1];
  __shared__ int s_item[kMaxBatch + 1];
  __shared__ int s_err[kMaxBatch];
  __shared__ int s_len[kMaxBatch];
  __shared__ int s_slot[kMaxBatch], s_dep[kMaxBatch];
  const int B = p.batch;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {   // the per-request loads, in parallel
    int slot = p.slots[b], k = p.depths[b], e = 0;
    if (d.dyn_ctrl) {                                    // dynamic-depth graph: this replay's batch
      slot = d.dyn_ctrl[b];
      k = d.dyn_ctrl[B + b];
      if (slot < 0 || slot >= d.max_slots) { slot = 0; e = 1; }
      if (k < 0 || k > d.max_depth) { k = 0; e = 1; }
    }
    s_slot[b] = slot;
    s_dep[b] = k;
    s_len[b] = d.len[slot];
    s_err[b] = e;
  }
  __syncthreads();
  if (threadIdx.x == 0) {                                // prefix sums over shared memory only
    int o = 0, it = 0;
    for (int b = 0; b < B; ++b) {
      s_off[b] = o;
      s_item[b] = it;
      o += s_dep[b] + 1;
      if (attn) it += num_splits(s_len[b]) * d.Hkv;
    }
    s_off[B] = o;
    s_item[B] = it;
    *d.n_items = it;
    *d.batch_n = B;
    *d.T_dev = o;
  }
  __syncthreads();
  for (int b = threadIdx.x; b <= B; b += blockDim.x) {
    d.row_off[b] = s_off[b];
    d.item_start[b] = s_item[b];
    if (b < B) {
      d.slots[b] = s_slot[b];
      d.depths[b] = s_dep[b];
    }
  }
  const int T = s_off[B];
  for (int r = threadIdx.x; r < T; r += blockDim.x) {
    int lo = 0, hi = B - 1;                      // last b with s_off[b] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int b = lo, j = r - s_off[b], slot = s_slot[b];
    int tok = j == 0 ? d.pending[slot] : draft_tokens[s_off[b] - b + j - 1];
    if (tok < 0 || tok >= d.V) {
      atomicOr(&s_err[b], 1);
      tok = 0;
    }
    // chain row j = node j: position L + depth(j), ancestor-or-self mask over the request's nodes
    // (a chain: depth j, nodes 0..j; a token tree: follow the parents, each in [0, n-1], R30)
    int depth = j;
    unsigned long long anc = j >= 63 ? ~0ull : (2ull << j) - 1ull;
    if (parents && j > 0) {
      const int* par = parents + (s_off[b] - b);     // parent of node n at par[n - 1]
      anc = 1ull << j;
      depth = 0;
      for (int n = j; n != 0; ++depth) {
        const int pn = par[n - 1];
        if (pn < 0 || pn >= n) {                       // not topological: the request is invalid
          atomicOr(&s_err[b], 4);
          break;
        }
        n = pn;
        anc |= 1ull << n;
      }
    }
    d.row_anc[r] = anc;
    int pos = s_len[b] + depth;
    if (pos >= d.max_pos) {                      // chain would run past the position table
      atomicOr(&s_err[b], 2);
      pos = d.max_pos - 1;                       // keep every read in range; the request is not committed
    }
    d.row_req[r] = b;
    d.row_pos[r] = pos;
    d.chain_tok[r] = tok;
    if (attn) d.row_comb[r] = make_int4(j, num_splits(s_len[b]), s_item[b], 0);   // the combine's one load
  }
  if (attn) {
    const int n_items = s_item[B];
    for (int it = threadIdx.x; it < n_items; it += blockDim.x) {
      int lo = 0, hi = B - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_item[mid] <= it) lo = mid; else hi = mid - 1;
      }
      const int b = lo, rel = it - s_item[b];
      const int ns = num_splits(s_len[b]);
      d.items[it] = make_int4(b, rel / ns, rel % ns, ns);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    d.req_err[b] = s_err[b];
    if (s_err[b] & 1) atomicOr(d.err, SV_DERR_BAD_TOKEN);
    if (s_err[b] & 2) atomicOr(d.err, SV_DERR_MAX_POS);
    if (s_err[b] & 4) atomicOr(d.err, SV_DERR_BAD_TREE);
  }
}

cudaError_t launch_plan(const LaneDev& d, const PlanArgs& p, const int* draft_tokens, const int* parents, bool attn,
                        cudaStream_t s) {
  SV_COUNT_LAUNCH();
  return launch_pdl(plan_kernel, dim3(1), dim3(1024), 0, s, 1, d, p, draft_tokens, parents, attn ? 1 : 0);
}

// ------------------------------------------------------------------ a2: embed + RMSNorm
// h0 = E[c]; a = bf16(RMSNorm(h0) * g), RMSNorm in fp32.
template <int NT>
__device__ float block_sum(float v) {
  __shared__ float red[NT / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(256) embed_norm_kernel(LaneDev d) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (r >= *d.T_dev) return;                       // launched for Tmax rows (dynamic-depth graph)
  const int tok = d.chain_tok[r];
  const bf16* e = d.embed + (size_t)tok * d.D;
  float* h = d.h0 + (size_t)r * d.D;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d.D; i += 256) {
    const float x = bf2f(e[i]);
    h[i] = x;
    ss += x * x;
  }
  const float rstd = 1.0f / sqrtf(block_sum<256>(ss) / float(d.D) + d.eps);
  for (int i = threadIdx.x; i < d.D; i += 256) d.a[(size_t)r * d.D + i] = f2bf(h[i] * rstd * bf2f(d.attn_norm[i]));
}

// Vectorised forms (D <= 8192, 16-byte aligned rows): each thread keeps its <= 4 eight-element
// vectors in registers between the sum of squares and the scaled store (one read of the input).
__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&x)[8]) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(p[i]);
    x[2 * i] = f.x;
    x[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 f32x8_to_bf16(const float (&x)[8]) {
  uint4 u;
  __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
  return u;
}

constexpr int kNormMaxVec = 4;   // 4 x 8 elements x 256 threads: D <= 8192

__global__ void __launch_bounds__(256) embed_norm_vec_kernel(LaneDev d) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int Tn = *d.T_dev, tok = d.chain_tok[r];   // both loads in flight together
  if (r >= Tn) return;                             // launched for Tmax rows (dynamic-depth graph)
  const int nv = d.D / 8;
  const uint4* e = reinterpret_cast<const uint4*>(d.embed + (size_t)tok * d.D);
  float4* h = reinterpret_cast<float4*>(d.h0 + (size_t)r * d.D);
  float x[kNormMaxVec][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int v = threadIdx.x + k * 256;
    if (v < nv) {
      bf16x8_to_f32(e[v], x[k]);
      h[2 * v] = make_float4(x[k][0], x[k][1], x[k][2], x[k][3]);
      h[2 * v + 1] = make_float4(x[k][4], x[k][5], x[k][6], x[k][7]);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += x[k][i] * x[k][i];
    }
  }
  const float rstd = 1.0f / sqrtf(block_sum<256>(ss) / float(d.D) + d.eps);
  const uint4* gw = reinterpret_cast<const uint4*>(d.attn_norm);
  uint4* out = reinterpret_cast<uint4*>(d.a + (size_t)r * d.D);
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int v = threadIdx.x + k * 256;
    if (v < nv) {
      float g[8], y[8];
      bf16x8_to_f32(gw[v], g);
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = x[k][i] * rstd * g[i];
      out[v] = f32x8_to_bf16(y);
    }
  }
}

__global__ void __launch_bounds__(256) rmsnorm_vec_kernel(const float* __restrict__ x, const bf16* __restrict__ g,
                                                          bf16* __restrict__ out, int D, float eps, const int* __restrict__ Tdev) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (Tdev && r >= *Tdev) return;                 // launched for Tmax rows (dynamic-depth graph)
  const int nv = D / 8;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)r * D);
  float v8[kNormMaxVec][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int v = threadIdx.x + k * 256;
    if (v < nv) {
      const float4 a = xr[2 * v], b = xr[2 * v + 1];
      v8[k][0] = a.x; v8[k][1] = a.y; v8[k][2] = a.z; v8[k][3] = a.w;
      v8[k][4] = b.x; v8[k][5] = b.y; v8[k][6] = b.z; v8[k][7] = b.w;
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += v8[k][i] * v8[k][i];
    }
  }
  const float rstd = 1.0f / sqrtf(block_sum<256>(ss) / float(D) + eps);
  const uint4* gw = reinterpret_cast<const uint4*>(g);
  uint4* o = reinterpret_cast<uint4*>(out + (size_t)r * D);
#pragma unroll
  for (int k = 0; k < kNormMaxVec; ++k) {
    const int v = threadIdx.x + k * 256;
    if (v < nv) {
      float gg[8], y[8];
      bf16x8_to_f32(gw[v], gg);
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = v8[k][i] * rstd * gg[i];
      o[v] = f32x8_to_bf16(y);
    }
  }
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// ------------------------------------------------------------------ a1 + a2 fused: plan + embed
// One CTA per chain row (Tmax rows for a dynamic-depth graph). Every CTA reads the batch's slots /
// depths (kernel parameters, or the graph's device copy) and lengths and scans them itself, so no CTA
// waits for another: row r finds its request, writes its row tables, gathers its token's embedding
// and normalises it (a2); the CTA of each request's first row also writes the request's tables, its
// split-KV work items and the request's error bits (every row of the request checked there, as
// plan_kernel does), and CTA 0 the batch totals. Same outputs as plan_kernel + embed_norm_vec_kernel.
__device__ __forceinline__ int block_excl_scan256(int v, int* s_w, int* total) {
  // exclusive scan over the 256 threads of the block (8 warps)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  int off = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    off += i < w ? s_w[i] : 0;
    tot += s_w[i];
  }
  __syncthreads();
  *total = tot;
  return off + x - v;
}

__global__ void __launch_bounds__(256) plan_embed_kernel(LaneDev d, PlanArgs p, const int* __restrict__ draft_tokens,
                                                         const int* __restrict__ parents, int allow_wide) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_off[kMaxBatch + 1], s_item[kMaxBatch + 1], s_len[kMaxBatch], s_slot[kMaxBatch];
  __shared__ int s_w[8], s_err, s_minL;
  const int B = p.batch, tid = threadIdx.x;
  if (tid == 0) s_minL = 0x7fffffff;
  // per-request state: thread t < B holds request t (B <= kMaxBatch = 256)
  int k1 = 0, nit = 0;
  if (tid < B) {
    int slot = p.slots[tid], k = p.depths[tid];
    if (d.dyn_ctrl) {
      slot = d.dyn_ctrl[tid];
      k = d.dyn_ctrl[B + tid];
      if (slot < 0 || slot >= d.max_slots) slot = 0;
      if (k < 0 || k > d.max_depth) k = 0;
    }
    const int L = d.len[slot];
    s_slot[tid] = slot;
    s_len[tid] = L;
    k1 = k + 1;
  }
  __syncthreads();
  if (tid < B) atomicMin(&s_minL, s_len[tid]);
  __syncthreads();
  // wide (2048-key) splits when every context holds at least two of them: half the items, half the
  // split-KV partials the combine reads (ns 4096-token contexts); shorter or mixed contexts keep
  // 1024-key items, which balance better over the persistent grid (c3: 1-2k contexts measured worse wide)
  const int wide = allow_wide && s_minL >= 4 * kSplitKeys ? 1 : 0;
  const int sk = kSplitKeys << wide;
  if (tid < B) nit = num_splits_k(s_len[tid], sk) * d.Hkv;
  int T = 0, NI = 0;
  const int off = block_excl_scan256(k1, s_w, &T);
  const int ito = block_excl_scan256(nit, s_w, &NI);
  if (tid < B) {
    s_off[tid] = off;
    s_item[tid] = ito;
  }
  if (tid == 0) {
    s_off[B] = T;
    s_item[B] = NI;
  }
  __syncthreads();
  const int r = blockIdx.x;
  if (r == 0 && tid == 0) {
    *d.n_items = NI;
    *d.batch_n = B;
    *d.T_dev = T;
    d.row_off[B] = T;
    d.item_start[B] = NI;
  }
  if (r >= T) return;                              // launched for Tmax rows (dynamic-depth graph)
  int lo = 0, hi = B - 1;                          // last b with s_off[b] <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_off[mid] <= r) lo = mid; else hi = mid - 1;
  }
  const int b = lo, j = r - s_off[b], slot = s_slot[b], L = s_len[b];
  const int R = s_off[b + 1] - s_off[b];
  const int doff = s_off[b] - b;                   // first draft token of request b
  // this CTA's row (thread 0) and, for the request's first row, every row's validity (threads t < R)
  if (tid == 0) s_err = 0;
  __syncthreads();
  auto row_info = [&](int jj, int& tok, int& pos, unsigned long long& anc, int& e) {
    e = 0;
    tok = jj == 0 ? d.pending[slot] : draft_tokens[doff + jj - 1];
    if (tok < 0 || tok >= d.V) {
      e |= 1;
      tok = 0;
    }
    int depth = jj;
    anc = jj >= 63 ? ~0ull : (2ull << jj) - 1ull;
    if (parents && jj > 0) {
      const int* par = parents + doff;               // parent of node n at par[n - 1]
      anc = 1ull << jj;
      depth = 0;
      for (int n = jj; n != 0; ++depth) {
        const int pn = par[n - 1];
        if (pn < 0 || pn >= n) {                     // not topological: the request is invalid
          e |= 4;
          break;
        }
        n = pn;
        anc |= 1ull << n;
      }
    }
    pos = L + depth;
    if (pos >= d.max_pos) {
      e |= 2;
      pos = d.max_pos - 1;
    }
  };
  __shared__ int s_tok;
  if (j == 0) {
    if (tid < R) {
      int tok, pos, e;
      unsigned long long anc;
      row_info(tid, tok, pos, anc, e);
      if (e) atomicOr(&s_err, e);
    }
    if (tid == 0) {
      int e0 = 0;
      if (d.dyn_ctrl) {
        const int s0 = d.dyn_ctrl[b], k0 = d.dyn_ctrl[B + b];
        if (s0 < 0 || s0 >= d.max_slots || k0 < 0 || k0 > d.max_depth) e0 = 1;
      }
      if (e0) atomicOr(&s_err, e0);
      d.row_off[b] = s_off[b];
      d.item_start[b] = s_item[b];
      d.slots[b] = slot;
      d.depths[b] = R - 1;
    }
    const int ns = num_splits_k(L, sk);
    for (int i = tid; i < ns * d.Hkv; i += blockDim.x)
      d.items[s_item[b] + i] = make_int4(b, i / ns, i % ns, ns | (wide << kItemWideShift));
  }
  if (tid == 0) {
    int tok, pos, e;
    unsigned long long anc;
    row_info(j, tok, pos, anc, e);
    d.row_anc[r] = anc;
    d.row_req[r] = b;
    d.row_pos[r] = pos;
    d.chain_tok[r] = tok;
    d.row_comb[r] = make_int4(j, num_splits_k(L, sk), s_item[b], 0);
    s_tok = tok;
  }
  __syncthreads();
  if (j == 0 && tid == 0) {
    const int e = s_err;
    d.req_err[b] = e;
    if (e & 1) atomicOr(d.err, SV_DERR_BAD_TOKEN);
    if (e & 2) atomicOr(d.err, SV_DERR_MAX_POS);
    if (e & 4) atomicOr(d.err, SV_DERR_BAD_TREE);
  }
  // a2: h0 = E[c]; a = bf16(RMSNorm(h0) * g)
  const int nv = d.D / 8;
  const uint4* e = reinterpret_cast<const uint4*>(d.embed + (size_t)s_tok * d.D);
  float4* h = reinterpret_cast<float4*>(d.h0 + (size_t)r * d.D);
  float x[kNormMaxVec][8];
  float ss = 0.f;
#pragma unroll
  for (int kk = 0; kk < kNormMaxVec; ++kk) {
    const int v = tid + kk * 256;
    if (v < nv) {
      bf16x8_to_f32(e[v], x[kk]);
      h[2 * v] = make_float4(x[kk][0], x[kk][1], x[kk][2], x[kk][3]);
      h[2 * v + 1] = make_float4(x[kk][4], x[kk][5], x[kk][6], x[kk][7]);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += x[kk][i] * x[kk][i];
    }
  }
  const float rstd = 1.0f / sqrtf(block_sum<256>(ss) / float(d.D) + d.eps);
  const uint4* gw = reinterpret_cast<const uint4*>(d.attn_norm);
  uint4* out = reinterpret_cast<uint4*>(d.a + (size_t)r * d.D);
#pragma unroll
  for (int kk = 0; kk < kNormMaxVec; ++kk) {
    const int v = tid + kk * 256;
    if (v < nv) {
      float g[8], y[8];
      bf16x8_to_f32(gw[v], g);
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = x[kk][i] * rstd * g[i];
      out[v] = f32x8_to_bf16(y);
    }
  }
}

bool plan_embed_supported(const LaneDev& d) {
  return d.D <= 256 * 8 * kNormMaxVec && (d.D % 8) == 0 && aligned16(d.embed) && aligned16(d.attn_norm);
}

cudaError_t launch_plan_embed(const LaneDev& d, const PlanArgs& p, const int* draft_tokens, const int* parents,
                              int rows, bool allow_wide, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  return launch_pdl(plan_embed_kernel, dim3(rows), dim3(256), 0, s, 1, d, p, draft_tokens, parents, allow_wide ? 1 : 0);
}

cudaError_t launch_embed_norm(const LaneDev& d, int T, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  if (d.D <= 256 * 8 * kNormMaxVec && aligned16(d.embed) && aligned16(d.attn_norm))
    return launch_pdl(embed_norm_vec_kernel, dim3(T), dim3(256), 0, s, 1, d);
  else
    return launch_pdl(embed_norm_kernel, dim3(T), dim3(256), 0, s, 1, d);
}

__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x, const bf16* __restrict__ g,
                                                      bf16* __restrict__ out, int D, float eps, const int* __restrict__ Tdev) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (Tdev && r >= *Tdev) return;                 // launched for Tmax rows (dynamic-depth graph)
  const float* xr = x + (size_t)r * D;
  float ss = 0.f;
  for (int i = threadIdx.x; i < D; i += 256) ss += xr[i] * xr[i];
  const float rstd = 1.0f / sqrtf(block_sum<256>(ss) / float(D) + eps);
  for (int i = threadIdx.x; i < D; i += 256) out[(size_t)r * D + i] = f2bf(xr[i] * rstd * bf2f(g[i]));
}

cudaError_t launch_rmsnorm(const LaneDev& d, const float* x, const bf16* g, bf16* out, int T, cudaStream_t s,
                           bool bound_by_T_dev) {
  SV_COUNT_LAUNCH();
  const int* Tdev = bound_by_T_dev ? d.T_dev : nullptr;
  if (d.D <= 256 * 8 * kNormMaxVec && aligned16(g))
    return launch_pdl(rmsnorm_vec_kernel, dim3(T), dim3(256), 0, s, 1, x, g, out, d.D, d.eps, Tdev);
  else
    return launch_pdl(rmsnorm_kernel, dim3(T), dim3(256), 0, s, 1, x, g, out, d.D, d.eps, Tdev);
}

// ------------------------------------------------------------------ a2: QKV + RoPE epilogue
// rotate_half RoPE at position row_pos[r] with the fp32 cos/sin table.
__global__ void qkv_rope_kernel(LaneDev d, int layer) {
  const int r = blockIdx.x;
  const int half = d.dh / 2;
  const int pos = d.row_pos[r];
  const float* c = d.cbuf + (size_t)r * d.qkv_rows;
  const float* cs = d.rope_cos + (size_t)pos * half;
  const float* sn = d.rope_sin + (size_t)pos * half;
  const int nq = d.Hq * d.dh, nk = d.Hkv * d.dh;
  bf16* kc = d.kc + ((size_t)layer * d.Tmax + r) * nk;
  bf16* vc = d.vc + ((size_t)layer * d.Tmax + r) * nk;
  for (int i = threadIdx.x; i < (d.Hq + d.Hkv) * half; i += blockDim.x) {
    const int head = i / half, m = i % half;
    const float* src = c + head * d.dh;
    const float x1 = src[m], x2 = src[m + half];
    const float o1 = x1 * cs[m] - x2 * sn[m];
    const float o2 = x2 * cs[m] + x1 * sn[m];
    bf16* dst = head < d.Hq ? d.q + (size_t)r * nq + head * d.dh : kc + (head - d.Hq) * d.dh;
    dst[m] = f2bf(o1);
    dst[m + half] = f2bf(o2);
  }
  for (int i = threadIdx.x; i < nk; i += blockDim.x) vc[i] = f2bf(c[nq + nk + i]);
}

cudaError_t launch_qkv_rope_epilogue(const LaneDev& d, int layer, int T, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  qkv_rope_kernel<<<T, 256, 0, s>>>(d, layer);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a4: residual / SwiGLU epilogues
__global__ void residual_kernel(const float* __restrict__ hin, const float* __restrict__ c, float* __restrict__ hout,
                                size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    hout[i] = hin[i] + c[i];
}

cudaError_t launch_residual_epilogue(const float* hin, const float* c, float* hout, int T, int D, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  residual_kernel<<<148 * 4, 256, 0, s>>>(hin, c, hout, (size_t)T * D);
  return cudaGetLastError();
}

// u = bf16(silu(gate) * up), gate = C[:, j], up = C[:, F + j]
__global__ void swiglu_kernel(LaneDev d, int T) {
  const size_t n = (size_t)T * d.F;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / d.F, j = i % d.F;
    const float g = d.cbuf[r * 2 * d.F + j], up = d.cbuf[r * 2 * d.F + d.F + j];
    d.u[i] = f2bf(g / (1.0f + expf(-g)) * up);
  }
}

cudaError_t launch_swiglu_epilogue(const LaneDev& d, int T, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  swiglu_kernel<<<148 * 4, 256, 0, s>>>(d, T);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a5: vocab-tile statistics
// One warp per (row, kVocabTile-wide tile): m = max(l * inv_temp), s = sum exp(l * inv_temp - m),
// argmax = lowest index attaining the max of l * inv_temp.
__global__ void tile_stats_kernel(LaneDev d, int T, float inv_temp) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= T * d.nt) return;
  const int r = warp / d.nt, t = warp % d.nt;
  const float* row = d.logits + (size_t)r * d.V;
  const int x0 = t * kVocabTile;
  float v[kVocabTile / 32];
  float m = -INFINITY;
  int am = 0x7fffffff;
#pragma unroll
  for (int i = 0; i < kVocabTile / 32; ++i) {
    const int x = x0 + i * 32 + lane;
    v[i] = x < d.V ? row[x] * inv_temp : -INFINITY;
    if (v[i] > m) { m = v[i]; am = x; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const int oa = __shfl_xor_sync(0xffffffffu, am, o);
    if (om > m || (om == m && oa < am)) { m = om; am = oa; }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kVocabTile / 32; ++i) s += expf(v[i] - m);
  s = warp_sum(s);
  if (lane == 0) {
    d.tile_max[(size_t)r * d.nt + t] = m;
    d.tile_sum[(size_t)r * d.nt + t] = s;
    d.tile_arg[(size_t)r * d.nt + t] = am;
  }
}

cudaError_t launch_tile_stats(const LaneDev& d, int T, float inv_temp, cudaStream_t s) {
  const int warps = T * d.nt;
  SV_COUNT_LAUNCH();
  tile_stats_kernel<<<(warps + 7) / 8, 256, 0, s>>>(d, T, inv_temp);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ test / fixture kernels
__global__ void debug_uniforms_kernel(uint64_t seed, uint64_t rid, uint32_t z, int purpose, int x0, int n,
                                      float* u) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = x0 + i;
  if (purpose == PURPOSE_ACCEPT) {
    u[i] = uniform_accept(seed, rid, z);      // x ignored (ACCEPT uses x = 0)
  } else {
    const u32x4 w = race_words(seed, rid, z, uint32_t(x) >> 2);
    const uint32_t ww = (x & 3) == 0 ? w.x : (x & 3) == 1 ? w.y : (x & 3) == 2 ? w.z : w.w;
    u[i] = word_to_uniform(ww);
  }
}

cudaError_t launch_debug_uniforms(uint64_t seed, uint64_t rid, uint32_t z, int purpose, int x0, int n, float* u,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  SV_COUNT_LAUNCH();
  debug_uniforms_kernel<<<(n + 255) / 256, 256, 0, s>>>(seed, rid, z, purpose, x0, n, u);
  return cudaGetLastError();
}

// planted-successor drafter (bench fixture): one thread per request
__global__ void draft_planted_kernel(LaneDev d, PlanArgs p, const int* __restrict__ succ,
                                     const uint8_t* __restrict__ mask, const int* __restrict__ dev_tok,
                                     const int* __restrict__ parents, int* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= p.batch) return;
  const int* dep = d.dyn_ctrl ? d.dyn_ctrl + p.batch : p.depths;   // dynamic-depth graph: device copies
  const int* slt = d.dyn_ctrl ? d.dyn_ctrl : p.slots;
  int off = 0;
  for (int i = 0; i < b; ++i) off += min(max(dep[i], 0), d.max_depth);
  const int kb = min(max(dep[b], 0), d.max_depth);
  int tok[kMaxDepth + 1];                          // node tokens (node 0 = the pending token)
  const int sl = slt[b];
  tok[0] = d.pending[sl >= 0 && sl < d.max_slots ? sl : 0];
  for (int j = 0; j < kb; ++j) {
    int par = parents ? parents[off + j] : j;      // tree: the node's parent; chain: the previous node
    if (par < 0 || par > j) par = j;               // (the verify flags a bad tree; keep reads in range)
    int t = succ[tok[par]];
    if (mask[off + j]) t = dev_tok[off + j];
    out[off + j] = t;
    tok[j + 1] = t;
  }
}

cudaError_t launch_draft_planted(const LaneDev& d, const PlanArgs& p, const int* succ, const uint8_t* mask,
                                 const int* dev_tok, const int* parents, int* draft_tokens, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  return launch_pdl(draft_planted_kernel, dim3((p.batch + 127) / 128), dim3(128), 0, s, 1, d, p, succ, mask, dev_tok,
                    parents, draft_tokens);
}

// ------------------------------------------------------------------ lane state init
__global__ void init_state_kernel(LaneDev d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d.n_pages) d.free_list[i] = d.n_pages - 1 - i;     // pop order 0, 1, 2, ...
  if (i < d.max_slots) { d.len[i] = 0; d.pending[i] = 0; d.rid[i] = 0ull; }
  if (i < kNumStats) d.stats[i] = 0ull;
  if (i == 0) { d.free_top[0] = d.n_pages; d.free_top[1] = 0; *d.err = 0; }   // [1]: free-list lock
}

cudaError_t launch_init_state(const LaneDev& d, cudaStream_t s) {
  int n = d.n_pages;
  if (d.max_slots > n) n = d.max_slots;
  if (kNumStats > n) n = kNumStats;
  SV_COUNT_LAUNCH();
  init_state_kernel<<<(n + 255) / 256, 256, 0, s>>>(d);
  return cudaGetLastError();
}

}  // namespace sv
