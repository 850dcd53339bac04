// NEXT-3 chunked prefill with long chunks (eq:prefill_computation; R29):
// a chunk of C prompt tokens (C up to the workspace's Tmax rows) of one slot runs through the layer
// stack as C rows at positions L .. L+C-1 (L = the slot's committed length):
//   prefill_plan   rows, positions, tokens, page pops for the chunk, attention work items
//   (per layer) QKV GEMM + RoPE -> prefill_kv copies the chunk's K/V rows into their pages ->
//               attn_prefill (k_attn_prefill.cu) reads every key from the pages with a per-row causal
//               limit -> O-proj, MLP
//   (last chunk) final RMSNorm + lm-head of the LAST row only (its argmax is the next token)
//   prefill_finish len += C; pending = the next prompt token, or the argmax of the last row.
#include "common.cuh"
#include "lane.h"
#include "../../include/sv.h"

namespace sv {

// free-list lock (k_kv.cu)
SV_DEV void pf_lock(const LaneDev& d) {
  while (atomicCAS(d.free_top + 1, 0, 1) != 0) __nanosleep(32);
  __threadfence();
}
SV_DEV void pf_unlock(const LaneDev& d) {
  __threadfence();
  atomicExch(d.free_top + 1, 0);
}

// One CTA. Work items (0, h, qb, 0), longest first (qb descending), RB = 128 / G rows per block.
__global__ void __launch_bounds__(256) prefill_plan_kernel(LaneDev d, int slot, const int* __restrict__ tokens, int C) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_L, s_old, s_cnt, s_first, s_bad;
  if (threadIdx.x == 0) {
    const int L = d.len[slot];
    const int have = (L + d.page - 1) / d.page, need = (L + C + d.page - 1) / d.page;
    s_L = L;
    s_bad = 0;
    s_cnt = 0;
    s_first = have;
    if (L + C > d.max_pos || need > d.max_pages_per_slot) {
      atomicOr(d.err, SV_DERR_MAX_POS);
      s_bad = 1;
    } else if (need > have) {
      pf_lock(d);
      const int old = *reinterpret_cast<volatile int*>(d.free_top);
      if (old < need - have) {
        pf_unlock(d);
        atomicOr(d.err, SV_DERR_NO_PAGES);
        s_bad = 1;
      } else {
        s_old = old;
        s_cnt = need - have;
      }
    }
    d.row_off[0] = 0;
    d.row_off[1] = C;
    d.slots[0] = slot;
    d.depths[0] = C - 1;
    *d.batch_n = 1;
    *d.T_dev = C;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_cnt; i += blockDim.x)
    d.page_table[slot * d.max_pages_per_slot + s_first + i] = d.free_list[s_old - s_cnt + i];
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt > 0) {
    *d.free_top = s_old - s_cnt;
    pf_unlock(d);
  }
  for (int r = threadIdx.x; r < C; r += blockDim.x) {
    int tok = tokens[r];
    if (tok < 0 || tok >= d.V) {
      atomicOr(d.err, SV_DERR_BAD_TOKEN);
      tok = 0;
    }
    d.row_req[r] = 0;
    d.row_pos[r] = s_bad ? 0 : s_L + r;
    d.chain_tok[r] = tok;
  }
  const int G = d.Hq / d.Hkv, RB = 128 / G, nqb = (C + RB - 1) / RB;
  const int n_items = s_bad ? 0 : d.Hkv * nqb;
  for (int it = threadIdx.x; it < n_items; it += blockDim.x) {
    const int qb = nqb - 1 - it / d.Hkv, h = it % d.Hkv;
    d.items[it] = make_int4(0, h, qb, 0);
  }
  if (threadIdx.x == 0) *d.n_items = n_items;
}

cudaError_t launch_prefill_plan(const LaneDev& d, int slot, const int* tokens, int C, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  return launch_pdl(prefill_plan_kernel, dim3(1), dim3(256), 0, s, 1, d, slot, tokens, C);
}

// The chunk's K/V rows of one layer (chain scratch kc / vc rows 0..C-1) -> pages at L .. L+C-1.
// One warp per (row, K|V) set, page looked up once, all loads before the stores.
__global__ void __launch_bounds__(256) prefill_kv_kernel(LaneDev d, int layer, int C) {
  pdl_trigger();
  pdl_wait();
  if (*d.n_items == 0) return;                          // the plan refused the chunk
  const int slot = d.slots[0], L = d.len[slot];
  const int vpr = d.dh / 8, nvec = d.Hkv * vpr;
  const size_t nkv = (size_t)d.Hkv * d.dh;
  const int lane = threadIdx.x & 31, nwarps = (gridDim.x * blockDim.x) >> 5;
  const bf16* kc = d.kc + (size_t)layer * d.Tmax * nkv;
  const bf16* vc = d.vc + (size_t)layer * d.Tmax * nkv;
  for (int set = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; set < 2 * C; set += nwarps) {
    const int kv = set & 1, c = set >> 1, t = L + c;
    const int page = d.page_table[slot * d.max_pages_per_slot + t / d.page];
    bf16* dst0 = d.pool + (((((size_t)layer * d.n_pages + page) * 2 + kv) * d.Hkv) * d.page + t % d.page) * d.dh;
    const bf16* src0 = (kv ? vc : kc) + (size_t)c * nkv;
    for (int e0 = 0; e0 < nvec; e0 += 32 * 8) {
      uint4 buf[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) buf[u] = *reinterpret_cast<const uint4*>(src0 + (size_t)e * 8);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) {
          const int h = e / vpr, v8 = e - h * vpr;
          *reinterpret_cast<uint4*>(dst0 + (size_t)h * d.page * d.dh + v8 * 8) = buf[u];
        }
      }
    }
  }
}

cudaError_t launch_prefill_kv(const LaneDev& d, int layer, int C, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  int blocks = (2 * C + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  return launch_pdl(prefill_kv_kernel, dim3(blocks), dim3(256), 0, s, 1, d, layer, C);
}

// len += C; pending = next_token (>= 0), or the lowest-index argmax of lm-head row 0 (vocab-tile
// statistics: the first tile holding the row maximum, its lowest argmax) -> also *y_out.
__global__ void __launch_bounds__(256) prefill_finish_kernel(LaneDev d, int C, int next_token, int* y_out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float s_v[256];
  __shared__ int s_t[256];
  const int slot = d.slots[0];
  int y = next_token;
  if (next_token < 0) {
    float best = -INFINITY;
    int bt = 0x7fffffff;
    for (int t = threadIdx.x; t < d.nt; t += blockDim.x) {
      const float v = d.tile_max[t];
      if (v > best || (v == best && t < bt)) { best = v; bt = t; }
    }
    s_v[threadIdx.x] = best;
    s_t[threadIdx.x] = bt;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        const float v = s_v[threadIdx.x + w];
        const int t = s_t[threadIdx.x + w];
        if (v > s_v[threadIdx.x] || (v == s_v[threadIdx.x] && t < s_t[threadIdx.x])) {
          s_v[threadIdx.x] = v;
          s_t[threadIdx.x] = t;
        }
      }
      __syncthreads();
    }
    y = s_t[0] < d.nt ? d.tile_arg[s_t[0]] : 0;
  }
  if (threadIdx.x == 0) {
    if (*d.n_items == 0) {                              // refused chunk: nothing committed
      *y_out = -1;
      return;
    }
    d.len[slot] += C;
    d.pending[slot] = y;
    *y_out = y;
  }
}

cudaError_t launch_prefill_finish(const LaneDev& d, int C, int next_token, int* y_out, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  return launch_pdl(prefill_finish_kernel, dim3(1), dim3(256), 0, s, 1, d, C, next_token, y_out);
}

}  // namespace sv
