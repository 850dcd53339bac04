// KV-cache state kernels:
//   a8  commit / rollback compaction (eq:kv_concatenation): chain rows
//       0..n-1 of kc/vc -> pages at positions L..L+n-1, pages popped from the device free list
//   a9  append (sv_append_kv / hand-off receive): context K/V -> newly popped pages
//   release: pages back to the free list; hand-off wire packing.
// Device free list: a stack free_list[0 .. top-1]; pops take [top-n, top), pushes append. Every
// mutation holds a spin lock (free_top[1]): the hand-off receive pops pages on the lane's comm
// stream while commits (pops) and releases (pushes) run on the lane stream. The holder is always a
// running thread, so waiters only spin for one short critical section.
#include "common.cuh"
#include "lane.h"
#include "../../include/sv.h"

namespace sv {

SV_DEV size_t pool_row(const LaneDev& d, int layer, int page, int kv, int h, int off) {
  return ((((size_t)layer * d.n_pages + page) * 2 + kv) * d.Hkv + h) * d.page + off;
}

// acquire / release atomics (no full fences): the critical section's reads see the previous holder's
// writes, and its own writes are visible to the next holder
SV_DEV void fl_lock(const LaneDev& d) {
  int old;
  for (;;) {
    asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], 0, 1;" : "=r"(old) : "l"(d.free_top + 1) : "memory");
    if (old == 0) break;
    __nanosleep(32);
  }
}
SV_DEV void fl_unlock(const LaneDev& d) {
  asm volatile("st.release.gpu.global.b32 [%0], 0;" ::"l"(d.free_top + 1) : "memory");
}
SV_DEV int fl_top(const LaneDev& d) { return *reinterpret_cast<volatile int*>(d.free_top); }

// pop `n` pages for `slot` whose first new page index is `first` (one thread); false on exhaustion
SV_DEV bool pop_pages(const LaneDev& d, int slot, int first, int n) {
  if (n <= 0) return true;
  fl_lock(d);
  const int old = fl_top(d);
  const bool ok = old >= n;
  if (ok) {
    for (int i = 0; i < n; ++i) d.page_table[slot * d.max_pages_per_slot + first + i] = d.free_list[old - n + i];
    *d.free_top = old - n;
  }
  fl_unlock(d);
  if (!ok) atomicOr(d.err, SV_DERR_NO_PAGES);
  return ok;
}

// ------------------------------------------------------------------ a8 commit
__global__ void __launch_bounds__(256) commit_kernel(LaneDev d, const int* __restrict__ n_keep) {
  pdl_trigger();
  pdl_wait();
  // Loads that do not depend on each other are issued together (latency-bound kernel: every dependent
  // global round trip is ~1 us): the request's row offset, the accepted path and emitted tokens (K1
  // words each) with the slot; the slot's length; then the page-table words of the <= 8 pages the new
  // tokens can touch, in parallel with thread 0's page pop (the pops write the new page ids to s_pg too)
  __shared__ int s_n, s_ok;
  __shared__ int s_row[kMaxDepth + 1], s_tok[kMaxDepth + 1];
  __shared__ int s_pg[8];
  const int b = blockIdx.x, tid = threadIdx.x;
  const int K1 = d.max_depth + 1;
  const int slot = d.slots[b];
  const int row0 = d.row_off[b];
  if (tid < K1) {
    s_row[tid] = row0 + d.path_int[(size_t)b * K1 + tid];   // the accepted path's chain rows (R30)
    s_tok[tid] = d.tok_int[(size_t)b * K1 + tid];
  }
  const int L = d.len[slot];
  const int have = (L + d.page - 1) / d.page, pg0 = L / d.page;
  if (tid >= 32 && tid < 40) {                         // pages already owned (new ones: thread 0)
    const int idx = pg0 + tid - 32;
    if (idx < have) s_pg[tid - 32] = d.page_table[slot * d.max_pages_per_slot + idx];
  }
  if (tid == 0) {
    int n = d.acc_int[b] + 1;                          // acc_int = -1 on error -> n = 0
    if (n > 0 && n_keep) {
      const int nk = n_keep[b];
      if (nk < 1) { atomicOr(d.err, SV_DERR_BAD_KEEP); n = 0; }
      else if (nk < n) n = nk;
    }
    int ok = n > 0;
    if (ok) {
      const int need = (L + n + d.page - 1) / d.page;
      if (L + n > d.max_pos || need > d.max_pages_per_slot) {
        atomicOr(d.err, SV_DERR_MAX_POS);
        ok = 0;
      } else if (need > have) {
        const int cnt = need - have;
        fl_lock(d);
        const int old = fl_top(d);
        ok = old >= cnt;
        if (ok) {
          for (int i = 0; i < cnt; ++i) {
            const int id = d.free_list[old - cnt + i];
            d.page_table[slot * d.max_pages_per_slot + have + i] = id;
            s_pg[have + i - pg0] = id;
          }
          *d.free_top = old - cnt;
        }
        fl_unlock(d);
        if (!ok) atomicOr(d.err, SV_DERR_NO_PAGES);
      }
    }
    s_n = n;
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return;
  const int n = s_n;
  const int vec_per_row = d.dh / 8;              // 16-byte vectors per (token, kv head)
  const int per_tok = 2 * d.Hkv * vec_per_row;
  const size_t nkv = (size_t)d.Hkv * d.dh;
  const int total = d.n_layers * n * per_tok;
  constexpr int U = 4;                           // loads of U vectors in flight before their stores
  for (int i0 = tid; i0 < total; i0 += U * blockDim.x) {
    uint4 v[U];
    bf16* dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      dst[u] = nullptr;
      if (i >= total) continue;
      const int layer = i / (n * per_tok), li = i % (n * per_tok);
      const int c = li / per_tok, rem = li % per_tok;
      const int kv = rem / (d.Hkv * vec_per_row), h = (rem / vec_per_row) % d.Hkv, v8 = rem % vec_per_row;
      const int t = L + c;
      const bf16* src = (kv ? d.vc : d.kc) + ((size_t)layer * d.Tmax + s_row[c]) * nkv + (size_t)h * d.dh + v8 * 8;
      v[u] = *reinterpret_cast<const uint4*>(src);
      dst[u] = d.pool + pool_row(d, layer, s_pg[t / d.page - pg0], kv, h, t % d.page) * d.dh + v8 * 8;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u]) *reinterpret_cast<uint4*>(dst[u]) = v[u];
  }
  if (tid == 0) {
    d.len[slot] = L + n;
    d.pending[slot] = s_tok[n - 1];
  }
}

cudaError_t launch_commit(const LaneDev& d, const int* n_keep, int batch, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  return launch_pdl(commit_kernel, dim3(batch), dim3(256), 0, s, 1, d, n_keep);
}

// ------------------------------------------------------------------ append (alloc + copy)
// scratch int: d.batch_n is reused? no — a dedicated word: item_start[kMaxBatch] region is per
// verify; append keeps its old length in n_items[1] (workspace word reserved for it).
__global__ void append_alloc_kernel(LaneDev d, int slot, unsigned long long rid, int n, int pending,
                                    const int* pending_dev, int* scratch) {
  // thread 0 checks and reserves the pages (one atomic on the free-list top); the block copies the
  // popped page ids into the slot's table in parallel (a long prompt pops hundreds of pages)
  __shared__ int s_old, s_cnt, s_first;
  if (threadIdx.x == 0) {
    const int L = d.len[slot];
    const int have = (L + d.page - 1) / d.page, need = (L + n + d.page - 1) / d.page;
    int ok = 1, cnt = need - have, old = 0;
    if (L + n > d.max_pos || need > d.max_pages_per_slot) { atomicOr(d.err, SV_DERR_MAX_POS); ok = 0; }
    if (ok && cnt > 0) {
      fl_lock(d);                                    // released below, after the block copied the ids
      old = fl_top(d);
      if (old < cnt) {
        fl_unlock(d);
        atomicOr(d.err, SV_DERR_NO_PAGES);
        ok = 0;
      }
    }
    int pend = pending_dev ? *pending_dev : pending;
    if (pend < 0 || pend >= d.V) { atomicOr(d.err, SV_DERR_BAD_TOKEN); pend = 0; }
    scratch[0] = L;
    scratch[1] = ok;
    if (ok) {
      d.len[slot] = L + n;
      d.pending[slot] = pend;
      d.rid[slot] = rid;
    }
    s_old = old;
    s_cnt = ok ? cnt : 0;
    s_first = have;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_cnt; i += blockDim.x)
    d.page_table[slot * d.max_pages_per_slot + s_first + i] = d.free_list[s_old - s_cnt + i];
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt > 0) {
    *d.free_top = s_old - s_cnt;
    fl_unlock(d);
  }
}

// The KV copies below move "row sets": the Hkv x d_h/8 16-byte vectors of one (layer, token, K|V).
// One warp per row set: the page is looked up once (a broadcast load), all of the warp's loads are
// issued before its stores, and the packed side is one contiguous segment (Hkv * d_h * 2 bytes).
constexpr int KV_U = 8;                          // vectors per lane in flight (row sets <= 256 vectors per pass)

__global__ void append_copy_kernel(LaneDev d, int slot, const bf16* __restrict__ k, const bf16* __restrict__ v,
                                   int n, int packed, const int* __restrict__ scratch) {
  if (!scratch[1]) return;
  const int L = scratch[0];
  const int vpr = d.dh / 8, nvec = d.Hkv * vpr, nsets = d.n_layers * n * 2;
  const size_t nkv = (size_t)d.Hkv * d.dh;
  const int lane = threadIdx.x & 31, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int set = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; set < nsets; set += nwarps) {
    const int kv = set & 1, lt = set >> 1, layer = lt / n, c = lt - layer * n, t = L + c;
    const int page = d.page_table[slot * d.max_pages_per_slot + t / d.page];
    bf16* dst0 = d.pool + pool_row(d, layer, page, kv, 0, t % d.page) * d.dh;
    const bf16* src0 = packed ? k + (((size_t)layer * n + c) * 2 + kv) * nkv : (kv ? v : k) + ((size_t)layer * n + c) * nkv;
    for (int e0 = 0; e0 < nvec; e0 += 32 * KV_U) {
      uint4 buf[KV_U];
#pragma unroll
      for (int u = 0; u < KV_U; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) buf[u] = *reinterpret_cast<const uint4*>(src0 + (size_t)e * 8);
      }
#pragma unroll
      for (int u = 0; u < KV_U; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) {
          const int h = e / vpr, v8 = e - h * vpr;
          *reinterpret_cast<uint4*>(dst0 + (size_t)h * d.page * d.dh + v8 * 8) = buf[u];
        }
      }
    }
  }
}

static int kv_copy_grid(int nsets) {                // 8 warps per block, at most 8 blocks per SM
  const int blocks = (nsets + 7) / 8;
  return blocks < 148 * 8 ? (blocks > 0 ? blocks : 1) : 148 * 8;
}

cudaError_t launch_append(const LaneDev& d, int slot, unsigned long long rid, const bf16* k, const bf16* v, int n,
                          int pending, const int* pending_dev, int packed, cudaStream_t s) {
  int* scratch = d.n_items + 1;                  // two spare workspace words
  SV_COUNT_LAUNCH();
  append_alloc_kernel<<<1, 256, 0, s>>>(d, slot, rid, n, pending, pending_dev, scratch);
  if (n > 0) {
    SV_COUNT_LAUNCH();
    append_copy_kernel<<<kv_copy_grid(d.n_layers * n * 2), 256, 0, s>>>(d, slot, k, v, n, packed, scratch);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a9 batched hand-off: page pop
// One CTA per received request: pops ceil(n / page) pages for the (EMPTY, len 0) slot, writes its
// page-table row, len = n and the request id. The pages and the pending token are then written by
// the NCCL receives (sv_kv_recv_slots); the host checked the free list beforehand.
__global__ void handoff_alloc_kernel(LaneDev d, const int* __restrict__ slots, const unsigned long long* __restrict__ rids,
                                     const int* __restrict__ ns) {
  __shared__ int s_old, s_cnt;
  const int slot = slots[blockIdx.x], n = ns[blockIdx.x];
  if (threadIdx.x == 0) {
    const int cnt = (n + d.page - 1) / d.page;
    fl_lock(d);
    const int old = fl_top(d);
    if (old < cnt) {
      fl_unlock(d);
      atomicOr(d.err, SV_DERR_NO_PAGES);
      s_cnt = -1;
    } else {
      s_cnt = cnt;
      d.len[slot] = n;
      d.rid[slot] = rids[blockIdx.x];
    }
    s_old = old;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_cnt; i += blockDim.x)
    d.page_table[slot * d.max_pages_per_slot + i] = d.free_list[s_old - s_cnt + i];
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt >= 0) {
    *d.free_top = s_old - s_cnt;
    fl_unlock(d);
  }
}

cudaError_t launch_handoff_alloc(const LaneDev& d, const int* slots, const unsigned long long* rids, const int* ns,
                                 int n, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  handoff_alloc_kernel<<<n, 256, 0, s>>>(d, slots, rids, ns);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a9 batched hand-off: block gather / scatter
// Staging layout (sv_host.cpp "batched page-block hand-off"): block b of the batch = request i
// (bstart[i] <= b < bstart[i + 1]), layer = (b - bstart[i]) / m_i, page index p = (b - bstart[i]) % m_i
// (m_i = ceil(n_i / page)); then the n pending tokens. A block is [2][Hkv][page][d_h] bf16, contiguous
// in the pool at (layer, page id); CTAs copy whole blocks with 16-byte vectors, U in flight per thread.
SV_DEV void handoff_block(const LaneDev& d, const int* slots, const int* ns, const int* bstart, int n, int b,
                          int* slot, int* layer, int* p) {
  int lo = 0, hi = n - 1;                          // last i with bstart[i] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bstart[mid] <= b) lo = mid; else hi = mid - 1;
  }
  const int m = (ns[lo] + d.page - 1) / d.page, rel = b - bstart[lo];
  *slot = slots[lo];
  *layer = rel / m;
  *p = rel - *layer * m;
}

template <bool GATHER>
__global__ void __launch_bounds__(256) handoff_copy_kernel(LaneDev d, const int* __restrict__ slots,
                                                           const int* __restrict__ ns, const int* __restrict__ bstart,
                                                           int n, char* __restrict__ staging) {
  const int nb = bstart[n];
  const size_t bvec = (size_t)2 * d.Hkv * d.page * d.dh / 8;     // 16-byte vectors per block
  constexpr int U = 8;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    int slot, layer, p;
    handoff_block(d, slots, ns, bstart, n, b, &slot, &layer, &p);
    const int page = d.page_table[slot * d.max_pages_per_slot + p];
    uint4* pg = reinterpret_cast<uint4*>(d.pool + ((size_t)layer * d.n_pages + page) * bvec * 8);
    uint4* st = reinterpret_cast<uint4*>(staging) + (size_t)b * bvec;
    const uint4* src = GATHER ? pg : st;
    uint4* dst = GATHER ? st : pg;
    for (size_t v0 = threadIdx.x; v0 < bvec; v0 += (size_t)U * blockDim.x) {
      uint4 buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = v0 + (size_t)u * blockDim.x;
        if (v < bvec) buf[u] = src[v];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t v = v0 + (size_t)u * blockDim.x;
        if (v < bvec) dst[v] = buf[u];
      }
    }
  }
  if (blockIdx.x == 0) {
    int* tail = reinterpret_cast<int*>(staging + (size_t)nb * bvec * 16);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (GATHER) tail[i] = d.pending[slots[i]];
      else d.pending[slots[i]] = tail[i];
    }
  }
}

static int handoff_grid(const LaneDev& d) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return 4 * sms;                                  // 4 CTAs of 256 threads per SM, grid-stride over blocks
}

cudaError_t launch_handoff_gather(const LaneDev& d, const int* slots, const int* ns, const int* bstart, int n,
                                  char* staging, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  handoff_copy_kernel<true><<<handoff_grid(d), 256, 0, s>>>(d, slots, ns, bstart, n, staging);
  return cudaGetLastError();
}

cudaError_t launch_handoff_scatter(const LaneDev& d, const int* slots, const int* ns, const int* bstart, int n,
                                   const char* staging, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  handoff_copy_kernel<false><<<handoff_grid(d), 256, 0, s>>>(d, slots, ns, bstart, n, const_cast<char*>(staging));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ release
__global__ void release_kernel(LaneDev d, int slot) {
  const int L = d.len[slot];
  const int n = (L + d.page - 1) / d.page;
  __shared__ int s_old;
  if (threadIdx.x == 0) {
    fl_lock(d);
    s_old = fl_top(d);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    d.free_list[s_old + i] = d.page_table[slot * d.max_pages_per_slot + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    *d.free_top = s_old + n;
    fl_unlock(d);
    d.len[slot] = 0; d.pending[slot] = 0; d.rid[slot] = 0ull;
  }
}

cudaError_t launch_release(const LaneDev& d, int slot, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  release_kernel<<<1, 256, 0, s>>>(d, slot);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ hand-off packing
__global__ void kv_pack_kernel(const bf16* __restrict__ k, const bf16* __restrict__ v, int n_layers, int Hkv, int dh,
                               int n, int pending, bf16* __restrict__ out) {
  const int nvec = Hkv * dh / 8, nsets = n_layers * n * 2;
  const size_t nkv = (size_t)Hkv * dh;
  const int lane = threadIdx.x & 31, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int set = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; set < nsets; set += nwarps) {
    const int kv = set & 1, lt = set >> 1;             // lt = layer * n + token
    const bf16* src0 = (kv ? v : k) + (size_t)lt * nkv;
    bf16* dst0 = out + (size_t)set * nkv;               // [layer][token][kv] = set
    for (int e0 = 0; e0 < nvec; e0 += 32 * KV_U) {
      uint4 buf[KV_U];
#pragma unroll
      for (int u = 0; u < KV_U; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) buf[u] = *reinterpret_cast<const uint4*>(src0 + (size_t)e * 8);
      }
#pragma unroll
      for (int u = 0; u < KV_U; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) *reinterpret_cast<uint4*>(dst0 + (size_t)e * 8) = buf[u];
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int* trailer = reinterpret_cast<int*>(out + (size_t)nsets * nkv);
    trailer[0] = pending;
    trailer[1] = trailer[2] = trailer[3] = 0;
  }
}

cudaError_t launch_kv_pack(const bf16* k, const bf16* v, int n_layers, int Hkv, int dh, int n, int pending,
                           void* packed, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  kv_pack_kernel<<<kv_copy_grid(n_layers * n * 2), 256, 0, s>>>(k, v, n_layers, Hkv, dh, n, pending,
                                                                reinterpret_cast<bf16*>(packed));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ a9 prefill side: pack a slot
// Committed rows 0..n-1 of `slot` (all layers, from its pages) + its pending token -> the wire
// format [n_layers][n][2][Hkv][dh] bf16 + 16-byte trailer. n > len sets SV_DERR_MAX_POS.
__global__ void kv_pack_slot_kernel(LaneDev d, int slot, int n, bf16* __restrict__ out) {
  const int L = d.len[slot];
  if (n > L) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(d.err, SV_DERR_MAX_POS);
    return;
  }
  const int vpr = d.dh / 8, nvec = d.Hkv * vpr, nsets = d.n_layers * n * 2;
  const size_t nkv = (size_t)d.Hkv * d.dh;
  const int lane = threadIdx.x & 31, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int set = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; set < nsets; set += nwarps) {
    const int kv = set & 1, lt = set >> 1, layer = lt / n, t = lt - layer * n;
    const int page = d.page_table[slot * d.max_pages_per_slot + t / d.page];
    const bf16* src0 = d.pool + pool_row(d, layer, page, kv, 0, t % d.page) * d.dh;
    bf16* dst0 = out + (size_t)set * nkv;
    for (int e0 = 0; e0 < nvec; e0 += 32 * KV_U) {
      uint4 buf[KV_U];
#pragma unroll
      for (int u = 0; u < KV_U; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) {
          const int h = e / vpr, v8 = e - h * vpr;
          buf[u] = *reinterpret_cast<const uint4*>(src0 + (size_t)h * d.page * d.dh + v8 * 8);
        }
      }
#pragma unroll
      for (int u = 0; u < KV_U; ++u) {
        const int e = e0 + lane + 32 * u;
        if (e < nvec) *reinterpret_cast<uint4*>(dst0 + (size_t)e * 8) = buf[u];
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int* trailer = reinterpret_cast<int*>(out + (size_t)nsets * nkv);
    trailer[0] = d.pending[slot];
    trailer[1] = trailer[2] = trailer[3] = 0;
  }
}

cudaError_t launch_kv_pack_slot(const LaneDev& d, int slot, int n, void* packed, cudaStream_t s) {
  SV_COUNT_LAUNCH();
  kv_pack_slot_kernel<<<kv_copy_grid(d.n_layers * n * 2), 256, 0, s>>>(d, slot, n, reinterpret_cast<bf16*>(packed));
  return cudaGetLastError();
}

}  // namespace sv
