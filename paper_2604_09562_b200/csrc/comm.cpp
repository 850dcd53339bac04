// a9: prefill -> decode KV hand-off over NCCL point-to-point (NVLink 5 / NVSwitch).
// Replaces the paper's NIXL GPU-direct P2P transfer.
// One message per request: packed KV [n_layers][n][2][Hkv][d_h] bf16 + 16-byte trailer.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <vector>

#include "../../include/sv.h"

sv_status sv_internal_append_packed(sv_ctx* c, int32_t slot, uint64_t request_id, const void* packed,
                                    int32_t n_tokens);
sv_status sv_internal_append_check(sv_ctx* c, int32_t slot, uint64_t request_id, const void* packed,
                                   int32_t n_tokens);
cudaStream_t sv_internal_stream(sv_ctx* c);
cudaStream_t sv_internal_comm_stream(sv_ctx* c);
sv_status sv_internal_comm_posted(sv_ctx* c, cudaStream_t on, int32_t n, const int32_t* slots);
sv_status sv_internal_config(sv_ctx* c, sv_config* out);
sv_status sv_internal_send_prepare(sv_ctx* c, int32_t n, const int32_t* slots, const int32_t* ntok, void* staging,
                                   size_t* bytes);
sv_status sv_internal_recv_prepare(sv_ctx* c, int32_t n, const int32_t* slots, const uint64_t* rids,
                                   const int32_t* ntok, void* staging, size_t* bytes);
sv_status sv_internal_recv_finish(sv_ctx* c, int32_t n, const void* staging);
size_t sv_internal_packed_bytes(sv_ctx* c, int32_t n_tokens);
size_t sv_kv_packed_bytes(const sv_config* cfg, int32_t n_tokens);

static sv_status nccl_ok(ncclResult_t r) {
  if (r != ncclSuccess) {
    fprintf(stderr, "[sv] NCCL error: %s\n", ncclGetErrorString(r));
    return SV_ENCCL;
  }
  return SV_OK;
}

extern "C" {

sv_status sv_nccl_unique_id(uint8_t id[128]) {
  if (!id) return SV_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  sv_status s = nccl_ok(ncclGetUniqueId(&u));
  if (s) return s;
  memcpy(id, &u, 128);
  return SV_OK;
}

sv_status sv_nccl_comm_init(int nranks, const uint8_t id[128], int rank, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return SV_EINVAL;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclComm_t c;
  sv_status s = nccl_ok(ncclCommInitRank(&c, nranks, u, rank));
  if (s) return s;
  *comm = c;
  return SV_OK;
}

sv_status sv_nccl_comm_destroy(void* comm) {
  if (!comm) return SV_EINVAL;
  return nccl_ok(ncclCommDestroy((ncclComm_t)comm));
}

sv_status sv_kv_send(const void* kv_packed, int32_t n_layers, int32_t n_kv_heads, int32_t head_dim, int32_t n_tokens,
                     int peer, void* nccl_comm, sv_stream_t stream) {
  if (!kv_packed || !nccl_comm || n_layers < 1 || n_kv_heads < 1 || head_dim < 1 || n_tokens < 0 || peer < 0)
    return SV_EINVAL;
  const size_t bytes = (size_t)n_layers * n_tokens * 2 * n_kv_heads * head_dim * 2 + 16;
  sv_status s = nccl_ok(ncclGroupStart());
  if (s) return s;
  s = nccl_ok(ncclSend(kv_packed, bytes, ncclUint8, peer, (ncclComm_t)nccl_comm, (cudaStream_t)stream));
  sv_status s2 = nccl_ok(ncclGroupEnd());
  return s ? s : s2;
}

sv_status sv_kv_recv_append(sv_ctx* ctx, int32_t slot, uint64_t request_id, int32_t n_tokens, void* staging,
                            int peer, void* nccl_comm) {
  if (!ctx || !staging || !nccl_comm || n_tokens < 0 || peer < 0) return SV_EINVAL;
  const sv_status chk = sv_internal_append_check(ctx, slot, request_id, staging, n_tokens);
  if (chk) return chk;
  const size_t bytes = sv_internal_packed_bytes(ctx, n_tokens);
  // the receive runs on the lane's comm stream (it overlaps a verify already enqueued); the append
  // copy that follows on the lane stream waits for it
  cudaStream_t st = sv_internal_comm_stream(ctx);
  sv_status s = nccl_ok(ncclGroupStart());
  if (s) return s;
  s = nccl_ok(ncclRecv(staging, bytes, ncclUint8, peer, (ncclComm_t)nccl_comm, st));
  sv_status s2 = nccl_ok(ncclGroupEnd());
  if (s || s2) return s ? s : s2;
  if ((s = sv_internal_comm_posted(ctx, st, 1, &slot))) return s;
  return sv_internal_append_packed(ctx, slot, request_id, staging, n_tokens);
}

sv_status sv_kv_append_packed(sv_ctx* ctx, int32_t slot, uint64_t request_id, int32_t n_tokens,
                              const void* kv_packed) {
  if (!ctx || !kv_packed || n_tokens < 0 || ((uintptr_t)kv_packed & 15)) return SV_EINVAL;
  return sv_internal_append_packed(ctx, slot, request_id, kv_packed, n_tokens);
}

sv_status sv_kv_loopback_append(sv_ctx* ctx, int32_t slot, uint64_t request_id, int32_t n_tokens,
                                const void* kv_packed, void* staging, int rank, void* nccl_comm) {
  if (!ctx || !kv_packed || !staging || !nccl_comm || n_tokens < 0 || rank < 0) return SV_EINVAL;
  if (((uintptr_t)kv_packed | (uintptr_t)staging) & 15) return SV_EINVAL;
  const sv_status chk = sv_internal_append_check(ctx, slot, request_id, staging, n_tokens);
  if (chk) return chk;
  const size_t bytes = sv_internal_packed_bytes(ctx, n_tokens);
  cudaStream_t st = sv_internal_stream(ctx);
  sv_status s = nccl_ok(ncclGroupStart());
  if (s) return s;
  sv_status s1 = nccl_ok(ncclSend(kv_packed, bytes, ncclUint8, rank, (ncclComm_t)nccl_comm, st));
  sv_status s2 = nccl_ok(ncclRecv(staging, bytes, ncclUint8, rank, (ncclComm_t)nccl_comm, st));
  sv_status s3 = nccl_ok(ncclGroupEnd());
  if (s1 || s2 || s3) return s1 ? s1 : (s2 ? s2 : s3);
  return sv_internal_append_packed(ctx, slot, request_id, staging, n_tokens);
}

// ---- batched hand-off (wire format: sv_host.cpp "batched page-block hand-off"): one NCCL op per batch
sv_status sv_kv_send_slots(sv_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* n_tokens, void* staging,
                           int peer, void* nccl_comm) {
  if (!nccl_comm || peer < 0) return SV_EINVAL;
  size_t bytes = 0;
  sv_status s = sv_internal_send_prepare(ctx, n, slots, n_tokens, staging, &bytes);
  if (s) return s;
  cudaStream_t st = sv_internal_comm_stream(ctx);
  if ((s = nccl_ok(ncclGroupStart()))) return s;
  s = nccl_ok(ncclSend(staging, bytes, ncclUint8, peer, (ncclComm_t)nccl_comm, st));
  const sv_status s2 = nccl_ok(ncclGroupEnd());
  if (s || s2) return s ? s : s2;
  return sv_internal_comm_posted(ctx, st, n, slots);
}

sv_status sv_kv_recv_slots(sv_ctx* ctx, int32_t n, const int32_t* slots, const uint64_t* request_ids,
                           const int32_t* n_tokens, void* staging, int peer, void* nccl_comm) {
  if (!nccl_comm || peer < 0) return SV_EINVAL;
  size_t bytes = 0;
  sv_status s = sv_internal_recv_prepare(ctx, n, slots, request_ids, n_tokens, staging, &bytes);
  if (s) return s;
  cudaStream_t st = sv_internal_comm_stream(ctx);
  if ((s = nccl_ok(ncclGroupStart()))) return s;
  s = nccl_ok(ncclRecv(staging, bytes, ncclUint8, peer, (ncclComm_t)nccl_comm, st));
  const sv_status s2 = nccl_ok(ncclGroupEnd());
  if (s || s2) return s ? s : s2;
  if ((s = sv_internal_recv_finish(ctx, n, staging))) return s;
  return sv_internal_comm_posted(ctx, st, n, slots);
}

sv_status sv_kv_loopback_slots(sv_ctx* src, sv_ctx* dst, int32_t n, const int32_t* src_slots,
                               const int32_t* dst_slots, const uint64_t* request_ids, const int32_t* n_tokens,
                               void* src_staging, void* dst_staging, int rank, void* nccl_comm) {
  if (!src || !dst || src == dst || !nccl_comm || rank < 0) return SV_EINVAL;
  sv_config a, b;
  sv_internal_config(src, &a);
  sv_internal_config(dst, &b);
  if (a.n_layers != b.n_layers || a.n_kv_heads != b.n_kv_heads || a.head_dim != b.head_dim ||
      a.page_size != b.page_size)
    return SV_EINVAL;
  size_t sb = 0, rb = 0;
  sv_status s = sv_internal_send_prepare(src, n, src_slots, n_tokens, src_staging, &sb);
  if (s) return s;
  if ((s = sv_internal_recv_prepare(dst, n, dst_slots, request_ids, n_tokens, dst_staging, &rb))) return s;
  // both halves on dst's comm stream, after src's gather
  cudaStream_t st = sv_internal_comm_stream(dst);
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return SV_ECUDA;
  cudaEventRecord(ev, sv_internal_comm_stream(src));
  cudaStreamWaitEvent(st, ev, 0);
  cudaEventDestroy(ev);
  if ((s = nccl_ok(ncclGroupStart()))) return s;
  s = nccl_ok(ncclSend(src_staging, sb, ncclUint8, rank, (ncclComm_t)nccl_comm, st));
  if (!s) s = nccl_ok(ncclRecv(dst_staging, rb, ncclUint8, rank, (ncclComm_t)nccl_comm, st));
  const sv_status s2 = nccl_ok(ncclGroupEnd());
  if (s || s2) return s ? s : s2;
  if ((s = sv_internal_recv_finish(dst, n, dst_staging))) return s;
  if ((s = sv_internal_comm_posted(src, st, n, src_slots))) return s;
  return sv_internal_comm_posted(dst, st, n, dst_slots);
}

}  // extern "C"
