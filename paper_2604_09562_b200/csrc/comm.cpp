// a9: prefill -> decode KV hand-off over NCCL point-to-point (NVLink 5 / NVSwitch).
// Replaces the paper's NIXL GPU-direct P2P transfer.
// One message per request: packed KV [n_layers][n][2][Hkv][d_h] bf16 + 16-byte trailer.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include "../../include/sv.h"

sv_status sv_internal_append_packed(sv_ctx* c, int32_t slot, uint64_t request_id, const void* packed,
                                    int32_t n_tokens);
sv_status sv_internal_append_check(sv_ctx* c, int32_t slot, uint64_t request_id, const void* packed,
                                   int32_t n_tokens);
cudaStream_t sv_internal_stream(sv_ctx* c);
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
  cudaStream_t st = sv_internal_stream(ctx);
  sv_status s = nccl_ok(ncclGroupStart());
  if (s) return s;
  s = nccl_ok(ncclRecv(staging, bytes, ncclUint8, peer, (ncclComm_t)nccl_comm, st));
  sv_status s2 = nccl_ok(ncclGroupEnd());
  if (s || s2) return s ? s : s2;
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

}  // extern "C"
