// tcgen05 verify attention (k_attn_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "lane.h"

namespace sv {
int attn_tc_smem_bytes(int dh);
// map_q: 3-D (d_h, Hq, Tmax) over the Q buffer, box (64, 1, q_box_tokens) = one q head's chain rows;
// map_kv: 2-D (d_h, pool rows), box (64, 64) = one page of one kv head; both bf16, 128-byte swizzle.
// Requires page_size 64, d_h in {64, 128}, G = Hq / Hkv <= 4 and max_depth + 1 <= q_box_tokens <= 32.
cudaError_t launch_attention_tc(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                int num_sms, int q_box_tokens, cudaStream_t s);
// keys-on-lanes variant (k_attn_tc2.cu), d_h = 128 only. map_q: 3-D (d_h, Hq, Tmax), box (64, G, 64 / G)
// = the 64 query slots j*G + g of one kv head; map_kv as above. Requires (max_depth + 1) * G <= 64.
int attn_tc2_smem_bytes();
cudaError_t launch_attention_tc2(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                 int num_sms, cudaStream_t s);
// long-chunk prefill attention (k_attn_prefill.cu): map_q 3-D (d_h, Hq, Tmax), box (64, 1, 128 / G);
// every key from the pages (the chunk's rows committed first), per-row causal limit, normalised O.
cudaError_t launch_attention_prefill(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                     int n_items, int num_sms, cudaStream_t s);
}  // namespace sv
