// tcgen05 verify attention (k_attn_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "lane.h"

namespace sv {
int attn_tc_smem_bytes(int dh);
// map_q: 3-D (d_h, Hq, Tmax) over the Q buffer, box (64, G, 64 / G); map_kv: 2-D (d_h, pool rows),
// box (64, 64); both bf16 with 128-byte swizzle.
cudaError_t launch_attention_tc(const CUtensorMap& map_q, const CUtensorMap& map_kv, const LaneDev& d, int layer,
                                int num_sms, cudaStream_t s);
}  // namespace sv
