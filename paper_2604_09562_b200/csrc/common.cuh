// Shared device helpers for the sv kernels (sm_100a). Product code: no oracle code here.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define SV_DEV __device__ __forceinline__

namespace sv {

// ---------------------------------------------------------------- programmatic dependent launch
// (lane.h launch_pdl): wait = every earlier kernel of the stream has finished and its writes are
// visible; trigger = the next kernel may be scheduled now.
SV_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SV_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based RNG (north_star "counter-based Philox RNG"); constants of
// Random123 / cuRAND. Key = (seed_lo, seed_hi); counter =
// (z, rid_lo, rid_hi, purpose << 28 | x >> 2); R7.
struct u32x4 { uint32_t x, y, z, w; };

SV_DEV u32x4 philox10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

// U = ((w >> 9) + 0.5) * 2^-23, exact in fp32 (R7).
SV_DEV float word_to_uniform(uint32_t w) { return (float(w >> 9) + 0.5f) * 1.1920928955078125e-07f; }

enum { PURPOSE_ACCEPT = 0, PURPOSE_RACE = 1 };

SV_DEV float uniform_accept(uint64_t seed, uint64_t rid, uint32_t z) {
  u32x4 c{z, uint32_t(rid), uint32_t(rid >> 32), uint32_t(PURPOSE_ACCEPT) << 28};
  return word_to_uniform(philox10(c, uint32_t(seed), uint32_t(seed >> 32)).x);
}

// accept uniform of the s-th sibling tried at sequence index z (token trees, R30):
// counter word s >> 2, lane s & 3; s = 0 is uniform_accept
SV_DEV float uniform_accept_rank(uint64_t seed, uint64_t rid, uint32_t z, uint32_t s) {
  u32x4 c{z, uint32_t(rid), uint32_t(rid >> 32), (uint32_t(PURPOSE_ACCEPT) << 28) | (s >> 2)};
  const u32x4 w = philox10(c, uint32_t(seed), uint32_t(seed >> 32));
  const uint32_t l = s & 3;
  return word_to_uniform(l == 0 ? w.x : (l == 1 ? w.y : (l == 2 ? w.z : w.w)));
}

// four race uniforms for x = 4m .. 4m+3
SV_DEV u32x4 race_words(uint64_t seed, uint64_t rid, uint32_t z, uint32_t m) {
  u32x4 c{z, uint32_t(rid), uint32_t(rid >> 32), (uint32_t(PURPOSE_RACE) << 28) | m};
  return philox10(c, uint32_t(seed), uint32_t(seed >> 32));
}

// ---------------------------------------------------------------- bf16 helpers
SV_DEV float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
SV_DEV __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

SV_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SV_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace sv
