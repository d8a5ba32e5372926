// keys.cuh — 64-bit token keys (total order of R7 as one integer), warp-distributed sorted top-K
// lists and the online-softmax push, shared by the single-row step kernels (cstep.cu, gstep.cu).
#pragma once
#include "common.cuh"

namespace ds {

// ---------------------------------------------------------------- total order as one 64-bit key
// key = ord_key(z) << 32 | ~id: a larger key is a larger logit, or an equal logit with a lower
// token id (R7, R23: -0 folded into +0).  0 is below every valid key (padding).
__device__ __forceinline__ unsigned long long tok_key(float z, int id) {
  return ((unsigned long long)ord_key(z) << 32) | (unsigned long long)(~(uint32_t)id);
}
__device__ __forceinline__ float key_value(unsigned long long k) {
  const uint32_t u = (uint32_t)(k >> 32);
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ __forceinline__ int key_id(unsigned long long k) { return (int)(~(uint32_t)k); }

// Warp-distributed sorted list (lane r < K holds the r-th best key; 0 = empty).  `kth` mirrors
// lane K-1's entry, so a candidate that cannot enter costs one compare.
__device__ __forceinline__ void list_insert(unsigned long long& mine, unsigned long long& kth, unsigned long long x,
                                            int K, int lane) {
  if (x <= kth) return;  // warp-uniform
  const uint32_t lanes = K >= 32 ? 0xffffffffu : ((1u << K) - 1u);
  const int pos = __popc(__ballot_sync(0xffffffffu, mine > x) & lanes);
  const unsigned long long up = __shfl_up_sync(0xffffffffu, mine, 1);
  if (lane > pos) mine = up;
  else if (lane == pos) mine = x;
  kth = __shfl_sync(0xffffffffu, mine, K - 1);
}

// Online softmax accumulation of one logit (warp-uniform state).
__device__ __forceinline__ void lse_push(float& m, float& s, float z) {
  if (z > m) {
    s = s * expf(m - z) + 1.f;
    m = z;
  } else {
    s += expf(z - m);
  }
}

}  // namespace ds
