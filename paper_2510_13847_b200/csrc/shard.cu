// shard.cu — cluster-sharded head across GPUs (SURVEY §8(e) option 2).
//
// Rank g owns the contiguous cluster range [m_lo, m_hi) (one contiguous block of W_perm rows).
// The router and the selection run replicated (bit-identical on every rank); each rank restricts
// every row's selection to its clusters (restrict_selection), runs the gathered head over them
// and emits one fixed-size record per row — (max, sum exp, top-k_t (logit, id)) — instead of the
// final outputs; the records are all-gathered (NCCL, by the caller) and merged in rank order
// (merge_records) into the same lse / top-k the unsharded head produces (the softmax over V_S is
// the combination of the per-shard (max, sum) pairs).
#include <algorithm>

#include "head_impl.cuh"
#include "internal.h"

namespace ds {

// One warp per row: keep the selected clusters inside [m_lo, m_hi) (ascending order preserved)
// and rebuild the exclusive scan of their sizes.
__global__ void restrict_selection_kernel(const int32_t* __restrict__ sel, const int32_t* __restrict__ cnt,
                                          int rows, int M, const int32_t* __restrict__ offsets, int m_lo, int m_hi,
                                          int32_t* __restrict__ osel, int32_t* __restrict__ ocnt,
                                          int32_t* __restrict__ ooff) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int n = cnt[r];
  int base = 0, run = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const int m = i < n ? sel[(size_t)r * M + i] : -1;
    const bool keep = m >= m_lo && m < m_hi;
    const uint32_t b = __ballot_sync(0xffffffffu, keep);
    const int pos = base + __popc(b & ((1u << lane) - 1u));
    const int sz = keep ? offsets[m + 1] - offsets[m] : 0;
    int inc = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (keep) {
      osel[(size_t)r * M + pos] = m;
      ooff[(size_t)r * (M + 1) + pos] = run + inc - sz;
    }
    base += __popc(b);
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {
    ocnt[r] = base;
    ooff[(size_t)r * (M + 1) + base] = run;
  }
}

// One CTA per row: merge the G rank records of the row (rank-major input [G][B][rec]).
__global__ void __launch_bounds__(256) merge_records_kernel(const float* __restrict__ records, int G, int B, int K,
                                                            int32_t* top_ids, float* top_logits, float* top_logp,
                                                            float* lse) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int rec = 2 + 2 * K;
  const int r = blockIdx.x;
  float* pm = reinterpret_cast<float*>(smem);
  float* ps = pm + G;
  float* cv = ps + G;
  int* ci = reinterpret_cast<int*>(cv + G * K);
  float* sv = reinterpret_cast<float*>(ci + G * K);
  int* si = reinterpret_cast<int*>(sv + G * K);
  float* red = reinterpret_cast<float*>(si + G * K);
  int* misc = reinterpret_cast<int*>(red + 64);
  for (int idx = threadIdx.x; idx < G * rec; idx += blockDim.x) {
    const int g = idx / rec, f = idx - g * rec;
    const float v = records[((size_t)g * B + r) * rec + f];
    if (f == 0) pm[g] = v;
    else if (f == 1) ps[g] = v;
    else if ((f & 1) == 0) cv[((f - 2) >> 1) * G + g] = v;
    else ci[((f - 3) >> 1) * G + g] = __float_as_int(v);
  }
  __syncthreads();
  HeadArgs a = {};
  a.k_t = K;
  a.top_ids = top_ids;
  a.top_logits = top_logits;
  a.top_logp = top_logp;
  a.lse = lse;
  a.record_out = nullptr;
  HeadCtx c = {};
  c.red = red;
  c.misc = misc;
  merge_finish(a, c, G, r, pm, ps, cv, ci, sv, si, true, nullptr);
}

cudaError_t launch_restrict(const int32_t* sel, const int32_t* cnt, int rows, int M, const int32_t* offsets, int m_lo,
                            int m_hi, int32_t* osel, int32_t* ocnt, int32_t* ooff, cudaStream_t st) {
  const int wpb = 4;
  restrict_selection_kernel<<<(rows + wpb - 1) / wpb, 32 * wpb, 0, st>>>(sel, cnt, rows, M, offsets, m_lo, m_hi,
                                                                          osel, ocnt, ooff);
  return cudaGetLastError();
}

size_t merge_records_smem(int G, int K) { return (size_t)(2 * G + 4 * G * K) * 4 + 64 * 4 + 16 * 4; }

cudaError_t launch_merge_records(const float* records, int G, int B, int K, int32_t* top_ids, float* top_logits,
                                 float* top_logp, float* lse, cudaStream_t st) {
  const size_t smem = merge_records_smem(G, K);
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(merge_records_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  merge_records_kernel<<<B, 256, smem, st>>>(records, G, B, K, top_ids, top_logits, top_logp, lse);
  return cudaGetLastError();
}

}  // namespace ds
