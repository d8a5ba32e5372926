// select_impl.cuh — S3/S4 cluster selection + router layer 2 building blocks (any blockDim).
//
// K = TopK_k(s) under (score desc, id asc) (R7), emitted in ascending cluster id (R8);
// sl_offsets = exclusive scan of |C_m| over K (|V_S| = sum |C_m|).
#pragma once
#include "common.cuh"

namespace ds {

// flags[m] |= rank(m) < k; rank(m) = #{j : s_j > s_m or (s_j == s_m and j < m)}.  s in smem.
__device__ __forceinline__ void rank_select(const float* s, int M, int k, uint8_t* flags) {
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const float key = s[m] + 0.0f;  // -0 -> +0 (R23)
    int rank = 0;
    int j = 0;
    for (; j + 4 <= M; j += 4) {
      const float4 o = *reinterpret_cast<const float4*>(s + j);
      rank += ((o.x + 0.0f) > key) || ((o.x + 0.0f) == key && j < m);
      rank += ((o.y + 0.0f) > key) || ((o.y + 0.0f) == key && j + 1 < m);
      rank += ((o.z + 0.0f) > key) || ((o.z + 0.0f) == key && j + 2 < m);
      rank += ((o.w + 0.0f) > key) || ((o.w + 0.0f) == key && j + 3 < m);
    }
    for (; j < M; ++j) {
      const float o = s[j] + 0.0f;
      rank += (o > key) || (o == key && j < m);
    }
    if (rank < k) flags[m] = 1;
  }
}

// Compact flags into ascending ids + exclusive scan of cluster sizes.
__device__ __forceinline__ void emit_selection(const uint8_t* flags, int M, const int32_t* offsets, int32_t* sel,
                                               int32_t* sel_count, int32_t* sl_off, int* scratch) {
  const int nt = blockDim.x;
  const int per = (M + nt - 1) / nt;
  const int m0 = threadIdx.x * per;
  int cnt = 0, sz = 0;
  for (int j = 0; j < per; ++j) {
    const int m = m0 + j;
    if (m < M && flags[m]) {
      ++cnt;
      sz += offsets[m + 1] - offsets[m];
    }
  }
  int tot_cnt, tot_sz;
  int pos = block_excl_scan_dyn(cnt, scratch, tot_cnt);
  int off = block_excl_scan_dyn(sz, scratch, tot_sz);
  for (int j = 0; j < per; ++j) {
    const int m = m0 + j;
    if (m < M && flags[m]) {
      sel[pos] = m;
      sl_off[pos] = off;
      ++pos;
      off += offsets[m + 1] - offsets[m];
    }
  }
  if (threadIdx.x == 0) {
    *sel_count = tot_cnt;
    sl_off[tot_cnt] = tot_sz;
  }
}

// a1[u] = act(sum_{ks} part[ks][b][u] + b1[u]) in fixed split order (act = ReLU if h_r > 0).
__device__ __forceinline__ void router_hidden(const float* part, int KS, int B, int b, int rows1, const float* b1,
                                              bool relu, float* a1) {
  for (int u = threadIdx.x; u < rows1; u += blockDim.x) {
    float acc = 0.f;
    for (int ks = 0; ks < KS; ++ks) acc += __ldcg(part + ((size_t)ks * B + b) * rows1 + u);
    acc += b1[u];
    a1[u] = relu ? fmaxf(acc, 0.f) : acc;
  }
}

// s[m] = sum_u W2[m][u] a1[u] + b2[m]: warp per score, 16-byte loads of W2 (smem or global).
// b2 must already be staged (smem or registers-resident): no dependent global load per score.
template <typename T>
__device__ __forceinline__ void router_out(const T* W2, const float* a1, const float* b2, int M, int h_r, float* s) {
  constexpr int E = Elem<T>::kPer16B;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int m = warp; m < M; m += nw) {
    const T* w = W2 + (size_t)m * h_r;
    float acc = 0.f;
    for (int c = lane * E; c < h_r; c += 32 * E) {
      float wf[E];
      widen16(*reinterpret_cast<const uint4*>(w + c), wf, w);
#pragma unroll
      for (int j = 0; j < E; ++j) acc = fmaf(wf[j], a1[c + j], acc);
    }
    acc = warp_sum(acc) + b2[m];
    if (lane == 0) s[m] = acc;
  }
}

}  // namespace ds
