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

namespace ds {

// ---------------------------------------------------------------- fast variants (fused step)

// Order-preserving map float -> uint32 (larger float => larger key); -0 folded into +0 (R23).
__device__ __forceinline__ uint32_t ord_key(float x) {
  const uint32_t u = __float_as_uint(x + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// s[m] = W2[m] . a1 + b2[m] with L = (h_r / E rounded up to a power of two, <= 32) lanes per
// score, so a warp produces 32 / L scores per pass (W2, a1, b2 in shared memory).
template <typename T>
__device__ __forceinline__ void router_scores_fast(const T* W2, const float* a1, const float* b2, int M, int h_r,
                                                   float* sc) {
  constexpr int E = Elem<T>::kPer16B;
  const int chunks = h_r / E;
  int L = 1;
  while (L < chunks && L < 32) L <<= 1;
  const int spw = 32 / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int sub = lane % L, slot = lane / L;
  for (int m0 = warp * spw; m0 < M; m0 += nw * spw) {
    const int m = m0 + slot;
    float acc = 0.f;
    if (m < M) {
      const T* w = W2 + (size_t)m * h_r;
      for (int ch = sub; ch < chunks; ch += L) {
        float wf[E];
        widen16(*reinterpret_cast<const uint4*>(w + ch * E), wf, w);
#pragma unroll
        for (int j = 0; j < E; ++j) acc = fmaf(wf[j], a1[ch * E + j], acc);
      }
    }
    for (int o = L / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (sub == 0 && m < M) sc[m] = acc + b2[m];
  }
}

// TopK_k of sc[0..M) under (score desc, id asc) as a bit mask (R7): 4-pass radix select
// of the k-th largest order key, then every key above it plus the lowest-id ties.
// Smem: mask [ceil(M/32)] words, hist [256], sh [2].  All threads of the block participate.
__device__ __forceinline__ void radix_topk_mask(const float* sc, int M, int k, uint32_t* mask, int* hist, int* sh) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  uint32_t prefix = 0, pmask = 0;
  int kk = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nt) hist[i] = 0;
    __syncthreads();
    for (int m = tid; m < M; m += nt) {
      const uint32_t key = ord_key(sc[m]);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
    }
    __syncthreads();
    if (warp == 0) {
      int cnt[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[j] = hist[255 - 8 * lane - j];
        tot += cnt[j];
      }
      int inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int exc = inc - tot;
      if (exc < kk && kk <= inc) {
        int run = exc;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (run + cnt[j] >= kk) {
            sh[0] = 255 - 8 * lane - j;
            sh[1] = kk - run;
            break;
          }
          run += cnt[j];
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)sh[0] << shift;
    pmask |= 255u << shift;
    kk = sh[1];
    __syncthreads();
  }
  if (warp == 0) {
    int running = 0;
    for (int c = 0; c * 32 < M; ++c) {
      const int m = c * 32 + lane;
      const uint32_t key = m < M ? ord_key(sc[m]) : 0u;
      const bool gt = m < M && key > prefix;
      const bool eq = m < M && key == prefix;
      const uint32_t eb = __ballot_sync(0xffffffffu, eq);
      const int r = running + __popc(eb & ((1u << lane) - 1u));
      const uint32_t mb = __ballot_sync(0xffffffffu, gt || (eq && r < kk));
      if (lane == 0) mask[c] = mb;
      running += __popc(eb);
    }
  }
  __syncthreads();
}

// One warp: ascending ids of the set bits + exclusive scan of |C_m| (sl_offsets).
__device__ __forceinline__ void emit_mask_warp(const uint32_t* mask, int M, const int32_t* offs, int32_t* sel,
                                               int32_t* cnt_out, int32_t* sl_off) {
  const int lane = threadIdx.x & 31;
  int base = 0, run = 0;
  for (int c = 0; c * 32 < M; ++c) {
    const int m = c * 32 + lane;
    const bool f = m < M && ((mask[c] >> lane) & 1u);
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    const int pos = base + __popc(b & ((1u << lane) - 1u));
    const int sz = f ? offs[m + 1] - offs[m] : 0;
    int inc = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (f) {
      sel[pos] = m;
      sl_off[pos] = run + inc - sz;
    }
    base += __popc(b);
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {
    *cnt_out = base;
    sl_off[base] = run;
  }
}

}  // namespace ds
