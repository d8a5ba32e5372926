// select_impl.cuh — S3/S4 cluster selection + router layer 2 building blocks (any blockDim).
//
// K = TopK_k(s) under (score desc, id asc) (R7), emitted in ascending cluster id (R8);
// sl_offsets = exclusive scan of |C_m| over K (|V_S| = sum |C_m|).
#pragma once
#include "common.cuh"

namespace ds {

// a1[u] = act(sum_{ks} part[ks][b][u] + b1[u]) in fixed split order (act = ReLU if h_r > 0).
__device__ __forceinline__ void router_hidden(const float* part, int KS, int B, int b, int rows1, const float* b1,
                                              bool relu, float* a1) {
  for (int u = threadIdx.x; u < rows1; u += blockDim.x) {
    float acc = 0.f;
    int ks = 0;
    for (; ks + 8 <= KS; ks += 8) {  // 8 independent loads in flight, summed in split order (R19)
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(part + ((size_t)(ks + j) * B + b) * rows1 + u);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j];
    }
    for (; ks < KS; ++ks) acc += __ldcg(part + ((size_t)ks * B + b) * rows1 + u);
    acc += b1[u];
    a1[u] = relu ? fmaxf(acc, 0.f) : acc;
  }
}

}  // namespace ds

namespace ds {

// ---------------------------------------------------------------- fast variants (fused step)

// ord_key (order-preserving float -> uint32): common.cuh

// One thread per score: s[m] = W2[m] . a1 + b2[m].  Thread m walks its 16-byte chunks starting at
// chunk (m mod chunks), so the 8 threads of an LDS.128 phase hit 8 different bank groups.
template <typename T>
__device__ __forceinline__ void router_scores_thread(const T* W2, const float* a1, const float* b2, int M, int h_r,
                                                     float* sc) {
  constexpr int E = Elem<T>::kPer16B;
  const int chunks = h_r / E;
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const T* w = W2 + (size_t)m * h_r;
    float acc0 = 0.f, acc1 = 0.f;
    const int c0 = m % chunks;
    int i = 0;
    for (; i + 8 <= chunks; i += 8) {  // 8 independent 16-byte loads in flight, then the FMAs in order
      uint4 raw[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int c = c0 + i + u;
        c = c >= chunks ? c - chunks : c;
        raw[u] = *reinterpret_cast<const uint4*>(w + c * E);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int c = c0 + i + u;
        c = c >= chunks ? c - chunks : c;
        float wf[E];
        widen16(raw[u], wf, w);
        const float* av = a1 + c * E;
#pragma unroll
        for (int j = 0; j < E; j += 2) {
          acc0 = fmaf(wf[j], av[j], acc0);
          acc1 = fmaf(wf[j + 1], av[j + 1], acc1);
        }
      }
    }
    for (; i < chunks; ++i) {
      int c = c0 + i;
      c = c >= chunks ? c - chunks : c;
      float wf[E];
      widen16(*reinterpret_cast<const uint4*>(w + c * E), wf, w);
      const float* av = a1 + c * E;
#pragma unroll
      for (int j = 0; j < E; j += 2) {
        acc0 = fmaf(wf[j], av[j], acc0);
        acc1 = fmaf(wf[j + 1], av[j + 1], acc1);
      }
    }
    sc[m] = (acc0 + acc1) + b2[m];
  }
}

// TopK_k of sc[0..M) as a bit mask by counting ranks in one pass: rank(m) = #{j : s_j > s_m or
// (s_j == s_m and j < m)} (R7), selected iff rank < k.  mask has ceil(M/32) words.
__device__ __forceinline__ void rank_mask(const float* sc, int M, int k, uint32_t* mask) {
  const int lane = threadIdx.x & 31;
  const int Mr = (M + 31) & ~31;
  for (int m = threadIdx.x; m < Mr; m += blockDim.x) {
    bool sel = false;
    if (m < M) {
      const float key = sc[m] + 0.0f;
      int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
      int j = 0;
      for (; j + 4 <= M; j += 4) {
        const float4 o = *reinterpret_cast<const float4*>(sc + j);
        const float o0 = o.x + 0.0f, o1 = o.y + 0.0f, o2 = o.z + 0.0f, o3 = o.w + 0.0f;
        r0 += (o0 > key) | ((o0 == key) & (j < m));
        r1 += (o1 > key) | ((o1 == key) & (j + 1 < m));
        r2 += (o2 > key) | ((o2 == key) & (j + 2 < m));
        r3 += (o3 > key) | ((o3 == key) & (j + 3 < m));
      }
      for (; j < M; ++j) {
        const float o = sc[j] + 0.0f;
        r0 += (o > key) | ((o == key) & (j < m));
      }
      sel = (r0 + r1 + r2 + r3) < k;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) mask[m >> 5] = b;
  }
}

// TopK_k of sc[0..M) under (score desc, id asc) (R7) as a bit mask, by an MSB-first radix select on
// the order-preserving 32-bit keys (4 passes of 8-bit digits: a shared-memory histogram each, one warp
// finds the digit where the count from the top crosses k): T = the k-th largest key and need = how
// many keys equal to T are taken (the lowest ids).  O(M) work per pass instead of rank_mask's O(M^2):
// the router's layer-2 kernel at M = 512 spent most of its time ranking.  Same selection bit for bit.
// hist: shared [256 + 8] u32.  Ends with a __syncthreads (mask complete).
__device__ __forceinline__ void radix_mask(const float* sc, int M, int k, uint32_t* mask, uint32_t* hist) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* st = hist + 256;  // [0] prefix, [1] prefix mask, [2] remaining k, [3] equal-key budget
  if (threadIdx.x == 0) {
    st[0] = 0u;
    st[1] = 0u;
    st[2] = (uint32_t)k;
  }
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const uint32_t pre = st[0], pm = st[1];
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
      const uint32_t key = ord_key(sc[m] + 0.0f);
      if ((key & pm) == pre) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (warp == 0) {  // digits 255..0 from the top: lane l holds digits 255 - 8l .. 248 - 8l
      uint32_t c[8], tot = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * lane - j];
        tot += c[j];
      }
      uint32_t inc = tot;  // inclusive scan over lanes (from the top digit down)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t kk = st[2];
      const uint32_t before = inc - tot;  // keys in higher digits than this lane's
      if (before < kk && inc >= kk) {     // exactly one lane: the crossing digit is here
        uint32_t run = before;
        int j = 0;
        for (; j < 8; ++j) {
          if (run + c[j] >= kk) break;
          run += c[j];
        }
        const uint32_t digit = 255u - 8u * (uint32_t)lane - (uint32_t)j;
        st[0] = pre | (digit << shift);
        st[1] = pm | (255u << shift);
        st[2] = kk - run;  // still to take among keys with this prefix
      }
    }
    __syncthreads();
  }
  // T = st[0]: keys > T are in; keys == T: the st[2] lowest ids
  const uint32_t T = st[0], need = st[2];
  const int Mr = (M + 31) & ~31;
  uint32_t taken = 0u;  // equal keys in earlier words, per thread (words are handled in order by warp 0)
  if (warp == 0) {
    for (int m0 = 0; m0 < Mr; m0 += 32) {
      const int m = m0 + lane;
      const uint32_t key = m < M ? ord_key(sc[m] + 0.0f) : 0u;
      const uint32_t eq = __ballot_sync(0xffffffffu, m < M && key == T);
      const uint32_t rank_eq = taken + __popc(eq & ((1u << lane) - 1u));
      const bool in = m < M && (key > T || (key == T && rank_eq < need));
      const uint32_t b = __ballot_sync(0xffffffffu, in);
      if (lane == 0) mask[m0 >> 5] = b;
      taken += __popc(eq);
    }
  }
  __syncthreads();
}

// Ascending ids of the set bits (position = popcount of the lower bits) and sl_offsets = exclusive
// scan of |C_m| over them (one warp scan per 32 selected clusters).  tmp: smem [M] ints.
__device__ __forceinline__ void emit_fast(const uint32_t* mask, int M, const int32_t* offs, int32_t* sel,
                                          int32_t* cnt_out, int32_t* sl_off, int32_t* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int words = (M + 31) >> 5;
  int total = 0;
  for (int w = 0; w < words; ++w) total += __popc(mask[w]);
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const int w = m >> 5;
    const uint32_t bits = mask[w];
    if ((bits >> (m & 31)) & 1u) {
      int pos = __popc(bits & ((1u << (m & 31)) - 1u));
      for (int u = 0; u < w; ++u) pos += __popc(mask[u]);
      sel[pos] = m;
      tmp[pos] = offs[m + 1] - offs[m];
    }
  }
  __syncthreads();
  if (warp == 0) {
    int run = 0;
    for (int p0 = 0; p0 < total; p0 += 32) {
      const int p = p0 + lane;
      const int sz = p < total ? tmp[p] : 0;
      int inc = sz;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (p < total) sl_off[p] = run + inc - sz;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      *cnt_out = total;
      sl_off[total] = run;
    }
  }
}

}  // namespace ds
