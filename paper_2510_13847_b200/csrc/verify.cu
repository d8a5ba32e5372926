// verify.cu — NEXT-4: lossless verification of drafted chains against the target's full-vocabulary
// logits (Eq. 3, and the speculative-sampling rule its footnote cites; SPEC S:454-464;
// reading R25), plus the shortlist-id materialisation (S4) that embeds the drafter's q in V.
//
// Two launches, both HBM-streaming over the target logits (no contraction: CUDA cores, 16 B loads):
//   verify_lse_kernel      grid (B (gamma+1), chunks): per-chunk (max, sum exp) of every target row;
//                          the last CTA of a row folds the chunks into lse_p[row]; the last row of a
//                          chain takes the accept decisions u_i < p_i(x_i) / q_i(x_i), finds the first
//                          rejection j and scatters q_j into the chain's dense q buffer.
//   verify_residual_kernel grid (B, chunks): per-chunk sums of w = (p_j - q_j)_+ (the bonus case j =
//                          gamma has q = 0, so w = p_gamma); the last CTA of a chain locates the chunk
//                          whose cumulative weight crosses u_res * Z, rescans it in id order for the
//                          token (R25) and clears the scattered q entries (the buffer stays zero).
#include <algorithm>

#include "head_impl.cuh"
#include "internal.h"

namespace ds {

constexpr int kVT = 256;                 // threads per CTA
constexpr int kVChunk = 8192;            // vocabulary entries per CTA
constexpr int kVPer = kVChunk / kVT;     // 32 values per thread

struct VerifyArgs {
  const void* p_logits;  // [B][gamma+1][V]
  int64_t V;
  int B, gamma, nchunk;
  const int32_t* q_ids;
  const float* q_logits;
  int64_t q_stride;
  const int32_t* q_count;
  const float* q_lse;
  const int32_t* x;
  const int32_t* x_slot;
  const float* u_acc;
  const float* u_res;
  int32_t* accepted;
  int32_t* committed;
  float2* part;         // [B (gamma+1)][nchunk] (max, sum exp)
  float* lse_p;         // [B (gamma+1)]
  float* wpart;         // [B][nchunk]
  int32_t* jrow;        // [B]
  float* qbuf;          // [B][V], zero between calls
  unsigned* ctr_row;    // [B (gamma+1)]
  unsigned* ctr_chain;  // [B]
  unsigned* ctr_res;    // [B]
};

__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }

// Coalesced 16 B loads: element e of vector k of this thread is lo + (k kVT + tid) VEC + e.
template <typename T>
__device__ __forceinline__ void load_chunk(const T* row, int64_t lo, int64_t hi, float* v) {
  constexpr int VEC = 16 / sizeof(T);
#pragma unroll
  for (int k = 0; k < kVPer / VEC; ++k) {
    const int64_t x = lo + (int64_t)(k * kVT + threadIdx.x) * VEC;
    if (x < hi) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + x);
      widen16(u, v + k * VEC, (const T*)nullptr);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) v[k * VEC + e] = -INFINITY;
    }
  }
}

template <typename T>
__device__ __forceinline__ void load_q(const float* q, int64_t lo, int64_t hi, float* out) {
  constexpr int VEC = 16 / sizeof(T);
#pragma unroll
  for (int k = 0; k < kVPer / VEC; ++k) {
    const int64_t x = lo + (int64_t)(k * kVT + threadIdx.x) * VEC;
#pragma unroll
    for (int h = 0; h < VEC / 4; ++h) {
      const float4 f = x < hi ? *reinterpret_cast<const float4*>(q + x + 4 * h) : make_float4(0.f, 0.f, 0.f, 0.f);
      out[k * VEC + 4 * h] = f.x;
      out[k * VEC + 4 * h + 1] = f.y;
      out[k * VEC + 4 * h + 2] = f.z;
      out[k * VEC + 4 * h + 3] = f.w;
    }
  }
}

// Accept decisions of chain b (warp 0) and the q_j scatter (whole CTA).
template <typename T>
__device__ void verify_decide(const VerifyArgs& a, int b, int* sh) {
  const int lane = threadIdx.x & 31, g = a.gamma, g1 = g + 1;
  if (threadIdx.x < 32) {
    bool valid = false, acc = false;
    if (lane < g) {
      const int pi = b * g + lane;
      const int xi = a.x[pi], slot = a.x_slot[pi], cnt = a.q_count[pi];
      valid = xi >= 0 && xi < a.V && slot >= 0 && slot < cnt && a.q_ids[(size_t)pi * a.q_stride + slot] == xi;
      if (valid) {
        const T* l = static_cast<const T*>(a.p_logits) + ((size_t)b * g1 + lane) * a.V;
        const float p = expf(to_f(l[xi]) - __ldcg(&a.lse_p[b * g1 + lane]));
        const float q = expf(a.q_logits[(size_t)pi * a.q_stride + slot] - a.q_lse[pi]);
        acc = a.u_acc[pi] < p / q;  // Eq. 3: accept with probability min(1, p/q)
      }
    }
    const unsigned stop = __ballot_sync(0xffffffffu, lane < g && !(valid && acc));
    const int j = stop ? __ffs(stop) - 1 : g;
    const bool bad = j < g && !__shfl_sync(0xffffffffu, valid, j & 31);
    if (!bad && lane < j) a.committed[(size_t)b * g1 + lane] = a.x[b * g + lane];
    if (lane == 0) {
      a.jrow[b] = bad ? -1 : j;
      a.accepted[b] = bad ? -1 : j;
      if (bad) a.committed[(size_t)b * g1] = -1;
      a.ctr_chain[b] = 0;
      sh[0] = bad ? -1 : j;
    }
  }
  __syncthreads();
  const int j = sh[0];
  if (j < 0 || j >= g) return;
  const int pi = b * g + j;
  const int n = a.q_count[pi];
  const float qs = a.q_lse[pi];
  const int32_t* ids = a.q_ids + (size_t)pi * a.q_stride;
  const float* ql = a.q_logits + (size_t)pi * a.q_stride;
  float* qb = a.qbuf + (size_t)b * a.V;
  for (int s = threadIdx.x; s < n; s += blockDim.x) qb[ids[s]] = expf(ql[s] - qs);
}

template <typename T>
__global__ void __launch_bounds__(kVT) verify_lse_kernel(const VerifyArgs a) {
  __shared__ float red[32];
  __shared__ int sh[2];
  const int row = blockIdx.x, chunk = blockIdx.y, g1 = a.gamma + 1, b = row / g1;
  const T* l = static_cast<const T*>(a.p_logits) + (size_t)row * a.V;
  const int64_t lo = (int64_t)chunk * kVChunk, hi = min(a.V, lo + kVChunk);
  float v[kVPer];
  load_chunk<T>(l, lo, hi, v);
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < kVPer; ++i) m = fmaxf(m, v[i]);
  m = block_max(m, red);
  float s = 0.f;
  if (m != -INFINITY) {
#pragma unroll
    for (int i = 0; i < kVPer; ++i) s += expf(v[i] - m);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    a.part[(size_t)row * a.nchunk + chunk] = make_float2(m, s);
    fence_acq_rel_gpu();
    sh[0] = atomicAdd(&a.ctr_row[row], 1u) == (unsigned)(a.nchunk - 1);
  }
  __syncthreads();
  if (!sh[0]) return;
  fence_acq_rel_gpu();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    float M = -INFINITY, S = 0.f;
    for (int c = lane; c < a.nchunk; c += 32) {
      const float2 p = __ldcg(&a.part[(size_t)row * a.nchunk + c]);
      lse_combine(M, S, p.x, p.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float M2 = __shfl_xor_sync(0xffffffffu, M, o), S2 = __shfl_xor_sync(0xffffffffu, S, o);
      lse_combine(M, S, M2, S2);
    }
    if (lane == 0) {
      a.lse_p[row] = M + logf(S);
      a.ctr_row[row] = 0;
      fence_acq_rel_gpu();
      sh[1] = atomicAdd(&a.ctr_chain[b], 1u) == (unsigned)(g1 - 1);
    }
  }
  __syncthreads();
  if (!sh[1]) return;
  fence_acq_rel_gpu();
  verify_decide<T>(a, b, sh);
}

template <typename T>
__global__ void __launch_bounds__(kVT) verify_residual_kernel(const VerifyArgs a) {
  __shared__ float red[32];
  __shared__ float fsh[2];
  __shared__ int ish[4];
  const int b = blockIdx.x, chunk = blockIdx.y, g1 = a.gamma + 1;
  const int j = a.jrow[b];
  if (j < 0) return;
  const int row = b * g1 + j;
  const float lse = a.lse_p[row];
  const T* l = static_cast<const T*>(a.p_logits) + (size_t)row * a.V;
  const float* qb = a.qbuf + (size_t)b * a.V;
  const int64_t lo = (int64_t)chunk * kVChunk, hi = min(a.V, lo + kVChunk);
  float v[kVPer], q[kVPer];
  load_chunk<T>(l, lo, hi, v);
  load_q<T>(qb, lo, hi, q);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kVPer; ++i) s += fmaxf(expf(v[i] - lse) - q[i], 0.f);
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    a.wpart[(size_t)b * a.nchunk + chunk] = s;
    fence_acq_rel_gpu();
    ish[0] = atomicAdd(&a.ctr_res[b], 1u) == (unsigned)(a.nchunk - 1);
  }
  __syncthreads();
  if (!ish[0]) return;
  fence_acq_rel_gpu();
  // ---- last CTA of the chain: inverse CDF in id order (R25)
  if (threadIdx.x == 0) {
    float Z = 0.f;
    for (int c = 0; c < a.nchunk; ++c) Z += __ldcg(&a.wpart[(size_t)b * a.nchunk + c]);
    const int usep = !(Z > 0.f);  // R25: p == q numerically -> sample from p
    if (usep) {
      Z = 0.f;
      for (int c = 0; c < a.nchunk; ++c) {
        const float2 p = __ldcg(&a.part[(size_t)row * a.nchunk + c]);
        Z += p.y * expf(p.x - lse);
      }
    }
    const float target = a.u_res[b] * Z;
    float cum = 0.f, base = 0.f, last_base = 0.f;
    int cstar = -1, last_pos = 0;
    for (int c = 0; c < a.nchunk; ++c) {
      float wc;
      if (usep) {
        const float2 p = __ldcg(&a.part[(size_t)row * a.nchunk + c]);
        wc = p.y * expf(p.x - lse);
      } else {
        wc = __ldcg(&a.wpart[(size_t)b * a.nchunk + c]);
      }
      if (wc > 0.f) {
        last_pos = c;
        last_base = cum;
      }
      if (cstar < 0 && cum + wc > target) {
        cstar = c;
        base = cum;
      }
      cum += wc;
    }
    if (cstar < 0) {
      cstar = last_pos;
      base = last_base;
    }
    ish[1] = cstar;
    ish[2] = usep;
    ish[3] = INT32_MAX;
    fsh[0] = base;
    fsh[1] = target;
  }
  __syncthreads();
  const int cstar = ish[1], usep = ish[2];
  const float base = fsh[0], target = fsh[1];
  // thread t owns the contiguous ids [clo + 32 t, clo + 32 t + 32) of chunk c*
  const int64_t clo = (int64_t)cstar * kVChunk + (int64_t)threadIdx.x * kVPer;
  float w[kVPer];
  float tot = 0.f;
  int lastx = -1;
#pragma unroll
  for (int i = 0; i < kVPer; ++i) {
    const int64_t x = clo + i;
    float wi = 0.f;
    if (x < a.V) {
      const float p = expf(to_f(l[x]) - lse);
      wi = usep ? p : fmaxf(p - qb[x], 0.f);
    }
    w[i] = wi;
    tot += wi;
    if (wi > 0.f) lastx = (int)x;
  }
  // exclusive scan of the thread totals (warp shuffles, then warp totals in index order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __shared__ float wtot[kVT / 32];
  __shared__ int lastmax;
  if (threadIdx.x == 0) lastmax = -1;
  if (lane == 31) wtot[warp] = inc;
  __syncthreads();
  float wbase = 0.f;
  for (int k = 0; k < warp; ++k) wbase += wtot[k];
  float cum = base + wbase + inc - tot;
  int found = INT32_MAX;
#pragma unroll
  for (int i = 0; i < kVPer; ++i) {
    cum += w[i];
    if (found == INT32_MAX && w[i] > 0.f && cum > target) found = (int)(clo + i);
  }
  if (found != INT32_MAX) atomicMin(&ish[3], found);
  if (lastx >= 0) atomicMax(&lastmax, lastx);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int xs = ish[3] != INT32_MAX ? ish[3] : (lastmax >= 0 ? lastmax : (int)((int64_t)cstar * kVChunk));
    a.committed[(size_t)b * g1 + j] = xs;
    a.ctr_res[b] = 0;
  }
  if (j < a.gamma) {  // leave the q buffer zero for the next call
    const int pi = b * a.gamma + j;
    const int n = a.q_count[pi];
    const int32_t* ids = a.q_ids + (size_t)pi * a.q_stride;
    float* qw = a.qbuf + (size_t)b * a.V;
    for (int s2 = threadIdx.x; s2 < n; s2 += blockDim.x) qw[ids[s2]] = 0.f;
  }
}

// ------------------------------------------------------------------ shortlist ids (S4)

// One CTA per row, one warp per selected cluster: ids[r][sl_off[r][i] + u] = perm[offsets[m_i] + u].
__global__ void shortlist_ids_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ offsets, int M,
                                     const int32_t* __restrict__ sel, const int32_t* __restrict__ cnt,
                                     const int32_t* __restrict__ sl_off, int64_t stride, int32_t* __restrict__ ids) {
  const int r = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = cnt[r];
  for (int i = warp; i < n; i += nw) {
    const int m = sel[(size_t)r * M + i];
    const int o0 = offsets[m], sz = offsets[m + 1] - o0;
    const int base = sl_off[(size_t)r * (M + 1) + i];
    for (int u = lane; u < sz; u += 32) ids[(size_t)r * stride + base + u] = perm[o0 + u];
  }
}

// ------------------------------------------------------------------ host side

struct VerifyLayout {
  size_t part, lse, wpart, jrow, ctr_row, ctr_chain, ctr_res, qbuf, total;
};

static VerifyLayout verify_layout(int64_t V, int B, int gamma) {
  const int nchunk = (int)((V + kVChunk - 1) / kVChunk);
  const size_t rows = (size_t)B * (gamma + 1);
  VerifyLayout L;
  size_t o = 0;
  auto take = [&](size_t n) {
    const size_t at = o;
    o = align_up(o + n, 256);
    return at;
  };
  L.ctr_row = take(rows * 4);
  L.ctr_chain = take((size_t)B * 4);
  L.ctr_res = take((size_t)B * 4);
  L.qbuf = take((size_t)B * V * 4);
  L.part = take(rows * nchunk * 8);
  L.lse = take(rows * 4);
  L.wpart = take((size_t)B * nchunk * 4);
  L.jrow = take((size_t)B * 4);
  L.total = o;
  return L;
}

size_t verify_ws_bytes(int64_t V, int B, int gamma) { return verify_layout(V, B, gamma).total; }

cudaError_t launch_verify(const void* p_logits, int dtype, int64_t V, int B, int gamma, const int32_t* q_ids,
                          const float* q_logits, int64_t q_stride, const int32_t* q_count, const float* q_lse,
                          const int32_t* x, const int32_t* x_slot, const float* u_acc, const float* u_res,
                          int32_t* accepted, int32_t* committed, void* ws, cudaStream_t st) {
  const VerifyLayout L = verify_layout(V, B, gamma);
  uint8_t* w = static_cast<uint8_t*>(ws);
  VerifyArgs a;
  a.p_logits = p_logits;
  a.V = V;
  a.B = B;
  a.gamma = gamma;
  a.nchunk = (int)((V + kVChunk - 1) / kVChunk);
  a.q_ids = q_ids;
  a.q_logits = q_logits;
  a.q_stride = q_stride;
  a.q_count = q_count;
  a.q_lse = q_lse;
  a.x = x;
  a.x_slot = x_slot;
  a.u_acc = u_acc;
  a.u_res = u_res;
  a.accepted = accepted;
  a.committed = committed;
  a.part = reinterpret_cast<float2*>(w + L.part);
  a.lse_p = reinterpret_cast<float*>(w + L.lse);
  a.wpart = reinterpret_cast<float*>(w + L.wpart);
  a.jrow = reinterpret_cast<int32_t*>(w + L.jrow);
  a.qbuf = reinterpret_cast<float*>(w + L.qbuf);
  a.ctr_row = reinterpret_cast<unsigned*>(w + L.ctr_row);
  a.ctr_chain = reinterpret_cast<unsigned*>(w + L.ctr_chain);
  a.ctr_res = reinterpret_cast<unsigned*>(w + L.ctr_res);
  const dim3 g1(B * (gamma + 1), a.nchunk), g2(B, a.nchunk);  // rows in x (no 65535 limit)
  if (dtype == DS_BF16) {
    verify_lse_kernel<__nv_bfloat16><<<g1, kVT, 0, st>>>(a);
    verify_residual_kernel<__nv_bfloat16><<<g2, kVT, 0, st>>>(a);
  } else {
    verify_lse_kernel<float><<<g1, kVT, 0, st>>>(a);
    verify_residual_kernel<float><<<g2, kVT, 0, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_shortlist_ids(const ds_clusters* c, int rows, const int32_t* sel, const int32_t* cnt,
                                 const int32_t* sl_off, int64_t stride, int32_t* ids, cudaStream_t st) {
  shortlist_ids_kernel<<<rows, 256, 0, st>>>(c->perm, c->offsets, c->M, sel, cnt, sl_off, stride, ids);
  return cudaGetLastError();
}

}  // namespace ds
