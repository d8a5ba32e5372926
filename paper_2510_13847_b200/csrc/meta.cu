// meta.cu — S1 meta-classifier r_theta and S3/S4 cluster selection (stream S_m).
//
// s = W2 ReLU(W1 [h_prev || e] + b1) + b2          (§4.2 "Low-cost router"; R4, R5)
// K = TopK_k(s), ascending ids; sl_offsets = scan  (Alg. 1 line 8)
//
// Layer 1 is a skinny GEMV (h_r x 2d weights, 2 MB at Llama-3) and is HBM/latency bound:
// it is split over (h_r / 8) x KS CTAs, each warp owning one hidden unit and one K-chunk,
// holding its W1 slice in registers and reusing it for all B rows; x = [h_prev||e] is
// staged in shared memory.  Partials go to the workspace (no float atomics) and layer 2
// (one CTA per row) reduces them in fixed split order, applies b1 + ReLU, computes the M
// scores (warp per score) and then selects in the same CTA — selection never leaves the
// chip.  Shared (tree) mode: the last row-CTA (atomic ticket) forms the union selection.
#include <limits.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "select_impl.cuh"

namespace ds {

constexpr int kMetaThreads = 256;
constexpr int kMetaUnitsPerCTA = kMetaThreads / 32;
constexpr int kSelThreads = 256;

__global__ void __launch_bounds__(kSelThreads) select_kernel(const float* __restrict__ scores, int B, int M,
                                                             const int32_t* __restrict__ offsets, int k,
                                                             const int32_t* __restrict__ k_per_row, int shared,
                                                             int32_t* sel, int32_t* sel_count, int32_t* sl_off) {
  __shared__ __align__(16) float s[kMaxM];
  __shared__ uint32_t mask[kMaxM / 32], acc[kMaxM / 32];
  __shared__ int32_t tmp[kMaxM];
  __shared__ int32_t offs[kMaxM + 1];
  const int words = (M + 31) / 32;
  for (int m = threadIdx.x; m <= M; m += blockDim.x) offs[m] = offsets[m];
  for (int w = threadIdx.x; w < words; w += blockDim.x) acc[w] = 0u;
  const int r_lo = shared ? 0 : blockIdx.x, r_hi = shared ? B : blockIdx.x + 1;
  for (int r = r_lo; r < r_hi; ++r) {
    __syncthreads();
    for (int m = threadIdx.x; m < M; m += blockDim.x) s[m] = scores[(size_t)r * M + m];
    __syncthreads();
    rank_mask(s, M, k_per_row ? k_per_row[r] : k, mask);
    __syncthreads();
    for (int w = threadIdx.x; w < words; w += blockDim.x) acc[w] |= mask[w];
  }
  __syncthreads();
  const int o = shared ? 0 : blockIdx.x;
  emit_fast(acc, M, offs, sel + (size_t)o * M, sel_count + o, sl_off + (size_t)o * (M + 1), tmp);
}

// ------------------------------------------------------------------ layer 1: split-K partials

template <typename T>
__global__ void __launch_bounds__(kMetaThreads) meta_l1_kernel(const T* __restrict__ W1, const T* __restrict__ h_prev,
                                                               const T* __restrict__ e, int B, int d, int rows1,
                                                               int KC, int RB, float* __restrict__ part, int pdl) {
  constexpr int E = Elem<T>::kPer16B;
  extern __shared__ __align__(16) uint8_t msm[];
  T* xs = reinterpret_cast<T*>(msm);  // [RB][KC]: rows [b0, b0 + nb) of this CTA's row block
  const int b0 = blockIdx.z * RB, nb = min(RB, B - b0);
  const int dr = 2 * d;
  const int k0 = blockIdx.y * KC;
  const int kn = min(KC, dr - k0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * kMetaUnitsPerCTA + warp;

  // W1 slice of this warp -> registers (independent of upstream kernels: load before the PDL wait)
  constexpr int kMaxChunks = 4;  // KC <= 32 * E * kMaxChunks
  uint4 wv[kMaxChunks];
#pragma unroll
  for (int i = 0; i < kMaxChunks; ++i) {
    const int c = lane * E + i * 32 * E;
    wv[i] = (u < rows1 && c < kn) ? __ldg(reinterpret_cast<const uint4*>(W1 + (size_t)u * dr + k0 + c))
                                  : make_uint4(0, 0, 0, 0);
  }
  if (pdl) pdl_wait();
  // stage x = [h_prev || e][:, k0:k0+kn]; a 16-byte chunk never straddles h/e since d % E == 0
  const int cpr = kn / E;
  for (int idx = threadIdx.x; idx < nb * cpr; idx += blockDim.x) {
    const int b = idx / cpr, c = (idx - b * cpr) * E;
    const int k = k0 + c;
    const T* src = k < d ? h_prev + (size_t)(b0 + b) * d + k : e + (size_t)(b0 + b) * d + (k - d);
    *reinterpret_cast<uint4*>(xs + (size_t)b * KC + c) = *reinterpret_cast<const uint4*>(src);
  }
  __syncthreads();
  if (pdl) pdl_launch_dependents();
  if (u >= rows1) return;
  float wf[kMaxChunks][E];
#pragma unroll
  for (int i = 0; i < kMaxChunks; ++i) widen16(wv[i], wf[i], W1);
  // 8 rows at a time: lane partials, then one transpose-reduction (9 shuffles for 8 rows instead of
  // 8 x 5): after it lane L holds row 4 b4 + 2 b3 + b2 (bits of L) summed over all 32 lanes
  for (int bb = 0; bb < nb; bb += 8) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float acc = 0.f;
      if (bb + q < nb) {
#pragma unroll
        for (int i = 0; i < kMaxChunks; ++i) {
          const int c = lane * E + i * 32 * E;
          if (c < kn) {
            float xf[E];
            widen16(*reinterpret_cast<const uint4*>(xs + (size_t)(bb + q) * KC + c), xf, W1);
#pragma unroll
            for (int j = 0; j < E; ++j) acc = fmaf(wf[i][j], xf[j], acc);
          }
        }
      }
      v[q] = acc;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool hi = lane & 16;
      const float send = hi ? v[j] : v[j + 4], keep = hi ? v[j + 4] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const bool hi = lane & 8;
      const float send = hi ? v[j] : v[j + 2], keep = hi ? v[j + 2] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
      const bool hi = lane & 4;
      const float send = hi ? v[0] : v[1], keep = hi ? v[1] : v[0];
      v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int q = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && bb + q < nb) part[((size_t)blockIdx.y * B + b0 + bb + q) * rows1 + u] = v[0];
  }
}

// ------------------------------------------------------------------ layer 2 + select (CTA per row)

template <typename T>
__global__ void __launch_bounds__(kMetaThreads) meta_l2_kernel(const float* __restrict__ part, int KS, int B,
                                                               int rows1, const float* __restrict__ b1,
                                                               const T* __restrict__ W2, const float* __restrict__ b2,
                                                               int h_r, int M, float* __restrict__ scores,
                                                               const int32_t* __restrict__ offsets, int k,
                                                               const int32_t* __restrict__ k_per_row, int shared,
                                                               int32_t* sel, int32_t* sel_count, int32_t* sl_off,
                                                               unsigned* counter, int pdl, unsigned long long* trace) {
  __shared__ __align__(16) float a1[kMaxM];
  __shared__ __align__(16) float s[kMaxM];
  __shared__ uint32_t mask[kMaxM / 32], acc[kMaxM / 32];
  __shared__ int32_t tmp[kMaxM];
  __shared__ int is_last;
  __shared__ float b1s[kMaxM];
  __shared__ float b2s[kMaxM];
  __shared__ int32_t offs[kMaxM + 1];
  __shared__ uint32_t rhist[256 + 8];
  const int b = blockIdx.x;
  // constants first (they do not depend on the upstream kernel)
  for (int u = threadIdx.x; u < rows1; u += blockDim.x) b1s[u] = b1[u];
  for (int m = threadIdx.x; m < M; m += blockDim.x) b2s[m] = h_r > 0 ? b2[m] : 0.f;
  if (offsets)
    for (int m = threadIdx.x; m <= M; m += blockDim.x) offs[m] = offsets[m];
  if (h_r > 0 && threadIdx.x == 0) {  // W2 into L2 while the upstream kernel finishes: slice b of B
    const size_t bytes = (size_t)M * h_r * sizeof(T);
    const size_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~(size_t)15;
    const size_t lo = (size_t)b * per;
    if (lo < bytes) bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(W2) + lo, (uint32_t)min(per, bytes - lo));
  }
  trace_mark(trace, 16);
  if (pdl) pdl_wait();
  __syncthreads();
  trace_mark(trace, 17);
  router_hidden(part, KS, B, b, rows1, b1s, h_r > 0, a1);
  __syncthreads();
  trace_mark(trace, 18);
  if (h_r > 0) {
    router_scores_thread<T>(W2, a1, b2s, M, h_r, s);
  } else {
    for (int m = threadIdx.x; m < M; m += blockDim.x) s[m] = a1[m];
  }
  __syncthreads();
  const int words = (M + 31) / 32;
  for (int m = threadIdx.x; m < M; m += blockDim.x) scores[(size_t)b * M + m] = s[m];
  if (sel == nullptr) return;
  if (pdl) pdl_launch_dependents();
  trace_mark(trace, 19);
  // O(M^2 / threads) rank count up to M = 256 (one score per thread: 0.5 us); radix select above
  if (M > 256) radix_mask(s, M, k_per_row ? k_per_row[b] : k, mask, rhist);
  else rank_mask(s, M, k_per_row ? k_per_row[b] : k, mask);
  __syncthreads();
  trace_mark(trace, 20);
  if (!shared) {
    emit_fast(mask, M, offs, sel + (size_t)b * M, sel_count + b, sl_off + (size_t)b * (M + 1), tmp);
    return;
  }
  // shared mode: every row-CTA publishes its TopK mask (workspace tail after the layer-1 partials);
  // the last row-CTA ORs the B masks into the union and emits it (R9)
  uint32_t* gmask = reinterpret_cast<uint32_t*>(const_cast<float*>(part) + (size_t)KS * B * rows1);
  for (int w = threadIdx.x; w < words; w += blockDim.x) gmask[(size_t)b * (kMaxM / 32) + w] = mask[w];
  __syncthreads();
  if (threadIdx.x == 0) is_last = release_add(counter, 1u) == (unsigned)(gridDim.x - 1);
  __syncthreads();
  trace_mark(trace, 21);
  if (!is_last) return;
  if (threadIdx.x == 0) fence_acq_rel_gpu();
  __syncthreads();
  for (int w = threadIdx.x; w < words; w += blockDim.x) {
    uint32_t u = 0u;
    for (int r = 0; r < B; ++r) u |= __ldcg(gmask + (size_t)r * (kMaxM / 32) + w);
    acc[w] = u;
  }
  __syncthreads();
  emit_fast(acc, M, offs, sel, sel_count, sl_off, tmp);
  if (threadIdx.x == 0) *counter = 0u;
  trace_mark(trace, 22);
}

// ------------------------------------------------------------------ host side

MetaPlan meta_plan(const ds_router* r, int B) {
  MetaPlan p;
  const int E = r->dtype == DS_BF16 ? 8 : 4;
  p.rows1 = r->h_r > 0 ? r->h_r : r->M;
  const int dr = 2 * r->d;
  // K-chunk: up to 4 x 16-byte chunks per lane; keep x staging <= 96 KB
  int KC = 4 * 32 * E;
  const int esz = r->dtype == DS_BF16 ? 2 : 4;
  while (KC > 32 * E && (size_t)B * KC * esz > 96 * 1024) KC /= 2;
  if (KC > dr) KC = ((dr + E - 1) / E) * E;
  p.KC = KC;
  // rows per layer-1 CTA (x staging <= 96 KB); more rows -> more row blocks (grid z)
  p.RB = std::max(1, std::min(B, (int)((96 * 1024) / ((size_t)KC * esz))));
  p.KS = (dr + KC - 1) / KC;
  // many bf16 rows: layer 1 on tcgen05 (meta_tc.cu) with its own split count
  int ks_tc = 0, kcp = 0;
  p.tc = meta_tc_plan(r, B, &ks_tc, &kcp) ? 1 : 0;
  p.KS_tc = ks_tc;
  p.kc_per_tc = kcp;
  const int ks_max = std::max(p.KS, p.tc ? p.KS_tc : 0);
  // layer-1 partials, then (shared mode) the rows' TopK masks
  p.part_bytes = (size_t)ks_max * B * p.rows1 * sizeof(float) + (size_t)B * (kMaxM / 32) * sizeof(uint32_t);
  return p;
}

template <typename T>
static cudaError_t launch_meta_t(const ds_router* r, const void* h_prev, const void* e, int B, float* scores,
                                 float* part, unsigned* counter, const int32_t* offsets, int k,
                                 const int32_t* k_per_row, int shared, int32_t* sel, int32_t* sel_count,
                                 int32_t* sl_offsets, cudaStream_t st, bool pdl) {
  const MetaPlan p = meta_plan(r, B);
  const size_t smem1 = (size_t)p.RB * p.KC * sizeof(T);
  if (smem1 > 48 * 1024) {
    cudaError_t ea = cudaFuncSetAttribute(meta_l1_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    if (ea != cudaSuccess) return ea;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;

  int KS = p.KS;
  const bool tc = p.tc && sizeof(T) == 2 && ((reinterpret_cast<uintptr_t>(h_prev) | reinterpret_cast<uintptr_t>(e) |
                                              reinterpret_cast<uintptr_t>(r->W1)) & 15u) == 0;
  if (tc) {
    KS = p.KS_tc;
    cudaError_t et = launch_meta_tc_l1(r, h_prev, e, B, part, p.KS_tc, p.kc_per_tc, st, pdl);
    if (et != cudaSuccess) return et;
  } else {
  cudaLaunchConfig_t c1 = {};
  c1.gridDim = dim3((p.rows1 + kMetaUnitsPerCTA - 1) / kMetaUnitsPerCTA, p.KS, (B + p.RB - 1) / p.RB);
  c1.blockDim = dim3(kMetaThreads);
  c1.dynamicSmemBytes = smem1;
  c1.stream = st;
  c1.attrs = attr;
  c1.numAttrs = pdl ? 1 : 0;
  cudaError_t err = cudaLaunchKernelEx(&c1, meta_l1_kernel<T>, static_cast<const T*>(r->W1),
                                       static_cast<const T*>(h_prev), static_cast<const T*>(e), B, r->d, p.rows1,
                                       p.KC, p.RB, part, pdl ? 1 : 0);
  if (err != cudaSuccess) return err;
  }
  cudaLaunchConfig_t c2 = {};
  c2.gridDim = dim3(B);
  c2.blockDim = dim3(kMetaThreads);
  c2.stream = st;
  c2.attrs = attr;
  c2.numAttrs = 1;  // layer 2 always follows layer 1 in-stream
  return cudaLaunchKernelEx(&c2, meta_l2_kernel<T>, (const float*)part, KS, B, p.rows1, r->b1,
                            static_cast<const T*>(r->W2), r->b2, r->h_r, r->M, scores, offsets, k, k_per_row,
                            shared, sel, sel_count, sl_offsets, counter, 1, debug_trace());
}

cudaError_t launch_meta(const ds_router* r, const void* h_prev, const void* e, int B, float* scores, float* part,
                        unsigned* counter, const int32_t* offsets, int k, const int32_t* k_per_row, int shared,
                        int32_t* sel, int32_t* sel_count, int32_t* sl_offsets, cudaStream_t st, bool pdl) {
  if (r->dtype == DS_BF16)
    return launch_meta_t<__nv_bfloat16>(r, h_prev, e, B, scores, part, counter, offsets, k, k_per_row, shared, sel,
                                        sel_count, sl_offsets, st, pdl);
  return launch_meta_t<float>(r, h_prev, e, B, scores, part, counter, offsets, k, k_per_row, shared, sel,
                              sel_count, sl_offsets, st, pdl);
}

cudaError_t launch_select(const float* scores, int B, int M, const int32_t* offsets, int k, const int32_t* k_per_row,
                          int shared, int32_t* sel, int32_t* sel_count, int32_t* sl_offsets, unsigned* /*counter*/,
                          cudaStream_t st) {
  select_kernel<<<shared ? 1 : B, kSelThreads, 0, st>>>(scores, B, M, offsets, k, k_per_row, shared, sel, sel_count,
                                                        sl_offsets);
  return cudaGetLastError();
}

}  // namespace ds
