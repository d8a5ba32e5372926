// step.cu — one DynaSpec draft step (Alg. 1 lines 8, 10, 11) in ONE persistent launch.
//
// When the router does not have a drafter core to hide behind (single-stream use), the
// B200-first choice is a single kernel with one CTA per SM:
//   phase A  every warp of every CTA: router layer 1 split-K partials of W1 [h_r][2d];
//            the selector CTA(s) meanwhile prefetch W2 into shared memory with a TMA bulk copy;
//   phase B  selector CTA(s) (row b on CTA b; the union on CTA 0 in shared mode), after all
//            partials have landed (global counter): b1 + ReLU, layer 2, TopK_k + ascending ids +
//            sl_offsets — published to global and signalled with a second counter;
//   phase C  all CTAs: the gathered head of head_impl.cuh over the published shortlist;
//   phase D  per-CTA (max, sum exp, top-k_t) partials, last-CTA merge + remap.
// The grid is #SM CTAs (1 per SM by shared-memory footprint), so every CTA is resident and the
// counter waits cannot deadlock; the counters are reset by the merging CTA.  No float atomics.
#include <algorithm>

#include "head_impl.cuh"
#include "internal.h"
#include "select_impl.cuh"

namespace ds {

constexpr int kStepCH = 2;  // 16-byte chunks per lane per layer-1 task

struct StepArgs {
  HeadArgs h;               // head part; h.sel / sel_count / sl_off point to the step outputs
  const void* W1;
  const float* b1;
  const void* W2;
  const float* b2;
  const void* h_prev;
  const void* e;
  float* scores;            // [B][M]
  float* mpart;             // [KS][B][rows1]
  int32_t B, h_r, rows1, KC, KS, k, w2_prefetch;
  unsigned* ctr;            // [0] merge ticket, [1] phase-A count, [2] selections published
  unsigned long long* trace;  // opt-in phase timestamps (nullptr)
};

template <typename T>
__device__ void step_phase_a(const StepArgs& s) {
  constexpr int E = Elem<T>::kPer16B;
  const int d = s.h.d, dr = 2 * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int tasks = s.rows1 * s.KS;
  const T* W1 = static_cast<const T*>(s.W1);
  const T* hp = static_cast<const T*>(s.h_prev);
  const T* ev = static_cast<const T*>(s.e);
  for (int t = blockIdx.x * nw + warp; t < tasks; t += gridDim.x * nw) {
    const int u = t % s.rows1, ks = t / s.rows1;
    const int k0 = ks * s.KC;
    uint4 wv[kStepCH];
#pragma unroll
    for (int j = 0; j < kStepCH; ++j) {
      const int k = k0 + lane * E + j * 32 * E;
      wv[j] = (k < dr && k < k0 + s.KC) ? __ldg(reinterpret_cast<const uint4*>(W1 + (size_t)u * dr + k))
                                        : make_uint4(0, 0, 0, 0);
    }
    for (int b = 0; b < s.B; ++b) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < kStepCH; ++j) {
        const int k = k0 + lane * E + j * 32 * E;
        if (k < dr && k < k0 + s.KC) {
          const T* src = k < d ? hp + (size_t)b * d + k : ev + (size_t)b * d + (k - d);
          float wf[E], xf[E];
          widen16(wv[j], wf, W1);
          widen16(__ldg(reinterpret_cast<const uint4*>(src)), xf, W1);
#pragma unroll
          for (int q = 0; q < E; ++q) acc = fmaf(wf[q], xf[q], acc);
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) s.mpart[((size_t)ks * s.B + b) * s.rows1 + u] = acc;
    }
  }
}

// Layer 2 + selection for the rows this CTA owns; returns after publishing.
template <typename T>
__device__ void step_phase_b(const StepArgs& s, const HeadCtx& c, uint64_t* w2bar) {
  const int M = s.h.M;
  float* a1 = reinterpret_cast<float*>(c.extra);
  float* sc = a1 + 1024;
  float* b1s = sc + 1024;
  float* b2s = b1s + 1024;
  int32_t* offs = reinterpret_cast<int32_t*>(b2s + 1024);
  uint8_t* flags = reinterpret_cast<uint8_t*>(offs + 1028);
  int* scratch = reinterpret_cast<int*>(flags + 1024);
  const T* W2 = s.w2_prefetch ? reinterpret_cast<const T*>(c.ring) : static_cast<const T*>(s.W2);
  if (threadIdx.x == 0) spin_until_geq(s.ctr + 1, gridDim.x);  // all layer-1 partials visible
  trace_mark(s.trace, 8);
  if (s.w2_prefetch) mbar_wait(w2bar, 0);
  __syncthreads();
  trace_mark(s.trace, 9);
  for (int m = threadIdx.x; m < M; m += blockDim.x) flags[m] = 0;
  const bool shared = s.h.shared != 0;
  const int b_lo = shared ? 0 : blockIdx.x;
  const int b_step = shared ? 1 : gridDim.x;
  int published = 0;
  for (int b = b_lo; b < s.B; b += b_step) {
    __syncthreads();
    router_hidden(s.mpart, s.KS, s.B, b, s.rows1, b1s, s.h_r > 0, a1);
    __syncthreads();
    if (s.h_r > 0) {
      router_out<T>(W2, a1, b2s, M, s.h_r, sc);
    } else {
      for (int m = threadIdx.x; m < M; m += blockDim.x) sc[m] = a1[m];
    }
    __syncthreads();
    for (int m = threadIdx.x; m < M; m += blockDim.x) s.scores[(size_t)b * M + m] = sc[m];
    rank_select(sc, M, s.k, flags);
    if (!shared) {
      __syncthreads();
      emit_selection(flags, M, offs, const_cast<int32_t*>(s.h.sel) + (size_t)b * M,
                     const_cast<int32_t*>(s.h.sel_count) + b, const_cast<int32_t*>(s.h.sl_off) + (size_t)b * (M + 1),
                     scratch);
      __syncthreads();
      for (int m = threadIdx.x; m < M; m += blockDim.x) flags[m] = 0;
      ++published;
    }
  }
  if (shared) {
    __syncthreads();
    emit_selection(flags, M, offs, const_cast<int32_t*>(s.h.sel), const_cast<int32_t*>(s.h.sel_count),
                   const_cast<int32_t*>(s.h.sl_off), scratch);
    published = 1;
  }
  __threadfence();
  __syncthreads();
  trace_mark(s.trace, 10);
  if (threadIdx.x == 0 && published) atomicAdd(s.ctr + 2, (unsigned)published);
}

template <typename T>
__global__ void __launch_bounds__((kMaxStages + 1) * 32, 1) step_kernel(const StepArgs s) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const HeadArgs& a = s.h;
  const HeadSmem L = head_smem(a.stages, a.stage_bytes, a.nrows, a.d, (int)sizeof(T), a.lcap, kStepExtra);
  const HeadCtx c = head_ctx(smem, L);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool shared = a.shared != 0;
  const int nsel_rows = shared ? 1 : s.B;
  const bool selector = shared ? blockIdx.x == 0 : (int)blockIdx.x < s.B;
  uint64_t* w2bar = c.full + 2 * kMaxStages;  // spare barrier slot
  if (threadIdx.x == 0) {
    head_init_barriers(c, a.stages);
    if (selector && s.w2_prefetch) {
      mbar_init(w2bar, 1);
      fence_mbar_init();
    }
  }
  __syncthreads();
  // Router constants do not depend on upstream work: stage them before waiting on the previous
  // kernel (W2 by TMA into the idle ring; b1, b2, offsets by plain loads into `extra`).
  if (selector) {
    if (s.w2_prefetch && threadIdx.x == 0) {
      mbar_arrive_expect_tx(w2bar, (uint32_t)s.w2_prefetch);
      bulk_g2s(c.ring, s.W2, (uint32_t)s.w2_prefetch, w2bar, policy_evict_last());
    }
    float* b1s = reinterpret_cast<float*>(c.extra) + 2048;
    float* b2s = b1s + 1024;
    int32_t* offs = reinterpret_cast<int32_t*>(b2s + 1024);
    for (int u = threadIdx.x; u < s.rows1; u += blockDim.x) b1s[u] = __ldg(s.b1 + u);
    for (int m = threadIdx.x; m < a.M; m += blockDim.x) b2s[m] = s.h_r > 0 ? __ldg(s.b2 + m) : 0.f;
    for (int m = threadIdx.x; m <= a.M; m += blockDim.x) offs[m] = __ldg(a.offsets + m);
  }
  trace_mark(s.trace, 0);
  if (a.pdl) pdl_wait();  // h_prev / e / h_new come from upstream kernels
  trace_mark(s.trace, 1);
  // h_new -> smem (consumer warps), layer-1 partials (all warps)
  head_load_h(a, c, (int)sizeof(T), threadIdx.x, blockDim.x);
  step_phase_a<T>(s);
  __threadfence();
  __syncthreads();
  trace_mark(s.trace, 2);
  if (threadIdx.x == 0) atomicAdd(s.ctr + 1, 1u);
  if (selector) step_phase_b<T>(s, c, w2bar);
  if (threadIdx.x == 0) spin_until_geq(s.ctr + 2, (unsigned)nsel_rows);  // selections published
  __syncthreads();
  trace_mark(s.trace, 3);
  if (selector && s.w2_prefetch) fence_proxy_async_smem();  // generic reads of W2 before TMA reuse
  head_segments(a, c);
  __syncthreads();
  trace_mark(s.trace, 4);
  if (warp == a.stages) {
    if (lane == 0) head_produce<T>(a, c);
  } else {
    head_consume<T>(a, c, warp, lane);
  }
  __syncthreads();
  trace_mark(s.trace, 5);
  if (a.pdl) pdl_launch_dependents();
  head_partials(a, c);
  trace_mark(s.trace, 6);
  if (!head_ticket(a, c)) return;
  head_merge(a, c, a.stages * a.stage_bytes);
  trace_mark(s.trace, 7);
  if (threadIdx.x == 0) {
    s.ctr[0] = 0u;
    s.ctr[1] = 0u;
    s.ctr[2] = 0u;
  }
}

// ------------------------------------------------------------------ host side

struct StepPlan {
  HeadPlan hp;
  int rows1, KC, KS;
  size_t mpart_bytes, scores_bytes, head_bytes, total;
  int w2_bytes;
};

static bool step_plan(const ds_clusters* c, const ds_router* r, int B, int k_t, int64_t max_shortlist, int shared,
                      StepPlan* p) {
  if (B > kMaxGroups) return false;
  if (r->M > 1024 || (r->h_r > 0 ? r->h_r : r->M) > 1024) return false;
  if (!head_plan_ex(c, B, k_t, max_shortlist, kStepExtra, kMaxGroups, &p->hp)) return false;
  if (p->hp.rows_per_launch < B) return false;  // one launch must hold every row
  if (!shared && B > p->hp.G) return false;
  const int E = r->dtype == DS_BF16 ? 8 : 4;
  const int esz = r->dtype == DS_BF16 ? 2 : 4;
  p->rows1 = r->h_r > 0 ? r->h_r : r->M;
  p->KC = kStepCH * 32 * E;
  p->KS = (2 * r->d + p->KC - 1) / p->KC;
  p->mpart_bytes = align_up((size_t)p->KS * B * p->rows1 * sizeof(float), 256);
  p->scores_bytes = align_up((size_t)B * r->M * sizeof(float), 256);
  p->head_bytes = align_up(p->hp.part_bytes, 256);
  p->total = 256 + p->mpart_bytes + p->scores_bytes + p->head_bytes;
  const size_t w2 = r->h_r > 0 ? (size_t)r->M * r->h_r * esz : 0;
  p->w2_bytes = (w2 > 0 && w2 % 16 == 0 && w2 <= (size_t)p->hp.stages * p->hp.stage_bytes) ? (int)w2 : 0;
  return true;
}

bool step_supported(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared, int64_t max_shortlist) {
  StepPlan p;
  return step_plan(c, r, B, k_t, max_shortlist, shared, &p);
}

size_t step_ws_bytes(const ds_clusters* c, const ds_router* r, int B, int k_t) {
  StepPlan p;
  if (!step_plan(c, r, B, k_t, 0, 0, &p) && !step_plan(c, r, B, k_t, 0, 1, &p)) return 0;
  return p.total;
}

template <typename T>
static cudaError_t launch_step_t(const StepArgs& s, size_t smem, int G, cudaStream_t st, bool pdl) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(step_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem_optin());
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3((s.h.stages + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, step_kernel<T>, s);
}

cudaError_t launch_step(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                        const void* h_new, int B, int k, int k_t, int shared, int64_t max_shortlist, float* scores,
                        int32_t* sel, int32_t* sel_count, int32_t* sl_offsets, int32_t* top_ids, float* top_logits,
                        float* top_logp, float* lse, float* z_out, int64_t z_stride, void* ws, cudaStream_t st,
                        bool pdl) {
  StepPlan p;
  if (!step_plan(c, r, B, k_t, max_shortlist, shared, &p)) return cudaErrorInvalidValue;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  unsigned* ctr = reinterpret_cast<unsigned*>(w8);
  float* mpart = reinterpret_cast<float*>(w8 + 256);
  float* sc = scores ? scores : reinterpret_cast<float*>(w8 + 256 + p.mpart_bytes);
  float* hpart = reinterpret_cast<float*>(w8 + 256 + p.mpart_bytes + p.scores_bytes);
  StepArgs s;
  fill_head_args(s.h, c, p.hp, h_new, 0, B, sel, sel_count, sl_offsets, shared, k_t, max_shortlist, top_ids,
                 top_logits, top_logp, lse, z_out, z_stride, hpart, ctr, pdl);
  s.W1 = r->W1;
  s.b1 = r->b1;
  s.W2 = r->W2;
  s.b2 = r->b2;
  s.h_prev = h_prev;
  s.e = e;
  s.scores = sc;
  s.mpart = mpart;
  s.B = B;
  s.h_r = r->h_r;
  s.rows1 = p.rows1;
  s.KC = p.KC;
  s.KS = p.KS;
  s.k = k;
  s.w2_prefetch = p.w2_bytes;
  s.ctr = ctr;
  s.trace = debug_trace();
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  const size_t smem = head_smem(p.hp.stages, p.hp.stage_bytes, B, c->d, esz, p.hp.lcap, kStepExtra).total;
  return c->dtype == DS_BF16 ? launch_step_t<__nv_bfloat16>(s, smem, p.hp.G, st, pdl)
                             : launch_step_t<float>(s, smem, p.hp.G, st, pdl);
}

}  // namespace ds
