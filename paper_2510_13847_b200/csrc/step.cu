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

// Shared-memory carve-up of the fused step's router/selection scratch (inside HeadSmem.extra).
struct StepExtra {
  uint32_t a1, sc, b1, b2, offs, mask, hist, sh, sel, sloff, cnt, tmp, sv, si, total;
};
__host__ __device__ inline StepExtra step_extra(int M, int rows1) {
  StepExtra X;
  uint32_t o = 0;
  auto take = [&](uint32_t bytes) {
    const uint32_t at = o;
    o = (o + bytes + 15u) & ~15u;
    return at;
  };
  X.a1 = take(4u * rows1);
  X.sc = take(4u * M);
  X.b1 = take(4u * rows1);
  X.b2 = take(4u * M);
  X.offs = take(4u * (M + 1));
  X.mask = take(4u * 32);
  X.hist = take(4u * 256);
  X.sh = take(16);
  X.sel = take(4u * M);
  X.sloff = take(4u * (M + 1));
  X.cnt = take(16);
  X.tmp = take(4u * M);
  X.sv = take(4u * M);
  X.si = take(4u * M);
  X.total = o;
  return X;
}

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
  uint32_t* maskbuf;        // [B][32] per-row selection masks (tree mode)
  int32_t B, h_r, rows1, KC, KS, k, w2_prefetch, extra_bytes;
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
  const uint64_t keep = policy_evict_last();
  for (int t = blockIdx.x * nw + warp; t < tasks; t += gridDim.x * nw) {
    const int u = t % s.rows1, ks = t / s.rows1;
    const int k0 = ks * s.KC;
    uint4 wv[kStepCH];
#pragma unroll
    for (int j = 0; j < kStepCH; ++j) {
      const int k = k0 + lane * E + j * 32 * E;
      wv[j] = (k < dr && k < k0 + s.KC) ? ld_evict_last_v4(W1 + (size_t)u * dr + k, keep)
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

// Router layer 2 + TopK mask of row b (whole CTA): a1 -> scores -> radix select.
template <typename T>
__device__ void step_row_select(const StepArgs& s, uint8_t* ex, const StepExtra& X, const T* W2, int b,
                                bool write_scores) {
  const int M = s.h.M;
  float* a1 = reinterpret_cast<float*>(ex + X.a1);
  float* sc = reinterpret_cast<float*>(ex + X.sc);
  router_hidden(s.mpart, s.KS, s.B, b, s.rows1, reinterpret_cast<const float*>(ex + X.b1), s.h_r > 0, a1);
  __syncthreads();
  trace_mark(s.trace, 11);
  if (s.h_r > 0) {
    router_scores_thread<T>(W2, a1, reinterpret_cast<const float*>(ex + X.b2), M, s.h_r, sc);
  } else {
    for (int m = threadIdx.x; m < M; m += blockDim.x) sc[m] = a1[m];
  }
  __syncthreads();
  trace_mark(s.trace, 12);
  if (write_scores)
    for (int m = threadIdx.x; m < M; m += blockDim.x) s.scores[(size_t)b * M + m] = sc[m];
  uint32_t* mask = reinterpret_cast<uint32_t*>(ex + X.mask);
  for (int w = threadIdx.x; w < (M + 31) / 32; w += blockDim.x) mask[w] = 0u;
  // TopK_k under (score desc, id asc) (R7): pruned rank count, bits set per winner
  block_topk(
      M, s.k, [&](int i, float& v, int& id) { v = sc[i] + 0.0f; id = i; },
      [&](int, float, int id) { atomicOr(&mask[id >> 5], 1u << (id & 31)); },
      reinterpret_cast<float*>(ex + X.sv), reinterpret_cast<int*>(ex + X.si), reinterpret_cast<int*>(ex + X.sh));
  trace_mark(s.trace, 13);
}

template <typename T>
__global__ void __launch_bounds__((kMaxStages + 1) * 32, 1) step_kernel(const StepArgs s) {
  extern __shared__ __align__(1024) uint8_t smem[];
  HeadArgs a = s.h;
  const HeadSmem L = head_smem(a.stages, a.stage_bytes, a.nrows, a.d, (int)sizeof(T), a.lcap, s.extra_bytes);
  const HeadCtx c = head_ctx(smem, L);
  const StepExtra X = step_extra(a.M, s.rows1);
  uint8_t* ex = c.extra;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = a.M;
  const bool shared = a.shared != 0;
  const bool local = !shared && s.B == 1;  // every CTA selects for itself: no publish round trip
  const bool row_cta = local || (int)blockIdx.x < s.B;
  uint64_t* w2bar = c.full + 2 * kMaxStages;  // spare barrier slot
  const bool prefetch = row_cta && s.w2_prefetch > 0;
  if (threadIdx.x == 0) {
    head_init_barriers(c, a.stages);
    if (prefetch) {
      mbar_init(w2bar, 1);
      fence_mbar_init();
    }
  }
  __syncthreads();
  trace_mark(s.trace, 0);
  if (a.pdl) pdl_wait();  // h_prev / e / h_new come from upstream kernels
  trace_mark(s.trace, 1);
  // Router constants (W2 by TMA into the idle ring; b1, b2, offsets by plain loads).  Issued after
  // the PDL wait so that the early-launched CTAs do not compete with the previous step's merge
  // for L2; they land while phase A runs.
  if (row_cta) {
    if (prefetch && threadIdx.x == 0) {
      mbar_arrive_expect_tx(w2bar, (uint32_t)s.w2_prefetch);
      bulk_g2s(c.ring, s.W2, (uint32_t)s.w2_prefetch, w2bar, policy_evict_last());
    }
    float* b1s = reinterpret_cast<float*>(ex + X.b1);
    float* b2s = reinterpret_cast<float*>(ex + X.b2);
    int32_t* offs_w = reinterpret_cast<int32_t*>(ex + X.offs);
    for (int u = threadIdx.x; u < s.rows1; u += blockDim.x) b1s[u] = __ldg(s.b1 + u);
    for (int m = threadIdx.x; m < M; m += blockDim.x) b2s[m] = s.h_r > 0 ? __ldg(s.b2 + m) : 0.f;
    for (int m = threadIdx.x; m <= M; m += blockDim.x) offs_w[m] = __ldg(a.offsets + m);
  }
  head_load_h(a, c, (int)sizeof(T), threadIdx.x, blockDim.x);
  step_phase_a<T>(s);  // router layer 1, split over every warp of every CTA
  __syncthreads();
  trace_mark(s.trace, 2);
  if (threadIdx.x == 0) release_add(s.ctr + 1, 1u);

  int32_t* sel_s = reinterpret_cast<int32_t*>(ex + X.sel);
  int32_t* sloff_s = reinterpret_cast<int32_t*>(ex + X.sloff);
  int32_t* cnt_s = reinterpret_cast<int32_t*>(ex + X.cnt);
  uint32_t* mask = reinterpret_cast<uint32_t*>(ex + X.mask);
  const int32_t* offs = reinterpret_cast<const int32_t*>(ex + X.offs);
  int32_t* tmp = reinterpret_cast<int32_t*>(ex + X.tmp);
  const int mwords = (M + 31) / 32;
  if (row_cta) {
    if (threadIdx.x == 0) acquire_wait_geq(s.ctr + 1, gridDim.x);  // all layer-1 partials visible
    trace_mark(s.trace, 8);
    if (prefetch) mbar_wait(w2bar, 0);
    __syncthreads();
    const T* W2 = prefetch ? reinterpret_cast<const T*>(c.ring) : static_cast<const T*>(s.W2);
    const int b = local ? 0 : (int)blockIdx.x;
    step_row_select<T>(s, ex, X, W2, b, !local || blockIdx.x == 0);
    if (local) {
      emit_fast(mask, M, offs, sel_s, cnt_s, sloff_s, tmp);
      if (blockIdx.x == 0) {  // CTA 0 also writes the caller's outputs
        __syncthreads();
        emit_fast(mask, M, offs, const_cast<int32_t*>(a.sel), const_cast<int32_t*>(a.sel_count),
                  const_cast<int32_t*>(a.sl_off), tmp);
      }
    } else if (shared) {
      for (int i = threadIdx.x; i < mwords; i += blockDim.x) s.maskbuf[(size_t)b * 32 + i] = mask[i];
    } else {
      emit_fast(mask, M, offs, const_cast<int32_t*>(a.sel) + (size_t)b * M, const_cast<int32_t*>(a.sel_count) + b,
                const_cast<int32_t*>(a.sl_off) + (size_t)b * (M + 1), tmp);
    }
    __syncthreads();
    trace_mark(s.trace, 10);
    if (!local && threadIdx.x == 0) release_add(s.ctr + 2, 1u);
  }
  if (!local) {
    if (threadIdx.x == 0) acquire_wait_geq(s.ctr + 2, (unsigned)s.B);  // every row's selection published
    __syncthreads();
    if (shared) {  // union over the depth's rows (R9), formed by every CTA
      int32_t* offs_g = reinterpret_cast<int32_t*>(ex + X.offs);
      if (!row_cta)
        for (int m = threadIdx.x; m <= M; m += blockDim.x) offs_g[m] = __ldg(a.offsets + m);
      for (int i = threadIdx.x; i < mwords; i += blockDim.x) {
        uint32_t u = 0;
        for (int b = 0; b < s.B; ++b) u |= __ldcg(s.maskbuf + (size_t)b * 32 + i);
        mask[i] = u;
      }
      __syncthreads();
      emit_fast(mask, M, offs, sel_s, cnt_s, sloff_s, tmp);
      if (blockIdx.x == 0) {
        __syncthreads();
        emit_fast(mask, M, offs, const_cast<int32_t*>(a.sel), const_cast<int32_t*>(a.sel_count),
                  const_cast<int32_t*>(a.sl_off), tmp);
      }
      __syncthreads();
    }
  } else {
    __syncthreads();
  }
  trace_mark(s.trace, 3);
  if (local || shared) {  // the head reads this CTA's own copy of the selection
    a.sel = sel_s;
    a.sel_count = cnt_s;
    a.sl_off = sloff_s;
  }
  if (prefetch) fence_proxy_async_smem();  // generic reads of W2 in the ring before TMA reuse
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
  head_partials(a, c, a.stages * a.stage_bytes);
  trace_mark(s.trace, 6);
  const int j = head_ticket(a, c);
  if (j < 0) return;
  trace_mark(s.trace, 14);
  trace_mark(s.trace, 15);  // back-to-back: the cost of one mark
  head_merge(a, c, a.stages * a.stage_bytes, s.trace, 0, j, min(a.nrows, (int)gridDim.x));
  trace_mark(s.trace, 7);
  head_merge_done(a, 2);  // also resets the phase counters ctr[1], ctr[2]
}

// ------------------------------------------------------------------ host side

struct StepPlan {
  HeadPlan hp;
  int rows1, KC, KS, extra;
  size_t mpart_bytes, scores_bytes, mask_bytes, head_bytes, total;
  int w2_bytes;
};

static bool step_plan(const ds_clusters* c, const ds_router* r, int B, int k_t, int64_t max_shortlist, int shared,
                      StepPlan* p) {
  if (B > kMaxGroups) return false;
  if (r->M > 1024 || (r->h_r > 0 ? r->h_r : r->M) > 1024) return false;
  if (B > num_sms()) return false;
  p->rows1 = r->h_r > 0 ? r->h_r : r->M;
  p->extra = (int)step_extra(r->M, p->rows1).total;
  if (!head_plan_ex(c, B, k_t, max_shortlist, p->extra, kMaxGroups, &p->hp)) return false;
  if (p->hp.rows_per_launch < B) return false;  // one launch must hold every row
  if (!shared && B > p->hp.G) return false;
  const int E = r->dtype == DS_BF16 ? 8 : 4;
  const int esz = r->dtype == DS_BF16 ? 2 : 4;
  p->KC = kStepCH * 32 * E;
  p->KS = (2 * r->d + p->KC - 1) / p->KC;
  p->mpart_bytes = align_up((size_t)p->KS * B * p->rows1 * sizeof(float), 256);
  p->scores_bytes = align_up((size_t)B * r->M * sizeof(float), 256);
  p->mask_bytes = align_up((size_t)B * 32 * sizeof(uint32_t), 256);
  p->head_bytes = align_up(p->hp.part_bytes, 256);
  p->total = kWsFixed + p->mpart_bytes + p->scores_bytes + p->mask_bytes + p->head_bytes;
  const size_t w2 = r->h_r > 0 ? (size_t)r->M * r->h_r * esz : 0;
  p->w2_bytes = (w2 > 0 && w2 % 16 == 0 && w2 <= (size_t)p->hp.stages * p->hp.stage_bytes) ? (int)w2 : 0;
  return true;
}

bool step_supported(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared, int64_t max_shortlist) {
  StepPlan p;
  return step_plan(c, r, B, k_t, max_shortlist, shared, &p);
}

// The cluster step's records live after the grid-wide step's scratch, so the two kernels never
// alias (the cluster step's merger relies on its record words reading 0 between launches).
// The workspace of the fused step does not depend on the shortlist bound (only its shared-memory
// plan does), so size it from any plan that fits: the unbounded one, else the tightest bound
// (a tree step of few clusters fits where the full-vocabulary bound does not).  Both modes.
static size_t grid_step_ws(const ds_clusters* c, const ds_router* r, int B, int k_t) {
  size_t need = 0;
  for (int64_t ms : {(int64_t)0, (int64_t)1})
    for (int sh = 0; sh < 2; ++sh) {
      StepPlan p;
      if (step_plan(c, r, B, k_t, ms, sh, &p)) need = std::max(need, align_up(p.total, 256));
    }
  return need;
}

bool step_rows_as_gsteps(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared) {
  const char* mv = getenv("DS_GSTEP_ROWS_MAX");
  const int bmax = mv && mv[0] ? atoi(mv) : 3;
  return !shared && B >= 2 && B <= bmax && gstep_supported(c, r, 1, k_t, 0);
}

size_t step_ws_bytes(const ds_clusters* c, const ds_router* r, int B, int k_t) {
  return grid_step_ws(c, r, B, k_t);  // the single-row step kernels use the fixed prefix (internal.h)
}

template <typename T>
static cudaError_t launch_step_t(const StepArgs& s, size_t smem, int G, cudaStream_t st, bool pdl) {
  static int configured[64] = {0};  // the attribute is per device
  {
    cudaError_t e = configure_max_smem(reinterpret_cast<const void*>(step_kernel<T>), configured);
    if (e != cudaSuccess) return e;
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
  // B = 1: the grid step (gstep.cu: router units over every CTA, no clusters) or, for shapes it does
  // not cover, the cluster step (cstep.cu); neither needs a grid-wide barrier before the head streams
  if (gstep_supported(c, r, B, k_t, shared) && gstep_pointers_ok(r, h_prev, e, h_new))
    return launch_gstep(c, r, h_prev, e, h_new, k, k_t, max_shortlist, scores, sel, sel_count, sl_offsets, top_ids,
                        top_logits, top_logp, lse, z_out, ws, st, pdl);
  // a few independent rows: one grid step per row, PDL-chained (Llama-3, us per draft step: B = 2
  // 39.2 vs 49.0 for the grid-wide multi-row step, B = 3 58.2 vs 60.3, B = 4 ~78 vs 71.2);
  // DS_GSTEP_ROWS_MAX (default 3)
  if (step_rows_as_gsteps(c, r, B, k_t, shared)) {
    const size_t esz = c->dtype == DS_BF16 ? 2 : 4, xr = (size_t)c->d * esz;
    for (int b = 0; b < B; ++b) {
      const uint8_t* hp = static_cast<const uint8_t*>(h_prev) + b * xr;
      const uint8_t* ee = static_cast<const uint8_t*>(e) + b * xr;
      const uint8_t* hn = static_cast<const uint8_t*>(h_new) + b * xr;
      if (!gstep_pointers_ok(r, hp, ee, hn)) return cudaErrorInvalidValue;
      const cudaError_t err = launch_gstep(
          c, r, hp, ee, hn, k, k_t, max_shortlist, scores ? scores + (size_t)b * c->M : nullptr,
          sel + (size_t)b * c->M, sel_count + b, sl_offsets + (size_t)b * (c->M + 1), top_ids + (size_t)b * k_t,
          top_logits + (size_t)b * k_t, top_logp + (size_t)b * k_t, lse + b, z_out ? z_out + (size_t)b * z_stride : nullptr,
          ws, st, b == 0 ? pdl : true);
      if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
  }
  if (cstep_supported(c, r, B, k_t, shared, max_shortlist) && cstep_pointers_ok(r, h_prev, e, h_new))
    return launch_cstep(c, r, h_prev, e, h_new, k, k_t, max_shortlist, scores, sel, sel_count, sl_offsets, top_ids,
                        top_logits, top_logp, lse, z_out, z_stride, ws, st, pdl);
  StepPlan p;
  if (!step_plan(c, r, B, k_t, max_shortlist, shared, &p)) return cudaErrorInvalidValue;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  unsigned* ctr = reinterpret_cast<unsigned*>(w8);
  float* mpart = reinterpret_cast<float*>(w8 + kWsFixed);
  float* sc = scores ? scores : reinterpret_cast<float*>(w8 + kWsFixed + p.mpart_bytes);
  uint32_t* maskbuf = reinterpret_cast<uint32_t*>(w8 + kWsFixed + p.mpart_bytes + p.scores_bytes);
  float* hpart = reinterpret_cast<float*>(w8 + kWsFixed + p.mpart_bytes + p.scores_bytes + p.mask_bytes);
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
  s.maskbuf = maskbuf;
  s.extra_bytes = p.extra;
  s.ctr = ctr;
  s.trace = debug_trace();
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  const size_t smem = head_smem(p.hp.stages, p.hp.stage_bytes, B, c->d, esz, p.hp.lcap, p.extra).total;
  return c->dtype == DS_BF16 ? launch_step_t<__nv_bfloat16>(s, smem, p.hp.G, st, pdl)
                             : launch_step_t<float>(s, smem, p.hp.G, st, pdl);
}

}  // namespace ds
