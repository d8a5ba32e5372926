// common.cuh — device helpers shared by the DynaSpec sm_100a kernels (product path only).
// PTX wrappers for mbarrier / bulk async copy (TMA 1D) / PDL, warp reductions, total orders.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dynaspec.h"
#include "internal.h"

namespace ds {

// ------------------------------------------------------------------ dtype helpers
template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> { static constexpr int kPer16B = 8; };
template <> struct Elem<float> { static constexpr int kPer16B = 4; };

// Widen 16 bytes of T into fp32 values (bf16 -> f32 is exact: the bf16 bits are the top half).
__device__ __forceinline__ void widen16(const uint4& v, float* out, const __nv_bfloat16*) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ void widen16(const uint4& v, float* out, const float*) {
  out[0] = __uint_as_float(v.x);
  out[1] = __uint_as_float(v.y);
  out[2] = __uint_as_float(v.z);
  out[3] = __uint_as_float(v.w);
}

// Order-preserving map float -> uint32 (larger float => larger key); -0 folded into +0 (R23).
__device__ __forceinline__ uint32_t ord_key(float x) {
  const uint32_t u = __float_as_uint(x + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ------------------------------------------------------------------ warp reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// (value desc, id asc) total order used for token top-k (R7): a beats b?
__device__ __forceinline__ bool beats(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}
// Warp-wide argmax under `beats`; every lane returns the winner.
__device__ __forceinline__ void warp_best(float& v, int& id, int& aux) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, id, o);
    int a2 = __shfl_xor_sync(0xffffffffu, aux, o);
    if (beats(v2, i2, v, id)) { v = v2; id = i2; aux = a2; }
  }
}

// ------------------------------------------------------------------ shared-memory / mbarrier PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Request [src, src + bytes) into L2 (bytes a multiple of 16, src 16-byte aligned); no completion.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// Non-blocking probe (test_wait never suspends the thread; try_wait may, for a time limit).
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// L2 eviction-priority policies for bulk copies.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 16-byte global load that keeps the line in L2 (router weights: reused by every draft step).
__device__ __forceinline__ uint4 ld_evict_last_v4(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
// TMA 1D bulk copy global -> shared, completion signalled as tx bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Programmatic dependent launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ float ld_cg_f32(const float* p) { return __ldcg(p); }

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Opt-in phase trace (dynaspec_debug_set_trace): [cta][slot] nanosecond timestamps.
__device__ __forceinline__ void trace_mark(unsigned long long* t, int slot) {
  if (t != nullptr && threadIdx.x == 0) {
    t[blockIdx.x * 64 + 32 + slot] = clock64();  // SM clock first: the %globaltimer read is not free
    t[blockIdx.x * 64 + slot] = globaltimer_ns();
    if (slot == 0) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      t[blockIdx.x * 64 + 31] = sm + 1u;  // trace slot 31: SM id + 1
      t[blockIdx.x * 64 + 30] = blockDim.x;  // trace slot 30: threads per CTA
    }
  }
}

// Same, from lane 0 of the calling warp (for code that only one warp of the CTA still runs).
__device__ __forceinline__ void trace_mark_w(unsigned long long* t, int slot) {
  if (t != nullptr && (threadIdx.x & 31) == 0) {
    t[blockIdx.x * 64 + slot] = globaltimer_ns();
    t[blockIdx.x * 64 + 32 + slot] = clock64();
  }
}

// Spin (one thread) until *ctr >= target, then acquire.
__device__ __forceinline__ void spin_until_geq(const unsigned* ctr, unsigned target) {
  while (ld_volatile_u32(ctr) < target) {
    __nanosleep(20);
  }
  __threadfence();
}

// Exclusive scan of one int per thread over the whole block (any blockDim multiple of 32, <= 1024).
__device__ __forceinline__ int block_excl_scan_dyn(int v, int* scratch /* >= 33 ints */, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < nw) ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) scratch[lane] = w;
  }
  __syncthreads();
  const int base = warp > 0 ? scratch[warp - 1] : 0;
  total = scratch[nw - 1];
  __syncthreads();
  return base + x - v;
}

// ------------------------------------------------------------------ block scan (int), blockDim = NT
// Exclusive scan of one value per thread; returns the exclusive prefix, writes the total.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* scratch /* >= NT/32 + 1 ints */, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < NT / 32) ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) scratch[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int base = warp > 0 ? scratch[warp - 1] : 0;
  total = scratch[NT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

}  // namespace ds

namespace ds {
// Release / acquire at GPU scope (lighter than the sequentially consistent __threadfence()).
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// One thread: publish this CTA's prior writes (ordered before it by a __syncthreads) and count.
__device__ __forceinline__ unsigned release_add(unsigned* ctr, unsigned v) {
  fence_acq_rel_gpu();
  return atomicAdd(ctr, v);
}
// One thread: wait until *ctr >= target with acquire semantics.
__device__ __forceinline__ void acquire_wait_geq(const unsigned* ctr, unsigned target) {
  while (ld_acquire_u32(ctr) < target) {
  }
  fence_acq_rel_gpu();
}
}  // namespace ds

namespace ds {
// Block-wide top-K of n items under (value desc, id asc) without a full O(n^2) rank:
//   T0 = the K-th best of the first S = min(n, max(64, 4K)) items (the K-th best of a subset is
//        never better than the K-th best of the whole set, so every member of the true top-K is
//        >= T0);  survivors = items not beaten by T0;  rank-count the survivors only.
// get(i) -> (v, id) for i < n (items with v == -inf are ignored); emit(rank, v, id) is called
// once for each rank < min(K, #valid items).  sv / si: smem scratch for up to n survivors.
// misc: 3 ints of smem.  All threads of the block must call it.
template <class Get, class Emit>
__device__ __forceinline__ void block_topk(int n, int K, Get get, Emit emit, float* sv, int* si, int* misc) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  const int S = min(n, max(64, 4 * K));
  if (tid == 0) {
    misc[0] = 0;
    misc[1] = __float_as_int(-INFINITY);
    misc[2] = INT_MAX;
  }
  __syncthreads();
  // rank of item i among the first S items, split over `sp` lanes (shallower chains)
  {
    int sp = 32;
    while (sp > 1 && S * sp > nt) sp >>= 1;
    const int groups = nt / sp;
    for (int base = 0; base < S; base += groups) {
      const int i = base + tid / sp, part = tid % sp;
      float v = -INFINITY;
      int id = INT_MAX;
      if (i < S && tid < groups * sp) get(i, v, id);
      int rank = 0;
      if (v > -INFINITY)
        for (int j = part; j < S; j += sp) {
          float v2;
          int id2;
          get(j, v2, id2);
          rank += beats(v2, id2, v, id);
        }
      for (int o = sp >> 1; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
      if (part == 0 && v > -INFINITY && rank == K - 1) {
        misc[1] = __float_as_int(v);
        misc[2] = id;
      }
    }
  }
  __syncthreads();
  const float tv = __int_as_float(misc[1]);
  const int tid0 = misc[2];
  for (int i0 = 0; i0 < n; i0 += nt) {
    const int i = i0 + tid;
    float v = -INFINITY;
    int id = INT_MAX;
    if (i < n) get(i, v, id);
    const bool keep = v > -INFINITY && !beats(tv, tid0, v, id);
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    int slot0 = 0;
    if (lane == 0 && bal) slot0 = atomicAdd(&misc[0], __popc(bal));
    slot0 = __shfl_sync(0xffffffffu, slot0, 0);
    if (keep) {
      const int slot = slot0 + __popc(bal & ((1u << lane) - 1u));
      sv[slot] = v;
      si[slot] = id;
    }
  }
  __syncthreads();
  const int ns = misc[0];
  {
    int sp = 32;
    while (sp > 1 && ns * sp > nt) sp >>= 1;
    const int groups = nt / sp;
    for (int base = 0; base < ns; base += groups) {
      const int s2 = base + tid / sp, part = tid % sp;
      const bool active = s2 < ns && tid < groups * sp;
      const float v = active ? sv[s2] : -INFINITY;
      const int id = active ? si[s2] : INT_MAX;
      int rank = 0;
      if (active)
        for (int t = part; t < ns; t += sp) rank += beats(sv[t], si[t], v, id);
      for (int o = sp >> 1; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
      if (active && part == 0 && rank < K) emit(rank, v, id);
    }
  }
  __syncthreads();
}

// Online-softmax pair combine: (m1, s1) + (m2, s2) -> (max, s1 e^{m1-M} + s2 e^{m2-M}).
__device__ __forceinline__ void lse_combine(float& m, float& s, float m2, float s2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    s = s2;
    return;
  }
  const float M = fmaxf(m, m2);
  s = s * expf(m - M) + s2 * expf(m2 - M);
  m = M;
}
// Block-wide (max, sum) combine with a fixed order (warp trees, then warps in index order).
__device__ __forceinline__ void block_lse(float& m, float& s, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_combine(m, s, m2, s2);
  }
  __syncthreads();
  if (lane == 0) {
    red[2 * warp] = m;
    red[2 * warp + 1] = s;
  }
  __syncthreads();
  m = red[0];
  s = red[1];
  for (int w = 1; w < nw; ++w) lse_combine(m, s, red[2 * w], red[2 * w + 1]);
}
}  // namespace ds

namespace ds {
// Warp-level counterpart of block_topk (one warp, no block barriers): pruned rank count.
// sv / si: this warp's smem scratch (>= n entries).  Returns the number of survivors.
template <class Get, class Emit>
__device__ __forceinline__ int warp_topk(int n, int K, Get get, Emit emit, float* sv, int* si) {
  const int lane = threadIdx.x & 31;
  const int S = min(n, max(32, 2 * K));
  float tv = -INFINITY;
  int tid0 = INT_MAX;
  bool found = false;
  for (int i = lane; i < S; i += 32) {
    float v;
    int id;
    get(i, v, id);
    if (v == -INFINITY) continue;
    int rank = 0;
    for (int j = 0; j < S; ++j) {
      float v2;
      int id2;
      get(j, v2, id2);
      rank += beats(v2, id2, v, id);
    }
    if (rank == K - 1) {
      tv = v;
      tid0 = id;
      found = true;
    }
  }
  const uint32_t who = __ballot_sync(0xffffffffu, found);
  if (who) {
    const int src = __ffs(who) - 1;
    tv = __shfl_sync(0xffffffffu, tv, src);
    tid0 = __shfl_sync(0xffffffffu, tid0, src);
  }
  int base = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    float v = -INFINITY;
    int id = INT_MAX;
    if (i < n) get(i, v, id);
    const bool keep = v > -INFINITY && !beats(tv, tid0, v, id);
    const uint32_t b = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int pos = base + __popc(b & ((1u << lane) - 1u));
      sv[pos] = v;
      si[pos] = id;
    }
    base += __popc(b);
  }
  __syncwarp();
  for (int s2 = lane; s2 < base; s2 += 32) {
    const float v = sv[s2];
    const int id = si[s2];
    int rank = 0;
    for (int t = 0; t < base; ++t) rank += beats(sv[t], si[t], v, id);
    if (rank < K) emit(rank, v, id);
  }
  __syncwarp();
  return base;
}

// Warp-level (max, sum exp(z - max)) of z[0..n).
__device__ __forceinline__ void warp_lse_items(const float* z, int n, float& m, float& s) {
  const int lane = threadIdx.x & 31;
  m = -INFINITY;
  s = 0.f;
  for (int j = lane; j < n; j += 32) {
    const float x = z[j];
    if (x == -INFINITY) continue;  // masked (not in this row's shortlist)
    if (x > m) {
      s = s * expf(m - x) + 1.f;
      m = x;
    } else {
      s += expf(x - m);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_combine(m, s, m2, s2);
  }
}
}  // namespace ds

namespace ds {
// ------------------------------------------------------------------ thread-block clusters (DSMEM)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// Address of the same shared-memory variable in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// 4-byte store into a cluster peer's shared memory that completes `bytes` = 4 on the peer's
// mbarrier (the receiver waits for the bytes it expects; no cluster-wide barrier).
__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
               "r"(rbar)
               : "memory");
}
// Wait for a phase of a local mbarrier completed by peers' st.async (cluster-scope acquire).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Cluster barrier (every thread of every CTA of the cluster; warp-converged).
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
}  // namespace ds

namespace ds {
// 64-bit store visible at GPU scope (one word: value and its "written" tag land together).
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// 16-byte read-only global load (inputs that no kernel writes while this one runs).
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
}  // namespace ds
