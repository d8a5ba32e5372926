// cstep.cu — one DynaSpec draft step for a single row (B = 1) with the router computed per
// thread-block CLUSTER, so the step needs no grid-wide barrier before the head streams.
//
// Why: at B = 1 the step is latency-bound (P:283 T_D model; SURVEY §8(d) latency budget).  The
// grid-wide variant (step.cu) spends ~2 us on a global counter handshake between router layer 1
// and layer 2 and ~5 us on single-CTA layer 2 + TopK.  Here every cluster of Q CTAs (Q = 16 when
// the GPU fits it, one CTA per SM) evaluates the whole router r_theta([h_prev ‖ e]) (P:198-199,
// Alg. 1 line 8) by itself:
//   * CTA q streams rows [q h_r/Q, (q+1) h_r/Q) of W1 by TMA into its ring — issued before the
//     PDL wait, since router weights do not depend on the upstream kernel — and dots them with
//     [h_prev ‖ e] (each W1 row = two d-element halves, so a half is exactly one head row);
//   * hidden activations a = ReLU(W1 x + b1) are broadcast into every CTA of the cluster through
//     distributed shared memory (st.shared::cluster) + one hardware cluster barrier;
//   * CTA q computes the scores s_m = W2_m . a + b2_m of its slice of M and broadcasts them;
//   * CTA q ranks its own slice against all M scores (rank < k <=> in TopK_k under (score desc,
//     id asc), R7) and broadcasts the selected ids; every CTA then forms the ascending
//     selection and shortlist offsets (R8) locally.  The scores are bit-identical in every
//     cluster (same code, same order), so all clusters agree on the shortlist.
// The gathered head: CTA g streams segment g of the shortlist through the TMA ring of
// head_impl.cuh, its producer lane deriving the segment from the TopK mask (no block-wide prefix
// sum on the critical path); each consumer warp folds its logits into an online (max, sum exp) and a lane-distributed sorted
// top-k_t list while the next slots are in flight.  Lists are merged in two levels
// without float atomics (R19): the CTA's warps, then the last CTA to take the global ticket merges
// the G per-CTA records (CTA order).
#include <algorithm>
#include <stdlib.h>

#include "head_impl.cuh"
#include "internal.h"
#include "select_impl.cuh"
#include "keys.cuh"

namespace ds {

constexpr int kCStepMaxKt = 32;  // one list entry per lane

// Poll a record word until it is non-zero.  Bounded: a record that has not landed 2 s after the merger
// started (a CTA of this grid could not become resident, e.g. SMs held by a concurrent kernel) raises
// DS_ERR_DEVICE_TIMEOUT in the workspace error word and returns a placeholder instead of hanging.
__device__ __noinline__ unsigned long long cstep_poll(const unsigned long long* p, unsigned long long t0,
                                                      unsigned* err) {
  for (unsigned n = 1;; ++n) {
    const unsigned long long v = ld_relaxed_u64(p);
    if (v != 0ull) return v;
    if ((n & 255u) == 0u && globaltimer_ns() - t0 > 2000000000ull) {
      atomicExch(err, (unsigned)DS_ERR_DEVICE_TIMEOUT);
      return 1ull;
    }
  }
}

struct CStepArgs {
  HeadArgs h;              // head part; sel / sel_count / sl_off are redirected to shared memory
  const void* W1;          // [rows1][2d]
  const float* b1;         // [rows1]
  const void* W2;          // [M][h_r] (h_r > 0)
  const float* b2;         // [M]
  const void* h_prev;      // [d]
  const void* e;           // [d]
  float* scores;           // [M] (nullable)
  int32_t* sel_out;        // [M]
  int32_t* cnt_out;        // [1]
  int32_t* sloff_out;      // [M+1]
  int32_t h_r, rows1, k, extra_bytes;
  unsigned long long* crec;  // [G][2 + k_t] per-CTA records (max | sum, count + 1, k_t keys); 0 = not yet
                             // written (the merger zeroes them after reading)
  unsigned* ctr;             // workspace error word: DS_ERR_DEVICE_TIMEOUT when a record never lands
  unsigned long long* trace;
  int xs_slot;  // ring slot holding [h_prev ‖ e] (-1: a separate shared-memory region)
  int head_only;  // 1: S1-S3 ran elsewhere (dynaspec_step_route); the TopK comes from h.sel / h.sel_count
};

// Shared-memory carve-up (inside HeadSmem.extra).
struct CExtra {
  uint32_t xs, p1, a1, sc, w2s, b1s, b2s, offs, selb, xb, mask, sel, sloff, cnt, tmp, wm, ws, wl, total;
};
// xs_in_ring: [h_prev ‖ e] lives in a ring slot after the router rows (free until streaming starts)
__host__ __device__ inline CExtra cstep_extra(int d, int esz, int M, int h_r, int rows1, int Q, int K, int S, int C,
                                             int xs_in_ring) {
  CExtra X;
  uint32_t o = 0;
  auto take = [&](uint32_t bytes) {
    const uint32_t at = o;
    o = (o + bytes + 15u) & ~15u;
    return at;
  };
  const int U = (rows1 + Q - 1) / Q;
  const int Ms = h_r > 0 ? (M + Q - 1) / Q : 0;
  X.xs = take(xs_in_ring ? 0u : 2u * d * esz);
  X.p1 = take(4u * 2 * U);
  X.a1 = take(4u * (h_r > 0 ? h_r : 1));
  X.sc = take(4u * ((M + 3) & ~3));
  X.w2s = take((uint32_t)Ms * (h_r > 0 ? h_r : 0) * esz);
  X.b1s = take(4u * U);
  X.b2s = take(4u * (Ms > 0 ? Ms : 1));
  X.offs = take(4u * (M + 1));
  X.selb = take(4u * M);  // u32 TopK flags (st.async writes 4-byte words)
  X.xb = take(3 * 8);     // mbarriers of the three cluster exchanges
  X.mask = take(4u * 32);
  X.sel = take(4u * M);
  X.sloff = take(4u * (M + 1));
  X.cnt = take(16);
  X.tmp = take(4u * M);
  X.wm = take(4u * S);
  X.ws = take(4u * S);
  X.wl = take(16u * S * K);
  X.total = o;
  return X;
}

// Two staged rows against two (possibly different) vectors: lane-parallel fp32 partials + warp
// trees (R18), as dot2 in head_impl.cuh.
template <typename T>
__device__ __forceinline__ void dot2x(const T* __restrict__ w0, const T* __restrict__ w1, const T* __restrict__ x0,
                                      const T* __restrict__ x1, int d, int lane, float& z0, float& z1) {
  constexpr int E = Elem<T>::kPer16B;
  float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 2
  for (int c = lane * E; c < d; c += 32 * E) {
    float xf[E], yf[E], uf[E], vf[E];
    widen16(*reinterpret_cast<const uint4*>(w0 + c), xf, w0);
    widen16(*reinterpret_cast<const uint4*>(w1 + c), yf, w0);
    widen16(*reinterpret_cast<const uint4*>(x0 + c), uf, w0);
    widen16(*reinterpret_cast<const uint4*>(x1 + c), vf, w0);
#pragma unroll
    for (int j = 0; j < E; j += 2) {
      a0 = fmaf(xf[j], uf[j], a0);
      b0 = fmaf(yf[j], vf[j], b0);
      a1 = fmaf(xf[j + 1], uf[j + 1], a1);
      b1 = fmaf(yf[j + 1], vf[j + 1], b1);
    }
  }
  z0 = warp_sum(a0 + a1);
  z1 = warp_sum(b0 + b1);
}

// Producer lane: the CTA's share of the virtual shortlist (the selected clusters in ascending id,
// R8; |V_S| = sum of their sizes), streamed as chunks of at most `stage_rows` whole W_perm
// rows that never cross a cluster boundary.  Chunk c (in shortlist order) goes to CTA c mod G, so
// at any moment the grid reads one contiguous window of the shortlist: per-CTA stream times no
// longer depend on which address range a CTA was given (a contiguous per-CTA segment made the
// slowest CTA ~1.2x the mean, the slowness following the address range, not the SM).
// info = (-, virtual shortlist position, rows, first W_perm row).
template <typename T>
__device__ void cstep_produce(const HeadArgs& a, const HeadCtx& c, const uint32_t* mask, const int32_t* offs, int g,
                              int G, uint32_t it0) {
  if ((threadIdx.x & 31) != 0) return;
  const int words = (a.M + 31) >> 5;
  const uint64_t pol = policy_evict_first();
  const uint32_t rowbytes = (uint32_t)a.d * (uint32_t)sizeof(T);
  const uint8_t* W = static_cast<const uint8_t*>(a.W);
  const uint32_t S = (uint32_t)a.stages;
  const int R = a.stage_rows;
  uint32_t it = it0;
  long long vpos = 0;  // virtual position of the current cluster's first row
  long long cb = 0;    // global index of the current cluster's first chunk
  long long cn = g;    // next chunk this CTA streams
  for (int w = 0; w < words; ++w) {
    for (uint32_t bits = mask[w]; bits; bits &= bits - 1u) {
      const int m = (w << 5) + __ffs(bits) - 1;
      const int beg = offs[m], sz = offs[m + 1] - beg;
      const long long nch = (sz + R - 1) / R;
      for (; cn < cb + nch; cn += G) {
        const int j0 = (int)(cn - cb) * R;
        const int n = min(R, sz - j0);
        const uint32_t sl = it % S;
        mbar_wait(&c.empty[sl], ((it / S) & 1u) ^ 1u);
        c.info[sl] = make_int4(0, (int)(vpos + j0), n, beg + j0);
        mbar_arrive_expect_tx(&c.full[sl], (uint32_t)n * rowbytes);
        bulk_g2s(c.ring + (size_t)sl * a.stage_bytes, W + (size_t)(beg + j0) * rowbytes, (uint32_t)n * rowbytes,
                 &c.full[sl], pol);
        ++it;
      }
      cb += nch;
      vpos += sz;
    }
  }
  for (uint32_t j = 0; j < S; ++j, ++it) {  // one end-of-stream marker per slot
    const uint32_t sl = it % S;
    mbar_wait(&c.empty[sl], ((it / S) & 1u) ^ 1u);
    c.info[sl] = make_int4(-1, 0, -1, 0);
    mbar_arrive(&c.full[sl]);
  }
}

// Consumer warp `w` (ring slot w): gathered-head logits of the CTA's segment folded on the fly into
// (m, s) and the warp's sorted top-K list.
template <typename T>
__device__ __forceinline__ void cstep_consume(const HeadArgs& a, const HeadCtx& c, int w, int lane, uint32_t k0,
                                              float& m, float& s, unsigned long long& mine) {
  const T* hs = static_cast<const T*>(c.hs);
  const int K = a.k_t;
  unsigned long long kth = 0ull;
  m = -INFINITY;
  s = 0.f;
  mine = 0ull;
  for (uint32_t k = k0;; ++k) {
    mbar_wait(&c.full[w], k & 1u);
    const int4 inf = c.info[w];
    if (inf.z < 0) break;
    const T* st = reinterpret_cast<const T*>(c.ring + (size_t)w * a.stage_bytes);
    const long long zbase = inf.y;  // virtual shortlist position of the slot's first row
    for (int rr = 0; rr < inf.z; rr += 2) {
      const bool two = rr + 1 < inf.z;
      const int tok0 = __ldg(a.perm + inf.w + rr);
      const int tok1 = two ? __ldg(a.perm + inf.w + rr + 1) : 0;
      const T* w0 = st + (size_t)rr * a.d;
      float z0, z1;
      dot2<T>(w0, two ? w0 + a.d : w0, hs, a.d, lane, z0, z1);
      lse_push(m, s, z0);
      list_insert(mine, kth, tok_key(z0, tok0), K, lane);
      if (two) {
        lse_push(m, s, z1);
        list_insert(mine, kth, tok_key(z1, tok1), K, lane);
      }
      if (a.z_out && lane == 0) {
        a.z_out[zbase + rr] = z0;
        if (two) a.z_out[zbase + rr + 1] = z1;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&c.empty[w]);
  }
}

template <typename T>
__global__ void __launch_bounds__((kMaxStages + 1) * 32, 1) cstep_kernel(const CStepArgs s) {
  extern __shared__ __align__(1024) uint8_t smem[];
  HeadArgs a = s.h;
  const HeadSmem L = head_smem(a.stages, a.stage_bytes, 1, a.d, (int)sizeof(T), a.lcap, s.extra_bytes);
  const HeadCtx c = head_ctx(smem, L);
  constexpr int E = Elem<T>::kPer16B;
  const int Q = (int)cluster_nctarank(), q = (int)cluster_ctarank();
  const int cid = (int)cluster_id_x(), C = (int)cluster_count_x();
  const int M = a.M, d = a.d, K = a.k_t, S = a.stages;
  const CExtra X = cstep_extra(d, (int)sizeof(T), M, s.h_r, s.rows1, Q, K, S, C, s.xs_slot >= 0);
  uint8_t* ex = c.extra;
  T* xs = reinterpret_cast<T*>(s.xs_slot >= 0 ? c.ring + (size_t)s.xs_slot * a.stage_bytes : ex + X.xs);
  float* p1 = reinterpret_cast<float*>(ex + X.p1);
  float* a1 = reinterpret_cast<float*>(ex + X.a1);
  float* sc = reinterpret_cast<float*>(ex + X.sc);
  T* w2s = reinterpret_cast<T*>(ex + X.w2s);
  float* b1s = reinterpret_cast<float*>(ex + X.b1s);
  float* b2s = reinterpret_cast<float*>(ex + X.b2s);
  int32_t* offs = reinterpret_cast<int32_t*>(ex + X.offs);
  uint32_t* selb = reinterpret_cast<uint32_t*>(ex + X.selb);
  uint64_t* xb = reinterpret_cast<uint64_t*>(ex + X.xb);  // [0] a, [1] scores, [2] TopK flags
  uint32_t* mask = reinterpret_cast<uint32_t*>(ex + X.mask);
  int32_t* sel_s = reinterpret_cast<int32_t*>(ex + X.sel);
  int32_t* sloff_s = reinterpret_cast<int32_t*>(ex + X.sloff);
  int32_t* cnt_s = reinterpret_cast<int32_t*>(ex + X.cnt);
  int32_t* tmp = reinterpret_cast<int32_t*>(ex + X.tmp);
  float* wm = reinterpret_cast<float*>(ex + X.wm);
  float* wsum = reinterpret_cast<float*>(ex + X.ws);
  unsigned long long* wl = reinterpret_cast<unsigned long long*>(ex + X.wl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  uint64_t* xbar = c.full + 2 * kMaxStages;  // spare barrier slots: x + h_new, W2 slice
  uint64_t* wbar = xbar + 1;

  // this CTA's router rows (layer-1 units) and score slice
  const int u0 = s.rows1 * q / Q, u1 = s.rows1 * (q + 1) / Q, U = u1 - u0;
  const int nh = 2 * U;                                   // half rows of W1 (d elements each)
  const int n1 = (nh + a.stage_rows - 1) / a.stage_rows;  // ring loads of router rows
  const int ms0 = s.h_r > 0 ? M * q / Q : u0, ms1 = s.h_r > 0 ? M * (q + 1) / Q : u1;  // score slice
  const uint32_t hb = (uint32_t)d * (uint32_t)sizeof(T);
  const uint32_t w2_bytes = (uint32_t)(ms1 - ms0) * (uint32_t)(s.h_r > 0 ? s.h_r : 0) * (uint32_t)sizeof(T);

  if (threadIdx.x == 0) {
    head_init_barriers(c, S);
    mbar_init(xbar, 1);
    mbar_init(wbar, 1);
    // the three exchanges: each CTA expects every value of the cluster-wide vector (own included)
    for (int i = 0; i < 3; ++i) mbar_init(&xb[i], 1);
    mbar_arrive_expect_tx(&xb[0], 4u * (uint32_t)s.rows1);
    if (s.h_r > 0) mbar_arrive_expect_tx(&xb[1], 4u * (uint32_t)M);
    mbar_arrive_expect_tx(&xb[2], 4u * (uint32_t)s.k);  // exactly k ranks are < k (distinct keys)
    fence_mbar_init();
  }
  for (int m = threadIdx.x; m < M; m += blockDim.x) selb[m] = 0;
  if (threadIdx.x < 32) mask[threadIdx.x] = 0u;
  __syncthreads();
  cluster_arrive_relaxed();  // paired with the wait before the first DSMEM store (barrier inits are fenced)
  trace_mark(s.trace, 0);
  if (s.head_only) {
    // S1-S3 ran on S_m (dynaspec_step_route): the TopK mask from the selection in global memory
    if (warp == S && lane == 0) {
      mbar_arrive_expect_tx(xbar, hb);
      bulk_g2s(c.hs, a.h, hb, xbar, policy_evict_first());
    }
    // a row whose |V_S| exceeds max_shortlist is not computed (dynaspec.h): an empty mask streams
    // nothing, so the merger emits ids -1 and lse NaN
    const int cnt = __ldg(a.sel_count);
    const bool fits = cnt >= 1 && cnt <= M && (long long)__ldg(a.sl_off + cnt) <= a.max_shortlist;
    for (int i = threadIdx.x; fits && i < cnt; i += blockDim.x) {
      const int m = __ldg(a.sel + i);
      if (m >= 0 && m < M) atomicOr(&mask[m >> 5], 1u << (m & 31));
    }
    for (int m = threadIdx.x; m <= M; m += blockDim.x) offs[m] = __ldg(a.offsets + m);
    cluster_wait_acquire();  // pairs the launch-time arrive (a one-CTA cluster: no peer)
    mbar_wait(xbar, 0);
    __syncthreads();
  } else {
  if (warp == S) {
    if (lane == 0) {
      // router weights are constants: stream them before the PDL wait (W2 slice, then W1 rows)
      const uint64_t keep = policy_evict_last();
      if (w2_bytes > 0) {
        mbar_arrive_expect_tx(wbar, w2_bytes);
        bulk_g2s(w2s, static_cast<const T*>(s.W2) + (size_t)ms0 * s.h_r, w2_bytes, wbar, keep);
      }
      const uint8_t* src = static_cast<const uint8_t*>(s.W1) + (size_t)u0 * 2 * hb;
      auto issue = [&](int it) {
        const int sl = it % S;
        mbar_wait(&c.empty[sl], ((uint32_t)(it / S) & 1u) ^ 1u);
        const int j0 = it * a.stage_rows, n = min(a.stage_rows, nh - j0);
        c.info[sl] = make_int4(j0, 0, n, 0);
        mbar_arrive_expect_tx(&c.full[sl], (uint32_t)n * hb);
        bulk_g2s(c.ring + (size_t)sl * a.stage_bytes, src + (size_t)j0 * hb, (uint32_t)n * hb, &c.full[sl], keep);
      };
      const int first = min(n1, S);
      for (int it = 0; it < first; ++it) issue(it);
      // activations come from upstream kernels: x = [h_prev ‖ e] and h_new, one barrier
      if (a.pdl) pdl_wait();
      mbar_arrive_expect_tx(xbar, 3u * hb);
      const uint64_t stream = policy_evict_first();
      bulk_g2s(xs, s.h_prev, hb, xbar, stream);
      bulk_g2s(reinterpret_cast<uint8_t*>(xs) + hb, s.e, hb, xbar, stream);
      bulk_g2s(c.hs, a.h, hb, xbar, stream);
      for (int it = first; it < n1; ++it) issue(it);
    }
    __syncwarp();
  } else {
    const int tid = threadIdx.x, nt = S * 32;
    if (s.h_r > 0)
      for (int i = tid; i < ms1 - ms0; i += nt) b2s[i] = __ldg(s.b2 + ms0 + i);
    for (int i = tid; i < U; i += nt) b1s[i] = __ldg(s.b1 + u0 + i);
    for (int m = tid; m <= M; m += nt) offs[m] = __ldg(a.offsets + m);
    mbar_wait(xbar, 0);
    trace_mark(s.trace, 1);
    // router layer 1 on this CTA's rows: half row j dots h_prev (j even) or e (j odd) (R4)
    for (uint32_t kk = 0;; ++kk) {
      const int it = (int)kk * S + warp;
      if (it >= n1) break;
      mbar_wait(&c.full[warp], kk & 1u);
      const int4 inf = c.info[warp];
      const T* st = reinterpret_cast<const T*>(c.ring + (size_t)warp * a.stage_bytes);
      for (int rr = 0; rr < inf.z; rr += 2) {
        const int j = inf.x + rr;
        const bool two = rr + 1 < inf.z;
        const T* w0 = st + (size_t)rr * d;
        float z0, z1;
        dot2x<T>(w0, two ? w0 + d : w0, xs + (size_t)(j & 1) * d, xs + (size_t)((j + 1) & 1) * d, d, lane, z0, z1);
        if (lane == 0) {
          p1[j] = z0;
          if (two) p1[j + 1] = z1;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.empty[warp]);
    }
  }
  __syncthreads();  // p1 complete (the producer lane has issued every router row by now)
  trace_mark(s.trace, 2);
  cluster_wait_acquire();  // every CTA of the cluster is running: DSMEM stores are safe
  // a = ReLU(W1 x + b1) for this CTA's units -> a1[] of every CTA in the cluster (linear router:
  // the units are the scores themselves)
  {
    float* dstv = s.h_r > 0 ? a1 : sc;
    for (int t = threadIdx.x; t < U * Q; t += blockDim.x) {
      const int u = t / Q, dst = t - u * Q;
      const float z = (p1[2 * u] + p1[2 * u + 1]) + b1s[u];
      st_async_u32(mapa_u32(smem_u32(dstv + u0 + u), (uint32_t)dst), __float_as_uint(s.h_r > 0 ? fmaxf(z, 0.f) : z),
                   mapa_u32(smem_u32(&xb[0]), (uint32_t)dst));
    }
  }
  mbar_wait_cluster(&xb[0], 0);
  trace_mark(s.trace, 8);
  if (s.h_r > 0) {  // layer 2 on this CTA's score slice -> every CTA's sc[]
    if (w2_bytes > 0) mbar_wait(wbar, 0);
    // lanes per score: h_r / E chunks of 16 bytes, at most 32, a power of two
    int sub = 32;
    while (sub > 1 && sub * E > s.h_r) sub >>= 1;
    const int per_warp = 32 / sub, part = lane % sub, slot = lane / sub;
    for (int m = ms0 + warp * per_warp + slot; m - slot < ms1; m += nwarps * per_warp) {
      float acc = 0.f;
      if (m < ms1) {
        const T* w = w2s + (size_t)(m - ms0) * s.h_r;
        for (int j = part * E; j < s.h_r; j += sub * E) {
          float wf[E];
          widen16(*reinterpret_cast<const uint4*>(w + j), wf, w);
#pragma unroll
          for (int u = 0; u < E; ++u) acc = fmaf(wf[u], a1[j + u], acc);
        }
      }
      for (int o = sub >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (m < ms1) {
        acc += b2s[m - ms0];
        for (int dst = part; dst < Q; dst += sub)
          st_async_u32(mapa_u32(smem_u32(sc + m), (uint32_t)dst), __float_as_uint(acc),
                       mapa_u32(smem_u32(&xb[1]), (uint32_t)dst));
      }
    }
    mbar_wait_cluster(&xb[1], 0);
  }
  trace_mark(s.trace, 12);
  // TopK_k under (score desc, id asc) (R7): rank this CTA's slice against all M scores
  // (sub lanes per score), broadcast the winners' flags
  {
    const int nsl = ms1 - ms0;
    int sub = 32;
    while (sub > 1 && sub * nsl > (int)blockDim.x) sub >>= 1;
    const int groups = blockDim.x / sub;
    for (int i0 = 0; i0 < nsl; i0 += groups) {
      const int i = i0 + threadIdx.x / sub, part = threadIdx.x % sub;
      const bool act = i < nsl && (int)threadIdx.x < groups * sub;
      const int m = ms0 + i;
      const float key = act ? sc[m] + 0.0f : 0.f;
      int rank = 0;
      if (act)
        for (int j = part; j < M; j += sub) {
          const float o = sc[j] + 0.0f;
          rank += (o > key) | ((o == key) & (j < m));
        }
      for (int o = sub >> 1; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
      if (act && rank < s.k)
        for (int dst = part; dst < Q; dst += sub)
          st_async_u32(mapa_u32(smem_u32(selb + m), (uint32_t)dst), 1u, mapa_u32(smem_u32(&xb[2]), (uint32_t)dst));
    }
  }
  mbar_wait_cluster(&xb[2], 0);
  trace_mark(s.trace, 13);
  {
    const int Mr = (M + 31) & ~31;
    for (int m = threadIdx.x; m < Mr; m += blockDim.x) {
      const uint32_t b = __ballot_sync(0xffffffffu, m < M && selb[m] != 0);
      if (lane == 0) mask[m >> 5] = b;
    }
  }
  __syncthreads();
  }
  fence_proxy_async_smem();  // the ring was read by generic loads (W1 rows) before TMA reuses it
  trace_mark(s.trace, 4);
  if (warp == S) {
    cstep_produce<T>(a, c, mask, offs, (int)blockIdx.x, (int)gridDim.x, (uint32_t)(s.head_only ? 0 : n1));
  } else {  // logits folded into per-warp (m, s) + a sorted top-K list while the ring streams
    float m, se;
    unsigned long long mine;
    const int it0 = s.head_only ? 0 : n1;
    cstep_consume<T>(a, c, warp, lane, it0 > warp ? (uint32_t)((it0 - 1 - warp) / S + 1) : 0u, m, se, mine);
    if (lane < K) wl[warp * K + lane] = mine;
    if (lane == 0) {
      wm[warp] = m;
      wsum[warp] = se;
    }
  }
  __syncthreads();
  trace_mark(s.trace, 5);
  if (a.pdl) pdl_launch_dependents();
  const int G = (int)gridDim.x, g = (int)blockIdx.x, rec = 2 + K;
  // CTA record = (max, sum exp) of the CTA's logits + its K best keys, sorted.  One pass, no further
  // block barrier: thread i ranks warp-list entry i against all S K entries (keys are distinct;
  // 0 = empty) and writes it to its rank if that is < K; the ranks >= the number of valid keys are
  // padding (1, below every key: a key's low word ~id has bit 31 set).  Warp S (the producer, idle
  // now) folds the S warp (max, sum) pairs: max as an order-preserving integer, sums by a fixed xor
  // tree (R19).  Record words are never 0, so the merger polls the data itself: no fence, no ticket.
  {
    unsigned long long* my = s.crec + (size_t)g * rec;
    const int n = S * K, nr = S * 32;  // the consumer warps rank; warp S folds (max, sum)
    int P = 1;                         // lanes per key (a power of two: shallower loops)
    while (P < 8 && n * (P * 2) <= nr) P <<= 1;
    if (threadIdx.x < (unsigned)nr)
      for (int v0 = 0; v0 < n * P; v0 += nr) {  // uniform trip count: every lane shuffles
        const int v = v0 + threadIdx.x, i = v / P, part = v % P;
        const bool act = i < n;
        const unsigned long long x = act ? wl[i] : 0ull;
        int rk = 0, nv = 0;
        if (act)
#pragma unroll 4
          for (int j = part; j < n; j += P) {
            const unsigned long long y = wl[j];
            rk += y > x;
            nv += y != 0ull;
          }
        for (int o = P >> 1; o > 0; o >>= 1) {
          rk += __shfl_xor_sync(0xffffffffu, rk, o);
          nv += __shfl_xor_sync(0xffffffffu, nv, o);
        }
        if (act && part == 0) {
          if (x != 0ull && rk < K) my[2 + rk] = x;
          if (i < K && i >= nv) my[2 + i] = 1ull;  // padding (R17)
          if (i == 0) my[1] = (unsigned long long)min(nv, K) + 1ull;
        }
      }
    if (warp == S) {
      const bool has = lane < S;
      const float mw = has ? wm[lane] : -INFINITY;
      const uint32_t mk = __reduce_max_sync(0xffffffffu, mw > -INFINITY ? ord_key(mw) : 0u);
      const float Mx = mk ? __uint_as_float((mk & 0x80000000u) ? (mk & 0x7fffffffu) : ~mk) : -INFINITY;
      const float sum = warp_sum(has && mw > -INFINITY ? wsum[lane] * expf(mw - Mx) : 0.f);
      if (lane == 0)
        my[0] = (unsigned long long)__float_as_uint(Mx) | ((unsigned long long)__float_as_uint(sum) << 32);
    }
  }
  trace_mark(s.trace, 9);
  if (!s.head_only && g == G - 1) {  // the caller's copies of scores / selection / offsets (S3 outputs), off the merger CTA
    emit_fast(mask, M, offs, sel_s, cnt_s, sloff_s, tmp);
    __syncthreads();
    const int cnt = *cnt_s;
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      if (s.scores) s.scores[i] = sc[i];
      if (i < cnt) s.sel_out[i] = sel_s[i];
    }
    for (int i = threadIdx.x; i <= cnt; i += blockDim.x) s.sloff_out[i] = sloff_s[i];
    if (threadIdx.x == 0) *s.cnt_out = cnt;
  }
  if (g != 0) return;

  // Merger (CTA 0).  (1) every thread polls record words (coalesced) until they land, staging them
  // in shared memory (record heads also contiguously) and folding max m_g as an order-preserving
  // integer.  (2) thread g ranks head g among the G heads: with r_g heads above it, key j of record
  // g has at least r_g + j keys above it (records are sorted), so only keys j < K - r_g can be in
  // the global top-K (every global top-K member is in its CTA's record) — at most K (K + 1) / 2
  // candidates; the same threads form the lse partials s_g e^{m_g - M} (fixed xor trees, R19).
  // (3) thread per candidate: rank, outputs.  Two block barriers.  Scratch: the ring.
  unsigned long long* raw = reinterpret_cast<unsigned long long*>(c.ring);  // [G][rec] the records
  unsigned long long* fsurv = raw + (size_t)G * rec;                       // [G*K] candidates
  const int G4 = (G + 3) & ~3;
  uint32_t* hh = reinterpret_cast<uint32_t*>(fsurv + (((size_t)G * K + 1) & ~(size_t)1));  // [G4] heads' high words (16 B aligned)
  int* fc = reinterpret_cast<int*>(hh + G4);                               // [G] valid keys per record
  float* fm = reinterpret_cast<float*>(fc + G);                            // [G]
  float* fs = fm + G;                                                      // [G]
  float* wps = fs + G;                                                     // [32] warp partial sums
  unsigned* sh = reinterpret_cast<unsigned*>(wps + 32);                    // [0] count [1] max key
  if (threadIdx.x == 0) {
    sh[0] = 0u;
    sh[1] = 0u;
  }
  for (int i = G + threadIdx.x; i < G4; i += blockDim.x) hh[i] = 0u;
  {  // (1a) stage the record words as they land (coalesced; small code: the fields are decoded once below)
    constexpr int kB = 8;
    const int nrec = G * rec, nt = blockDim.x;
    const unsigned long long t0 = globaltimer_ns();
    for (int i0 = threadIdx.x; i0 < nrec; i0 += kB * nt) {
      unsigned long long v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) v[u] = i0 + u * nt < nrec ? __ldcg(s.crec + i0 + u * nt) : 1ull;
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (v[u] == 0ull) v[u] = cstep_poll(s.crec + i0 + u * nt, t0, s.ctr);  // not written yet: poll L2
        if (i0 + u * nt < nrec) raw[i0 + u * nt] = v[u];
      }
    }
  }
  __syncthreads();
  // every record word is in shared memory: zero them for the next launch now (off the output path)
  for (int i = threadIdx.x; i < G * rec; i += blockDim.x) s.crec[i] = 0ull;
  {  // (1b) thread g: record g's (max, sum), valid count, head; the max over records
    unsigned mymk = 0u;
    for (int g2 = threadIdx.x; g2 < G; g2 += blockDim.x) {
      const unsigned long long w0 = raw[(size_t)g2 * rec], hd = raw[(size_t)g2 * rec + 2];
      const float m = __uint_as_float((uint32_t)w0);
      fm[g2] = m;
      fs[g2] = __uint_as_float((uint32_t)(w0 >> 32));
      fc[g2] = (int)raw[(size_t)g2 * rec + 1] - 1;
      hh[g2] = hd > 1ull ? (uint32_t)(hd >> 32) : 0u;
      if (m > -INFINITY) mymk = max(mymk, ord_key(m));
    }
    mymk = __reduce_max_sync(0xffffffffu, mymk);
    if (lane == 0 && mymk) atomicMax(&sh[1], mymk);
  }
  __syncthreads();
  trace_mark(s.trace, 14);
  const uint32_t Mk = sh[1];
  const float Mx = Mk ? __uint_as_float((Mk & 0x80000000u) ? (Mk & 0x7fffffffu) : ~Mk) : -INFINITY;
  {
    float part = 0.f;
    for (int t = threadIdx.x; t < G; t += blockDim.x) {
      // r = heads with a strictly larger logit (<= heads above head t: a valid count)
      const uint32_t h = hh[t];
      const uint4* h4 = reinterpret_cast<const uint4*>(hh);
      int r = 0;
#pragma unroll 4
      for (int j = 0; j < G4 / 4; ++j) {
        const uint4 q = h4[j];
        r += (int)(q.x > h) + (int)(q.y > h) + (int)(q.z > h) + (int)(q.w > h);
      }
      const int ne = min(K - r, fc[t]);
      if (ne > 0) {
        const int base = (int)atomicAdd(&sh[0], (unsigned)ne);
        for (int j = 0; j < ne; ++j) fsurv[base + j] = raw[(size_t)t * rec + 2 + j];
      }
      if (fm[t] > -INFINITY) part += fs[t] * expf(fm[t] - Mx);
    }
    part = warp_sum(part);  // sum_g s_g e^{m_g - M}: xor tree per warp, then the warps in order
    if (lane == 0) wps[warp] = part;
  }
  __syncthreads();
  trace_mark(s.trace, 15);
  const int ns = (int)sh[0];
  const bool ok = Mx > -INFINITY;
  float sum = 0.f;
  for (int w2 = 0; w2 < nwarps; ++w2) sum += wps[w2];
  const float lse = ok ? Mx + logf(sum) : __int_as_float(0x7fc00000);
  {
    int P = 1;  // lanes per candidate
    while (P < 8 && ns * (P * 2) <= (int)blockDim.x) P <<= 1;
    const int nrk = ((int)blockDim.x / 32) * 32;
    for (int v0 = 0; v0 < ns * P; v0 += nrk) {  // uniform trip count: every lane shuffles
      const int v = v0 + threadIdx.x, i = v / P, part = v % P;
      const bool act = i < ns;
      const unsigned long long x = act ? fsurv[i] : 0ull;
      int rk = 0;
      if (act)
#pragma unroll 4
        for (int j = part; j < ns; j += P) rk += fsurv[j] > x;
      for (int o = P >> 1; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
      if (act && part == 0 && rk < K) {
        const float z = key_value(x);
        a.top_ids[rk] = key_id(x);
        a.top_logits[rk] = z;
        a.top_logp[rk] = z - lse;
      }
    }
  }
  for (int r = ns + threadIdx.x; r < K; r += blockDim.x) {  // fewer valid keys than K: padding (R17)
    a.top_ids[r] = -1;
    a.top_logits[r] = -INFINITY;
    a.top_logp[r] = -INFINITY;
  }
  if (threadIdx.x == 0) a.lse[0] = lse;
  trace_mark(s.trace, 7);
}

// ------------------------------------------------------------------ host side

// Cluster size: DS_CLUSTER_Q (0 disables the cluster step), default 16 (non-portable; one cluster
// per GPC).  Clusters per launch: the hardware's co-residency limit at one CTA per SM.
// Cluster size: DS_CLUSTER_Q if set (0 disables the cluster step; 1: every CTA evaluates the whole
// router alone, no exchanges — measured slower even for the Tiny router, 16.96 vs 14.56 us, the
// 148 CTAs each pulling W1 from L2), default 16 (each CTA holds 1/16 of W1).
static int cluster_q(const ds_clusters*, const ds_router*) {
  const char* v = getenv("DS_CLUSTER_Q");
  if (v && v[0]) return atoi(v);
  return 16;
}

template <typename T>
static cudaError_t cstep_configure() {
  static int done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(cstep_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem_optin());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(cstep_kernel<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  done[dev] = 1;
  return cudaSuccess;
}

static int max_clusters(int Q) {
  static int cache[64][33];
  static bool init = false;
  if (!init) {
    for (auto& row : cache)
      for (int& x : row) x = -1;
    init = true;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || Q < 1 || Q > 32) return 0;
  if (cache[dev][Q] >= 0) return cache[dev][Q];
  int n = 0;
  if (cstep_configure<__nv_bfloat16>() == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(Q);
    cfg.blockDim = dim3((kMaxStages + 1) * 32);
    cfg.dynamicSmemBytes = max_smem_optin();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, cstep_kernel<__nv_bfloat16>, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();  // a refused query leaves no sticky error
  cache[dev][Q] = n;
  return n;
}

struct CStepPlan {
  HeadPlan hp;
  int Q, C, extra, rows1, xs_slot;
  size_t smem, total;
};

static bool cstep_plan(const ds_clusters* c, const ds_router* r, int B, int k_t, int64_t max_shortlist, int shared,
                       CStepPlan* p) {
  // r == nullptr: head-only launch (the selection comes from dynaspec_step_route): one CTA per SM,
  // no cluster exchanges
  if (B != 1 || shared || k_t > kCStepMaxKt) return false;
  const int Q = r ? cluster_q(c, r) : 1;
  if (r && (Q < 1 || Q > 16)) return false;
  const int C = max_clusters(Q);
  if (C < 1 || C * Q < 64) return false;  // too few SMs would stream the head slowly
  p->Q = Q;
  p->C = C;
  const int h_r = r ? r->h_r : 0;
  p->rows1 = r ? (r->h_r > 0 ? r->h_r : r->M) : 0;
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  const int x0 = (int)cstep_extra(c->d, esz, c->M, h_r, p->rows1, Q, k_t, kMaxStages, C, 0).total;
  if (!head_plan_ex(c, 1, k_t, max_shortlist, x0, 1, &p->hp, C * Q)) return false;
  // logits never touch shared memory here (online per-warp state): no per-CTA logit buffer, and
  // the freed bytes go back to the ring
  p->hp.lcap = 0;
  const int smax = max_smem_optin();
  // router rows per CTA occupy ring slots [0, n1); [h_prev ‖ e] takes the next slot(s) if free
  const int n1 = (2 * ((p->rows1 + Q - 1) / Q) + p->hp.stage_rows - 1) / p->hp.stage_rows;
  const int xs_slots = (int)((2 * (size_t)c->d * esz + p->hp.stage_bytes - 1) / p->hp.stage_bytes);
  // at most 11 ring slots: measured at Llama-3 (k = 32,32,8x6), us/step by slots 8..12 =
  // 24.3, 23.8, 23.4, 22.9, 23.4 (scripts/variants.sh DS_CSTEP_STAGES=n)
  const char* sv = getenv("DS_CSTEP_STAGES");
  const int smax_st = sv && sv[0] ? std::max(2, std::min(kMaxStages, atoi(sv))) : std::min(kMaxStages, 11);
  for (int st = smax_st; st >= 2; --st) {
    const int alias = n1 + xs_slots <= st;
    const int xb = (int)cstep_extra(c->d, esz, c->M, h_r, p->rows1, Q, k_t, st, C, alias).total;
    const size_t sm = head_smem(st, p->hp.stage_bytes, 1, c->d, esz, 0, xb).total;
    if (sm <= (size_t)smax) {
      p->xs_slot = alias ? n1 : -1;
      p->hp.stages = st;
      p->extra = xb;
      p->smem = sm;
      break;
    }
    if (st == 2) return false;
  }
  // the last CTA merges the G records inside its ring
  const size_t G = (size_t)C * Q;
  if (G * (8 * (2 + k_t) + 8 * k_t + 20) + 1024 > (size_t)p->hp.stages * p->hp.stage_bytes) return false;
  if (G * (2 + k_t) * sizeof(unsigned long long) > kWsGstepRec - kWsCstepRec) return false;  // the record region
  p->total = kWsFixed;
  return true;
}

bool cstep_supported(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared, int64_t max_shortlist) {
  CStepPlan p;
  return cstep_plan(c, r, B, k_t, max_shortlist, shared, &p);
}

size_t cstep_ws_bytes(const ds_clusters* c, const ds_router* r, int B, int k_t) {
  CStepPlan p;
  return cstep_plan(c, r, B, k_t, 0, 0, &p) ? p.total : 0;
}

template <typename T>
static cudaError_t launch_cstep_t(const CStepArgs& s, size_t smem, int Q, int C, cudaStream_t st, bool pdl) {
  cudaError_t e = cstep_configure<T>();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * Q);
  cfg.blockDim = dim3((s.h.stages + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Q;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, cstep_kernel<T>, s);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cudaError_t launch_cstep(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                         const void* h_new, int k, int k_t, int64_t max_shortlist, float* scores, int32_t* sel,
                         int32_t* sel_count, int32_t* sl_offsets, int32_t* top_ids, float* top_logits,
                         float* top_logp, float* lse, float* z_out, int64_t z_stride, void* ws, cudaStream_t st,
                         bool pdl) {
  CStepPlan p;
  if (!cstep_plan(c, r, 1, k_t, max_shortlist, 0, &p)) return cudaErrorInvalidValue;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  CStepArgs s;
  fill_head_args(s.h, c, p.hp, h_new, 0, 1, sel, sel_count, sl_offsets, 0, k_t, max_shortlist, top_ids, top_logits,
                 top_logp, lse, z_out, z_stride, nullptr, reinterpret_cast<unsigned*>(w8), pdl);
  s.W1 = r->W1;
  s.b1 = r->b1;
  s.W2 = r->W2;
  s.b2 = r->b2;
  s.h_prev = h_prev;
  s.e = e;
  s.scores = scores;
  s.sel_out = sel;
  s.cnt_out = sel_count;
  s.sloff_out = sl_offsets;
  s.h_r = r->h_r;
  s.rows1 = p.rows1;
  s.k = k;
  s.extra_bytes = p.extra;
  s.xs_slot = p.xs_slot;
  s.head_only = 0;
  s.crec = reinterpret_cast<unsigned long long*>(w8 + kWsCstepRec);
  s.ctr = reinterpret_cast<unsigned*>(w8 + kWsErrorWord);
  s.trace = debug_trace();
  return c->dtype == DS_BF16 ? launch_cstep_t<__nv_bfloat16>(s, p.smem, p.Q, p.C, st, pdl)
                             : launch_cstep_t<float>(s, p.smem, p.Q, p.C, st, pdl);
}

// Head-only cluster-kernel launch (P:262-264 after S1-S3 on S_m): B = 1, the selection in sel /
// sel_count (device), records in `rec` (zero-filled once; left zeroed).
bool cstep_head_supported(const ds_clusters* c, int k_t, int64_t max_shortlist) {
  CStepPlan p;
  const char* v = getenv("DS_CSTEP_HEAD");
  if (v && v[0] == '0') return false;
  return cstep_plan(c, nullptr, 1, k_t, max_shortlist, 0, &p);
}

size_t cstep_head_rec_bytes(const ds_clusters* c, int k_t) {
  CStepPlan p;
  return cstep_plan(c, nullptr, 1, k_t, 0, 0, &p) ? p.total : 0;
}

cudaError_t launch_cstep_head(const ds_clusters* c, const void* h_new, const int32_t* sel, const int32_t* sel_count,
                              const int32_t* sl_offsets, int k_t, int64_t max_shortlist, int32_t* top_ids,
                              float* top_logits, float* top_logp, float* lse, float* z_out, int64_t z_stride,
                              void* ws, cudaStream_t st) {
  CStepPlan p;
  if (!cstep_plan(c, nullptr, 1, k_t, max_shortlist, 0, &p)) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(h_new) & 15u) != 0) return cudaErrorInvalidValue;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  CStepArgs s = {};
  fill_head_args(s.h, c, p.hp, h_new, 0, 1, sel, sel_count, sl_offsets, 0, k_t, max_shortlist, top_ids, top_logits,
                 top_logp, lse, z_out, z_stride, nullptr, reinterpret_cast<unsigned*>(w8), false);
  s.k = 1;
  s.extra_bytes = p.extra;
  s.xs_slot = p.xs_slot;
  s.head_only = 1;
  s.crec = reinterpret_cast<unsigned long long*>(w8 + kWsCstepRec);
  s.ctr = reinterpret_cast<unsigned*>(w8 + kWsErrorWord);
  s.trace = debug_trace();
  return c->dtype == DS_BF16 ? launch_cstep_t<__nv_bfloat16>(s, p.smem, p.Q, p.C, st, false)
                             : launch_cstep_t<float>(s, p.smem, p.Q, p.C, st, false);
}

bool cstep_pointers_ok(const ds_router* r, const void* h_prev, const void* e, const void* h_new) {
  return aligned16(h_prev) && aligned16(e) && aligned16(h_new) && aligned16(r->W1) &&
         (r->h_r == 0 || aligned16(r->W2));
}

}  // namespace ds
