// gstep.cu — one DynaSpec draft step for a single row (B = 1) on the WHOLE grid: one CTA per SM,
// no thread-block clusters, no counters, one launch per draft position.
//
// Why (SURVEY §8(d) latency budget; P:283 T_D model): at B = 1 a step moves 33-131 MB of cluster
// blocks, 5-20 us at HBM speed, so every microsecond of fixed latency shows.  The cluster step
// (cstep.cu) evaluates the router once per 16-CTA cluster and streams on 112 SMs; its three DSMEM
// exchanges and its record merge cost ~7 us per step.  Here:
//   * Router layer 1 (Alg. 1 line 8): CTA g owns hidden unit(s) u = g, g + G of
//     a = ReLU(W1 [h_prev ‖ e] + b1) (R4, R5).  Its W1 row(s) are loaded into REGISTERS before the PDL
//     wait (router weights do not depend on the upstream kernel); after the wait every thread loads
//     its 16-byte chunks of x and the CTA reduces one dot product of 2d terms.  The unit value is
//     published as ONE 64-bit word (1 << 32 | bits(a_u)) — value and "written" tag land together,
//     so no fence and no counter are needed; a word is 0 until written (the merger zeroes the words
//     after every CTA has read them).
//   * Every CTA polls the h_r words, then evaluates layer 2 s = W2 a + b2 for ALL M clusters from its
//     own registers (W2 slice per lane loaded before the wait; a fixed reduction order, so every CTA
//     holds bit-identical scores) and TopK_k (R7) as a pruned rank count: T = the
//     smallest of the per-warp q-th best keys (q = ceil(k / key warps)) is below the k-th best key, so
//     only keys >= T are rank-counted.  No CTA waits for another after this point except the merger.
//   * The gathered head streams the shortlist (selected clusters ascending, R8) as chunks of
//     <= 16 KB whole W_perm rows that never cross a cluster; chunk c goes to CTA c mod G (all SMs),
//     through a TMA bulk-copy ring (one producer lane, one consumer warp per slot); each consumer
//     warp folds its logits into an online (max, sum exp) and a lane-distributed sorted top-k_t list
//      while the next slots are in flight.
//   * CTA record = (max, sum) + its k_t best keys: entry r of warp list w has rank r + sum over the
//     other lists of (#entries above it), a binary search each.  Record words are never 0, so CTA 0
//     (the merger) polls the data itself and merges the G records in CTA order (R19).
// Every spin is bounded (kSpinNs): a CTA that never arrives (e.g. a concurrent kernel holding SMs)
// raises DS_ERR_DEVICE_TIMEOUT in the workspace error word instead of hanging the GPU.
#include <algorithm>
#include <stdlib.h>

#include "head_impl.cuh"
#include "internal.h"
#include "keys.cuh"
#include "select_impl.cuh"

// The once-per-launch phases are inlined: a call costs ~400 cycles per phase here (measured with
// scripts/probe/phase_bench.cu), more than the instruction-fetch misses the larger body adds.
#ifndef DS_GSTEP_NOINLINE
#define DS_GSTEP_NOINLINE __forceinline__
#endif

namespace ds {

constexpr int kGWarps = 16;
constexpr int kGThreads = 32 * kGWarps;
constexpr int kGProducer = kGWarps - 1;  // warp 15: TMA producer (its lane 0)
constexpr int kGSlots = 12;              // ring slots == consumer warps 0..S-1 (S <= 12 < 15)
constexpr int kGUnits = 2;               // router layer-1 units per CTA
constexpr int kGXChunks = 4;             // 16-byte chunks of x = [h_prev ‖ e] per thread
constexpr int kGRows2 = 16;              // layer-2 rows per warp (M <= 256), 2 column words per lane:
                                         //   h_r <= 128 (bf16) / 64 (fp32)
constexpr int kGMaxM = kGWarps * kGRows2;
constexpr int kGHeadsPerLane = 5;       // merger: record headers per polling lane (G <= 160)
constexpr int kGKeyWarps = 8;
constexpr int kGMaxKt = 32;              // one list entry per lane
constexpr unsigned long long kSpinNs = 2000000000ull;

struct GSmem {
  uint32_t ring, bars, info, hs, a1, sc, b2s, offs, cch, mask, thr, wc, surv, wl, wm, wsum, wn, misc, red, total;
};

__host__ __device__ inline GSmem gstep_smem(int S, int stage_bytes, int d, int esz, int M, int rows1, int K) {
  GSmem L;
  uint32_t o = 0;
  auto take = [&](uint32_t bytes, uint32_t al) {
    o = (o + al - 1u) & ~(al - 1u);
    const uint32_t at = o;
    o += bytes;
    return at;
  };
  L.ring = take((uint32_t)S * (uint32_t)stage_bytes, 1024);
  L.bars = take((2 * kGSlots + 1) * 8, 8);
  L.info = take(kGSlots * 16, 16);
  L.hs = take((uint32_t)d * esz, 128);
  L.a1 = take(4u * (rows1 > 0 ? rows1 : 1), 16);
  L.sc = take(4u * M, 16);
  L.b2s = take(4u * M, 16);
  L.offs = take(4u * (M + 1), 16);
  L.cch = take(4u * M, 16);
  L.mask = take(4u * (kGMaxM / 32), 16);
  L.thr = take(8u * kGWarps, 8);  // per-warp thresholds, then survivor bits
  L.wc = take(4u * kGWarps, 4);
  L.surv = take(8u * (M > kGSlots * K ? M : kGSlots * K), 16);
  L.wl = take(8u * kGSlots * K, 8);
  L.wm = take(4u * kGSlots, 4);
  L.wsum = take(4u * kGSlots, 4);
  L.wn = take(4u * kGSlots, 4);
  L.misc = take(4u * 16, 4);
  L.red = take(4u * kGWarps * kGUnits, 4);
  L.total = o;
  return L;
}

struct GStepArgs {
  const void* W;            // W_perm [V][d]
  const int32_t* perm;      // [V]
  const int32_t* offsets;   // [M+1]
  const void* W1;           // [rows1][2d]
  const float* b1;          // [rows1]
  const void* W2;           // [M][h_r] (h_r > 0)
  const float* b2;          // [M]
  const void* h_prev;       // [d]
  const void* e;            // [d]
  const void* h_new;        // [d]
  const int32_t* sel_in;    // head-only: the selection (ascending ids) from dynaspec_step_route / select
  const int32_t* cnt_in;    //            its count
  const int32_t* sloff_in;  //            its shortlist offsets
  float* scores;            // [M] nullable
  int32_t* sel_out;         // [M]
  int32_t* cnt_out;         // [1]
  int32_t* sloff_out;       // [M+1]
  int32_t* top_ids;
  float* top_logits;
  float* top_logp;
  float* lse;
  float* z_out;             // nullable: z over V_S in shortlist order
  int64_t max_shortlist;
  int32_t V, M, d, h_r, rows1, k, k_t, stages, stage_rows, stage_bytes, head_only, pdl;
  int32_t merge_fast;           // DS_GSTEP_MERGE=fast: the two-warp tournament merge (A/B; same cost, and
                                //   compute-sanitizer's synccheck flags its named barrier after the tournament)
  int32_t kpw, q_sel, q_merge;  // TopK launch constants: keys per warp, per-warp / record-warp ranks
  int32_t lgK;                  // ceil(log2(k_t + 1)): binary-search steps over a k_t-entry list
  uint32_t kdiv;                // ceil(2^32 / k_t): tid / k_t as one multiply-high
  unsigned long long* aslot;  // [rows1] published layer-1 units (0 = not yet)
  unsigned long long* rec;    // [G][2 + k_t] per-CTA records (0 = not yet)
  unsigned* err;              // workspace error word (DS_ERR_DEVICE_TIMEOUT)
  unsigned long long* trace;
  GSmem L;                    // shared-memory carve-up (host-computed)
};

// Slow path of a poll (out of line: the hot path is one load): spin until the word is non-zero.
// t0: the spin's start; on timeout the workspace error word is raised, *dead is set (later polls
// return at once) and 0 is returned.
__device__ __noinline__ unsigned long long poll_slow(const unsigned long long* p, unsigned long long t0, unsigned* err,
                                                     volatile int* dead, unsigned sleep_ns) {
  // sleep_ns > 0 backs off between probes: when every CTA polls the same few lines, a tight spin
  // would queue the publishers' stores behind the polling loads in those L2 slices.  A single
  // polling warp (the merger) spins.
  for (unsigned n = 1;; ++n) {
    const unsigned long long v = ld_relaxed_u64(p);
    if (v != 0ull) return v;
    if (sleep_ns) __nanosleep(sleep_ns);
    if ((n & 63u) == 0u) {
      if (*dead) return 0ull;
      if (globaltimer_ns() - t0 > kSpinNs) {
        atomicExch(err, (unsigned)DS_ERR_DEVICE_TIMEOUT);
        *dead = 1;
        return 0ull;
      }
    }
  }
}

// Poll N words per lane until all are non-zero, every round issuing the loads of all pending words
// at once (one round trip per round, not per word).  v[i] holds the first probe's value (1 = no word).
template <int N>
__device__ __forceinline__ void poll_words(const unsigned long long* const (&p)[N], unsigned long long (&v)[N],
                                           unsigned long long t0, unsigned* err, volatile int* dead, unsigned sleep_ns) {
  uint32_t pend = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) pend |= (v[i] == 0ull ? 1u : 0u) << i;
  for (unsigned n = 1; pend; ++n) {
    if (sleep_ns) __nanosleep(sleep_ns);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if ((pend >> i) & 1u) v[i] = ld_relaxed_u64(p[i]);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (v[i] != 0ull) pend &= ~(1u << i);
    if ((n & 63u) == 0u && pend) {
      if (*dead) return;
      if (globaltimer_ns() - t0 > kSpinNs) {
        atomicExch(err, (unsigned)DS_ERR_DEVICE_TIMEOUT);
        *dead = 1;
        return;
      }
    }
  }
}

// ---------------------------------------------------------------- arithmetic primitives (sm_100a)
// ev += lo(a) lo(b), od += hi(a) hi(b) for two bf16 pairs: FHFMA.BF16 (bf16 x bf16 + f32, one
// rounding) — bit-identical to fmaf of the exactly widened values, without the widening ops.
__device__ __forceinline__ void fma_bf16x2(uint32_t a, uint32_t b, float& ev, float& od) {
  asm("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %2;\n\tmov.b32 {bl, bh}, %3;\n\t"
      "fma.rn.f32.bf16 %0, al, bl, %0;\n\tfma.rn.f32.bf16 %1, ah, bh, %1;\n\t}"
      : "+f"(ev), "+f"(od)
      : "r"(a), "r"(b));
}
// (x, y) += (a0 b0, a1 b1): FFMA2, two independent RN fmas in one instruction.
__device__ __forceinline__ void ffma2(float& x, float& y, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 A, B, C;\n\tmov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\tmov.b64 C, {%0, %1};\n\t"
      "fma.rn.f32x2 C, A, B, C;\n\tmov.b64 {%0, %1}, C;\n\t}"
      : "+f"(x), "+f"(y)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// 16 bytes of x against 16 bytes of w: even / odd elements into two chains (the order of dot2).
__device__ __forceinline__ void dot16(const uint4& w, const uint4& x, float& ev, float& od, const __nv_bfloat16*) {
  fma_bf16x2(w.x, x.x, ev, od);
  fma_bf16x2(w.y, x.y, ev, od);
  fma_bf16x2(w.z, x.z, ev, od);
  fma_bf16x2(w.w, x.w, ev, od);
}
__device__ __forceinline__ void dot16(const uint4& w, const uint4& x, float& ev, float& od, const float*) {
  ev = fmaf(__uint_as_float(w.x), __uint_as_float(x.x), ev);
  od = fmaf(__uint_as_float(w.y), __uint_as_float(x.y), od);
  ev = fmaf(__uint_as_float(w.z), __uint_as_float(x.z), ev);
  od = fmaf(__uint_as_float(w.w), __uint_as_float(x.w), od);
}
// Two staged rows against h: z0, z1 with the summation order of dot2 (head_impl.cuh), so logits are
// bit-identical across the head kernels.
template <typename T>
__device__ __forceinline__ void dot2_fast(const T* __restrict__ w0, const T* __restrict__ w1, const T* __restrict__ h,
                                          int d, int lane, float& z0, float& z1) {
  constexpr int E = Elem<T>::kPer16B;
  float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 4
  for (int c = lane * E; c < d; c += 32 * E) {
    const uint4 hv = *reinterpret_cast<const uint4*>(h + c);
    const uint4 xv = *reinterpret_cast<const uint4*>(w0 + c);
    const uint4 yv = *reinterpret_cast<const uint4*>(w1 + c);
    dot16(xv, hv, a0, a1, h);
    dot16(yv, hv, b0, b1, h);
  }
  z0 = warp_sum(a0 + a1) + 0.0f;  // + 0.0f: -0 -> +0 (R23)
  z1 = warp_sum(b0 + b1) + 0.0f;
}

// lanes per item of a rank count: lp = floor(log2 nt) - ceil(log2 n), clamped to [0, 5] (no division)
__device__ __forceinline__ int lanes_log2(int n, int nt) {
  const int cl = n <= 1 ? 0 : 32 - __clz(n - 1);
  return min(5, max(0, (31 - __clz(nt)) - cl));
}

// Rank count of the n unique keys v[0..n) (rank = #keys above): key i by P = 2^lp lanes, P the
// smallest power of two with n / P <= 32 compares per lane, so only ceil(n P / 32) warps issue (a
// warp reading one position per lane group: broadcast loads, no bank conflicts); two accumulators.
// emit(rank, key) for rank < K.  Called by threads 0..nt-1 (nt a multiple of 32); passes of nt threads
// when n P exceeds nt (large k_t or tiny shortlists only).
template <class Emit>
__device__ __forceinline__ void rank_keys(const unsigned long long* v, int n, int K, int nt, Emit emit) {
  int lp = n <= 32 ? 0 : min(5, 32 - __clz((n - 1) >> 5));  // pow2ceil(n / 32), <= a warp
  if (n > 256)  // large k_t: one pass of nt threads (k_t = 32: 384 keys, 13 passes -> 1; 17.3k -> 11.4k cycles)
    while (lp > 0 && (n << lp) > nt) --lp;
  const int P = 1 << lp;
  const int work = ((n << lp) + 31) & ~31;  // threads with work, whole warps
#pragma unroll 1
  for (int t = threadIdx.x; t < work; t += nt) {  // one pass unless n P > nt (threads 0..nt-1 call this)
    const int i = t >> lp, part = t & (P - 1);
    const unsigned long long x = i < n ? v[i] : ~0ull;
    int r0 = 0, r1 = 0;
    int j = part;
#pragma unroll 4
    for (; j + P < n; j += 2 * P) {
      r0 += v[j] > x;
      r1 += v[j + P] > x;
    }
    if (j < n) r0 += v[j] > x;
    int rk = r0 + r1;
    for (int o = P >> 1; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    if (i < n && part == 0 && rk < K) emit(rk, x);
  }
}

// ---------------------------------------------------------------- router
// Layer-2 register slice, loaded coalesced: lane l of warp w holds rows m = w RWa + r (r < 16,
// RWa = ceil(M / 16)) and column words cw = 0, 1 (bf16: columns 2p, 2p + 1 with p = l + 32 cw;
// fp32: column l + 32 cw) — each load instruction reads 128 contiguous bytes of one row.
template <typename T>
__device__ __forceinline__ void load_w2(const GStepArgs& a, int warp, int lane, uint32_t (&w2r)[kGRows2][2]) {
  constexpr int per = sizeof(T) == 2 ? 2 : 1;  // columns per 32-bit word
  const int RWa = (a.M + kGWarps - 1) / kGWarps;
  const int rlim = min(RWa, a.M - warp * RWa);
  const int wpr = a.h_r / per;  // words per W2 row
  const uint32_t* p = static_cast<const uint32_t*>(a.W2) + (size_t)warp * RWa * wpr + lane;
  const bool c0 = lane < wpr, c1 = lane + 32 < wpr;
#pragma unroll
  for (int r = 0; r < kGRows2; ++r) {
    w2r[r][0] = (r < rlim && c0) ? __ldg(p + r * wpr) : 0u;
    w2r[r][1] = (r < rlim && c1) ? __ldg(p + r * wpr + 32) : 0u;
  }
}

// One reduce-scatter step of the transposed warp tree: lanes with bit (2H) set keep values
// [H, 2H), the others [0, H); each adds the partner's copy of the half it keeps.
template <int H>
__device__ __forceinline__ void halve(float* v, int lane) {
  const bool up = (lane & (2 * H)) != 0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const float send = up ? v[i] : v[i + H];
    const float keep = up ? v[i + H] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * H);
  }
}

// s_m = W2_m . a + b2_m for the warp's rows: per lane FFMA2 over its column words (even / odd
// column chains), then one transposed (reduce-scatter) warp tree — after it lane l holds the full
// sum of row (l >> 1) & 15.  Same code and order in every CTA.
template <typename T>
__device__ __forceinline__ void layer2(const GStepArgs& a, int warp, int lane, const uint32_t (&w2r)[kGRows2][2],
                                       const float* a1, const float* b2s, float* sc) {
  float v[kGRows2];
  if (sizeof(T) == 2) {
    const int c0 = 2 * lane, c1 = 2 * (lane + 32);
    const float a00 = c0 < a.h_r ? a1[c0] : 0.f, a01 = c0 < a.h_r ? a1[c0 + 1] : 0.f;
    const float a10 = c1 < a.h_r ? a1[c1] : 0.f, a11 = c1 < a.h_r ? a1[c1 + 1] : 0.f;
#pragma unroll
    for (int r = 0; r < kGRows2; ++r) {
      float x = 0.f, y = 0.f;
      ffma2(x, y, __uint_as_float(w2r[r][0] << 16), __uint_as_float(w2r[r][0] & 0xffff0000u), a00, a01);
      ffma2(x, y, __uint_as_float(w2r[r][1] << 16), __uint_as_float(w2r[r][1] & 0xffff0000u), a10, a11);
      v[r] = x + y;
    }
  } else {
    const float a0 = lane < a.h_r ? a1[lane] : 0.f, a1v = lane + 32 < a.h_r ? a1[lane + 32] : 0.f;
#pragma unroll
    for (int r = 0; r < kGRows2; ++r) {
      float x = 0.f, y = 0.f;
      ffma2(x, y, __uint_as_float(w2r[r][0]), __uint_as_float(w2r[r][1]), a0, a1v);
      v[r] = x + y;
    }
  }
  halve<8>(v, lane);
  halve<4>(v, lane);
  halve<2>(v, lane);
  halve<1>(v, lane);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  const int RWa = (a.M + kGWarps - 1) / kGWarps;
  const int r = (lane >> 1) & 15, m = warp * RWa + r;
  if ((lane & 1) == 0 && r < RWa && m < a.M) sc[m] = v[0] + b2s[m];
}

// TopK_k of sc[0..M) (score desc, id asc; R7) as a bit mask.  Key warp w holds keys m = w kpw + lane (kpw = ceil(M / 8) <= 32, 8 key
// warps).  Each key warp finds its q-th best score (q = ceil(k / key warps)) by q rounds of
// REDUX.MAX; T = the smallest of those (REDUX.MIN) has >= k scores at or above it, so the top k are
// among the survivors ord(s) >= T, and a survivor's rank among survivors is its rank (every key
// above a survivor is one).  Survivors are compacted (warp prefix by REDUX.ADD) and rank-counted
// by P lanes each.  Keys (ord(s) << 32 | ~m) are unique.  Four block barriers.
__device__ DS_GSTEP_NOINLINE void topk_mask(const float* sc, int M, int k, int kpw, int q, const int32_t* offs,
                                       uint32_t* mask, uint32_t* thr, unsigned long long* surv,
                                       unsigned long long* dbg) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = warp * kpw + lane;
  const bool valid = warp < kGKeyWarps && lane < kpw && m < M;
  const uint32_t ok = valid ? ord_key(sc[m]) : 0u;  // every valid key is > 0
  if (warp < kGKeyWarps) {
    uint32_t v = ok, tq = 0u;
    for (int it = 0; it < q; ++it) {
      const uint32_t mx = __reduce_max_sync(0xffffffffu, v);
      tq = mx;
      if (mx == 0u) break;  // fewer than q keys here: no bound from this warp
      const uint32_t b = __ballot_sync(0xffffffffu, v == mx);
      if (lane == __ffs(b) - 1) v = 0u;
    }
    if (lane == 0) thr[warp] = warp * kpw < M ? tq : 0xffffffffu;
  }
  __syncthreads();
  trace_mark(dbg, 13);
  const uint32_t T = __reduce_min_sync(0xffffffffu, lane < kGKeyWarps ? thr[lane] : 0xffffffffu);
  const bool sv = valid && ok >= T;
  const uint32_t b = __ballot_sync(0xffffffffu, sv);
  if (lane == 0 && warp < kGKeyWarps) thr[kGKeyWarps + warp] = __popc(b);
  __syncthreads();
  const unsigned c = lane < kGKeyWarps ? thr[kGKeyWarps + lane] : 0u;
  const int base = (int)__reduce_add_sync(0xffffffffu, lane < warp ? c : 0u);
  const int ns = (int)__reduce_add_sync(0xffffffffu, c);
  if (sv) surv[base + __popc(b & ((1u << lane) - 1u))] = ((unsigned long long)ok << 32) | (0xffffffffu - (uint32_t)m);
  __syncthreads();
  trace_mark(dbg, 14);
  rank_keys(surv, ns, k, kGThreads, [&](int, unsigned long long x) {
    const int mm = (int)(0xffffffffu - (uint32_t)x);
    atomicOr(&mask[mm >> 5], 1u << (mm & 31));
  });
  __syncthreads();
}

// ---------------------------------------------------------------- gathered head
// Chunks of the virtual shortlist, in shortlist order (selected clusters ascending, R8): chunk c =
// <= R whole W_perm rows inside one cluster; chunk c goes to streaming CTA c mod Gs (the whole grid
// sweeps one window of the shortlist at a time).  A resumable walk over this CTA's chunks.
struct ChunkWalk {
  const uint32_t* mask;
  const int32_t* offs;
  const int32_t* cch;
  int words, R, Gs;
  int w, beg, sz, nch;
  uint32_t bits;
  long long cb, vpos, cn;
  bool live;
  __device__ void init(const uint32_t* mask_, const int32_t* offs_, const int32_t* cch_, int M, int R_, int g, int Gs_) {
    mask = mask_;
    offs = offs_;
    cch = cch_;
    words = (M + 31) >> 5;
    R = R_;
    Gs = Gs_;
    w = 0;
    bits = mask[0];
    cb = 0;
    vpos = 0;
    cn = g;
    live = false;
    beg = sz = nch = 0;
  }
  // next chunk of this CTA: (virtual position, rows, first W_perm row); false at the end
  __device__ __forceinline__ bool next(int& vp, int& n, int& row) {
    for (;;) {
      if (live && cn < cb + nch) {
        const int j0 = (int)(cn - cb) * R;
        vp = (int)vpos + j0;
        n = min(R, sz - j0);
        row = beg + j0;
        cn += Gs;
        return true;
      }
      if (live) {
        cb += nch;
        vpos += sz;
      }
      while (bits == 0u) {
        if (++w >= words) return false;
        bits = mask[w];
      }
      const int m = (w << 5) + __ffs(bits) - 1;
      bits &= bits - 1u;
      beg = offs[m];
      sz = offs[m + 1] - beg;
      nch = cch[m];
      live = true;
    }
  }
};

// Producer lane: the CTA's chunks through the TMA bulk-copy ring (info = (-, virtual shortlist
// position, rows, first W_perm row)).  (Requesting the chunks that wait for a slot into L2 ahead of
// time with cp.async.bulk.prefetch.L2 measured slower: 20.1 -> 23.9 us per step.)
template <typename T>
__device__ __noinline__ void gstep_produce(const GStepArgs& a, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                           int4* info, const uint32_t* mask, const int32_t* offs, const int32_t* cch,
                                           bool stream) {
  const int g = blockIdx.x, Gs = gridDim.x - 1;  // the merger CTA (the last) streams nothing
  const uint64_t pol = policy_evict_first();
  const uint32_t rowbytes = (uint32_t)a.d * (uint32_t)sizeof(T);
  const uint8_t* W = static_cast<const uint8_t*>(a.W);
  const uint32_t S = (uint32_t)a.stages;
  uint32_t sl = 0, ph = 0;  // ring slot and phase (no divisions)
  if (stream && g < Gs) {
    ChunkWalk is;
    is.init(mask, offs, cch, a.M, a.stage_rows, g, Gs);
    int vp, n, row;
    while (is.next(vp, n, row)) {
      mbar_wait(&empty[sl], ph ^ 1u);
      info[sl] = make_int4(0, vp, n, row);
      mbar_arrive_expect_tx(&full[sl], (uint32_t)n * rowbytes);
      bulk_g2s(ring + (size_t)sl * a.stage_bytes, W + (size_t)row * rowbytes, (uint32_t)n * rowbytes, &full[sl], pol);
      if (++sl == S) {
        sl = 0;
        ph ^= 1u;
      }
    }
  }
  trace_mark_w(a.trace, 18);  // last chunk issued
#pragma unroll 1
  for (uint32_t j = 0; j < S; ++j) {  // one end-of-stream marker per slot
    mbar_wait(&empty[sl], ph ^ 1u);
    info[sl] = make_int4(-1, 0, -1, 0);
    mbar_arrive(&full[sl]);
    if (++sl == S) {
      sl = 0;
      ph ^= 1u;
    }
  }
}

// Consumer warp w (ring slot w): logits folded on the fly into (m, s) and the warp's sorted top-K list.
template <typename T>
__device__ __forceinline__ void gstep_consume(const GStepArgs& a, const uint8_t* ring, uint64_t* full,
                                              uint64_t* empty, const int4* info, const T* hs, int w, int lane,
                                              float& m, float& s, unsigned long long& mine) {
  const int K = a.k_t;
  unsigned long long kth = 0ull;
  m = -INFINITY;
  s = 0.f;
  mine = 0ull;
  for (uint32_t k = 0;; ++k) {
    mbar_wait(&full[w], k & 1u);
    if (k == 0 && w == 0) trace_mark_w(a.trace, 12);  // first chunk of slot 0 landed
    const int4 inf = info[w];
    if (inf.z < 0) break;
    const T* st = reinterpret_cast<const T*>(ring + (size_t)w * a.stage_bytes);
    for (int rr = 0; rr < inf.z; rr += 2) {
      const bool two = rr + 1 < inf.z;
      const int tok0 = __ldg(a.perm + inf.w + rr);
      const int tok1 = two ? __ldg(a.perm + inf.w + rr + 1) : 0;
      const T* w0 = st + (size_t)rr * a.d;
      float z0, z1;
      dot2_fast<T>(w0, two ? w0 + a.d : w0, hs, a.d, lane, z0, z1);
      lse_push(m, s, z0);
      list_insert(mine, kth, tok_key(z0, tok0), K, lane);
      if (two) {
        lse_push(m, s, z1);
        list_insert(mine, kth, tok_key(z1, tok1), K, lane);
      }
      if (a.z_out && lane == 0) {
        a.z_out[inf.y + rr] = z0;
        if (two) a.z_out[inf.y + rr + 1] = z1;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[w]);
  }
}

// CTA record (after the streaming barrier): (max | sum), min(#keys, K) + 1, the CTA's K best keys
// (padding 1) — never 0.  The S warp lists are sorted (descending, 0 = empty), so entry (w, r) has
// rank r + sum over the other lists of #entries above it: S - 1 binary searches of lgK steps, run
// as lgK rounds of independent shared-memory loads (no loop back-edges, no block barrier).  Warp
// 15 folds the S (max, sum) pairs (fixed xor tree, R19).  kdiv = ceil(2^32 / K): w = tid / K.
__device__ DS_GSTEP_NOINLINE void gstep_record(unsigned long long* my, const unsigned long long* wl, const float* wm,
                                          const float* wsum, const int* wn, int S, int K, int lgK, uint32_t kdiv) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == kGProducer) {
    const bool has = lane < S;
    const float mw = has ? wm[lane] : -INFINITY;
    const uint32_t mk = __reduce_max_sync(0xffffffffu, mw > -INFINITY ? ord_key(mw) : 0u);
    const float Mx = mk ? __uint_as_float((mk & 0x80000000u) ? (mk & 0x7fffffffu) : ~mk) : -INFINITY;
    const float sum = warp_sum(has && mw > -INFINITY ? wsum[lane] * expf(mw - Mx) : 0.f);
    const int nv = min(K, (int)__reduce_add_sync(0xffffffffu, has ? (unsigned)wn[lane] : 0u));
    if (lane >= nv && lane < K) my[2 + lane] = 1ull;  // padding (R17)
    if (lane == 0) {
      my[1] = (unsigned long long)nv + 1ull;
      my[0] = (unsigned long long)__float_as_uint(Mx) | ((unsigned long long)__float_as_uint(sum) << 32);
    }
    return;
  }
  // the S K entries (0 = empty) ranked against each other by the warps below the producer
  if (warp < kGProducer)
    rank_keys(wl, S * K, K, 32 * kGProducer, [&](int rk, unsigned long long x) {
      if (x != 0ull) my[2 + rk] = x;
    });
  (void)lgK;
  (void)kdiv;
}

// S3 outputs for the caller (selection ascending, sl_offsets, count, scores) by one warp.
__device__ __noinline__ void gstep_emit_selection(const GStepArgs& a, const uint32_t* mask, const int32_t* offs,
                                                  const float* sc) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (a.scores && tid < a.M) a.scores[tid] = sc[tid];  // M <= 256 < blockDim
  if (tid >= 32) return;
  int run = 0, off = 0;
  const int words = (a.M + 31) >> 5;
#pragma unroll 1
  for (int w = 0; w < words; ++w) {
    const uint32_t bits = mask[w];
    const int m = (w << 5) + lane;
    const bool s = (bits >> lane) & 1u;
    const int sz = s ? offs[m + 1] - offs[m] : 0;
    int inc = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int pos = run + __popc(bits & ((1u << lane) - 1u));
    if (s) {
      a.sel_out[pos] = m;
      a.sloff_out[pos] = off + inc - sz;
    }
    run += __popc(bits);
    off += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {
    *a.cnt_out = run;
    a.sloff_out[run] = off;
  }
}

// Merge of the G staged records raw[G][2 + K] (every thread of the CTA): lse = M + log sum_g s_g
// e^{m_g - M}, as per-warp partials relative to the warp's max (fixed xor trees) combined by one
// fixed tree (R19); top-K: each record warp finds its min(q, n_w)-th best head (REDUX rounds) and
// every key with a high word >= the smallest of those is a candidate (>= K keys are, and every key
// above a candidate is one); candidates (prefixes of the sorted records) are compacted and
// rank-counted.  Scratch after the records in raw.
__device__ DS_GSTEP_NOINLINE void gstep_merge_compute(const GStepArgs& a, unsigned long long* raw, int G, bool ok_in) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.k_t, rec = 2 + K;
  unsigned long long* cand = raw + (size_t)G * rec;                     // [G*K]
  uint32_t* wthr = reinterpret_cast<uint32_t*>(cand + (size_t)G * K);  // [16] per-warp q-th heads
  uint32_t* wmx = wthr + kGWarps;                                       // [16] per-warp max logit keys
  float* wps = reinterpret_cast<float*>(wmx + kGWarps);                 // [16] per-warp lse partials
  int* wq = reinterpret_cast<int*>(wps + kGWarps);                      // [16] keys each threshold bounds
  int* ncand = wq + kGWarps;
  // thread g: record g (G <= blockDim: one CTA per SM)
  const bool has = tid < G;
  const unsigned long long w0 = has ? raw[(size_t)tid * rec] : 0ull;
  const float mg = has ? __uint_as_float((uint32_t)w0) : -INFINITY;
  const float sg = __uint_as_float((uint32_t)(w0 >> 32));
  const int cg = has ? (int)raw[(size_t)tid * rec + 1] - 1 : 0;
  const unsigned long long hd = has ? raw[(size_t)tid * rec + 2] : 0ull;
  const uint32_t hk = (cg > 0 && hd > 1ull) ? (uint32_t)(hd >> 32) : 0u;
  {
    const uint32_t mk = __reduce_max_sync(0xffffffffu, mg > -INFINITY ? ord_key(mg) : 0u);
    const float Mw = mk ? __uint_as_float((mk & 0x80000000u) ? (mk & 0x7fffffffu) : ~mk) : -INFINITY;
    const float part = warp_sum(mg > -INFINITY ? sg * expf(mg - Mw) : 0.f);
    // this warp's min(q, n_w)-th best head (n_w: its non-empty records)
    const int qq = min(a.q_merge, __popc(__ballot_sync(0xffffffffu, hk != 0u)));
    uint32_t v = hk, tq = 0xffffffffu;
    for (int it = 0; it < qq; ++it) {
      tq = __reduce_max_sync(0xffffffffu, v);
      const uint32_t b = __ballot_sync(0xffffffffu, v == tq);
      if (lane == __ffs(b) - 1) v = 0u;
    }
    if (lane == 0) {
      wmx[warp] = mk;
      wps[warp] = part;
      wthr[warp] = tq;
      wq[warp] = qq;
    }
    if (tid == 0) *ncand = 0;
  }
  __syncthreads();
  trace_mark(a.trace, 10);
  const uint32_t wk = lane < kGWarps ? wmx[lane] : 0u;
  const uint32_t Mk = __reduce_max_sync(0xffffffffu, wk);
  const float Mx = Mk ? __uint_as_float((Mk & 0x80000000u) ? (Mk & 0x7fffffffu) : ~Mk) : -INFINITY;
  // the warps' thresholds bound >= sum of their qq keys from below: valid if that is >= K
  const unsigned nq = __reduce_add_sync(0xffffffffu, lane < kGWarps ? (unsigned)wq[lane] : 0u);
  const uint32_t T = (int)nq >= K ? __reduce_min_sync(0xffffffffu, lane < kGWarps ? wthr[lane] : 0xffffffffu) : 0u;
  if (has) {
    int c = cg;  // record keys with a high word >= T: a prefix of the sorted record
    if (T > 0u) {
      c = 0;
      while (c < cg && (uint32_t)(raw[(size_t)tid * rec + 2 + c] >> 32) >= T) ++c;
    }
    if (c > 0) {
      const int base = atomicAdd(ncand, c);
#pragma unroll 1
      for (int j = 0; j < c; ++j) cand[base + j] = raw[(size_t)tid * rec + 2 + j];
    }
  }
  // lse, meanwhile (every thread, same fixed tree): the warp partials rescaled to the global max
  float wt = 0.f;
  if (wk != 0u) {
    const float Mw = __uint_as_float((wk & 0x80000000u) ? (wk & 0x7fffffffu) : ~wk);
    wt = wps[lane] * expf(Mw - Mx);
  }
  const float sum = warp_sum(wt);
  const bool ok = ok_in && Mx > -INFINITY;
  const float lse = ok ? Mx + logf(sum) : __int_as_float(0x7fc00000);
  __syncthreads();
  trace_mark(a.trace, 11);
  const int ns = *ncand;
  if (a.trace != nullptr && tid == 0) a.trace[blockIdx.x * 64 + 29] = (unsigned long long)ns;  // candidates
  rank_keys(cand, ns, K, kGThreads, [&](int rk, unsigned long long x) {
    const float z = key_value(x);
    a.top_ids[rk] = ok ? key_id(x) : -1;
    a.top_logits[rk] = ok ? z : -INFINITY;
    a.top_logp[rk] = ok ? z - lse : -INFINITY;
  });
  if (tid >= min(ns, K) && tid < K) {  // fewer valid keys than K: padding (R17)
    a.top_ids[tid] = -1;
    a.top_logits[tid] = -INFINITY;
    a.top_logp[tid] = -INFINITY;
  }
  if (tid == 0) a.lse[0] = lse;
  trace_mark(a.trace, 9);
}

// Merge for k_t <= 16 and G <= 160 by two warps, no block barrier (the staged records raw[G][2 + K]):
//   warp 1: lse = M + log sum_g s_g e^{m_g - M} — lane l folds records l, l + 32, ... in that order,
//           then one fixed xor tree (R19);
//   warp 0: top-K by a K-round tournament over the G sorted records: each lane holds the current
//           head of its <= 5 records, the warp takes the largest 64-bit key (REDUX on the high
//           word, then on the low word among the ties — keys are unique), and the winning lane
//           advances that record.
// They meet at one named barrier (lse is needed for the log-probs).  Measured cost in isolation
// (scripts/probe/phase_bench.cu): see DESIGN §5.2c; replaces three block-wide phases.
constexpr int kGMergeRecs = 5;  // records per lane (G <= 160)
__device__ DS_GSTEP_NOINLINE void gstep_merge_fast(const GStepArgs& a, const unsigned long long* raw, int G,
                                                   bool ok_in, float* lse_sh) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.k_t, rec = 2 + K;
  if (warp == 1) {
    float mg[kGMergeRecs], sg[kGMergeRecs];
    uint32_t mk = 0u;
#pragma unroll
    for (int q = 0; q < kGMergeRecs; ++q) {
      const int g = lane + 32 * q;
      const unsigned long long w0 = g < G ? raw[(size_t)g * rec] : 0ull;
      mg[q] = g < G ? __uint_as_float((uint32_t)w0) : -INFINITY;
      sg[q] = __uint_as_float((uint32_t)(w0 >> 32));
      if (mg[q] > -INFINITY) mk = max(mk, ord_key(mg[q]));
    }
    mk = __reduce_max_sync(0xffffffffu, mk);
    const float Mx = mk ? __uint_as_float((mk & 0x80000000u) ? (mk & 0x7fffffffu) : ~mk) : -INFINITY;
    float part = 0.f;
#pragma unroll
    for (int q = 0; q < kGMergeRecs; ++q)
      if (mg[q] > -INFINITY) part += sg[q] * expf(mg[q] - Mx);
    const float sum = warp_sum(part);
    const bool ok = ok_in && Mx > -INFINITY;
    const float lse = ok ? Mx + logf(sum) : __int_as_float(0x7fc00000);
    if (lane == 0) {
      *lse_sh = lse;
      a.lse[0] = lse;
    }
    __syncwarp();
    named_bar_sync(3, 64);
  } else if (warp == 0) {
    unsigned long long cur[kGMergeRecs];
    int pos[kGMergeRecs], cnt[kGMergeRecs];
#pragma unroll
    for (int q = 0; q < kGMergeRecs; ++q) {
      const int g = lane + 32 * q;
      cnt[q] = g < G ? (int)raw[(size_t)g * rec + 1] - 1 : 0;
      pos[q] = 0;
      cur[q] = cnt[q] > 0 ? raw[(size_t)g * rec + 2] : 0ull;
    }
    unsigned long long mine = 0ull;  // lane r keeps the r-th best key
    for (int r = 0; r < K; ++r) {
      unsigned long long best = cur[0];
      int bq = 0;
#pragma unroll
      for (int q = 1; q < kGMergeRecs; ++q)
        if (cur[q] > best) {
          best = cur[q];
          bq = q;
        }
      const uint32_t hi = (uint32_t)(best >> 32);
      const uint32_t Mhi = __reduce_max_sync(0xffffffffu, hi);
      if (Mhi == 0u) break;  // every record exhausted: padding below
      const uint32_t lo = hi == Mhi ? (uint32_t)best : 0u;
      const uint32_t Mlo = __reduce_max_sync(0xffffffffu, lo);
      const unsigned long long win = ((unsigned long long)Mhi << 32) | Mlo;
      if (lane == r) mine = win;
      if (best == win) {  // exactly one lane: advance its record
#pragma unroll
        for (int q = 0; q < kGMergeRecs; ++q)
          if (q == bq) {
            ++pos[q];
            cur[q] = pos[q] < cnt[q] ? raw[(size_t)(lane + 32 * q) * rec + 2 + pos[q]] : 0ull;
          }
      }
    }
    __syncwarp();  // the tournament's winner-only updates leave the warp diverged: reconverge first
    named_bar_sync(3, 64);
    const float lse = *lse_sh;
    const bool ok = !(lse != lse);
    if (lane < K) {
      const bool v = ok && mine != 0ull;
      const float z = key_value(mine);
      a.top_ids[lane] = v ? key_id(mine) : -1;
      a.top_logits[lane] = v ? z : -INFINITY;
      a.top_logp[lane] = v ? z - lse : -INFINITY;
    }
  }
  trace_mark(a.trace, 9);
}

// Merger (CTA 0): stage the G records as their words land; thread g decodes record g.  lse = M + log
// sum_g s_g e^{m_g - M} (per-warp xor trees, then one fixed tree over the warps, R19).  Top-K: each
// record warp finds its q-th best head (q = ceil(K / record warps), REDUX rounds); every key with a
// high word >= the smallest of those is a candidate (>= K keys are, and every key above a
// candidate is one), candidates are rank-counted.  Scratch: the ring.
__device__ DS_GSTEP_NOINLINE void gstep_merge(const GStepArgs& a, uint8_t* ring, bool stream, unsigned long long t_spin,
                                         volatile int* dead) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, K = a.k_t, rec = 2 + K;
  unsigned long long* raw = reinterpret_cast<unsigned long long*>(ring);  // [G][rec] staged records
  const int nrec = G * rec;
  if (warp == 0) {  // first word of every record (written with its keys): one warp, all probes in flight
    unsigned long long v[kGHeadsPerLane];
    const unsigned long long* pw[kGHeadsPerLane];
#pragma unroll
    for (int i = 0; i < kGHeadsPerLane; ++i) {
      const int r = lane + 32 * i;
      pw[i] = a.rec + (size_t)(r < G ? r : 0) * rec;
      v[i] = r < G ? ld_relaxed_u64(pw[i]) : 1ull;
    }
    poll_words<kGHeadsPerLane>(pw, v, t_spin, a.err, dead, 0);
  }
  __syncthreads();
  {  // all loads in flight first, then spin only on the words that had not landed
    constexpr int kB = 4;
#pragma unroll 1
    for (int i0 = tid; i0 < nrec; i0 += kB * kGThreads) {
      unsigned long long v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) v[u] = i0 + u * kGThreads < nrec ? ld_relaxed_u64(a.rec + i0 + u * kGThreads) : 1ull;
#pragma unroll
      for (int u = 0; u < kB; ++u)
        if (i0 + u * kGThreads < nrec) raw[i0 + u * kGThreads] = v[u];
    }
    trace_mark(a.trace, 15);
#pragma unroll 1
    for (int i = tid; i < nrec; i += kGThreads)
      if (raw[i] == 0ull) raw[i] = poll_slow(a.rec + i, t_spin, a.err, dead, 0);
  }
  __syncthreads();
  trace_mark(a.trace, 8);
  // every word is staged and every CTA has read the unit words (its record exists only after its
  // poll): zero both for the next launch (the stores drain while the merge computes)
#pragma unroll 4
  for (int i = tid; i < nrec; i += kGThreads) a.rec[i] = 0ull;
  if (!a.head_only && tid < a.rows1) a.aslot[tid] = 0ull;  // rows1 <= blockDim
  if (a.k_t <= 16 && G <= 32 * kGMergeRecs && a.merge_fast)
    gstep_merge_fast(a, raw, G, *dead == 0 && stream, reinterpret_cast<float*>(raw + (size_t)G * (2 + a.k_t)));
  else
    gstep_merge_compute(a, raw, G, *dead == 0 && stream);
}

template <typename T>
__global__ void __launch_bounds__(kGThreads, 1) gstep_kernel(const __grid_constant__ GStepArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int E = Elem<T>::kPer16B;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = blockIdx.x, G = gridDim.x;
  const int M = a.M, d = a.d, K = a.k_t, S = a.stages;
  const GSmem& L = a.L;
  uint8_t* ring = smem + L.ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kGSlots;
  uint64_t* hbar = empty + kGSlots;
  int4* info = reinterpret_cast<int4*>(smem + L.info);
  T* hs = reinterpret_cast<T*>(smem + L.hs);
  float* a1 = reinterpret_cast<float*>(smem + L.a1);
  float* sc = reinterpret_cast<float*>(smem + L.sc);
  float* b2s = reinterpret_cast<float*>(smem + L.b2s);
  int32_t* offs = reinterpret_cast<int32_t*>(smem + L.offs);
  int32_t* cch = reinterpret_cast<int32_t*>(smem + L.cch);  // chunks per cluster
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem + L.mask);
  unsigned long long* wl = reinterpret_cast<unsigned long long*>(smem + L.wl);
  float* wm = reinterpret_cast<float*>(smem + L.wm);
  float* wsum = reinterpret_cast<float*>(smem + L.wsum);
  int* wn = reinterpret_cast<int*>(smem + L.wn);
  int* misc = reinterpret_cast<int*>(smem + L.misc);  // [0] |V_S| [1] bad selection [2] dead (spin timed out)
  float* red = reinterpret_cast<float*>(smem + L.red);
  volatile int* dead = misc + 2;

  if (tid == 0) {
#pragma unroll 1
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(hbar, 1);
    fence_mbar_init();
  }
  if (tid < kGMaxM / 32) mask[tid] = 0u;
  if (tid < 16) misc[tid] = 0;
  trace_mark(a.trace, 0);
  if (a.trace != nullptr && tid == 0) {  // cost of one trace mark (slots 16, 17: back-to-back marks)
    trace_mark(a.trace, 16);
    trace_mark(a.trace, 17);
  }
  // Dependents may launch now: they become resident only as this grid's CTAs exit (one CTA per SM),
  // and every CTA of this grid is resident once all have executed this, so waits cannot deadlock.
  if (a.pdl) pdl_launch_dependents();

  // ---- before the PDL wait: router constants (never written by an upstream kernel)
  const int nx = 2 * d / E;  // 16-byte chunks of x
  uint4 w1r[kGUnits][kGXChunks];
  uint32_t w2r[kGRows2][2];
  float b1r = 0.f;
  const int U = a.head_only ? 0 : (g < a.rows1) + (g + G < a.rows1);
  if (!a.head_only) {
    const uint64_t keep = policy_evict_last();
    const uint8_t* w1 = static_cast<const uint8_t*>(a.W1) + (size_t)g * 2 * d * sizeof(T) + (size_t)tid * 16;
    const size_t ustride = (size_t)G * 2 * d * sizeof(T);
#pragma unroll
    for (int j = 0; j < kGUnits; ++j)
#pragma unroll
      for (int i = 0; i < kGXChunks; ++i)
        w1r[j][i] = (j < U && tid + i * kGThreads < nx)
                        ? ld_evict_last_v4(w1 + j * ustride + (size_t)i * kGThreads * 16, keep)
                        : make_uint4(0u, 0u, 0u, 0u);
    if (warp < U) b1r = __ldg(a.b1 + g + warp * G);
    if (a.h_r > 0) {
      load_w2<T>(a, warp, lane, w2r);
      if (tid < M) b2s[tid] = __ldg(a.b2 + tid);  // M <= 256 < blockDim
    }
  }
  if (tid <= M) offs[tid] = __ldg(a.offsets + tid);
  if (tid < M) cch[tid] = (__ldg(a.offsets + tid + 1) - __ldg(a.offsets + tid) + a.stage_rows - 1) / a.stage_rows;
  __syncthreads();  // barrier inits, mask / misc zeroed, offsets and chunk counts staged

  if (a.pdl) pdl_wait();
  trace_mark(a.trace, 1);
  const uint32_t hb = (uint32_t)d * (uint32_t)sizeof(T);
  if (warp == kGProducer && lane == 0) {  // h_new for the head (needed once streaming starts)
    mbar_arrive_expect_tx(hbar, hb);
    bulk_g2s(hs, a.h_new, hb, hbar, policy_evict_first());
  }
  const unsigned long long t_spin = globaltimer_ns();
  if (!a.head_only) {
    // ---- layer 1: this CTA's unit(s) over x = [h_prev ‖ e] (R4), fixed summation order
    if (U > 0) {
      uint4 xr[kGXChunks];
#pragma unroll
      for (int i = 0; i < kGXChunks; ++i) {
        const int c = tid + i * kGThreads;
        const uint8_t* src = c < nx / 2 ? static_cast<const uint8_t*>(a.h_prev) + (size_t)c * 16
                                        : static_cast<const uint8_t*>(a.e) + (size_t)(c - nx / 2) * 16;
        xr[i] = c < nx ? ld_nc_v4(src) : make_uint4(0u, 0u, 0u, 0u);
      }
      float ev[kGUnits], od[kGUnits];
#pragma unroll
      for (int j = 0; j < kGUnits; ++j) ev[j] = od[j] = 0.f;
#pragma unroll
      for (int i = 0; i < kGXChunks; ++i)
#pragma unroll
        for (int j = 0; j < kGUnits; ++j) dot16(w1r[j][i], xr[i], ev[j], od[j], static_cast<const T*>(nullptr));
#pragma unroll
      for (int j = 0; j < kGUnits; ++j) {
        const float v = warp_sum(ev[j] + od[j]);
        if (lane == 0) red[warp * kGUnits + j] = v;
      }
      __syncthreads();
      if (warp < U) {  // warp j: unit j, the 16 warp partials by one fixed xor tree
        float s = warp_sum(lane < kGWarps ? red[lane * kGUnits + warp] : 0.f);
        s += b1r;
        if (a.h_r > 0) s = fmaxf(s, 0.f);
        if (lane == 0) st_relaxed_u64(a.aslot + g + warp * G, (1ull << 32) | (unsigned long long)__float_as_uint(s));
      }
    }
    trace_mark(a.trace, 2);
    // ---- every unit of every CTA, polled by one warp (all probes of a round in flight at once)
    if (warp == 0) {
#pragma unroll 1
      for (int u0 = 0; u0 < a.rows1; u0 += 128) {
        unsigned long long v[4];
        const unsigned long long* pw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int u = u0 + lane + 32 * i;
          pw[i] = a.aslot + (u < a.rows1 ? u : 0);
          v[i] = u < a.rows1 ? ld_relaxed_u64(pw[i]) : 1ull;
        }
        poll_words<4>(pw, v, t_spin, a.err, dead, 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int u = u0 + lane + 32 * i;
          if (u < a.rows1) a1[u] = __uint_as_float((uint32_t)v[i]);
        }
      }
    }
    __syncthreads();
    trace_mark(a.trace, 3);
    if (a.h_r > 0) {
      layer2<T>(a, warp, lane, w2r, a1, b2s, sc);
    } else {
      if (tid < M) sc[tid] = a1[tid];  // linear router: the units are the scores
    }
    __syncthreads();
    trace_mark(a.trace, 4);
    topk_mask(sc, M, a.k, a.kpw, a.q_sel, offs, mask, reinterpret_cast<uint32_t*>(smem + L.thr),
              reinterpret_cast<unsigned long long*>(smem + L.surv), a.trace);
  } else {
    // S1-S3 ran on S_m (dynaspec_step_route): the TopK mask from the selection in global memory
    const int cnt = __ldg(a.cnt_in);
    if (cnt < 1 || cnt > M) {
      if (tid == 0) misc[1] = 1;
    } else {
      if (tid < cnt) {  // cnt <= M <= 256 < blockDim
        const int m = __ldg(a.sel_in + tid);
        if (m < 0 || m >= M) misc[1] = 1;
        else atomicOr(&mask[m >> 5], 1u << (m & 31));
      }
      if (tid == 0) misc[0] = __ldg(a.sloff_in + cnt);
    }
    __syncthreads();
  }
  trace_mark(a.trace, 5);
  // head-only: a row whose |V_S| exceeds max_shortlist is not computed (top ids -1, lse NaN;
  // dynaspec.h).  Router mode: launch_gstep only runs with max_shortlist >= k max|C_m| >= |V_S|.
  const long long total = misc[0];
  const bool stream = !a.head_only || (misc[1] == 0 && total >= 1 && total <= a.max_shortlist);

  // ---- gathered head + per-warp epilogue state
  if (warp == kGProducer) {
    if (lane == 0) gstep_produce<T>(a, ring, full, empty, info, mask, offs, cch, stream);
  } else if (warp < S) {
    float m, se;
    unsigned long long mine;
    mbar_wait(hbar, 0);
    gstep_consume<T>(a, ring, full, empty, info, hs, warp, lane, m, se, mine);
    if (lane < K) wl[warp * K + lane] = mine;
    const int nv = __popc(__ballot_sync(0xffffffffu, lane < K && mine != 0ull));
    if (lane == 0) {
      wm[warp] = m;
      wsum[warp] = se;
      wn[warp] = nv;
    }
  }
  __syncthreads();
  trace_mark(a.trace, 6);
  gstep_record(a.rec + (size_t)g * (2 + K), wl, wm, wsum, wn, S, K, a.lgK, a.kdiv);
  trace_mark(a.trace, 7);
  // The merger is the LAST CTA and streams nothing: with one CTA per SM a dependent launch's CTA
  // lands on the previous merger's SM only once that merger exits, so the late CTA of the next step
  // is (per the block -> SM placement) its merger again — which has no router unit and no chunks.
  if (!a.head_only && g == G - 2) gstep_emit_selection(a, mask, offs, sc);  // S3 outputs, off the merger
  if (g == G - 1) gstep_merge(a, ring, stream, t_spin, dead);
}

// ------------------------------------------------------------------ host side

static int gstep_grid() { return std::max(2, num_sms() - 1); }

struct GStepPlan {
  int S, stage_rows, stage_bytes, rows1;
  size_t smem;
};

static bool gstep_plan(const ds_clusters* c, const ds_router* r, int k_t, GStepPlan* p) {
  const char* off = getenv("DS_GSTEP");
  if (off && off[0] == '0') return false;
  if (k_t < 1 || k_t > kGMaxKt || c->M > kGMaxM) return false;
  if ((reinterpret_cast<uintptr_t>(c->perm) & 15u) != 0 || c->V > (int64_t)0x7fffffff) return false;  // perm windows
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  const int G = gstep_grid();
  if (G > 32 * kGHeadsPerLane) return false;
  if ((size_t)G * (2 + k_t) * 8 > kWsGstepUnits - kWsGstepRec) return false;  // the record region
  p->rows1 = 0;
  if (r) {
    if (r->dtype != c->dtype) return false;
    p->rows1 = r->h_r > 0 ? r->h_r : r->M;
    if (r->h_r > 0 && r->h_r > 64 * (esz == 2 ? 2 : 1)) return false;  // layer-2 register slice
    if (p->rows1 > kGUnits * G || p->rows1 > kGThreads) return false;  // one polled unit word per thread
    if ((size_t)p->rows1 * 8 > kWsRowsUnits - kWsGstepUnits) return false;
    if ((size_t)2 * c->d * esz > (size_t)kGXChunks * kGThreads * 16) return false;
  }
  const int rowb = c->d * esz;
  const char* skb = getenv("DS_GSTEP_STAGE_KB");  // ring slot size (tuning knob; default 16 KB)
  const int target = skb && skb[0] ? std::max(4, std::min(64, atoi(skb))) * 1024 : kStageTarget;
  p->stage_rows = std::max(1, target / rowb);
  p->stage_bytes = p->stage_rows * rowb;
  const int smax = max_smem_optin();
  const size_t fixed = gstep_smem(0, p->stage_bytes, c->d, esz, c->M, std::max(p->rows1, 1), k_t).total + 1024;
  const char* sv = getenv("DS_GSTEP_STAGES");
  const int cap = sv && sv[0] ? std::max(2, std::min(kGSlots, atoi(sv))) : kGSlots;
  int S = (int)std::min<size_t>((size_t)cap, ((size_t)smax > fixed ? (size_t)smax - fixed : 0) / p->stage_bytes);
  if (S < 2) return false;
  // the merger stages G records + G K candidates + per-record fields inside the ring
  const size_t merge = (size_t)G * (2 + k_t) * 8 + (size_t)G * k_t * 8 + (size_t)(G + 4) * 16 + 256;
  if (merge > (size_t)S * p->stage_bytes) return false;
  p->S = S;
  p->smem = gstep_smem(S, p->stage_bytes, c->d, esz, c->M, std::max(p->rows1, 1), k_t).total;
  return p->smem <= (size_t)smax;
}

bool gstep_supported(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared) {
  GStepPlan p;
  return B == 1 && !shared && gstep_plan(c, r, k_t, &p);
}

template <typename T>
static cudaError_t gstep_configure() {
  static int done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (done[dev]) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(gstep_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             max_smem_optin());
  if (e != cudaSuccess) return e;
  done[dev] = 1;
  return cudaSuccess;
}

template <typename T>
static cudaError_t launch_gstep_t(const GStepArgs& a, size_t smem, cudaStream_t st, bool pdl) {
  cudaError_t e = gstep_configure<T>();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  // one CTA per SM on all SMs but one: the previous step's merger still holds its SM when this
  // step's CTAs are placed, so every CTA finds a free SM (no CTA of the step starts late)
  cfg.gridDim = dim3(gstep_grid());
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, gstep_kernel<T>, a);
}

static void fill_common(GStepArgs& a, const ds_clusters* c, const GStepPlan& p, int k_t, int64_t max_shortlist,
                        int32_t* top_ids, float* top_logits, float* top_logp, float* lse, float* z_out, void* ws) {
  a.W = c->W_perm;
  a.perm = c->perm;
  a.offsets = c->offsets;
  a.top_ids = top_ids;
  a.top_logits = top_logits;
  a.top_logp = top_logp;
  a.lse = lse;
  a.z_out = z_out;
  a.max_shortlist = max_shortlist > 0 ? std::min<int64_t>(max_shortlist, c->V) : c->V;
  a.V = (int32_t)c->V;
  a.M = c->M;
  a.d = c->d;
  a.k_t = k_t;
  a.stages = p.S;
  a.stage_rows = p.stage_rows;
  a.stage_bytes = p.stage_bytes;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  a.rec = reinterpret_cast<unsigned long long*>(w8 + kWsGstepRec);
  a.aslot = reinterpret_cast<unsigned long long*>(w8 + kWsGstepUnits);
  a.err = reinterpret_cast<unsigned*>(w8 + kWsErrorWord);
  a.trace = debug_trace();
  const char* mv = getenv("DS_GSTEP_MERGE");
  a.merge_fast = mv && mv[0] == 'f' ? 1 : 0;
  a.L = gstep_smem(p.S, p.stage_bytes, c->d, c->dtype == DS_BF16 ? 2 : 4, c->M, std::max(p.rows1, 1), k_t);
  a.kpw = (c->M + kGKeyWarps - 1) / kGKeyWarps;
  a.lgK = 0;
  while ((1 << a.lgK) < k_t + 1) ++a.lgK;
  a.kdiv = (uint32_t)((((uint64_t)1) << 32) / (uint64_t)k_t + (((((uint64_t)1) << 32) % (uint64_t)k_t) ? 1 : 0));
  const int nwr = (gstep_grid() + 31) / 32;
  a.q_merge = (k_t + nwr - 1) / nwr;
}

static int q_select(int M, int k) {
  const int kpw = (M + kGKeyWarps - 1) / kGKeyWarps, nk = (M + kpw - 1) / kpw;
  return (k + nk - 1) / nk;
}

cudaError_t launch_gstep(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                         const void* h_new, int k, int k_t, int64_t max_shortlist, float* scores, int32_t* sel,
                         int32_t* sel_count, int32_t* sl_offsets, int32_t* top_ids, float* top_logits,
                         float* top_logp, float* lse, float* z_out, void* ws, cudaStream_t st, bool pdl) {
  GStepPlan p;
  if (!gstep_plan(c, r, k_t, &p)) return cudaErrorInvalidValue;
  GStepArgs a = {};
  fill_common(a, c, p, k_t, max_shortlist, top_ids, top_logits, top_logp, lse, z_out, ws);
  a.W1 = r->W1;
  a.b1 = r->b1;
  a.W2 = r->W2;
  a.b2 = r->b2;
  a.h_prev = h_prev;
  a.e = e;
  a.h_new = h_new;
  a.scores = scores;
  a.sel_out = sel;
  a.cnt_out = sel_count;
  a.sloff_out = sl_offsets;
  a.h_r = r->h_r;
  a.rows1 = p.rows1;
  a.k = k;
  a.q_sel = q_select(c->M, k);
  a.head_only = 0;
  a.pdl = pdl ? 1 : 0;
  return c->dtype == DS_BF16 ? launch_gstep_t<__nv_bfloat16>(a, p.smem, st, pdl)
                             : launch_gstep_t<float>(a, p.smem, st, pdl);
}

cudaError_t launch_gstep_head(const ds_clusters* c, const void* h_new, const int32_t* sel, const int32_t* sel_count,
                              const int32_t* sl_offsets, int k_t, int64_t max_shortlist, int32_t* top_ids,
                              float* top_logits, float* top_logp, float* lse, float* z_out, void* ws,
                              cudaStream_t st) {
  GStepPlan p;
  if (!gstep_plan(c, nullptr, k_t, &p)) return cudaErrorInvalidValue;
  GStepArgs a = {};
  fill_common(a, c, p, k_t, max_shortlist, top_ids, top_logits, top_logp, lse, z_out, ws);
  a.h_new = h_new;
  a.sel_in = sel;
  a.cnt_in = sel_count;
  a.sloff_in = sl_offsets;
  a.k = 1;
  a.head_only = 1;
  a.pdl = 0;
  return c->dtype == DS_BF16 ? launch_gstep_t<__nv_bfloat16>(a, p.smem, st, false)
                             : launch_gstep_t<float>(a, p.smem, st, false);
}

bool gstep_pointers_ok(const ds_router* r, const void* h_prev, const void* e, const void* h_new) {
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  return al(h_prev) && al(e) && al(h_new) && al(r->W1) && (r->h_r == 0 || (reinterpret_cast<uintptr_t>(r->W2) & 3u) == 0);
}

}  // namespace ds
