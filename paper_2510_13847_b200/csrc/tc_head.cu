// tc_head.cu — S5' shared-shortlist head on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Tree drafting (R9, Alg. 1 line 8/10: one index set I for all k_t beam rows of a depth) makes the
// head a dense contraction Z[R x |V_S|] = H[R x d] W_S^T with R rows sharing V_S (P:262, P:286
// "computes on Tensor Cores").  Swap-AB so the vocabulary dimension is MMA-M = 128 and the rows
// are MMA-N (R padded to 16):  D[128 tokens x N] (fp32, TMEM) += A[128 x 64] (W_perm rows, smem)
// * B[N x 64]^T (h rows, smem), K = 16 per instruction (kind::f16, bf16 inputs).
//
// Per CTA (one per SM) the even segment of the shortlist (split rows, not clusters) is cut
// into 16-row boxes that never cross a cluster run; 8 boxes form one 128-row MMA tile.  Roles:
//   warp 0 lane 0   TMA producer: per (tile, 64-wide K chunk) 8 x 2-D boxes of W_perm (128B
//                   swizzle, evict_first) + one box of H into a ring slot (mbarrier tx count)
//   warp 1 lane 0   MMA issuer: 4 x tcgen05.mma per K chunk into a double-buffered TMEM
//                   accumulator; tcgen05.commit frees the slot / publishes the tile
//   warps 2..5      epilogue: tcgen05.ld 32x32b (one token per thread, R logits), remap via perm,
//                   logits to shared memory; then the shared per-CTA partial + last-CTA merge.
// Exactness: bf16 x bf16 products are exact in fp32; the exact-regime tests keep every partial
// sum an integer below 2^24, so any accumulation order reproduces the oracle bit for bit.
#include <cuda.h>

#include <algorithm>

#include "head_impl.cuh"
#include "internal.h"
#include "select_impl.cuh"
#include "tc_common.cuh"

namespace ds {

constexpr int kTcBoxRows = 16;
constexpr int kTcBoxes = 8;              // boxes per 128-row tile
constexpr int kTcK = 64;                 // K elements per stage (128 bytes: one swizzle span)
constexpr int kTcKPS = 2;                 // 64-wide K chunks per ring stage (one commit per stage)
constexpr int kTcABytes = 128 * kTcK * 2 * kTcKPS;  // A bytes of one stage
constexpr int kTcThreads = 6 * 32;
constexpr int kTcMaxBoxes = 2048;

struct TcArgs {
  HeadArgs h;
  int32_t N;        // MMA N (rows padded to 16)
  int32_t S;        // ring stages
  int32_t kchunks;  // ceil(d / 64)
  int32_t tmem_cols;
  int32_t online;   // 1: per-row running (max, sum, top-k) per tile instead of on-chip logit buffers
  const uint32_t* rowmask;  // nullable [nrows][32]: clusters each row selected (per-row batched mode)
  unsigned long long* trace;  // opt-in phase trace (dynaspec_debug_set_trace)
  int32_t box_cap;            // box table entries (ceil(lcap / 16) + M)
};

struct TcSmem {
  uint32_t a, b, bars, slot, misc, red, sega, segn, segi, boxes, zl, zid, stage, tokid, cid, runm, runs, lst, scr,
      total;
};

constexpr int kTcScr = 128 + kMaxKt;  // per-warp warp_topk scratch entries (online mode)

__host__ __device__ inline TcSmem tc_smem(int S, int N, int rows, int lcap, int online = 0, int K = 0,
                                          int box_cap = kTcMaxBoxes) {
  TcSmem L;
  uint32_t o = 0;
  L.a = o;
  o += (uint32_t)S * kTcABytes;
  L.b = o;
  o += (uint32_t)S * N * 128 * kTcKPS;
  o = (o + 1023u) & ~1023u;
  L.bars = o;
  o += (2 * 16 + 4) * 8;
  L.slot = o;
  o += 16;
  L.misc = o;
  o += 16 * 4;
  L.red = o;
  o += 64 * 4;
  L.sega = o;
  o += kMaxGroups * 8;
  L.segn = o;
  o += kMaxGroups * 4;
  L.segi = o;
  o += kMaxGroups * 4;
  o = (o + 15u) & ~15u;
  L.boxes = o;
  o += (uint32_t)box_cap * 16;
  L.zl = o;
  o += online ? 0u : (uint32_t)rows * lcap * 4;
  L.zid = o;
  o += online ? 0u : (uint32_t)rows * lcap * 4;
  L.stage = o;
  o += online ? (uint32_t)rows * 128 * 4 : 0u;
  L.tokid = o;
  o += online ? 128u * 4 : 0u;
  L.cid = o;
  o += online ? 128u * 4 : 0u;
  L.runm = o;
  o += online ? (uint32_t)rows * 4 : 0u;
  L.runs = o;
  o += online ? (uint32_t)rows * 4 : 0u;
  o = (o + 15u) & ~15u;
  L.lst = o;
  o += online ? 2u * rows * K * 8 : 0u;
  L.scr = o;
  o += online ? 4u * kTcScr * 8 : 0u;
  L.total = o;
  return L;
}

// ------------------------------------------------------------------ kernel
// W_perm views with box heights 16, 32, 64 and 128 rows (one TMA op per contiguous box group)
struct TcMaps {
  CUtensorMap w[4];
};

__global__ void __launch_bounds__(kTcThreads, 1) tc_head_kernel(const __grid_constant__ TcMaps tmWs,
                                                                const __grid_constant__ CUtensorMap tmH,
                                                                const TcArgs t) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const HeadArgs& a = t.h;
  const TcSmem L = tc_smem(t.S, t.N, a.nrows, a.lcap, t.online, a.k_t, t.box_cap);
  uint8_t* sa = smem + L.a;
  uint8_t* sb = smem + L.b;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + 16;
  uint64_t* tfull = empty + 16;
  uint64_t* tempty = tfull + 2;
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + L.slot);
  int4* boxes = reinterpret_cast<int4*>(smem + L.boxes);
  HeadCtx c;
  c.ring = sa;
  c.full = full;
  c.empty = empty;
  c.info = nullptr;
  c.misc = reinterpret_cast<int*>(smem + L.misc);
  c.red = reinterpret_cast<float*>(smem + L.red);
  c.sega = reinterpret_cast<long long*>(smem + L.sega);
  c.segn = reinterpret_cast<int*>(smem + L.segn);
  c.segi = reinterpret_cast<int*>(smem + L.segi);
  c.hs = nullptr;
  c.zl = reinterpret_cast<float*>(smem + L.zl);
  c.zid = reinterpret_cast<int*>(smem + L.zid);
  c.extra = nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < t.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
    for (int i = 0; i < 4; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmWs.w[i])) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
  }
  if (warp == 1) {  // TMEM accumulators: 2 x N fp32 columns, owned (and freed) by warp 1
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "r"(t.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  trace_mark(t.trace, 0);
  if (a.pdl) pdl_wait();
  head_segments(a, c);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;

  // boxes of <= 16 rows covering the segment, never crossing a cluster boundary
  if (threadIdx.x == 0) {
    int nb = 0;
    const int n = c.segn[0];
    if (n > 0) {
      const long long s0 = c.sega[0], s1 = s0 + n;
      const int32_t* so = a.sl_off;
      int i = c.segi[0];
      long long cl_beg = __ldcg(so + i), cl_end = __ldcg(so + i + 1);
      long long base = __ldg(a.offsets + __ldcg(a.sel + i));
      long long pos = s0;
      while (pos < s1 && nb < t.box_cap) {
        const long long lim = cl_end < s1 ? cl_end : s1;
        const int m = (int)min((long long)kTcBoxRows, lim - pos);
        boxes[nb++] = make_int4((int)(base + (pos - cl_beg)), (int)(pos - s0), m, __ldcg(a.sel + i));
        pos += m;
        if (pos == cl_end && pos < s1) {
          ++i;
          cl_beg = cl_end;
          cl_end = __ldcg(so + i + 1);
          base = __ldg(a.offsets + __ldcg(a.sel + i));
        }
      }
      if (pos < s1) nb = -1;  // segment too long for the box table: flag (host sizes lcap to avoid)
    }
    c.misc[1] = nb;
  }
  __syncthreads();
  const int nboxes = c.misc[1];
  const int ntiles = nboxes > 0 ? (nboxes + kTcBoxes - 1) / kTcBoxes : 0;
  const uint32_t S = (uint32_t)t.S;
  trace_mark(t.trace, 1);
  if (t.trace && threadIdx.x == 0) t.trace[blockIdx.x * 64 + 29] = (unsigned long long)ntiles;

  if (warp == 0) {
    if (lane == 0 && ntiles > 0) {
      const uint64_t pol_w = policy_evict_first(), pol_h = policy_evict_last();
      uint32_t it = 0;
      for (int tile = 0; tile < ntiles; ++tile) {
        const int b0 = tile * kTcBoxes, b1 = min(nboxes, b0 + kTcBoxes);
        // a tile of 8 full, consecutive 16-row boxes (inside one cluster run: most tiles) is one
        // 128-row box: the same swizzled shared-memory image with 8x fewer TMA operations.  (Splitting
        // partial tiles into 64/32-row groups measured +2.5% on the Qwen tree, -2.4% on Gemma.)
        bool contig = b1 - b0 == kTcBoxes;
        for (int b = b0; contig && b < b1; ++b)
          contig = boxes[b].z == kTcBoxRows && boxes[b].x == boxes[b0].x + (b - b0) * kTcBoxRows;
        const uint32_t bytes = (uint32_t)(b1 - b0) * kTcBoxRows * kTcK * 2 + (uint32_t)t.N * kTcK * 2;
        for (int kc0 = 0; kc0 < t.kchunks; kc0 += kTcKPS, ++it) {
          const uint32_t s = it % S;
          const int nk = min(kTcKPS, t.kchunks - kc0);
          mbar_wait(&empty[s], ((it / S) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], bytes * (uint32_t)nk);
          for (int j = 0; j < nk; ++j) {
            const int kc = kc0 + j;
            uint8_t* sa_j = sa + (size_t)s * kTcABytes + (size_t)j * (kTcABytes / kTcKPS);
            if (contig)
              tma_load_2d(sa_j, &tmWs.w[3], kc * kTcK, boxes[b0].x, &full[s], pol_w);
            else
              for (int b = b0; b < b1; ++b)
                tma_load_2d(sa_j + (size_t)(b - b0) * kTcBoxRows * 128, &tmWs.w[0], kc * kTcK, boxes[b].x, &full[s],
                            pol_w);
            tma_load_2d(sb + ((size_t)s * kTcKPS + j) * t.N * 128, &tmH, kc * kTcK, 0, &full[s], pol_h);
          }
        }
      }
      trace_mark_w(t.trace, 2);
    }
  } else if (warp == 1) {
    if (lane == 0 && ntiles > 0) {
      // instruction descriptor: D f32, A/B bf16, K-major both, N >> 3, M = 128 >> 4
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(t.N >> 3) << 17) | (8u << 24);
      uint32_t it = 0;
      for (int tile = 0; tile < ntiles; ++tile) {
        const int buf = tile & 1;
        mbar_wait(&tempty[buf], (((uint32_t)tile >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + (uint32_t)(buf * t.N);
        for (int kc0 = 0; kc0 < t.kchunks; kc0 += kTcKPS, ++it) {
          const uint32_t s = it % S;
          const int nk = min(kTcKPS, t.kchunks - kc0);
          mbar_wait(&full[s], (it / S) & 1u);
          tc_fence_after();
          for (int j = 0; j < nk; ++j) {
            const uint32_t abase = smem_u32(sa + (size_t)s * kTcABytes + (size_t)j * (kTcABytes / kTcKPS));
            const uint32_t bbase = smem_u32(sb + ((size_t)s * kTcKPS + j) * t.N * 128);
#pragma unroll
            for (int k = 0; k < kTcK / 16; ++k)
              tc_mma_bf16(d_tmem, sw128_desc(abase + k * 32), sw128_desc(bbase + k * 32), idesc,
                          (kc0 + j + k) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);  // slot reusable once these MMAs have read it
        }
        tc_commit(&tfull[buf]);  // accumulator complete
      }
      trace_mark_w(t.trace, 3);
    }
    __syncwarp();
  } else if (!t.online) {
    // epilogue warps 2..5: TMEM lane quarter q = warp % 4 holds tokens 32q .. 32q + 31 of a tile
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const int nr = a.nrows;
    for (int tile = 0; tile < ntiles; ++tile) {
      const int buf = tile & 1;
      mbar_wait(&tfull[buf], ((uint32_t)tile >> 1) & 1u);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * t.N);
      const int bi = tile * kTcBoxes + row / kTcBoxRows, r = row % kTcBoxRows;
      int local = -1, tok = 0;
      if (bi < nboxes) {
        const int4 bx = boxes[bi];
        if (r < bx.z) {
          local = bx.y + r;
          tok = __ldg(a.perm + bx.x + r);
        }
      }
      const long long vpos = c.sega[0] + local;
      for (int c0 = 0; c0 < t.N; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
        if (local >= 0) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int rr = c0 + j;
            if (rr < nr) {
              const float z = v[j] + 0.0f;
              c.zl[rr * a.lcap + local] = z;
              c.zid[rr * a.lcap + local] = tok;
              if (a.z_out) a.z_out[(size_t)rr * a.z_stride + vpos] = z;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
    if (warp == 2) trace_mark_w(t.trace, 4);
  } else {
    // online epilogue: stage the tile's logits (masked to each row's own clusters), then warp
    // ew = warp - 2 folds rows ew, ew + 4, ... into their running (max, sum exp) and top-k_t.
    const int q = warp & 3, ew = warp - 2;
    const int row = 32 * q + lane;
    const int nr = a.nrows, K = a.k_t;
    float* stage = reinterpret_cast<float*>(smem + L.stage);
    int* tokid = reinterpret_cast<int*>(smem + L.tokid);
    float* runm = reinterpret_cast<float*>(smem + L.runm);
    float* runs = reinterpret_cast<float*>(smem + L.runs);
    float2* lst = reinterpret_cast<float2*>(smem + L.lst);  // [2][nr][K] (value, id bits)
    float* sv = reinterpret_cast<float*>(smem + L.scr) + (size_t)ew * 2 * kTcScr;
    int* si = reinterpret_cast<int*>(sv + kTcScr);
    for (int i = threadIdx.x - 64; i < nr * K; i += 128) lst[i] = make_float2(-INFINITY, __int_as_float(INT_MAX));
    for (int i = threadIdx.x - 64; i < nr; i += 128) {
      runm[i] = -INFINITY;
      runs[i] = 0.f;
    }
    named_bar_sync(2, 128);
    long long cw = 0, cs = 0, cr = 0;
    for (int tile = 0; tile < ntiles; ++tile) {
      const int buf = tile & 1;
      const long long q0 = clock64();
      mbar_wait(&tfull[buf], ((uint32_t)tile >> 1) & 1u);
      tc_fence_after();
      const long long q1 = clock64();
      cw += q1 - q0;
      const int bi = tile * kTcBoxes + row / kTcBoxRows, r = row % kTcBoxRows;
      bool valid = false;
      int tok = INT_MAX, cl = 0;
      if (bi < nboxes) {
        const int4 bx = boxes[bi];
        if (r < bx.z) {
          valid = true;
          tok = __ldg(a.perm + bx.x + r);
          cl = bx.w;
        }
      }
      tokid[row] = tok;
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * t.N);
      for (int c0 = 0; c0 < t.N; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int rr = c0 + j;
          if (rr < nr) {
            bool ok = valid;
            if (ok && t.rowmask) ok = (__ldg(t.rowmask + (size_t)rr * 32 + (cl >> 5)) >> (cl & 31)) & 1u;
            stage[rr * 128 + row] = ok ? v[j] + 0.0f : -INFINITY;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      named_bar_sync(2, 128);
      const long long q2 = clock64();
      cs += q2 - q1;
      const int cur = tile & 1, nxt = cur ^ 1;
      for (int rr = ew; rr < nr; rr += 4) {
        const float* zr = stage + rr * 128;
        // tile (max, sum exp) of the row: max as one order-preserving integer reduction, then one
        // exp per logit against it and a fixed xor tree (R19); masked logits are -inf (exp = 0)
        const float x0 = zr[lane], x1 = zr[lane + 32], x2 = zr[lane + 64], x3 = zr[lane + 96];
        const uint32_t km = max(max(ord_key(x0), ord_key(x1)), max(ord_key(x2), ord_key(x3)));
        const uint32_t Km = __reduce_max_sync(0xffffffffu, km);
        const float m = __uint_as_float((Km & 0x80000000u) ? (Km & 0x7fffffffu) : ~Km);
        float se = 0.f;
        if (m != -INFINITY) se = warp_sum((expf(x0 - m) + expf(x1 - m)) + (expf(x2 - m) + expf(x3 - m)));
        if (lane == 0) {
          float M0 = runm[rr], S0 = runs[rr];
          lse_combine(M0, S0, m, se);
          runm[rr] = M0;
          runs[rr] = S0;
        }
        const float2* lc = lst + ((size_t)cur * nr + rr) * K;
        float2* ln = lst + ((size_t)nxt * nr + rr) * K;
        // a tile logit can enter the row's top-K only if >= its current K-th value (-inf: not full)
        if (m == -INFINITY || m < lc[K - 1].x) {
          for (int qq = lane; qq < K; qq += 32) ln[qq] = lc[qq];
          __syncwarp();
          continue;
        }
        const int nsv = warp_topk(
            128 + K, K,
            [&](int i, float& v, int& id) {
              if (i < 128) {
                v = zr[i];
                id = tokid[i];
              } else {
                v = lc[i - 128].x;
                id = __float_as_int(lc[i - 128].y);
              }
            },
            [&](int rank, float v, int id) { ln[rank] = make_float2(v, __int_as_float(id)); }, sv, si);
        for (int qq = nsv + lane; qq < K; qq += 32) ln[qq] = make_float2(-INFINITY, __int_as_float(INT_MAX));
        __syncwarp();
      }
      named_bar_sync(2, 128);
      cr += clock64() - q2;
    }
    if (t.trace && threadIdx.x == 64) {
      t.trace[blockIdx.x * 64 + 20] = cw;
      t.trace[blockIdx.x * 64 + 21] = cs;
      t.trace[blockIdx.x * 64 + 22] = cr;
    }
    // per-CTA partial records [row][cta][rec]
    const int fin = ntiles & 1;  // buffer holding the latest lists
    const int rec = 2 + 2 * K;
    for (int rr = ew; rr < nr; rr += 4) {
      float* P = a.part + ((size_t)rr * gridDim.x + blockIdx.x) * rec;
      const float2* lf = lst + ((size_t)fin * nr + rr) * K;
      for (int qq = lane; qq < K; qq += 32) {
        P[2 + 2 * qq] = lf[qq].x;
        P[3 + 2 * qq] = lf[qq].y;
      }
      if (lane == 0) {
        P[0] = runm[rr];
        P[1] = runs[rr];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(t.tmem_cols) : "memory");
  }
  trace_mark(t.trace, 5);
  if (a.pdl) pdl_launch_dependents();
  if (!t.online) head_partials(a, c, t.S * kTcABytes);
  trace_mark(t.trace, 6);
  const int j = head_ticket(a, c);
  if (j < 0) return;
  head_merge(a, c, t.S * kTcABytes, t.trace, 0, j, min(a.nrows, (int)gridDim.x));
  head_merge_done(a, 0);
  trace_mark(t.trace, 7);
}

// Union of B rows' selections (one CTA): per-row cluster bit masks + the ascending union with
// its sl_offsets — the shortlist the batched head streams once for all rows.
__global__ void __launch_bounds__(256) union_kernel(const int32_t* __restrict__ sel, const int32_t* __restrict__ cnt,
                                                    int B, int M, const int32_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ rowmask, int32_t* usel, int32_t* ucnt,
                                                    int32_t* usloff) {
  extern __shared__ __align__(16) uint32_t us[];
  pdl_wait();                 // the rows' selections come from the router (or the previous batch's head)
  pdl_launch_dependents();    // the head kernel may start its prologue; it waits for this grid
  uint32_t* acc = us;                                   // [32]
  uint32_t* rm = us + 32;                               // [B][32]
  int32_t* offs = reinterpret_cast<int32_t*>(rm + B * 32);  // [M+1]
  int32_t* tmp = offs + M + 1;                          // [M]
  for (int i = threadIdx.x; i < 32 + B * 32; i += blockDim.x) us[i] = 0u;
  for (int m = threadIdx.x; m <= M; m += blockDim.x) offs[m] = offsets[m];
  __syncthreads();
  // all rows at once (independent loads): entry i of row r for (r, i) in [0, B) x [0, M)
  for (int idx = threadIdx.x; idx < B * M; idx += blockDim.x) {
    const int r = idx / M, i = idx - r * M;
    if (i < __ldg(cnt + r)) {
      const int m = __ldg(sel + (size_t)r * M + i);
      atomicOr(&acc[m >> 5], 1u << (m & 31));
      atomicOr(&rm[r * 32 + (m >> 5)], 1u << (m & 31));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B * 32; i += blockDim.x) rowmask[i] = rm[i];
  emit_fast(acc, M, offs, usel, ucnt, usloff, tmp);
}

// ------------------------------------------------------------------ host side

struct TcPlan {
  HeadPlan hp;  // G, lcap, rec, part_bytes
  int N, S, tmem_cols, online, box_cap;
  size_t smem;
};

static bool tc_plan(const ds_clusters* c, int R, int k_t, int64_t max_shortlist, TcPlan* p, int online = 0) {
  if (c->dtype != DS_BF16 || R < 1 || R > (online ? 128 : 64) || (c->d % 8) != 0) return false;
  p->online = online;
  p->N = ((R + 15) / 16) * 16;
  p->tmem_cols = 32;
  while (p->tmem_cols < 2 * p->N) p->tmem_cols *= 2;
  p->hp.G = num_sms();
  const int64_t ms = (max_shortlist > 0 && max_shortlist < c->V) ? max_shortlist : c->V;
  p->hp.lcap = (int)((ms + p->hp.G - 1) / p->hp.G);
  p->box_cap = (p->hp.lcap + kTcBoxRows - 1) / kTcBoxRows + c->M;
  if (p->box_cap > kTcMaxBoxes) return false;
  if (online && k_t > kMaxKt) return false;
  p->hp.rec = 2 + 2 * k_t;
  p->hp.rows_per_launch = R;
  p->hp.launches = 1;
  p->hp.part_bytes = (size_t)p->hp.G * R * p->hp.rec * sizeof(float);
  const int smax = max_smem_optin();
  p->S = 0;
  for (int S = 12; S >= 3; --S) {
    if (S * kTcABytes < merge_smem_bytes(p->hp.G, k_t, kTcThreads / 32) || p->hp.G > 32 * (kTcThreads / 32)) break;
    if ((int)tc_smem(S, p->N, R, p->hp.lcap, online, k_t, p->box_cap).total <= smax) {
      p->S = S;
      break;
    }
  }
  if (p->S == 0) return false;
  p->smem = tc_smem(p->S, p->N, R, p->hp.lcap, online, k_t, p->box_cap).total;
  return encode_fn() != nullptr;
}

// Batched per-row mode: rows with their own selections, streamed once as their union.
constexpr int kTcBatchRows = 128;

bool tc_batched_supported(const ds_clusters* c, int B, int k_t) {
  TcPlan p;
  return c->M <= 1024 && tc_plan(c, std::min(B, kTcBatchRows), k_t, 0, &p, 1);
}

size_t tc_batched_ws_bytes(const ds_clusters* c, int B, int k_t) {
  TcPlan p;
  if (!tc_plan(c, std::min(B, kTcBatchRows), k_t, 0, &p, 1)) return 0;
  const int rows = std::min(B, kTcBatchRows);
  return align_up(p.hp.part_bytes, 256) + align_up((size_t)rows * 32 * 4, 256) +
         align_up((size_t)(2 * c->M + 8) * 4, 256);
}

static bool make_maps(TcMaps* m, const ds_clusters* c) {
  for (int j = 0; j < 4; ++j)
    if (!make_map(&m->w[j], c->W_perm, (uint64_t)c->V, (uint64_t)c->d, (uint32_t)(kTcBoxRows << j))) return false;
  return true;
}

static cudaError_t launch_tc_kernel(const TcPlan& p, const TcMaps& mw, const CUtensorMap& mh, const TcArgs& t,
                                    cudaStream_t st, bool pdl) {
  static int configured[64] = {0};  // the attribute is per device
  {
    cudaError_t e = configure_max_smem(reinterpret_cast<const void*>(tc_head_kernel), configured);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.hp.G);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, tc_head_kernel, mw, mh, t);
}

cudaError_t launch_tc_batched(const ds_clusters* c, const void* h_new, int B, const int32_t* sel,
                              const int32_t* sel_count, int k_t, int32_t* top_ids, float* top_logits,
                              float* top_logp, float* lse, void* ws, unsigned* counter, cudaStream_t st) {
  const int esz = 2;
  for (int r0 = 0; r0 < B; r0 += kTcBatchRows) {
    const int nr = std::min(kTcBatchRows, B - r0);
    TcPlan p;
    if (!tc_plan(c, nr, k_t, 0, &p, 1)) return cudaErrorInvalidValue;
    uint8_t* w8 = static_cast<uint8_t*>(ws);
    float* part = reinterpret_cast<float*>(w8);
    uint32_t* rowmask = reinterpret_cast<uint32_t*>(w8 + align_up(p.hp.part_bytes, 256));
    int32_t* usel = reinterpret_cast<int32_t*>(w8 + align_up(p.hp.part_bytes, 256) +
                                               align_up((size_t)std::min(B, kTcBatchRows) * 32 * 4, 256));
    int32_t* ucnt = usel + c->M;
    int32_t* usloff = ucnt + 4;
    const size_t usm = (size_t)(32 + nr * 32) * 4 + (size_t)(2 * c->M + 1) * 4;
    cudaLaunchConfig_t uc = {};
    uc.gridDim = dim3(1);
    uc.blockDim = dim3(256);
    uc.dynamicSmemBytes = usm;
    uc.stream = st;
    cudaLaunchAttribute ua[1];
    ua[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ua[0].val.programmaticStreamSerializationAllowed = 1;
    uc.attrs = ua;
    uc.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&uc, union_kernel, sel + (size_t)r0 * c->M, sel_count + r0, nr, c->M,
                                       (const int32_t*)c->offsets, rowmask, usel, ucnt, usloff);
    if (e != cudaSuccess) return e;
    TcMaps mw;
    CUtensorMap mh;
    if (!make_maps(&mw, c)) return cudaErrorInvalidValue;
    const void* h0 = static_cast<const uint8_t*>(h_new) + (size_t)r0 * c->d * esz;
    if (!make_map(&mh, h0, (uint64_t)nr, (uint64_t)c->d, (uint32_t)p.N)) return cudaErrorInvalidValue;
    TcArgs t;
    fill_head_args(t.h, c, p.hp, h0, 0, nr, usel, ucnt, usloff, 1, k_t, 0, top_ids + (size_t)r0 * k_t,
                   top_logits + (size_t)r0 * k_t, top_logp + (size_t)r0 * k_t, lse + r0, nullptr, 0, part, counter,
                   true);
    t.h.h = h0;
    t.N = p.N;
    t.S = p.S;
    t.kchunks = (c->d + kTcK - 1) / kTcK;
    t.tmem_cols = p.tmem_cols;
    t.online = 1;
    t.rowmask = rowmask;
    t.trace = debug_trace();
    t.box_cap = p.box_cap;
    e = launch_tc_kernel(p, mw, mh, t, st, true);  // PDL after the union kernel
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

bool tc_head_supported(const ds_clusters* c, int R, int k_t, int64_t max_shortlist) {
  TcPlan p;
  return th_supported(c, R, k_t) || tc_plan(c, R, k_t, max_shortlist, &p);
}

size_t tc_head_part_bytes(const ds_clusters* c, int R, int k_t) {
  TcPlan p;
  return std::max(tc_plan(c, R, k_t, 0, &p) ? p.hp.part_bytes : (size_t)0, th_ws_bytes(c, R, k_t));
}

cudaError_t launch_tc_head(const ds_clusters* c, const void* h_new, int R, const int32_t* sel,
                           const int32_t* sel_count, const int32_t* sl_offsets, int k_t, int64_t max_shortlist,
                           int32_t* top_ids, float* top_logits, float* top_logp, float* lse, float* z_out,
                           int64_t z_stride, float* part, unsigned* counter, cudaStream_t st, bool pdl) {
  // shared (tree) mode keeps the logits on chip for the per-CTA partial: at tree-depth shortlists a
  // CTA holds 1-2 tiles, where the online per-tile epilogue measured slower (Qwen tree 89 vs 97 us)
  // Epilogue choice by the per-CTA logit bound lcap: <= 4 tiles keep the logits on chip for one
  // per-CTA partial (Qwen tree depths: 94 vs 96 us online); more use the online per-tile running
  // (max, sum, top-k) (dense k = M on the Qwen head: 255 vs 526+ us).  z_out needs the logits.
  // <= 16 tree rows: the balanced tree head (th.cu)
  if (th_supported(c, R, k_t))
    return launch_th(c, h_new, R, sel, sel_count, sl_offsets, k_t, max_shortlist, top_ids, top_logits, top_logp, lse,
                     z_out, z_stride, part, counter, st, pdl);
  TcPlan p;
  if (!tc_plan(c, R, k_t, max_shortlist, &p, 0)) return cudaErrorInvalidValue;
  const char* ov = getenv("DS_TC_ONLINE");  // "0" / "1": force (tuning)
  const bool force = ov && (ov[0] == '0' || ov[0] == '1');
  const bool online = !z_out && (force ? ov[0] == '1' : p.hp.lcap > 4 * 128);
  if (online) {
    TcPlan po;
    if (tc_plan(c, R, k_t, max_shortlist, &po, 1)) p = po;
  }
  TcMaps mw;
  CUtensorMap mh;
  if (!make_maps(&mw, c)) return cudaErrorInvalidValue;
  if (!make_map(&mh, h_new, (uint64_t)R, (uint64_t)c->d, (uint32_t)p.N)) return cudaErrorInvalidValue;
  TcArgs t;
  fill_head_args(t.h, c, p.hp, h_new, 0, R, sel, sel_count, sl_offsets, 1, k_t, max_shortlist, top_ids, top_logits,
                 top_logp, lse, z_out, z_stride, part, counter, pdl);
  t.N = p.N;
  t.S = p.S;
  t.kchunks = (c->d + kTcK - 1) / kTcK;
  t.tmem_cols = p.tmem_cols;
  t.online = p.online;
  t.rowmask = nullptr;
  t.trace = debug_trace();
  t.box_cap = p.box_cap;
  return launch_tc_kernel(p, mw, mh, t, st, pdl);
}

}  // namespace ds
