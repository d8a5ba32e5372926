// th.cu — S5' for tree rows: R <= 16 draft rows sharing ONE shortlist (Alg. 1 line 8: one index
// set I for all beam rows of a depth; line 10 P:262; "computes on Tensor Cores").
//
// Z[R x |V_S|] = H[R x d] W_S^T with swap-AB (vocabulary = MMA-M = 128, rows = MMA-N = 16): per CTA
//   D[128 tokens x 16] (fp32, TMEM, two buffers) += A[128 x 64] (W_perm rows, SW128) B[16 x 64]^T (H).
//
// Why a second tree head (tc_head.cu is the general one): at tree depths the union is 6-25k rows,
// i.e. 40-200 rows per SM, so what costs is not the contraction but how the rows are fetched and
// everything around the stream.  Here:
//   * CTA ranges snapped to clusters: cluster i of the union owns CTAs [s_i, s_(i+1)),
//     s_i = round(G so_i / |V_S|), its 8-row groups split evenly over them (a cluster too small for a
//     CTA of its own goes whole to CTA min(s_i, G - 1)); found per CTA by one division-free binary
//     search.  Every tile (<= 128 rows) is one contiguous W_perm row range, loaded with ONE 3-D TMA
//     box {64, h, c} per 32 KB ring slot — c K chunks at once (16 maps, h = 8..128); small 2-D boxes
//     per K chunk measured ~125 ns of fixed cost per op.
//   * H (<= 16 rows x d) loaded ONCE by one 3-D box and kept in shared memory (8 rows per K chunk
//     when R <= 8: the MMA's upper 8-row atom is then the next chunk's, garbage in unused D columns).
//   * roles: warp 0 lane 0 TMA producer; warp 1 lane 0 MMA issuer (4 x K = 16 per chunk,
//     tcgen05.commit frees the slot / publishes the tile); warps 2-5 drain TMEM (tcgen05.ld
//     32x32b, one vocabulary row per thread, the R logits in registers) and write z[r][pos]
//     (z_out, or workspace scratch); warps 6-9 join the tail.
//   * tail: keys (logit, token id) staged in the freed ring + H, one warp per row reduces the CTA's
//     record (max, sum exp, k_t best keys: direct rank count, or a lane-maximum threshold + rank
//     count); a 64-bit epoch arrival ticket makes the last R CTAs per-row mergers (bounded spin until
//     all G arrived): lse by a fixed fold over the records in CTA order (R19), top-k_t by a head
//     threshold + rank count.
//   * modes: shared (tree rows; the union either staged from the router's selection or formed here
//     from the rows' published masks — deferred union) and rows (independent rows, R9 shared = 0:
//     the union of their clusters streamed once, per-tile row masks, each row over its own clusters).
// Exactness: bf16 x bf16 products are exact in fp32; in the exact regime every partial sum is an
// integer below 2^24, so the logits equal the oracle's bit for bit whatever the MMA order.
#include <cuda.h>

#include <algorithm>

#include "internal.h"
#include "keys.cuh"
#include "tc_common.cuh"

namespace ds {

constexpr int kThThreads = 320;          // 10 warps: 0 TMA, 1 MMA, 2-5 epilogue; all 10 in the tail
constexpr int kThWarps = kThThreads / 32;
constexpr int kThN = 16;                 // MMA N: rows padded to 16
constexpr int kThSlot = 32768;           // ring slot bytes
constexpr int kThMaxPieces = 256;
constexpr int kThMaxKt = 16;
constexpr int kThMaxG = 160;             // merge: <= 5 records per lane

constexpr int kThMaps = 16;              // 3-D W_perm views, box heights 8 (j + 1)

// K chunks per TMA box (and ring slot) for a tile of h rows: h x c x 128 B <= 32 KB, c <= 8
__host__ __device__ constexpr int th_cpc(int h) { return 256 / h < 8 ? 256 / h : 8; }

struct ThMaps {
  CUtensorMap w[kThMaps];  // W_perm as (64 elements, rows, K chunk): box {64, h, th_cpc(h)}
};

struct ThArgs {
  const int32_t* sel;        // shared: [M] union; rows mode: [R][M] per-row selections
  const int32_t* sel_count;  // shared: [1]; rows mode: [R]
  unsigned long long* umask;        // shared mode, deferred union (nullable): the R rows' TopK masks as
                                    // published by the few-row router ([R][32] tagged words); the union,
                                    // sel / sel_count / sl_offsets are then built (and written) here
  int32_t* usel;                    // deferred union outputs (CTA 0 writes them)
  int32_t* ucnt;
  int32_t* usloff;
  const int32_t* sl_off;
  const int32_t* offsets;
  const int32_t* perm;
  int32_t R, kchunks, K, S, cap, M;
  int32_t hr;  // H rows stored per K chunk (8 when R <= 8, else 16)
  int64_t V;  // cap: union positions per CTA (token-id buffer)
  int32_t rstride;                   // record words per row (G (2 + K), even)
  int64_t max_shortlist;          // > 0: a union longer than this is not computed (dynaspec.h)
  float* z;                       // [R][z_stride] logits by union position
  int64_t z_stride;
  int32_t* top_ids;
  float* top_logits;
  float* top_logp;
  float* lse;
  unsigned long long* rec;  // [R][G][2 + K] (row stride rstride words)
  unsigned* counter;        // 64-bit arrival count (8-byte aligned), never reset: epoch = count / G
  unsigned* err;            // workspace error word
  int32_t rows;  // 1: independent rows (R9 shared = 0): stream the union of the rows' clusters once,
                 // each row's (max, sum, top-k_t) over its OWN clusters only (per-tile row masks)
  int32_t pdl;
  int32_t dbg;  // DS_TH_DBG (timing experiments): 1 = no MMAs
  unsigned long long* trace;
};

struct ThSmem {
  uint32_t ring, h, bars, misc, pieces, ppos, cmask, tmask, rtot, sel, slo, off, tok, total;
};

__host__ __device__ inline ThSmem th_smem(int S, int kchunks, int cap, int M, int hr) {
  ThSmem L;
  uint32_t o = 0;
  L.ring = o;
  o += (uint32_t)S * kThSlot;
  L.h = o;  // directly after the ring: the MMA's 128-row reads of a short tile spill into H (harmless)
  o += (uint32_t)kchunks * hr * 128;  // H rows stored per K chunk: 8 (R <= 8) or 16
  o = (o + 1023u) & ~1023u;
  if (o < L.h + kThSlot) o = L.h + kThSlot;  // the spill window exists even for tiny d
  L.bars = o;
  o += (2 * 16 + 8) * 8;
  L.misc = o;
  o += 64 * 4;
  L.pieces = o;
  o += kThMaxPieces * 16;
  L.ppos = o;
  o += kThMaxPieces * 4;
  L.cmask = o;  // [M] rows that selected cluster m (rows mode)
  o += (uint32_t)M * 4;
  L.tmask = o;  // [kThMaxPieces] row mask of each tile
  o += kThMaxPieces * 4;
  L.rtot = o;   // [16] per-row |V_S,r| (rows mode)
  o += 16 * 4;
  L.sel = o;
  o += (uint32_t)M * 4;
  L.slo = o;
  o += (uint32_t)(M + 1) * 4;
  L.off = o;
  o += (uint32_t)(M + 1) * 4;
  L.total = o;
  (void)cap;
  return L;
}

// largest key strictly below `below` among n keys of v (lane-strided); 0 if none
__device__ __forceinline__ unsigned long long th_best_below(const unsigned long long* v, int n, int lane,
                                                            unsigned long long below) {
  unsigned long long b = 0ull;
  for (int i = lane; i < n; i += 32) {
    const unsigned long long x = v[i];
    if (x < below && x > b) b = x;
  }
  return b;
}

// warp max of unique 64-bit keys (two REDUX rounds)
__device__ __forceinline__ unsigned long long th_warp_max64(unsigned long long x) {
  const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(x >> 32));
  const uint32_t lo = __reduce_max_sync(0xffffffffu, (uint32_t)(x >> 32) == hi ? (uint32_t)x : 0u);
  return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ float ord_to_float(uint32_t mk) {
  return mk ? __uint_as_float((mk & 0x80000000u) ? (mk & 0x7fffffffu) : ~mk) : -INFINITY;
}


// The K best of n unique nonzero keys v[0..n) by one warp, written to out[0..K) in descending order
// (0-padded): T = the K-th largest of the 32 lane maxima (each lane's maximum is a distinct key, so
// >= K keys are >= T), the keys >= T are compacted to cand[] and each is rank-counted against the
// others.  No sequential rounds.  Zero keys are ignored.  Returns min(#nonzero keys, K).
__device__ __forceinline__ int th_warp_topk(const unsigned long long* v, int n, int K, int lane,
                                            unsigned long long* cand, unsigned long long* out) {
  if (n <= 96) {  // short lists: every nonzero key rank-counted against all n directly (no threshold)
    int nz = 0;
    for (int i = lane; i < n; i += 32) {
      const unsigned long long x = v[i];
      nz += x != 0ull;
      if (x == 0ull) continue;
      int r0 = 0, r1 = 0;
      int j = 0;
#pragma unroll 4
      for (; j + 1 < n; j += 2) {
        r0 += v[j] > x ? 1 : 0;
        r1 += v[j + 1] > x ? 1 : 0;
      }
      if (j < n) r0 += v[j] > x ? 1 : 0;
      if (r0 + r1 < K) out[r0 + r1] = x;
    }
    nz = (int)__reduce_add_sync(0xffffffffu, (unsigned)nz);
    const int nv = min(nz, K);
    for (int j = nv + lane; j < K; j += 32) out[j] = 0ull;
    __syncwarp();
    return nv;
  }
  unsigned long long lm = 0ull;
#pragma unroll 4
  for (int i = lane; i < n; i += 32) lm = v[i] > lm ? v[i] : lm;
  int rk = 0;  // rank of this lane's maximum among the lane maxima
#pragma unroll 8
  for (int o = 0; o < 32; ++o) rk += __shfl_sync(0xffffffffu, lm, o) > lm ? 1 : 0;
  const unsigned sel = __ballot_sync(0xffffffffu, lm != 0ull && rk == K - 1);
  const unsigned long long T = sel ? __shfl_sync(0xffffffffu, lm, __ffs(sel) - 1) : 0ull;
  int c = 0, nz = 0;  // zero keys (positions outside the row's own clusters) never count
#pragma unroll 4
  for (int i = lane; i < n; i += 32) {
    c += (v[i] >= T && v[i] != 0ull) ? 1 : 0;
    nz += v[i] != 0ull ? 1 : 0;
  }
  nz = (int)__reduce_add_sync(0xffffffffu, (unsigned)nz);
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const int nc = __shfl_sync(0xffffffffu, inc, 31);
  int w = inc - c;
  for (int i = lane; i < n; i += 32)
    if (v[i] >= T && v[i] != 0ull) cand[w++] = v[i];
  __syncwarp();
  for (int i = lane; i < nc; i += 32) {
    const unsigned long long x = cand[i];
    int r = 0;
#pragma unroll 8
    for (int j = 0; j < nc; ++j) r += cand[j] > x ? 1 : 0;
    if (r < K) out[r] = x;
  }
  const int nv = min(nz, K);
  for (int j = nv + lane; j < K; j += 32) out[j] = 0ull;
  __syncwarp();
  return nv;
}

constexpr unsigned long long kThSpinNs = 2000000000ull;

__global__ void __launch_bounds__(kThThreads, 1) th_kernel(const __grid_constant__ ThMaps tmW,
                                                           const __grid_constant__ CUtensorMap tmH,
                                                           const __grid_constant__ ThArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const ThSmem L = th_smem(a.S, a.kchunks, a.cap, a.M, a.hr);
  uint8_t* ring = smem + L.ring;
  uint8_t* hs = smem + L.h;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + 16;
  uint64_t* hbar = empty + 16;
  uint64_t* tfull = hbar + 1;   // [2]
  uint64_t* tempty = tfull + 2; // [2]
  int* misc = reinterpret_cast<int*>(smem + L.misc);
  int4* pc = reinterpret_cast<int4*>(smem + L.pieces);  // tiles: (W_perm row, union position, rows loaded, valid)
  int* ssel = reinterpret_cast<int*>(smem + L.sel);
  int* sslo = reinterpret_cast<int*>(smem + L.slo);
  int* soff = reinterpret_cast<int*>(smem + L.off);
  uint32_t* cmask = reinterpret_cast<uint32_t*>(smem + L.cmask);
  uint32_t* tmask = reinterpret_cast<uint32_t*>(smem + L.tmask);
  int* rtot = reinterpret_cast<int*>(smem + L.rtot);
  int* rcnt = reinterpret_cast<int*>(smem + L.misc) + 32;  // [16]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, b = blockIdx.x, R = a.R, K = a.K, M = a.M;

  if (tid == 0) {
    for (int s = 0; s < a.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(hbar, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
    for (int i = 0; i < kThMaps; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW.w[i])) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
  }
  if (warp == 1) {  // TMEM: 2 x 16 fp32 columns, owned (and freed) by warp 1
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(misc)), "r"(32)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // cluster offsets are static (not produced upstream): staged before the dependency wait
  for (int i = tid; i <= M; i += kThThreads) soff[i] = __ldg(a.offsets + i);
  for (int i = tid; i < M; i += kThThreads) cmask[i] = 0u;
  trace_mark(a.trace, 0);
  if (a.pdl) pdl_wait();
  trace_mark(a.trace, 13);  // dependency released
  __syncthreads();  // barriers initialised
  if (tid == 0) {  // H (produced upstream) as soon as the wait is over: ONE 3-D box, all K chunks
    mbar_arrive_expect_tx(hbar, (uint32_t)a.kchunks * a.hr * 128);
    tma_load_3d(hs, &tmH, 0, 0, 0, hbar, policy_evict_last());
  }
  if (!a.rows && a.umask) {
    // tree rows, deferred union: OR the rows' masks (one round of loads), then the union in
    // ascending id with its offsets — the router's union step, done where it is consumed
    if (tid < 32) {
      uint32_t u = 0u;
      const int words = (M + 31) >> 5;
      if (tid < words)
        for (int r = 0; r < R; ++r) u |= (uint32_t)__ldcg(a.umask + (size_t)r * 32 + tid);
      rcnt[tid] = (int)u;  // scratch: union word tid
    }
    __syncthreads();
    for (int m = tid; m < M; m += kThThreads) cmask[m] = ((uint32_t)rcnt[m >> 5] >> (m & 31)) & 1u ? ~0u : 0u;
    __syncthreads();
  }
  if (!a.rows && !a.umask) {
    // the selection (count, ids, offsets) in one round of loads, whatever the count
    if (tid == 32) misc[7] = __ldcg(a.sel_count);
#pragma unroll 4
    for (int i = tid; i < 2 * M + 1; i += kThThreads) {
      if (i < M) ssel[i] = __ldcg(a.sel + i);
      else sslo[i - M] = __ldcg(a.sl_off + (i - M));
    }
    __syncthreads();
  } else {
    // independent rows: cluster m -> the rows that selected it; then the union in ascending id
    // (R8) with its offsets, exactly as a shared selection (deferred union: cmask is set above)
    if (a.rows && tid < R) {
      const int cr = __ldcg(a.sel_count + tid);
      rcnt[tid] = cr;
      rtot[tid] = cr > 0 ? __ldcg(a.sl_off + (size_t)tid * (M + 1) + cr) : 0;
    }
    __syncthreads();
    if (a.rows) {
#pragma unroll 4
      for (int idx = tid; idx < R * M; idx += kThThreads) {
        const int r = idx / M, i = idx - r * M;
        if (i < rcnt[r]) atomicOr(&cmask[__ldcg(a.sel + idx)], 1u << r);
      }
      __syncthreads();
    }
    // the union in ascending id with its offsets: 32-cluster chunks over all warps (per-chunk count
    // and size, then each chunk's base from the chunks before it)
    int* ccnt = reinterpret_cast<int*>(ring);  // [32] (the ring is idle until the plan)
    int* csz = ccnt + 32;
    const int nchunk = (M + 31) >> 5;
    for (int ch = warp; ch < nchunk; ch += kThWarps) {
      const int m = ch * 32 + lane;
      const bool f = m < M && cmask[m] != 0u;
      const int sz = f ? soff[m + 1] - soff[m] : 0;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      const int tot = (int)__reduce_add_sync(0xffffffffu, (unsigned)sz);
      if (lane == 0) {
        ccnt[ch] = __popc(bal);
        csz[ch] = tot;
      }
    }
    __syncthreads();
    for (int ch = warp; ch < nchunk; ch += kThWarps) {
      int run = 0, off = 0;
      for (int c2 = 0; c2 < ch; ++c2) {
        run += ccnt[c2];
        off += csz[c2];
      }
      const int m = ch * 32 + lane;
      const bool f = m < M && cmask[m] != 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      const int sz = f ? soff[m + 1] - soff[m] : 0;
      int inc = sz;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (f) {
        const int pos = run + __popc(bal & ((1u << lane) - 1u));
        ssel[pos] = m;
        sslo[pos] = off + inc - sz;
      }
      if (ch == nchunk - 1 && lane == 0) {
        misc[7] = run + __popc(bal);
        sslo[run + __popc(bal)] = off + csz[ch];
      }
    }
    __syncthreads();
    if (!a.rows && b == 0) {  // deferred union: the S3/S4 outputs of the step
      const int cnt = misc[7];
      for (int i = tid; i <= cnt; i += kThThreads) {
        if (i < cnt) a.usel[i] = ssel[i];
        a.usloff[i] = sslo[i];
      }
      if (tid == 0) *a.ucnt = cnt;
    }
  }
  trace_mark(a.trace, 14);  // selection staged

  // ---- plan (warp 0): this CTA's tiles.  Cluster i of the union (positions [so_i, so_i + n_i))
  // owns CTAs [s_i, s_(i+1)), s_i = round(G so_i / |V_S|); its 8-row groups are split evenly over
  // them, so a CTA's rows come from ONE cluster — one W_perm row range, one 3-D TMA box per stage.
  // A cluster too small for a CTA of its own (s_i = s_(i+1)) goes whole to CTA min(s_i, G - 1).
  // Tiles: <= 128 rows of one cluster (the last reads up to 7 rows past it, masked).
  if (warp == 0) {
    const int cnt = misc[7];
    const int total = cnt > 0 ? sslo[cnt] : 0;
    const bool fits = cnt > 0 && cnt <= M &&
                      (a.rows || a.max_shortlist <= 0 || (long long)total <= a.max_shortlist);
    const int ncl = fits ? cnt : 0;
    const unsigned NU = total > 0 ? (unsigned)total : 1u;  // 2 G |V_S| + |V_S| < 2^32 (host: V G < 2^30)
    // s(i) is monotone, so this CTA's clusters are a contiguous index range found by one binary
    // search (lane 0): i* = the last cluster with s(i*) <= b, then back over the clusters with
    // s(i) = s(i*) = b (small clusters rounded onto b; at b = G - 1 also s(i) = G).
    int nt = 0, p0 = INT_MAX, p1 = 0;
    if (lane == 0 && ncl > 0) {
      auto sidx = [&](int i) -> int {
        return i >= ncl ? G : (int)(((unsigned)G * (unsigned)sslo[i] * 2u + NU) / (2u * NU));
      };
      // min(s(i), G - 1) <= b  <=>  b = G - 1, or 2 G so_i < (2 b + 1) |V_S| (division-free)
      const unsigned long long lim = (unsigned long long)(2 * b + 1) * NU;
      int lo = 0, hi = ncl - 1;  // s(0) = 0 <= b
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b == G - 1 || 2ull * (unsigned long long)G * (unsigned)sslo[mid] < lim) lo = mid;
        else hi = mid - 1;
      }
      const int istar = lo;
      int first = istar;
      while (first > 0 && min(sidx(first - 1), G - 1) == b && min(sidx(first), G - 1) == b) --first;
      for (int i = first; i <= istar; ++i) {
        const int so = sslo[i], n = sslo[i + 1] - so, m = ssel[i];
        const int si = sidx(i), sn = sidx(i + 1);
        int r0 = 0, r1 = 0;
        if (sn > si) {
          if (b >= si && b < sn) {
            const int c = sn - si, j = b - si, ng = (n + 7) >> 3;
            r0 = min(n, 8 * (int)(((unsigned)j * (unsigned)ng) / (unsigned)c));
            r1 = min(n, 8 * (int)(((unsigned)(j + 1) * (unsigned)ng) / (unsigned)c));
          }
        } else if (min(si, G - 1) == b) {
          r1 = n;
        }
        if (r1 > r0) {
          const int wbase = soff[m];
          for (int r = r0; r < r1 && nt < kThMaxPieces; r += 128, ++nt) {
            const int len = min(128, r1 - r);
            pc[nt] = make_int4(wbase + r, so + r, (len + 7) & ~7, len);  // (W_perm row, position, rows, valid)
            tmask[nt] = a.rows ? cmask[m] : 0xffffffffu;
          }
          p0 = min(p0, so + r0);
          p1 = max(p1, so + r1);
        }
      }
    }
    const int P0 = (int)__reduce_min_sync(0xffffffffu, (unsigned)p0);
    const int P1 = (int)__reduce_max_sync(0xffffffffu, (unsigned)p1);
    if (lane == 0) {
      const bool over = nt > kThMaxPieces || (nt > 0 && P1 - P0 > a.cap);
      misc[1] = over ? 0 : nt;
      misc[3] = nt > 0 ? P0 : 0;  // first union position
      misc[4] = nt > 0 ? P1 : 0;  // one past the last
      misc[5] = fits ? 1 : 0;
      if (over) atomicExch(a.err, (unsigned)DS_ERR_UNSUPPORTED);  // plan bounds (host sizes cap)
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = (uint32_t)misc[0];
  const int ntiles = misc[1], P0 = misc[3];
  const int P1 = ntiles > 0 ? misc[4] : P0;
  const uint32_t S = (uint32_t)a.S;
  trace_mark(a.trace, 1);
  if (warp == 2) {  // token ids of this CTA's rows into L2 now (read by the record phase after the stream)
    for (int t = lane; t < ntiles; t += 32) {
      const int4 tq = pc[t];
      const uintptr_t lo = reinterpret_cast<uintptr_t>(a.perm + tq.x) & ~(uintptr_t)15;
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(a.perm + tq.x + tq.w) + 15) & ~(uintptr_t)15;
      bulk_prefetch_l2(reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo));
    }
  }

  if (warp == 0) {
    if (lane == 0 && ntiles > 0) {
      const uint64_t pol_w = policy_evict_first();
      uint32_t it = 0;
      for (int tile = 0; tile < ntiles; ++tile) {
        const int4 tq = pc[tile];
        const int h = tq.z, cpc = th_cpc(h);
        const CUtensorMap* map = &tmW.w[(h >> 3) - 1];
        for (int kc0 = 0; kc0 < a.kchunks; kc0 += cpc, ++it) {
          const uint32_t s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], (uint32_t)(cpc * h * 128));  // out-of-range chunks count (zero fill)
          tma_load_3d(ring + (size_t)s * kThSlot, map, 0, tq.x, kc0, &full[s], pol_w);
        }
      }
      trace_mark_w(a.trace, 7);  // last load issued
    }
  } else if (warp == 1) {
    if (lane == 0 && ntiles > 0) {
      // instruction descriptor: D f32, A/B bf16, K-major both, N >> 3, M = 128 >> 4
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kThN >> 3) << 17) | (8u << 24);
      mbar_wait(hbar, 0);
      tc_fence_after();
      trace_mark_w(a.trace, 5);  // H landed
      uint32_t it = 0;
      for (int tile = 0; tile < ntiles; ++tile) {
        const int buf = tile & 1;
        const int r8 = pc[tile].z;
        const int cpc = th_cpc(r8);
        mbar_wait(&tempty[buf], (((uint32_t)tile >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + (uint32_t)(buf * kThN);
        for (int kc0 = 0; kc0 < a.kchunks; kc0 += cpc, ++it) {
          const uint32_t s = it % S;
          const int nk = min(cpc, a.kchunks - kc0);
          mbar_wait(&full[s], (it / S) & 1u);
          tc_fence_after();
          if (it == 0) trace_mark_w(a.trace, 6);  // first slot landed
          if (a.dbg & 1) {
            tc_commit(&empty[s]);
            continue;
          }
          for (int j = 0; j < nk; ++j) {
            const uint32_t abase = smem_u32(ring + (size_t)s * kThSlot + (size_t)j * r8 * 128);
            // B = 16 H rows at SBO 1024: with 8 stored rows per chunk the upper atom is the next
            // chunk's (or the region after H): garbage in D columns 8..15, which no row reads
            const uint32_t bbase = smem_u32(hs + (size_t)(kc0 + j) * a.hr * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_bf16(d_tmem, sw128_desc(abase + k * 32), sw128_desc(bbase + k * 32), idesc,
                          (kc0 + j + k) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);  // the slot is free once these MMAs have read it
        }
        tc_commit(&tfull[buf]);  // accumulator complete
      }
      trace_mark_w(a.trace, 8);  // last MMA issued
    }
    __syncwarp();
  } else if (warp < 6) {
    // warps 2..5: TMEM lane quarter q = warp % 4 holds rows 32q .. 32q + 31 of a tile
    const int q = warp & 3;
    for (int tile = 0; tile < ntiles; ++tile) {
      const int buf = tile & 1;
      mbar_wait(&tfull[buf], ((uint32_t)tile >> 1) & 1u);
      tc_fence_after();
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * kThN), v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      const int4 tq = pc[tile];
      const int i = 32 * q + lane;
      if (i < tq.w) {
        const int pos = tq.y + i;
#pragma unroll
        for (int r = 0; r < kThN; ++r)
          if (r < R) a.z[(size_t)r * a.z_stride + pos] = v[r] + 0.0f;  // -0 -> +0 (R23)
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32) : "memory");
  }
  trace_mark(a.trace, 2);

  if (a.trace && tid == 0) a.trace[b * 64 + 12] = (unsigned long long)(P1 - P0);  // positions of this CTA
  // ---- per-CTA record of every row (layout [R][G][rec]).  Phase A: all threads stage the keys
  // (logit, token id) of rb rows x n positions in the free ring + H (one round of loads); phase B:
  // warp w reduces rows w, w + 6, ... of the batch from shared memory.
  const int n = P1 - P0;
  const int rec = 2 + K;
  const size_t rstride = (size_t)a.rstride;  // words per row: G rec rounded up to even
  {
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(ring);
    // rb rows of keys + one candidate buffer of n keys per warp
    // one row per warp when the staging holds R rows of keys + a candidate buffer per warp, else
    // six record warps (the host sizes the staging for rows of keys + 6 candidate buffers)
    const size_t stage_keys = (size_t)(L.bars - L.ring) / 8;
    const int nwr = (n > 0 && (size_t)(R + kThWarps) * n > stage_keys) ? 6 : kThWarps;
    const int rb = n > 0 ? min(R, (int)(stage_keys / (size_t)n) - nwr) : R;
    unsigned long long* cand = keys + (size_t)rb * n;
    for (int rb0 = 0; rb0 < R; rb0 += rb) {
      const int nr = min(rb, R - rb0);
      __syncthreads();  // the previous batch's keys are consumed
      constexpr int kB = 8;  // loads in flight per thread: every (z, token) pair of a batch first
      for (int base = tid; base < nr * n; base += kB * kThThreads) {
        float z[kB];
        int tok[kB];
        bool in[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int idx = base + u * kThThreads;
          z[u] = 0.f;
          tok[u] = 0;
          in[u] = false;
          if (idx < nr * n) {
            const int rr = idx / n, i = idx - rr * n;
            const int pos = P0 + i;
            int t = 0;  // the CTA's tiles cover [P0, P1) in position order
            while (t + 1 < ntiles && pc[t + 1].y <= pos) ++t;
            in[u] = (tmask[t] >> (rb0 + rr)) & 1u;  // rows mode: only the row's own clusters
            if (in[u]) {
              z[u] = __ldcg(a.z + (size_t)(rb0 + rr) * a.z_stride + pos);
              tok[u] = __ldg(a.perm + pc[t].x + (pos - pc[t].y));
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int idx = base + u * kThThreads;
          if (idx < nr * n) keys[idx] = in[u] ? tok_key(z[u], tok[u]) : 0ull;
        }
      }
      __syncthreads();
      if (rb0 == 0) trace_mark(a.trace, 10);  // keys staged
      for (int rr = warp; rr < nr && warp < nwr; rr += nwr) {
        const unsigned long long* kr = keys + (size_t)rr * n;
        uint32_t mk = 0u;
#pragma unroll 4
        for (int i = lane; i < n; i += 32) mk = max(mk, (uint32_t)(kr[i] >> 32));
        mk = __reduce_max_sync(0xffffffffu, mk);
        const float mx = ord_to_float(mk);
        float s = 0.f;
#pragma unroll 4
        for (int i = lane; i < n; i += 32)
          if (kr[i] != 0ull) s += expf(key_value(kr[i]) - mx);
        s = warp_sum(s);
        unsigned long long* out = a.rec + (size_t)(rb0 + rr) * rstride + (size_t)b * rec;
        const int nv = (a.dbg & 16) ? 0 : th_warp_topk(kr, n, K, lane, cand + (size_t)warp * n, out + 2);
        if (lane == 0) {
          out[0] = (unsigned long long)__float_as_uint(mx) | ((unsigned long long)__float_as_uint(s) << 32);
          out[1] = (unsigned long long)nv;
        }
      }
    }
  }
  // ---- ticket: the last R CTAs to arrive merge one row each (row G - 1 - ticket)
  __syncthreads();
  trace_mark(a.trace, 9);  // records written
  // 64-bit arrival count, never re-armed: launch e sees tickets [e G, (e + 1) G), so its mergers
  // wait for the count to reach (e + 1) G (no end-of-kernel reset atomics)
  unsigned long long* ticket = reinterpret_cast<unsigned long long*>(a.counter);
  if (tid == 0) {
    fence_acq_rel_gpu();
    const unsigned long long tk = atomicAdd(ticket, 1ull);
    misc[8] = G - 1 - (int)(tk % (unsigned long long)G);
    reinterpret_cast<unsigned long long*>(misc + 14)[0] = (tk / (unsigned long long)G + 1ull) * (unsigned long long)G;
  }
  __syncthreads();
  const int row = misc[8];
  if (row >= R) return;
  if (tid == 0) {  // every CTA's records: spin (bounded) until all G have arrived
    const unsigned long long t0 = globaltimer_ns();
    const unsigned long long target = reinterpret_cast<unsigned long long*>(misc + 14)[0];
    int dead = 0;
    for (unsigned k = 1; ld_acquire_u64(ticket) < target; ++k) {
      if ((k & 63u) == 0u && globaltimer_ns() - t0 > kThSpinNs) {
        atomicExch(a.err, (unsigned)DS_ERR_DEVICE_TIMEOUT);
        dead = 1;
        break;
      }
    }
    fence_acq_rel_gpu();
    misc[9] = dead;
  }
  __syncthreads();
  // deferred union: every CTA read the masks before its ticket, so the first merger clears them
  // (a later router launch that polls for its rows' masks must not see these)
  if (a.umask && row == 0)
    for (int i = tid; i < R * 32; i += kThThreads) a.umask[i] = 0ull;
  trace_mark(a.trace, 3);
  unsigned long long* st = reinterpret_cast<unsigned long long*>(ring);  // [G][rec] of this row
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.rec + (size_t)row * rstride);
    uint4* dst = reinterpret_cast<uint4*>(st);
    const int nv4 = (int)(rstride / 2);
#pragma unroll 8
    for (int i = tid; i < nv4; i += kThThreads) dst[i] = __ldcg(src + i);
  }
  __syncthreads();
  trace_mark(a.trace, 5);  // merger: records staged
  float* lse_sh = reinterpret_cast<float*>(st + rstride);
  const bool ok_all = misc[5] != 0 && misc[9] == 0 &&
                     (!a.rows || a.max_shortlist <= 0 || (long long)rtot[row] <= a.max_shortlist);
  // top-K: T = the K-th best record head (the K best heads are distinct keys, so >= K keys are
  // >= T); every record's keys >= T (a prefix of the sorted record) are candidates; rank-count them.
  unsigned long long* hd = st + rstride + 2;       // [G] heads
  unsigned long long* cnd = hd + G;                // [G K] candidates
  int* ncnd = reinterpret_cast<int*>(cnd + (size_t)G * K);
  if (tid < G) hd[tid] = st[(size_t)tid * rec + 1] > 0 ? st[(size_t)tid * rec + 2] : 0ull;
  if (tid == 0) *ncnd = 0;
  __syncthreads();
  if (warp == kThThreads / 32 - 1) {  // the last warp (no head: G <= 160), alongside the head ranking
    // lse: lane l folds records l, l + 32, ... in order, then one fixed xor tree (R19)
    uint32_t mk = 0u;
    for (int g = lane; g < G; g += 32) {
      const float m = __uint_as_float((uint32_t)st[(size_t)g * rec]);
      if (m > -INFINITY) mk = max(mk, ord_key(m));
    }
    mk = __reduce_max_sync(0xffffffffu, mk);
    const float Mx = ord_to_float(mk);
    float part = 0.f;
    for (int g = lane; g < G; g += 32) {
      const unsigned long long w0 = st[(size_t)g * rec];
      const float m = __uint_as_float((uint32_t)w0);
      if (m > -INFINITY) part += __uint_as_float((uint32_t)(w0 >> 32)) * expf(m - Mx);
    }
    const float sum = warp_sum(part);
    const bool ok = ok_all && Mx > -INFINITY;
    const float lse = ok ? Mx + logf(sum) : __int_as_float(0x7fc00000);
    if (lane == 0) {
      *lse_sh = lse;
      a.lse[row] = lse;
    }
  }  // lse_sh is read after the barriers below
  if (tid < G) {
    const unsigned long long h = hd[tid];
    int rk0 = 0, rk1 = 0;
#pragma unroll 8
    for (int g = 0; g < G - 1; g += 2) {
      rk0 += hd[g] > h ? 1 : 0;
      rk1 += hd[g + 1] > h ? 1 : 0;
    }
    if (G & 1) rk0 += hd[G - 1] > h ? 1 : 0;
    if (h != 0ull && rk0 + rk1 == K - 1) misc[10] = tid;
  }
  // records with a key: >= K of them means misc[10] holds the K-th best head's record
  const int nz = __syncthreads_count(tid < G && hd[tid] != 0ull);
  trace_mark(a.trace, 6);  // merger: heads ranked
  {
    const unsigned long long T = nz >= K ? hd[misc[10]] : 1ull;
    if (tid < G) {
      const int cg = (int)st[(size_t)tid * rec + 1];
      int c = 0;
      while (c < cg && st[(size_t)tid * rec + 2 + c] >= T) ++c;
      if (c > 0) {
        const int base = atomicAdd(ncnd, c);
        for (int j = 0; j < c; ++j) cnd[base + j] = st[(size_t)tid * rec + 2 + j];
      }
    }
  }
  __syncthreads();
  trace_mark(a.trace, 7);  // merger: candidates compacted
  {
    const int nc = *ncnd;
    const float lse = *lse_sh;
    const bool ok = !(lse != lse);
    for (int i = tid; i < nc; i += kThThreads) {
      const unsigned long long x = cnd[i];
      int r = 0;
#pragma unroll 8
      for (int j = 0; j < nc; ++j) r += cnd[j] > x ? 1 : 0;
      if (r < K) {
        const float z = key_value(x);
        a.top_ids[(size_t)row * K + r] = ok ? key_id(x) : -1;
        a.top_logits[(size_t)row * K + r] = ok ? z : -INFINITY;
        a.top_logp[(size_t)row * K + r] = ok ? z - lse : -INFINITY;
      }
    }
    for (int j = min(nc, K) + tid; j < K; j += kThThreads) {  // fewer keys than K: padding (R17)
      a.top_ids[(size_t)row * K + j] = -1;
      a.top_logits[(size_t)row * K + j] = -INFINITY;
      a.top_logp[(size_t)row * K + j] = -INFINITY;
    }
  }
  trace_mark(a.trace, 4);
}

// ------------------------------------------------------------------ host
struct ThPlan {
  int S, cap, rstride, hr;
  size_t smem;
};

static bool th_plan(const ds_clusters* c, int R, int k_t, ThPlan* p) {
  const char* off = getenv("DS_TH");
  if (off && off[0] == '0') return false;
  // d % 64 == 0: the 3-D view's K chunks are whole (a partial chunk would read the next row)
  if (c->dtype != DS_BF16 || R < 1 || R > kThN || k_t < 1 || k_t > kThMaxKt || (c->d % 64) != 0) return false;
  if (c->M < 1 || c->M > kMaxM) return false;
  const int G = num_sms();
  if (G > kThMaxG || c->V * (int64_t)G >= (int64_t)1 << 30) return false;  // 32-bit CTA-range arithmetic
  if ((c->d + 63) / 64 > 256) return false;                                   // H box: <= 256 K chunks
  const int kchunks = (c->d + 63) / 64;
  // union positions per CTA: a share of its big cluster (< 2 shares) + the small clusters rounded
  // to it (< 1 share) + up to 7 rows of group rounding; a share is |V_S| / G <= V / G
  p->cap = (int)(3 * ((c->V + G - 1) / G) + 64);
  const char* h8 = getenv("DS_TH_H8");  // "0": always store 16 H rows (A/B)
  p->hr = (R <= 8 && !(h8 && h8[0] == '0')) ? 8 : 16;
  const int smax = max_smem_optin();
  p->S = 0;
  for (int S = 16; S >= 2; --S)
    if ((int)th_smem(S, kchunks, p->cap, c->M, p->hr).total <= smax) {
      p->S = S;
      break;
    }
  if (p->S == 0) return false;
  // staging after the stream (ring + H): >= one row of keys + six warps' candidates (cap x 8 B each);
  // one row's G records + heads + candidates
  const ThSmem L = th_smem(p->S, kchunks, p->cap, c->M, p->hr);
  const size_t stage = L.bars - L.ring;
  p->rstride = (G * (2 + k_t) + 1) & ~1;
  if ((size_t)p->cap * 8 * 7 > stage ||
      ((size_t)p->rstride + 2 + G + (size_t)G * k_t) * 8 + 16 > stage)
    return false;
  p->smem = th_smem(p->S, kchunks, p->cap, c->M, p->hr).total;
  return encode_fn() != nullptr;
}

bool th_supported(const ds_clusters* c, int R, int k_t) {
  ThPlan p;
  return th_plan(c, R, k_t, &p);
}

size_t th_ws_bytes(const ds_clusters* c, int R, int k_t) {
  ThPlan p;
  if (!th_plan(c, R, k_t, &p)) return 0;
  return align_up((size_t)R * p.rstride * 8, 256) + align_up((size_t)R * c->V * 4, 256);
}

cudaError_t launch_th(const ds_clusters* c, const void* h_new, int R, const int32_t* sel, const int32_t* sel_count,
                      const int32_t* sl_offsets, int k_t, int64_t max_shortlist, int32_t* top_ids,
                      float* top_logits, float* top_logp, float* lse, float* z_out, int64_t z_stride, void* ws,
                      unsigned* counter, cudaStream_t st, bool pdl, int rows, const void* umask_ws) {
  ThPlan p;
  if (rows && (z_out || R > 16)) return cudaErrorInvalidValue;  // rows mode: no packed per-row z_out
  if (!th_plan(c, R, k_t, &p)) return cudaErrorInvalidValue;
  ThMaps mw;
  for (int j = 0; j < kThMaps; ++j)
    if (!make_map_kchunks(&mw.w[j], c->W_perm, (uint64_t)c->V, (uint64_t)c->d, (uint32_t)(8 * (j + 1)),
                          (uint32_t)th_cpc(8 * (j + 1))))
      return cudaErrorInvalidValue;
  CUtensorMap mh;  // H as (64, R rows, K chunks): one box {64, 16, kchunks} = the whole [chunk][16][128 B] image
  if (!make_map_kchunks(&mh, h_new, (uint64_t)R, (uint64_t)c->d, (uint32_t)p.hr, (uint32_t)((c->d + 63) / 64)))
    return cudaErrorInvalidValue;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  ThArgs a;
  a.sel = sel;
  a.sel_count = sel_count;
  // deferred union: the few-row router left the rows' masks in the workspace prefix of umask_ws
  a.umask = (!rows && umask_ws) ? reinterpret_cast<unsigned long long*>(
                                     const_cast<uint8_t*>(static_cast<const uint8_t*>(umask_ws)) + kWsRowsMasks)
                                : nullptr;
  a.usel = const_cast<int32_t*>(sel);
  a.ucnt = const_cast<int32_t*>(sel_count);
  a.usloff = const_cast<int32_t*>(sl_offsets);
  a.sl_off = sl_offsets;
  a.offsets = c->offsets;
  a.perm = c->perm;
  a.R = R;
  a.kchunks = (c->d + 63) / 64;
  a.K = k_t;
  a.S = p.S;
  a.cap = p.cap;
  a.hr = p.hr;
  a.M = c->M;
  a.V = c->V;
  a.rstride = p.rstride;
  a.max_shortlist = max_shortlist;
  a.rec = reinterpret_cast<unsigned long long*>(w8);
  if (z_out) {
    a.z = z_out;
    a.z_stride = z_stride;
  } else {
    a.z = reinterpret_cast<float*>(w8 + align_up((size_t)R * p.rstride * 8, 256));
    a.z_stride = c->V;
  }
  a.top_ids = top_ids;
  a.top_logits = top_logits;
  a.top_logp = top_logp;
  a.lse = lse;
  a.counter = counter + 16;  // [16] arrivals, [17] finished mergers (no other kernel uses them)
  a.err = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(counter) + kWsErrorWord);
  const char* np_ = getenv("DS_TH_NOPDL");  // A/B: launch without programmatic dependent launch
  if (np_ && np_[0] == '1') pdl = false;
  a.rows = rows ? 1 : 0;
  a.pdl = pdl ? 1 : 0;
  const char* dbg = getenv("DS_TH_DBG");
  a.dbg = dbg ? atoi(dbg) : 0;
  a.trace = debug_trace();
  static int configured[64] = {0};
  cudaError_t e = configure_max_smem(reinterpret_cast<const void*>(th_kernel), configured);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(kThThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, th_kernel, mw, mh, a);  // (pdl false: plain stream order)
}

}  // namespace ds
