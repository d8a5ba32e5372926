// gh.cu — S5 for MANY independent rows on the tensor cores: the grouped, cluster-major head.
//
// B requests each with their own selection K_b (Alg. 1 line 8; shared = 0, R9).  Row b needs
// z_b[v] = <h_b, W_LM[:, v]> only for v in its own shortlist V_S,b = U_{m in K_b} C_m.  At
// batch (Gemma-3: B = 512, k = 64 of M = 512) the union of the rows' shortlists is the whole
// vocabulary, but each (row, cluster) pair is needed by only ~k/M of the rows.  Grouping by cluster
// turns the head into a grouped GEMM (SURVEY §8(d) "batched cluster-major", intensity B k / M flop/B):
//   for every selected cluster m:  Z_m [rows(m) x |C_m|] = H[rows(m)] W_perm[C_m]^T
// so every cluster block of W_perm is read from HBM ONCE per step whatever the number of rows that
// selected it, and no logit outside a row's own shortlist is computed.
//
// Kernels (one launch each, PDL-chained):
//   gh_group_kernel   cluster -> row lists (CSR), per-row record slots, the work items:
//                     item = (cluster m, vocabulary tile of <= 256 rows of C_m, <= 128 of its rows)
//   gh_head_kernel    persistent, one CTA per SM, items i = blockIdx.x + j G (address order of W_perm):
//                       warp 0      TMA: the item's W_perm tile, 64-wide K chunks (128B swizzle, <= 5
//                                   boxes of 256/128/64/32/16/8 rows for a ragged tile)
//                       warps 2-3   gather: the item's rows of h_new by cp.async (16 B each, written
//                                   in the SW128 image), proxy fence, mbarrier arrive
//                       warp 1      tcgen05.mma M = 128 (rows) x N = 256 (vocabulary) x K = 16, fp32
//                                   accumulator in TMEM, double-buffered across items (2 x 256 columns)
//                       warps 4-7   epilogue: TMEM lane = row, so every row's online (max, sum exp) and
//                                   its top-k_t over the tile are THREAD-LOCAL (tcgen05.ld 32x32b): one
//                                   record (max, sum, top-k_t) per (row, cluster tile)
//   gh_merge_kernel   one CTA per row: the row's records in a fixed order -> lse, top-k_t
// Why not the gather4 TMA for the rows: scripts/probe/gather4_probe.cu measured ~60 ns per 4-row
// gather op per SM (9 GB/s per SM), 4x slower than the W tile it has to keep up with.
// Exactness: bf16 x bf16 products are exact in fp32; in the exact regime every partial sum is an
// integer below 2^24, so the logits equal the oracle bit for bit whatever the accumulation order.
#include <algorithm>

#include "head_impl.cuh"
#include "internal.h"
#include "keys.cuh"
#include "tc_common.cuh"

namespace ds {

constexpr int kGhRows = 128;    // MMA M: rows of one item
constexpr int kGhVoc = 256;     // MMA N: vocabulary rows of one item
constexpr int kGhS = 4;         // ring stages: A 16 KB (rows) + B 32 KB (vocabulary) each
constexpr int kGhABytes = kGhRows * 128;
constexpr int kGhBBytes = kGhVoc * 128;
constexpr int kGhThreads = 256;  // 8 warps
constexpr int kGhLoaders = 64;   // warps 2-3
constexpr int kGhKMax = 32;
constexpr int kGhMaxM = 1024;

struct GhArgs {
  const __nv_bfloat16* h;    // h_new [B][d]
  const int32_t* perm;       // [V]
  const int4* items;         // [nitems] (v0, nv | part << 16, g0, n)
  const int32_t* nitems;     // device count (written by gh_group_kernel)
  const int32_t* grp_rows;   // [sum n_m] row of each (cluster, row) pair
  const int32_t* grp_rec;    // [sum n_m] record index of the pair's first vocabulary tile
  float* recs;               // [records][2 + 2 k_t]
  int32_t d, kchunks, k_t;
  int32_t dbg;  // DS_GH_DBG (timing experiments only; results wrong): 1 skip the MMAs, 2 skip the row gather
  unsigned long long* trace;
};

struct GhSmem {
  uint32_t a, b, bars, slot, perm, rows, total;
};

__host__ __device__ inline GhSmem gh_smem() {
  GhSmem L;
  uint32_t o = 0;
  L.a = o;
  o += kGhS * kGhABytes;
  L.b = o;
  o += kGhS * kGhBBytes;
  L.bars = o;
  o += (2 * kGhS + 4) * 8;
  L.slot = o;
  o += 16;
  L.perm = o;
  o += 2 * kGhVoc * 4;  // token ids of the item's vocabulary tile (double-buffered by item parity)
  L.rows = o;
  o += 2 * kGhRows * 4;  // the item's rows (loaders), double-buffered by item parity
  L.total = o;
  return L;
}

struct GhMaps {
  CUtensorMap w[6];  // W_perm views with box heights 256, 128, 64, 32, 16, 8 rows (64 columns)
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------- grouping
// One CTA.  The rows' selections are staged in shared memory (one coalesced pass; every later pass
// reads them on chip), then: cnt_m = #rows that selected cluster m; the vocabulary tile T (256, or
// 128 / 64 when the union is too small to give every SM two items); CSR of (cluster -> rows); per-row
// record slots: row b's records are [rowoff[b], rowoff[b + 1]) with, for its i-th selected cluster
// m_i, the nparts(m_i) = ceil(|C_m| / T) records of that cluster at rowoff[b] + sum_{i' < i} nparts.
// (T = 256 unless fewer than G / 2 items would result; the workspace bound below covers T < 256.)
constexpr int kGhStageMax = 40 * 1024;  // staged selection entries (160 KB); larger batches read L2

// Items in descending tile-size order (counting sort on nv; ties in any order: an item's records do
// not depend on the CTA that computes it), so gh_item's snake assignment (CTA b takes positions b,
// 2G - 1 - b, 2G + b, ...) gives every CTA nearly the same W bytes: with cluster-major round-robin the
// busiest CTA carried 1.15x (Gemma-3 B = 512) to 1.4x (Llama-3 B = 16-64) the mean.
// bins: shared scratch of T + 1 ints.  The whole CTA calls it; cm / go are in shared memory.
__device__ void gh_emit_items(int M, int T, const int32_t* __restrict__ offsets, const int* cm, const int* go,
                              int4* items, int* bins) {
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i <= T; i += blockDim.x) bins[i] = 0;
  __syncthreads();
  for (int m = tid; m < M; m += blockDim.x) {
    const int n = cm[m];
    if (n == 0) continue;
    const int sz = __ldg(offsets + m + 1) - __ldg(offsets + m), nrb = (n + kGhRows - 1) / kGhRows;
    if (sz >= T) atomicAdd(&bins[T], (sz / T) * nrb);
    if (sz % T) atomicAdd(&bins[sz % T], nrb);
  }
  __syncthreads();
  if (tid < 32) {  // bins[nv] <- number of items with a larger tile (one warp, T + 1 <= 257 bins)
    int carry = 0;
    for (int base = T; base >= 0; base -= 32) {
      const int nv = base - lane;
      const int v = nv >= 0 ? bins[nv] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (nv >= 0) bins[nv] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __syncthreads();
  for (int m = tid; m < M; m += blockDim.x) {
    const int n = cm[m];
    if (n == 0) continue;
    const int beg = __ldg(offsets + m), sz = __ldg(offsets + m + 1) - beg;
    const int nrb = (n + kGhRows - 1) / kGhRows, P = (sz + T - 1) / T;
    for (int p = 0; p < P; ++p) {
      const int nv = min(T, sz - p * T);
      for (int rb = 0; rb < nrb; ++rb)
        items[atomicAdd(&bins[nv], 1)] = make_int4(beg + p * T, nv | (p << 16), go[m] + rb * kGhRows,
                                                   min(kGhRows, n - rb * kGhRows));
    }
  }
}

__global__ void __launch_bounds__(1024) gh_group_kernel(const int32_t* __restrict__ sel,
                                                        const int32_t* __restrict__ cnt, int B, int M,
                                                        int shared, int kmax, int G,
                                                        const int32_t* __restrict__ offsets, int32_t* grp_rows,
                                                        int32_t* grp_rec, int32_t* rowoff, int4* items,
                                                        int32_t* nitems) {
  extern __shared__ __align__(16) int32_t stg[];  // [nsel rows][kmax] staged selections (when they fit)
  __shared__ int cm[kGhMaxM], go[kGhMaxM + 1], cur[kGhMaxM], np[kGhMaxM], io[kGhMaxM + 1], csz[kGhMaxM];
  __shared__ int wsum[32];
  __shared__ int red[3], tsel;
  pdl_wait();                // the selections come from the router kernel
  pdl_launch_dependents();   // the head kernel may run its prologue
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int nrows_sel = shared ? 1 : B;
  const bool staged = (int64_t)nrows_sel * kmax <= kGhStageMax;
  for (int m = tid; m < M; m += blockDim.x) {
    cm[m] = 0;
    cur[m] = 0;
    csz[m] = __ldg(offsets + m + 1) - __ldg(offsets + m);
  }
  if (tid < 3) red[tid] = 0;
  if (staged) {
#pragma unroll 4
    for (int e = tid; e < nrows_sel * kmax; e += blockDim.x) {
      const int r = e / kmax, i = e - r * kmax;
      stg[e] = i < __ldg(cnt + r) ? __ldg(sel + (size_t)r * M + i) : -1;
    }
  }
  __syncthreads();
  auto sel_at = [&](int r, int i) { return staged ? stg[r * kmax + i] : __ldg(sel + (size_t)r * M + i); };
  // cluster counts: a shared selection is every row's (n_m = B for each union cluster)
  if (shared) {
    const int n = __ldg(cnt);
    for (int i = tid; i < n; i += blockDim.x) cm[sel_at(0, i)] = B;
  } else {
    for (int b = warp; b < B; b += nw) {
      const int n = __ldg(cnt + b);
      for (int i = lane; i < n; i += 32) atomicAdd(&cm[sel_at(b, i)], 1);
    }
  }
  __syncthreads();
  // vocabulary tile: the largest T in {256, 128, 64} giving work to at least half of the SMs
  {
    int it[3] = {0, 0, 0};
    for (int m = tid; m < M; m += blockDim.x)
      if (cm[m] > 0) {
        const int rb = (cm[m] + kGhRows - 1) / kGhRows;
#pragma unroll
        for (int j = 0; j < 3; ++j) it[j] += rb * ((csz[m] + (kGhVoc >> j) - 1) / (kGhVoc >> j));
      }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int v = (int)__reduce_add_sync(0xffffffffu, (unsigned)it[j]);
      if (lane == 0 && v) atomicAdd(&red[j], v);
    }
  }
  __syncthreads();
  // a 256-row tile keeps ~128 KB of W in flight per SM, so it only pays to split tiles when fewer than
  // half of the SMs would get one (Llama-3 B = 8: T = 64 measured 160 vs 120 us per step)
  if (tid == 0) tsel = red[0] >= G / 2 ? kGhVoc : red[1] >= G / 2 ? kGhVoc / 2 : kGhVoc / 4;
  __syncthreads();
  const int T = tsel;
  for (int m = tid; m < M; m += blockDim.x) np[m] = (csz[m] + T - 1) / T;
  __syncthreads();
  // each row's record count
  for (int b = warp; b < B; b += nw) {
    const int sb = shared ? 0 : b;
    const int n = __ldg(cnt + sb);
    int nr = 0;
    for (int i = lane; i < n; i += 32) nr += np[sel_at(sb, i)];
    nr = (int)__reduce_add_sync(0xffffffffu, (unsigned)nr);
    if (lane == 0) rowoff[b + 1] = nr;
  }
  __syncthreads();
  // exclusive scans: cluster groups (go), items per cluster (io); rows' records (sequential chunks)
  auto block_scan = [&](auto get, auto put, int n) {  // exclusive scan of get(i), i < n; put(i, prefix); returns total
    int carry = 0;
    for (int base = 0; base < n; base += blockDim.x) {
      const int i = base + tid;
      const int v = i < n ? get(i) : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        int s = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, s, o);
          if (lane >= o) s += y;
        }
        wsum[lane] = s;  // inclusive over warps
      }
      __syncthreads();
      const int excl = carry + (warp > 0 ? wsum[warp - 1] : 0) + x - v;
      if (i < n) put(i, excl);
      const int tot = wsum[nw - 1];
      __syncthreads();
      carry += tot;
    }
    return carry;
  };
  const int tg = block_scan([&](int m) { return cm[m]; }, [&](int m, int e) { go[m] = e; }, M);
  const int ti = block_scan([&](int m) { return cm[m] > 0 ? np[m] * ((cm[m] + kGhRows - 1) / kGhRows) : 0; },
                            [&](int m, int e) { io[m] = e; }, M);
  const int tr = block_scan([&](int b) { return rowoff[b + 1]; }, [&](int b, int e) { rowoff[b] = e; }, B);
  if (tid == 0) {
    go[M] = tg;
    io[M] = ti;
    rowoff[B] = tr;
    *nitems = ti;
  }
  __syncthreads();
  // fill: warp per row; lane i's record base = rowoff[b] + prefix of nparts over the row's clusters
  for (int b = warp; b < B; b += nw) {
    const int sb = shared ? 0 : b;
    const int n = __ldg(cnt + sb);
    int base = rowoff[b];
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const int m = i < n ? sel_at(sb, i) : 0;
      const int p = i < n ? np[m] : 0;
      int x = p;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < n) {
        const int pos = go[m] + (shared ? b : atomicAdd(&cur[m], 1));
        grp_rows[pos] = b;
        grp_rec[pos] = base + x - p;
      }
      base += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  // items: part p, row block rb of every selected cluster, largest tiles first
  gh_emit_items(M, T, offsets, cm, go, items, io);
}

// Large independent batches (B >= kGhWideRows rows, T = 256): the grouping as three
// grid-wide kernels (the one-CTA kernel above spent 35 us on Gemma-3 B = 512, one SM working):
//   gh_count_kernel  warp per row: n_m by global atomics, each row's record count (fixed T = 256)
//   gh_scan_kernel   one CTA: scans of n_m (groups), items per cluster and rows' records; the items;
//                    n_m and the fill cursors zeroed for the fill and the next call
//   gh_fill_kernel   warp per row: CSR entries and record slots
// cnt_g / cur_g: [M] ints in the per-call head scratch (cnt_g zeroed by a memset before the count kernel,
// cur_g by the scan kernel before the fill).
constexpr int kGhWideRows = 128;

__global__ void __launch_bounds__(1024) gh_count_kernel(const int32_t* __restrict__ sel,
                                                        const int32_t* __restrict__ cnt, int B, int M,
                                                        const int32_t* __restrict__ offsets, int* cnt_g,
                                                        int32_t* rowoff) {
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int n = __ldg(cnt + b);
  int nr = 0;
  for (int i = lane; i < n; i += 32) {
    const int m = __ldg(sel + (size_t)b * M + i);
    atomicAdd(cnt_g + m, 1);
    nr += (__ldg(offsets + m + 1) - __ldg(offsets + m) + kGhVoc - 1) / kGhVoc;
  }
  nr = (int)__reduce_add_sync(0xffffffffu, (unsigned)nr);
  if (lane == 0) rowoff[b + 1] = nr;
}

__global__ void __launch_bounds__(1024) gh_scan_kernel(int B, int M, const int32_t* __restrict__ offsets, int* cnt_g,
                                                       int* cur_g, int32_t* go_g, int32_t* rowoff, int4* items,
                                                       int32_t* nitems) {
  __shared__ int cm[kGhMaxM], go[kGhMaxM + 1], io[kGhMaxM + 1];
  __shared__ int wsum[32];
  pdl_wait();
  pdl_launch_dependents();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int m = tid; m < M; m += blockDim.x) {
    cm[m] = __ldcg(cnt_g + m);
    cur_g[m] = 0;  // the fill cursors
  }
  __syncthreads();
  auto block_scan = [&](auto get, auto put, int n) {
    int carry = 0;
    for (int base = 0; base < n; base += blockDim.x) {
      const int i = base + tid;
      const int v = i < n ? get(i) : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        int s = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, s, o);
          if (lane >= o) s += y;
        }
        wsum[lane] = s;
      }
      __syncthreads();
      const int excl = carry + (warp > 0 ? wsum[warp - 1] : 0) + x - v;
      if (i < n) put(i, excl);
      const int tot = wsum[nw - 1];
      __syncthreads();
      carry += tot;
    }
    return carry;
  };
  auto np = [&](int m) { return (__ldg(offsets + m + 1) - __ldg(offsets + m) + kGhVoc - 1) / kGhVoc; };
  const int tg = block_scan([&](int m) { return cm[m]; }, [&](int m, int e) { go[m] = e; }, M);
  const int ti = block_scan([&](int m) { return cm[m] > 0 ? np(m) * ((cm[m] + kGhRows - 1) / kGhRows) : 0; },
                            [&](int m, int e) { io[m] = e; }, M);
  const int tr = block_scan([&](int b) { return __ldcg(rowoff + b + 1); }, [&](int b, int e) { rowoff[b] = e; }, B);
  if (tid == 0) {
    rowoff[B] = tr;
    *nitems = ti;
    go_g[M] = tg;
  }
  for (int m = tid; m < M; m += blockDim.x) go_g[m] = go[m];
  gh_emit_items(M, kGhVoc, offsets, cm, go, items, io);
}

__global__ void __launch_bounds__(1024) gh_fill_kernel(const int32_t* __restrict__ sel,
                                                       const int32_t* __restrict__ cnt, int B, int M,
                                                       const int32_t* __restrict__ offsets, const int32_t* go_g,
                                                       int* cur_g, const int32_t* rowoff, int32_t* grp_rows,
                                                       int32_t* grp_rec) {
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int n = __ldg(cnt + b);
  int base = __ldcg(rowoff + b);
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const int m = i < n ? __ldg(sel + (size_t)b * M + i) : 0;
    const int p = i < n ? (__ldg(offsets + m + 1) - __ldg(offsets + m) + kGhVoc - 1) / kGhVoc : 0;
    int x = p;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (i < n) {
      const int pos = __ldcg(go_g + m) + atomicAdd(cur_g + m, 1);
      grp_rows[pos] = b;
      grp_rec[pos] = base + x - p;
    }
    base += __shfl_sync(0xffffffffu, x, 31);
  }
}

// ---------------------------------------------------------------------------- head
// Thread-local sorted top-K list in KMAX registers: slots [0, KMAX - K) hold ~0 sentinels (never
// displaced), the K real entries (descending 64-bit keys, 0 = empty) are L[KMAX - K .. KMAX - 1], so
// the K-th best is always L[KMAX - 1] and every index is compile-time.  x bubbles down: the larger
// of carry / L[i] stays.
template <int KMAX>
__device__ __forceinline__ void topk_insert(unsigned long long (&L)[KMAX], unsigned long long x) {
  unsigned long long carry = x;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    const unsigned long long cur = L[i];
    const bool gt = carry > cur;
    L[i] = gt ? carry : cur;
    carry = gt ? cur : carry;
  }
}

// The j-th item of CTA b (items sorted by tile size, largest first): a snake over rounds of G items.
__device__ __forceinline__ int gh_item(int j, int G) {
  return j * G + ((j & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
}

template <int KMAX>
__global__ void __launch_bounds__(kGhThreads, 1) gh_head_kernel(const __grid_constant__ GhMaps maps,
                                                                const GhArgs g) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const GhSmem L = gh_smem();
  uint8_t* sa = smem + L.a;
  uint8_t* sb = smem + L.b;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kGhS;
  uint64_t* tfull = empty + kGhS;
  uint64_t* tempty = tfull + 2;
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + L.slot);
  int32_t* ptok = reinterpret_cast<int32_t*>(smem + L.perm);
  int32_t* prow = reinterpret_cast<int32_t*>(smem + L.rows);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGhS; ++s) {
      mbar_init(&full[s], 1 + kGhLoaders);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
    for (int i = 0; i < 6; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[i])) : "memory");
  }
  if (warp == 1) {  // TMEM: 2 x 256 fp32 columns (one accumulator per item parity), owned by warp 1
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  pdl_wait();  // items / row lists come from gh_group_kernel
  trace_mark(g.trace, 1);
  const int nitems = *g.nitems;
  // this CTA's J items, processed from a per-CTA rotation so that at any moment the CTAs work on a mix
  // of tile sizes (all CTAs on ragged tiles at once leave HBM idle while they wait on latency)
  int J = 0;
  while (gh_item(J, G) < nitems) ++J;
  const int rot = J > 0 ? (int)blockIdx.x % J : 0;
  auto order = [&](int li) { return li < J ? gh_item(li + rot < J ? li + rot : li + rot - J, G) : nitems; };
  const int KC = g.kchunks;
  const size_t rowbytes = (size_t)g.d * 2;

  if (warp == 0) {
    // ---- TMA producer: the W_perm tile of every item, K chunk by K chunk
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      for (int li = 0, item = order(0); item < nitems; item = order(++li)) {
        const int4 itm = __ldg(g.items + item);
        const int v0 = itm.x, nv = itm.y & 0xffff;
        const int nv8 = (nv + 7) & ~7;  // rows loaded (multiple of 8; the tail beyond nv is never read back)
        for (int kc = 0; kc < KC; ++kc, ++it) {
          const uint32_t s = it % kGhS;
          mbar_wait(&empty[s], ((it / kGhS) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], (uint32_t)nv8 * 128u);
          uint8_t* dst = sb + (size_t)s * kGhBBytes;
          int r = 0;
#pragma unroll 1
          for (int j = 0; j < 6 && r < nv8; ++j) {
            const int h = kGhVoc >> j;
            if (nv8 - r >= h) {
              tma_load_2d(dst + (size_t)r * 128, &maps.w[j], kc * 64, v0 + r, &full[s], pol);
              r += h;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    if (lane == 0) {
      uint32_t it = 0;
      int li = 0;
      for (int item = order(0); item < nitems; item = order(++li)) {
        const int4 itm = __ldg(g.items + item);
        const int nv = itm.y & 0xffff;
        const int N = (nv + 15) & ~15;
        // D f32, A / B bf16, both K-major, N >> 3, M = 128 >> 4
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        const int buf = li & 1;
        mbar_wait(&tempty[buf], (((uint32_t)li >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + (uint32_t)(buf * kGhVoc);
        for (int kc = 0; kc < KC; ++kc, ++it) {
          const uint32_t s = it % kGhS;
          mbar_wait(&full[s], (it / kGhS) & 1u);
          tc_fence_after();
          const uint32_t abase = smem_u32(sa + (size_t)s * kGhABytes);
          const uint32_t bbase = smem_u32(sb + (size_t)s * kGhBBytes);
          if (!(g.dbg & 1)) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_bf16(d_tmem, sw128_desc(abase + k * 32), sw128_desc(bbase + k * 32), idesc,
                          (kc | k) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ---- row gather: the item's rows of h_new into the SW128 K-major image, 16 B per cp.async.
    // Every loader thread runs its own pipeline (no barrier between the 64 threads): thread t copies
    // column chunk t & 7 of rows (t >> 3) + 8 u, so it needs only its own <= 16 row ids, loaded from
    // global memory at each item start.  It issues a stage whenever the stage's slot is free and fewer
    // than kPend stages are pending, and otherwise publishes its oldest pending stage (wait for those
    // copies, proxy fence, arrive) — so up to kPend stages of row copies are in flight and a stage is
    // published as soon as its copies have landed.  (Publishing stage s only after issuing s + 1 capped
    // the gather at one stage per half L2 round trip, ~4.7 TB/s of W at Gemma-3 B = 512; waiting for
    // s + 3 to issue coupled stage s to the MMA of s - 1: slower still.)
    constexpr int kPend = kGhS - 1;
    const int t = threadIdx.x - 64;  // 0..63
    const int r0 = t >> 3, cch = t & 7;
    constexpr int kRowsPerThread = kGhRows / 8;
    uint32_t it_i = 0, it_r = 0;  // stages issued / published by this thread
    int li = 0, item = order(0), kc = 0, n = 0;
    int rid[kRowsPerThread];
    const uint8_t* hb = reinterpret_cast<const uint8_t*>(g.h);
    for (;;) {
      const bool more = item < nitems;
      if (more && it_i - it_r < (uint32_t)kPend &&
          mbar_test_wait(&empty[it_i % kGhS], ((it_i / kGhS) & 1u) ^ 1u)) {
        if (kc == 0) {  // item start: this thread's row ids
          const int4 itm = __ldg(g.items + item);
          n = itm.w;
#pragma unroll
          for (int u = 0; u < kRowsPerThread; ++u) {
            const int j = r0 + 8 * u;
            rid[u] = j < n ? __ldg(g.grp_rows + itm.z + j) : 0;
          }
        }
        uint8_t* dst = sa + (size_t)(it_i % kGhS) * kGhABytes;
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
          const int j = r0 + 8 * u;
          if (j < n && !(g.dbg & 2))
            cp_async16(dst + j * 128 + ((cch ^ (j & 7)) << 4), hb + (size_t)rid[u] * rowbytes + (size_t)kc * 128 + cch * 16);
        }
        cp_async_commit();
        ++it_i;
        if (++kc == KC) {
          kc = 0;
          item = order(++li);
        }
      } else if (it_i != it_r) {  // publish the oldest pending stage once its copies have landed
        switch (it_i - it_r) {
          case 1: cp_async_wait<0>(); break;
          case 2: cp_async_wait<1>(); break;
          default: cp_async_wait<2>(); break;  // kPend = 3
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&full[it_r % kGhS]);
        ++it_r;
      } else if (!more) {
        break;
      } else {  // nothing pending and the next slot busy: sleep on it
        mbar_wait(&empty[it_i % kGhS], ((it_i / kGhS) & 1u) ^ 1u);
      }
    }
  } else {
    // ---- epilogue: TMEM lane quarter q = warp & 3 holds rows 32 q .. 32 q + 31 of the item
    const int q = warp & 3, row = 32 * q + lane, et = threadIdx.x - 128;  // et: 0..127
    const int K = g.k_t, rec = 2 + 2 * K;
    int li = 0;
    for (int item = order(0); item < nitems; item = order(++li)) {
      const int4 itm = __ldg(g.items + item);
      const int v0 = itm.x, nv = itm.y & 0xffff, part = itm.y >> 16, n = itm.w;
      const int buf = li & 1;
      int32_t* tok = ptok + buf * kGhVoc;
      for (int j = et; j < nv; j += 128) tok[j] = __ldg(g.perm + v0 + j);
      const int myrec = row < n ? __ldg(g.grp_rec + itm.z + row) + part : 0;
      named_bar_sync(2, 128);  // token ids staged
      mbar_wait(&tfull[buf], ((uint32_t)li >> 1) & 1u);
      tc_fence_after();
      unsigned long long lst[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) lst[i] = i < KMAX - K ? ~0ull : 0ull;
      float m = -INFINITY, se = 0.f;
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * kGhVoc);
      for (int c0 = 0; c0 < nv; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);  // warp-collective: every lane, whatever its row
        if (row < n) {
          const int lim = min(16, nv - c0);
          float bm = m;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < lim) bm = fmaxf(bm, v[j]);
          se *= expf(m - bm);  // m = -inf at the start: se = 0 * 0
          if (!(se == se)) se = 0.f;
          m = bm;
          unsigned long long key[16];
          uint32_t hit = 0u;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float z = v[j] + 0.0f;  // -0 -> +0 (R23)
            key[j] = j < lim ? tok_key(z, tok[c0 + j]) : 0ull;
            if (j < lim) se += expf(z - m);
            hit |= (key[j] > lst[KMAX - 1] ? 1u : 0u) << j;
          }
          while (hit) {  // rare after the first tiles: one insertion body, the key picked by selects
            const int jj = __ffs(hit) - 1;
            hit &= hit - 1u;
            unsigned long long x = key[0];
#pragma unroll
            for (int j = 1; j < 16; ++j) x = jj == j ? key[j] : x;
            if (x > lst[KMAX - 1]) topk_insert<KMAX>(lst, x);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (row < n) {
        float* R = g.recs + (size_t)myrec * rec;
        R[0] = m;
        R[1] = se;
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          if (i >= KMAX - K) {
            const int o = i - (KMAX - K);
            const bool ok = lst[i] != 0ull;
            R[2 + 2 * o] = ok ? key_value(lst[i]) : -INFINITY;
            R[3 + 2 * o] = __int_as_float(ok ? key_id(lst[i]) : INT_MAX);
          }
        }
      }
      named_bar_sync(2, 128);  // tok[] of this parity is reused two items later
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
  pdl_launch_dependents();
  trace_mark(g.trace, 5);
}

// ---------------------------------------------------------------------------- merge
// One CTA per row: the row's records [rowoff[b], rowoff[b + 1]) in their fixed order (selection
// order, then vocabulary tile) -> lse = M + log sum_g S_g e^{m_g - M}, top-k_t.
__global__ void __launch_bounds__(128) gh_merge_kernel(const float* __restrict__ recs,
                                                       const int32_t* __restrict__ rowoff, int K,
                                                       int32_t* top_ids, float* top_logits, float* top_logp,
                                                       float* lse) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_wait();
  const int r = blockIdx.x, rec = 2 + 2 * K;
  const int r0 = __ldg(rowoff + r), G = __ldg(rowoff + r + 1) - r0;
  float* pm = reinterpret_cast<float*>(smem);
  float* ps = pm + G;
  float* cv = ps + G;
  int* ci = reinterpret_cast<int*>(cv + G * K);
  float* sv = reinterpret_cast<float*>(ci + G * K);
  int* si = reinterpret_cast<int*>(sv + G * K);
  float* red = reinterpret_cast<float*>(si + G * K);
  int* misc = reinterpret_cast<int*>(red + 64);
  for (int idx = threadIdx.x; idx < G * rec; idx += blockDim.x) {
    const int gg = idx / rec, f = idx - gg * rec;
    const float v = recs[(size_t)(r0 + gg) * rec + f];
    if (f == 0) pm[gg] = v;
    else if (f == 1) ps[gg] = v;
    else if ((f & 1) == 0) cv[((f - 2) >> 1) * G + gg] = v;
    else ci[((f - 3) >> 1) * G + gg] = __float_as_int(v);
  }
  __syncthreads();
  HeadArgs a = {};
  a.k_t = K;
  a.top_ids = top_ids;
  a.top_logits = top_logits;
  a.top_logp = top_logp;
  a.lse = lse;
  a.record_out = nullptr;
  HeadCtx c = {};
  c.red = red;
  c.misc = misc;
  merge_finish(a, c, G, r, pm, ps, cv, ci, sv, si, G > 0, nullptr);
}

// ---------------------------------------------------------------------------- host
struct GhWs {
  size_t grp_rows, grp_rec, rowoff, items, nitems, cnt, cur, go, recs, total;
  int64_t max_recs_per_row, max_items;
};

// Records per row = sum over its selected clusters of ceil(|C_m| / 256) <= min(k ceil(max_size / 256),
// k + ceil(V / 256)) (each cluster adds at most one partial tile to |V_S| / 256).
static GhWs gh_ws(const ds_clusters* c, int B, int k_t, int kmax) {
  GhWs w;
  const int64_t P = (c->max_size + kGhVoc - 1) / kGhVoc;
  // T = 256: <= min(k P, k + V / 256); T < 256 is chosen only when the 2T items number < 2 G, so a row
  // has < 4 G + M records then
  w.max_recs_per_row = std::max(std::min<int64_t>((int64_t)kmax * P, (int64_t)kmax + (c->V + kGhVoc - 1) / kGhVoc),
                                std::min<int64_t>((int64_t)4 * num_sms() + c->M, (int64_t)kmax * ((c->max_size + 63) / 64)));
  const int64_t pairs = (int64_t)B * kmax;
  w.max_items = std::max(std::min<int64_t>((int64_t)c->M * P, (int64_t)c->M + (c->V + kGhVoc - 1) / kGhVoc) *
                             ((B + kGhRows - 1) / kGhRows),
                         (int64_t)4 * num_sms() + 2 * c->M);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  w.grp_rows = take((size_t)pairs * 4);
  w.grp_rec = take((size_t)pairs * 4);
  w.rowoff = take((size_t)(B + 1) * 4);
  w.items = take((size_t)w.max_items * 16);
  w.nitems = take(16);
  w.cnt = take((size_t)c->M * 4);  // per-cluster counts (zeroed by launch_gh), fill cursors, group offsets
  w.cur = take((size_t)c->M * 4);
  w.go = take((size_t)(c->M + 1) * 4);
  w.recs = take((size_t)B * w.max_recs_per_row * (2 + 2 * k_t) * 4);
  w.total = o;
  return w;
}

static size_t gh_merge_smem(int64_t G, int K) { return (size_t)(2 * G + 4 * G * K) * 4 + 64 * 4 + 16 * 4; }

bool gh_wide_grouping(int B, int shared) { return !shared && B >= kGhWideRows; }

bool gh_supported(const ds_clusters* c, int B, int k_t, int kmax) {
  const char* off = getenv("DS_GH");
  if (off && off[0] == '0') return false;
  if (c->dtype != DS_BF16 || c->d % 64 != 0 || c->M > kGhMaxM || k_t < 1 || k_t > kGhKMax || B < 1) return false;
  if (kmax < 1 || kmax > c->M || (reinterpret_cast<uintptr_t>(c->W_perm) & 15u) != 0) return false;
  if ((int64_t)gh_smem().total > max_smem_optin()) return false;
  const GhWs w = gh_ws(c, B, k_t, kmax);
  if ((int64_t)gh_merge_smem(w.max_recs_per_row, k_t) > max_smem_optin()) return false;
  return encode_fn() != nullptr;
}

size_t gh_ws_bytes(const ds_clusters* c, int B, int k_t, int kmax) { return gh_ws(c, B, k_t, kmax).total; }

template <int KMAX>
static cudaError_t launch_gh_head_t(const GhMaps& maps, const GhArgs& a, cudaStream_t st) {
  static int configured[64] = {0};
  cudaError_t e = configure_max_smem(reinterpret_cast<const void*>(gh_head_kernel<KMAX>), configured);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(kGhThreads);
  cfg.dynamicSmemBytes = gh_smem().total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gh_head_kernel<KMAX>, maps, a);
}

cudaError_t launch_gh(const ds_clusters* c, const void* h_new, int B, const int32_t* sel, const int32_t* sel_count,
                      int shared, int k_t, int kmax, int32_t* top_ids, float* top_logits, float* top_logp, float* lse, void* ws,
                      cudaStream_t st) {
  if (!gh_supported(c, B, k_t, kmax)) return cudaErrorInvalidValue;
  const GhWs w = gh_ws(c, B, k_t, kmax);
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  int32_t* grp_rows = reinterpret_cast<int32_t*>(w8 + w.grp_rows);
  int32_t* grp_rec = reinterpret_cast<int32_t*>(w8 + w.grp_rec);
  int32_t* rowoff = reinterpret_cast<int32_t*>(w8 + w.rowoff);
  int4* items = reinterpret_cast<int4*>(w8 + w.items);
  int32_t* nitems = reinterpret_cast<int32_t*>(w8 + w.nitems);
  float* recs = reinterpret_cast<float*>(w8 + w.recs);
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  if (gh_wide_grouping(B, shared)) {
    int* cnt_g = reinterpret_cast<int*>(w8 + w.cnt);
    int* cur_g = reinterpret_cast<int*>(w8 + w.cur);
    int32_t* go_g = reinterpret_cast<int32_t*>(w8 + w.go);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(1024);
    cfg.stream = st;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((B + 31) / 32);
    // the counters live in the per-call head scratch, which other head kernels also use: zero them here
    cudaError_t e = cudaMemsetAsync(cnt_g, 0, (size_t)c->M * 4, st);
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&cfg, gh_count_kernel, sel, sel_count, B, c->M, (const int32_t*)c->offsets,
                                       cnt_g, rowoff);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3(1);
    e = cudaLaunchKernelEx(&cfg, gh_scan_kernel, B, c->M, (const int32_t*)c->offsets, cnt_g, cur_g, go_g, rowoff,
                           items, nitems);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3((B + 31) / 32);
    e = cudaLaunchKernelEx(&cfg, gh_fill_kernel, sel, sel_count, B, c->M, (const int32_t*)c->offsets,
                           (const int32_t*)go_g, cur_g, (const int32_t*)rowoff, grp_rows, grp_rec);
    if (e != cudaSuccess) return e;
  } else {
    cudaLaunchConfig_t cfg = {};
    const int nrs = shared ? 1 : B;
    const size_t stg = (int64_t)nrs * kmax <= kGhStageMax ? (size_t)nrs * kmax * 4 : 0;
    if (stg > 16 * 1024) {  // static arrays (~25 KB) + staged selections above the 48 KB default: opt in
      cudaError_t e0 = cudaFuncSetAttribute(gh_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stg);
      if (e0 != cudaSuccess) return e0;
    }
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = stg;
    cfg.stream = st;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, gh_group_kernel, sel, sel_count, B, c->M, shared ? 1 : 0, kmax,
                                       num_sms(), (const int32_t*)c->offsets,
                                       grp_rows, grp_rec, rowoff, items, nitems);
    if (e != cudaSuccess) return e;
  }
  GhMaps maps;
  for (int j = 0; j < 6; ++j)
    if (!make_map(&maps.w[j], c->W_perm, (uint64_t)c->V, (uint64_t)c->d, (uint32_t)(kGhVoc >> j)))
      return cudaErrorInvalidValue;
  GhArgs a;
  a.h = static_cast<const __nv_bfloat16*>(h_new);
  a.perm = c->perm;
  a.items = items;
  a.nitems = nitems;
  a.grp_rows = grp_rows;
  a.grp_rec = grp_rec;
  a.recs = recs;
  a.d = c->d;
  a.kchunks = c->d / 64;
  a.k_t = k_t;
  a.trace = debug_trace();
  const char* dv = getenv("DS_GH_DBG");
  a.dbg = dv ? atoi(dv) : 0;
  cudaError_t e = k_t <= 8 ? launch_gh_head_t<8>(maps, a, st)
                  : k_t <= 16 ? launch_gh_head_t<16>(maps, a, st)
                              : launch_gh_head_t<32>(maps, a, st);
  if (e != cudaSuccess) return e;
  {
    static int configured[64] = {0};
    e = configure_max_smem(reinterpret_cast<const void*>(gh_merge_kernel), configured);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(B);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = gh_merge_smem(w.max_recs_per_row, k_t);
    cfg.stream = st;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, gh_merge_kernel, (const float*)recs, (const int32_t*)rowoff, k_t, top_ids,
                           top_logits, top_logp, lse);
  }
  return e;
}

}  // namespace ds
