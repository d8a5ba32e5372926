// head_impl.cuh — building blocks of the gathered head (S5) + fused epilogue (S6), shared by the
// standalone head kernel (head.cu) and the fused one-launch draft-step kernel (step.cu).
//
// Per CTA: a ring of `stages` shared-memory slots (16 KB each), filled by ONE producer lane with
// TMA 1D bulk copies of contiguous W_perm row runs (a selected cluster is one contiguous block,
// R12 layout) and drained by one consumer warp per slot, which dots two staged rows at a time with
// h_new (staged once in shared memory) in fp32.  Logits stay on chip; each CTA emits a
// (max, sum exp, top-k_t) partial per row and the last CTA merges the partials in CTA order.
#pragma once
#include <float.h>
#include <limits.h>

#include "common.cuh"

namespace ds {

constexpr int kMaxStages = 12;
constexpr int kStageTarget = 16384;          // bytes per ring slot (rounded to whole rows)
constexpr int kRingMax = kMaxStages * kStageTarget;
constexpr int kMaxGroups = 64;               // rows per launch
// fused step: a1, scores, b1, b2 (fp32, <= 1024 each) + offsets (<= 1025 ints) + flags + scan scratch
constexpr int kStepExtra = 4096 * 4 + 4112 + 1024 + 256;
// shared-memory bytes the last-CTA merge needs inside the ring
__host__ __device__ inline int merge_smem_bytes(int G, int k_t, int nwarps) {
  (void)nwarps;
  return G * (2 + 2 * k_t) * 4 + 2 * G * k_t * 4 + 256;
}

struct HeadArgs {
  const void* W;             // W_perm [V][d]
  const int32_t* perm;       // [V]
  const int32_t* offsets;    // [M+1]
  const int32_t* sel;        // [groups][M]
  const int32_t* sel_count;  // [groups]
  const int32_t* sl_off;     // [groups][M+1]
  const void* h;             // [nrows][d]
  int32_t M, nrows, d, k_t, shared, lcap, pdl;
  int32_t stages, stage_bytes, stage_rows;
  int64_t max_shortlist;
  int32_t* top_ids;
  float* top_logits;
  float* top_logp;
  float* lse;
  float* z_out;
  int64_t z_stride;
  float* part;               // [nrows][G][2 + 2 k_t]
  unsigned* counter;         // [0] = merge ticket (the fused step also uses [1], [2])
  float* record_out;         // nullable [nrows][2 + 2 k_t]: emit the merged (max, sum, top-k) record
};

void fill_head_args(HeadArgs& a, const ds_clusters* c, const HeadPlan& p, const void* h_new, int r0, int nr,
                    const int32_t* sel, const int32_t* sel_count, const int32_t* sl_offsets, int shared, int k_t,
                    int64_t max_shortlist, int32_t* top_ids, float* top_logits, float* top_logp, float* lse,
                    float* z_out, int64_t z_stride, float* part, unsigned* counter, bool pdl);

struct HeadSmem {
  uint32_t ring, bars, info, misc, red, sega, segn, segi, h, zl, zid, extra, total;
};

__host__ __device__ inline HeadSmem head_smem(int stages, int stage_bytes, int rows, int d, int esz, int lcap,
                                              int extra) {
  HeadSmem L;
  uint32_t o = 0;
  L.ring = o;
  o += (uint32_t)stages * stage_bytes;
  L.bars = o;
  o += (2 * kMaxStages + 2) * 8;
  L.info = o;
  o += kMaxStages * 16;
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
  o = (o + 127u) & ~127u;
  L.h = o;
  o += (uint32_t)rows * d * esz;
  o = (o + 15u) & ~15u;
  L.zl = o;
  o += (uint32_t)rows * lcap * 4;
  L.zid = o;
  o += (uint32_t)rows * lcap * 4;
  o = (o + 15u) & ~15u;
  L.extra = o;
  o += extra;
  L.total = o;
  return L;
}

struct HeadCtx {
  uint8_t* ring;
  uint64_t* full;
  uint64_t* empty;
  int4* info;
  int* misc;
  float* red;  // block-reduction scratch (64 floats)
  long long* sega;
  int* segn;
  int* segi;   // index (into the group's selection) of the cluster holding the segment start
  void* hs;
  float* zl;
  int* zid;
  uint8_t* extra;
};

__device__ __forceinline__ HeadCtx head_ctx(uint8_t* smem, const HeadSmem& L) {
  HeadCtx c;
  c.ring = smem + L.ring;
  c.full = reinterpret_cast<uint64_t*>(smem + L.bars);
  c.empty = c.full + kMaxStages;
  c.info = reinterpret_cast<int4*>(smem + L.info);
  c.misc = reinterpret_cast<int*>(smem + L.misc);
  c.red = reinterpret_cast<float*>(smem + L.red);
  c.sega = reinterpret_cast<long long*>(smem + L.sega);
  c.segn = reinterpret_cast<int*>(smem + L.segn);
  c.segi = reinterpret_cast<int*>(smem + L.segi);
  c.hs = smem + L.h;
  c.zl = reinterpret_cast<float*>(smem + L.zl);
  c.zid = reinterpret_cast<int*>(smem + L.zid);
  c.extra = smem + L.extra;
  return c;
}

__device__ __forceinline__ void head_init_barriers(const HeadCtx& c, int stages) {
  for (int s = 0; s < stages; ++s) {
    mbar_init(&c.full[s], 1);
    mbar_init(&c.empty[s], 1);
  }
  fence_mbar_init();
}

// sel / sel_count / sl_off may live in global memory (written by an earlier kernel, or by
// another CTA of this kernel before a fenced counter handshake) or in this CTA's shared memory
// (fused step): plain generic loads are valid for both.
__device__ __forceinline__ long long shortlist_len(const HeadArgs& a, int gi) {
  const int cnt = a.sel_count[gi];
  if (cnt < 1 || cnt > a.M) return -1;
  const long long N = a.sl_off[(size_t)gi * (a.M + 1) + cnt];
  return (N >= 1 && N <= a.max_shortlist) ? N : -1;
}

// Segment [N*g/G, N*(g+1)/G) of each group's virtual shortlist (even split by rows), and
// the selected cluster holding its first row (warp-parallel search: one L2 round trip per 32
// selected clusters instead of a dependent chain).  Warp w handles groups w, w + nwarps, ...
__device__ __forceinline__ void head_segments(const HeadArgs& a, const HeadCtx& c) {
  const int G = gridDim.x, g = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ngroups = a.shared ? 1 : a.nrows;
  for (int gi = warp; gi < ngroups; gi += nw) {
    const long long N = shortlist_len(a, gi);
    long long s0 = 0;
    int n = -1, idx = 0;
    if (N >= 0) {
      s0 = N * g / G;
      n = (int)(N * (g + 1) / G - s0);
      const int cnt = a.sel_count[gi];
      const int32_t* so = a.sl_off + (size_t)gi * (a.M + 1);
      // idx = number of i in [1, cnt) with so[i] <= s0  (so[0] = 0 <= s0 always)
      for (int i0 = 1; i0 < cnt; i0 += 32) {
        const int i = i0 + lane;
        const bool le = i < cnt && so[i] <= s0;
        idx += __popc(__ballot_sync(0xffffffffu, le));
      }
    }
    if (lane == 0) {
      c.sega[gi] = s0;
      c.segn[gi] = n;
      c.segi[gi] = idx;
    }
  }
}

// Producer (one lane): stream every segment as runs of whole rows, slot it % stages.
template <typename T>
__device__ void head_produce(const HeadArgs& a, const HeadCtx& c, uint32_t it0 = 0) {
  const uint64_t pol = policy_evict_first();
  const uint32_t rowbytes = (uint32_t)a.d * (uint32_t)sizeof(T);
  const uint8_t* W = static_cast<const uint8_t*>(a.W);
  const int ngroups = a.shared ? 1 : a.nrows;
  const uint32_t S = (uint32_t)a.stages;
  uint32_t it = it0;  // ring iterations already used by this launch (the cluster step's router rows)
  for (int gi = 0; gi < ngroups; ++gi) {
    const int nseg = c.segn[gi];
    if (nseg <= 0) continue;
    const long long s0 = c.sega[gi], s1 = s0 + nseg;
    const int32_t* so = a.sl_off + (size_t)gi * (a.M + 1);
    const int32_t* sl = a.sel + (size_t)gi * a.M;
    int i = c.segi[gi];  // cluster holding virtual position s0
    long long pos = s0;
    long long cl_beg = so[i], cl_end = so[i + 1];
    long long base = __ldg(a.offsets + sl[i]);
    while (pos < s1) {
      const long long lim = cl_end < s1 ? cl_end : s1;
      const int n = (int)min((long long)a.stage_rows, lim - pos);
      const long long wrow = base + (pos - cl_beg);
      const uint32_t s = it % S;
      mbar_wait(&c.empty[s], ((it / S) & 1u) ^ 1u);
      c.info[s] = make_int4(gi, (int)(pos - s0), n, (int)wrow);
      mbar_arrive_expect_tx(&c.full[s], (uint32_t)n * rowbytes);
      bulk_g2s(c.ring + (size_t)s * a.stage_bytes, W + (size_t)wrow * rowbytes, (uint32_t)n * rowbytes, &c.full[s],
               pol);
      ++it;
      pos += n;
      if (pos == cl_end && pos < s1) {
        ++i;
        cl_beg = cl_end;
        cl_end = so[i + 1];
        base = __ldg(a.offsets + sl[i]);
      }
    }
  }
  for (uint32_t j = 0; j < S; ++j, ++it) {  // one end-of-stream marker per slot
    const uint32_t s = it % S;
    mbar_wait(&c.empty[s], ((it / S) & 1u) ^ 1u);
    c.info[s] = make_int4(-1, 0, -1, 0);
    mbar_arrive(&c.full[s]);
  }
}

// Two staged rows at once against one h row: 4 independent fp32 FMA chains per lane, then warp
// trees (R18: lane-parallel partials).  `two == false` duplicates row 0 (result ignored).
template <typename T>
__device__ __forceinline__ void dot2(const T* __restrict__ w0, const T* __restrict__ w1, const T* __restrict__ h,
                                     int d, int lane, float& z0, float& z1) {
  constexpr int E = Elem<T>::kPer16B;
  float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 2
  for (int c = lane * E; c < d; c += 32 * E) {
    const uint4 hv = *reinterpret_cast<const uint4*>(h + c);
    const uint4 xv = *reinterpret_cast<const uint4*>(w0 + c);
    const uint4 yv = *reinterpret_cast<const uint4*>(w1 + c);
    float hf[E], xf[E], yf[E];
    widen16(hv, hf, h);
    widen16(xv, xf, h);
    widen16(yv, yf, h);
#pragma unroll
    for (int j = 0; j < E; j += 2) {
      a0 = fmaf(xf[j], hf[j], a0);
      b0 = fmaf(yf[j], hf[j], b0);
      a1 = fmaf(xf[j + 1], hf[j + 1], a1);
      b1 = fmaf(yf[j + 1], hf[j + 1], b1);
    }
  }
  z0 = warp_sum(a0 + a1) + 0.0f;  // + 0.0f: -0 -> +0 (R23)
  z1 = warp_sum(b0 + b1) + 0.0f;
}

// Consumer warp `w` owns ring slot `w`.
template <typename T>
__device__ void head_consume(const HeadArgs& a, const HeadCtx& c, int w, int lane, uint32_t k0 = 0) {
  const T* hs = static_cast<const T*>(c.hs);
  for (uint32_t k = k0;; ++k) {
    mbar_wait(&c.full[w], k & 1u);
    const int4 inf = c.info[w];
    if (inf.z < 0) break;
    const T* st = reinterpret_cast<const T*>(c.ring + (size_t)w * a.stage_bytes);
    const int gi = inf.x;
    const int r_lo = a.shared ? 0 : gi, r_hi = a.shared ? a.nrows : gi + 1;
    const long long zbase = c.sega[gi] + inf.y;
    for (int rr = 0; rr < inf.z; rr += 2) {
      const bool two = rr + 1 < inf.z;
      const T* w0 = st + (size_t)rr * a.d;
      const T* w1 = two ? w0 + a.d : w0;
      int tok0 = 0, tok1 = 0;
      if (lane == 0) {
        tok0 = __ldg(a.perm + inf.w + rr);
        tok1 = two ? __ldg(a.perm + inf.w + rr + 1) : 0;
      }
      for (int r = r_lo; r < r_hi; ++r) {
        float z0, z1;
        dot2<T>(w0, w1, hs + (size_t)r * a.d, a.d, lane, z0, z1);
        if (lane == 0) {
          const int li = inf.y + rr;
          c.zl[r * a.lcap + li] = z0;
          c.zid[r * a.lcap + li] = tok0;
          if (a.z_out) a.z_out[(size_t)r * a.z_stride + zbase + rr] = z0;
          if (two) {
            c.zl[r * a.lcap + li + 1] = z1;
            c.zid[r * a.lcap + li + 1] = tok1;
            if (a.z_out) a.z_out[(size_t)r * a.z_stride + zbase + rr + 1] = z1;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&c.empty[w]);
  }
}

// Stage h_new rows into shared memory (16-byte vectors).
__device__ __forceinline__ void head_load_h(const HeadArgs& a, const HeadCtx& c, int esz, int t0, int nt) {
  const size_t nvec = (size_t)a.nrows * a.d * esz / 16;
  const uint4* src = static_cast<const uint4*>(a.h);
  uint4* dst = reinterpret_cast<uint4*>(c.hs);
  for (size_t i = t0; i < nvec; i += nt) dst[i] = src[i];
}

// Block-wide max / sum with a fixed reduction order (warp trees, then warps in index order).
__device__ __forceinline__ float block_max(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float m = red[0];
  for (int w = 1; w < nw; ++w) m = fmaxf(m, red[w]);
  return m;
}
__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = red[0];
  for (int w = 1; w < nw; ++w) t += red[w];
  return t;
}

// Per-CTA partial per row: (max, sum exp(z - max), top-k_t by (logit desc, id asc)), computed by
// the whole block with shallow dependency chains (block_topk, block_lse).  Scratch: the ring.
__device__ inline void head_partials(const HeadArgs& a, const HeadCtx& c, int ring_bytes) {
  const int K = a.k_t, rec = 2 + 2 * K;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (a.nrows > 1 && (nt >> 5) * 8 * a.lcap <= ring_bytes) {
    // several rows: one warp per row, warp-level lse and pruned top-k (no block barriers)
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    float* sv = reinterpret_cast<float*>(c.ring) + (size_t)warp * 2 * a.lcap;
    int* si = reinterpret_cast<int*>(sv + a.lcap);
    for (int r = warp; r < a.nrows; r += nw) {
      const int gi = a.shared ? 0 : r;
      const int n = c.segn[gi] > 0 ? c.segn[gi] : 0;
      float* P = a.part + ((size_t)r * gridDim.x + blockIdx.x) * rec;
      const float* zr = c.zl + r * a.lcap;
      const int* ir = c.zid + r * a.lcap;
      float m, se;
      warp_lse_items(zr, n, m, se);
      warp_topk(
          n, K, [&](int i, float& v, int& id) { v = zr[i]; id = ir[i]; },
          [&](int rank, float v, int id) {
            P[2 + 2 * rank] = v;
            P[3 + 2 * rank] = __int_as_float(id);
          },
          sv, si);
      for (int q = n + lane; q < K; q += 32) {
        P[2 + 2 * q] = -INFINITY;
        P[3 + 2 * q] = __int_as_float(INT_MAX);
      }
      if (lane == 0) {
        P[0] = m;
        P[1] = se;
      }
    }
    return;
  }
  float* sv = reinterpret_cast<float*>(c.ring);
  int* si = reinterpret_cast<int*>(sv + a.lcap);
  if (a.nrows == 1 && c.segn[0] <= 1024) {
    // one row, few logits: one warp, no block barriers (barriers dominate at this size)
    if (tid < 32) {
      const int n = c.segn[0] > 0 ? c.segn[0] : 0;
      float* P = a.part + (size_t)blockIdx.x * rec;
      const float* zr = c.zl;
      const int* ir = c.zid;
      float m, se;
      warp_lse_items(zr, n, m, se);
      warp_topk(
          n, K, [&](int i, float& v, int& id) { v = zr[i]; id = ir[i]; },
          [&](int rank, float v, int id) {
            P[2 + 2 * rank] = v;
            P[3 + 2 * rank] = __int_as_float(id);
          },
          sv, si);
      for (int q = n + tid; q < K; q += 32) {
        P[2 + 2 * q] = -INFINITY;
        P[3 + 2 * q] = __int_as_float(INT_MAX);
      }
      if (tid == 0) {
        P[0] = m;
        P[1] = se;
      }
    }
    return;
  }
  for (int r = 0; r < a.nrows; ++r) {
    const int gi = a.shared ? 0 : r;
    const int n = c.segn[gi] > 0 ? c.segn[gi] : 0;
    float* P = a.part + ((size_t)r * gridDim.x + blockIdx.x) * rec;   // [row][cta][rec]
    const float* zr = c.zl + r * a.lcap;
    const int* ir = c.zid + r * a.lcap;
    float m = -INFINITY, se = 0.f;
    for (int j = tid; j < n; j += nt) {
      const float z = zr[j];
      if (z == -INFINITY) continue;
      if (z > m) {
        se = se * expf(m - z) + 1.f;
        m = z;
      } else {
        se += expf(z - m);
      }
    }
    block_lse(m, se, c.red);
    block_topk(
        n, K, [&](int i, float& v, int& id) { v = zr[i]; id = ir[i]; },
        [&](int rank, float v, int id) {
          P[2 + 2 * rank] = v;
          P[3 + 2 * rank] = __int_as_float(id);
        },
        sv, si, c.misc + 8);
    for (int q = n + tid; q < K; q += nt) {
      P[2 + 2 * q] = -INFINITY;
      P[3 + 2 * q] = __int_as_float(INT_MAX);
    }
    if (tid == 0) {
      P[0] = m;
      P[1] = se;
    }
  }
}

// Ticket: every CTA takes an arrival index (release: its partials are visible before).  The last
// nm = min(nrows, G) arrivals become mergers: each waits (acquire) until all G partials are in
// and merges rows j, j + nm, ... (j = its rank among the mergers), so R rows merge in parallel.
// Returns the merger rank j, or -1 for CTAs that only contributed partials.
__device__ __forceinline__ int head_ticket(const HeadArgs& a, const HeadCtx& c) {
  __syncthreads();
  const int G = gridDim.x;
  const int nm = min(a.nrows, G);
  if (threadIdx.x == 0) {
    const int t = (int)release_add(a.counter, 1u);
    int j = t - (G - nm);
    if (j >= 0) acquire_wait_geq(a.counter, (unsigned)G);
    c.misc[0] = j >= 0 ? j : -1;
  }
  __syncthreads();
  return c.misc[0];
}

// After merging: the last merger to finish resets the ticket (and `extra_ctrs` more counters that
// follow it: the fused step's phase counters) for the next launch.
__device__ __forceinline__ void head_merge_done(const HeadArgs& a, int extra_ctrs) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nm = min(a.nrows, (int)gridDim.x);
    unsigned* done = a.counter + 3;
    if ((int)release_add(done, 1u) == nm - 1) {
      fence_acq_rel_gpu();
      a.counter[0] = 0u;
      for (int i = 1; i <= extra_ctrs; ++i) a.counter[i] = 0u;
      *done = 0u;
    }
  }
}

// Merge step shared by the last-CTA merge and the cross-rank merge: staged per-partial (m_g, s_g)
// and K candidates per partial in rank-major order -> lse and top-k (or the merged record).
__device__ inline void merge_finish(const HeadArgs& a, const HeadCtx& c, int G, int r, const float* pm,
                                    const float* ps, const float* cv, const int* ci, float* sv, int* si,
                                    bool valid_row, unsigned long long* trace) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int K = a.k_t, rec = 2 + 2 * K;
  // block-parallel (measured faster than a single warp here: the G x K candidate set is wide)
  float mx = -INFINITY;
  for (int g = tid; g < G; g += nt) mx = fmaxf(mx, pm[g]);
  mx = block_max(mx, c.red);
  float S = 0.f;
  for (int g = tid; g < G; g += nt)
    if (pm[g] > -INFINITY) S += ps[g] * expf(pm[g] - mx);
  S = block_sum(S, c.red);
  trace_mark(trace, 17);
  const bool ok = valid_row && mx > -INFINITY;
  const float lse = ok ? mx + logf(S) : __int_as_float(0x7fc00000);
  auto emit = [&](int rank, float v, int id) {
    if (a.record_out) {
      a.record_out[(size_t)r * rec + 2 + 2 * rank] = v;
      a.record_out[(size_t)r * rec + 3 + 2 * rank] = __int_as_float(id);
    } else {
      a.top_ids[(size_t)r * K + rank] = ok ? id : -1;
      a.top_logits[(size_t)r * K + rank] = ok ? v : -INFINITY;
      a.top_logp[(size_t)r * K + rank] = ok ? v - lse : -INFINITY;
    }
  };
  if (G * (K - 1) < K * (K + 1) / 2) {  // few lists (cross-rank merge): the generic pruned top-k
    block_topk(
        G * K, K, [&](int e, float& v, int& id) { v = cv[e]; id = ci[e]; }, emit, sv, si, c.misc + 8);
  } else {
    // Candidates (rank-major staging: entry j of list g at [j * G + g], lists sorted): with r_g list
    // heads strictly above head g, entry j of list g has >= r_g + j entries beating it, so only
    // j < K - r_g can be in the top-K — at most K (K + 1) / 2 (+ ties) candidates, ranked once.
    // Head values as order-preserving integers in the tail of sv (candidates use its front).
    uint32_t* hk = reinterpret_cast<uint32_t*>(sv + (size_t)G * K - G);
    int* ncand = c.misc + 9;
    if (tid == 0) *ncand = 0;
    for (int g = tid; g < G; g += nt) hk[g] = cv[g] == -INFINITY ? 0u : ord_key(cv[g]);
    __syncthreads();
    for (int g = tid; g < G; g += nt) {
      const uint32_t h = hk[g];
      if (h == 0u) continue;  // empty list
      int rg = 0;
#pragma unroll 8
      for (int q = 0; q < G; ++q) rg += hk[q] > h;
      int ne = 0;
      while (ne < K - rg && cv[ne * G + g] != -INFINITY) ++ne;
      if (ne > 0) {
        const int base = atomicAdd(ncand, ne);
        for (int j = 0; j < ne; ++j) {
          sv[base + j] = cv[j * G + g];
          si[base + j] = ci[j * G + g];
        }
      }
    }
    __syncthreads();
    const int nc = *ncand;
    for (int e = tid; e < nc; e += nt) {
      const float v = sv[e];
      const int id = si[e];
      int rk = 0;
      for (int f = 0; f < nc; ++f) rk += beats(sv[f], si[f], v, id);
      if (rk < K) emit(rk, v, id);
    }
    if (tid == 0) c.misc[8] = min(nc, K);
    __syncthreads();
  }
  trace_mark(trace, 19);
  const int nvalid = c.misc[8];
  for (int q = nvalid + tid; q < K; q += nt) {
    if (a.record_out) {
      a.record_out[(size_t)r * rec + 2 + 2 * q] = -INFINITY;
      a.record_out[(size_t)r * rec + 3 + 2 * q] = __int_as_float(INT_MAX);
    } else {
      a.top_ids[(size_t)r * K + q] = -1;
      a.top_logits[(size_t)r * K + q] = -INFINITY;
      a.top_logp[(size_t)r * K + q] = -INFINITY;
    }
  }
  if (tid == 0) {
    if (a.record_out) {
      a.record_out[(size_t)r * rec] = mx;
      a.record_out[(size_t)r * rec + 1] = S;
    } else {
      a.lse[r] = lse;
    }
  }
}

// Last CTA: merge the G partials of every row -> lse, top ids (remapped), logp.
//  lse  = M + log sum_g S_g exp(m_g - M)            (fixed-order block reduction)
//  top  : T = the k_t-th best list head; only entries not beaten by T can be in the global
//         top-k_t (k_t heads are >= T), so rank-count just those survivors.
__device__ inline void head_merge(const HeadArgs& a, const HeadCtx& c, int ring_bytes,
                                  unsigned long long* trace = nullptr, int G_override = 0, int r_begin = 0,
                                  int r_step = 1) {
  const int G = G_override > 0 ? G_override : (int)gridDim.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int K = a.k_t, rec = 2 + 2 * K;
  const int per_row = G * rec;
  // staged records: per-CTA (m_g, s_g) and the K candidates of every CTA in rank-major order
  float* pm = reinterpret_cast<float*>(c.ring);   // [G]
  float* ps = pm + G;                             // [G]
  float* cv = ps + G;                             // [K][G] values
  int* ci = reinterpret_cast<int*>(cv + G * K);   // [K][G] ids
  float* sv = reinterpret_cast<float*>(ci + G * K);
  int* si = reinterpret_cast<int*>(sv + G * K);
  (void)ring_bytes;
  for (int r = r_begin; r < a.nrows; r += r_step) {
    const float* src = a.part + (size_t)r * per_row;  // this row's G records, contiguous
    if ((per_row & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0)) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      for (int q = tid; q < per_row / 4; q += nt) {
        const float4 v4 = __ldcg(s4 + q);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = 4 * q + u;
          const int gg = idx / rec, f = idx - gg * rec;
          if (f == 0) pm[gg] = vv[u];
          else if (f == 1) ps[gg] = vv[u];
          else if ((f & 1) == 0) cv[((f - 2) >> 1) * G + gg] = vv[u];
          else ci[((f - 3) >> 1) * G + gg] = __float_as_int(vv[u]);
        }
      }
    } else {
      for (int idx = tid; idx < per_row; idx += nt) {
        const float v = __ldcg(src + idx);
        const int gg = idx / rec, f = idx - gg * rec;
        if (f == 0) pm[gg] = v;
        else if (f == 1) ps[gg] = v;
        else if ((f & 1) == 0) cv[((f - 2) >> 1) * G + gg] = v;
        else ci[((f - 3) >> 1) * G + gg] = __float_as_int(v);
      }
    }
    __syncthreads();
    trace_mark(trace, 16);
    merge_finish(a, c, G, r, pm, ps, cv, ci, sv, si, shortlist_len(a, a.shared ? 0 : r) >= 0, trace);
    __syncthreads();
    trace_mark(trace, 20);
  }
}

}  // namespace ds
