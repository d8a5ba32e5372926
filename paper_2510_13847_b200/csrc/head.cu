// head.cu — S5+S6: gathered LM head over the shortlist + fused log-softmax / top-k_t / remap.
//
// z_r[j] = <h_new_r, W_LM[:, V_S,r[j]]>              (Alg. 1 line 10, "FUSED_INDEX_GEMM")
// p = log_softmax(z); TopK_{k_t}(p); remap2realid   (Alg. 1 line 11)
//
// B200 design.  The shortlist is never materialised: row r's virtual
// shortlist is the concatenation of the selected clusters' row blocks of W_perm (each
// cluster one contiguous block, P:193-196 + R12 layout), addressed through sl_offsets.
// A persistent grid of G = #SM CTAs splits every row's virtual shortlist evenly (clusters
// are unbalanced, so we split rows, not clusters).  In each CTA one producer lane
// streams its segment from HBM with TMA 1D bulk copies (cp.async.bulk) into a 4-stage
// shared-memory ring guarded by mbarriers; 8 consumer warps dot each staged W row with
// h_new (staged once in shared memory) in fp32 and keep the logits on chip.  The epilogue
// computes per-CTA (max, sum exp, top-k_t) partials; the last CTA to finish (atomic ticket)
// merges them in CTA-index order and writes ids (remapped through perm), logits, logp, lse.
// No floating-point atomics: the result is deterministic for a fixed grid.
#include <float.h>
#include <limits.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace ds {

constexpr int kHeadConsumerWarps = 8;
constexpr int kHeadWarps = kHeadConsumerWarps + 1;  // + 1 producer warp
constexpr int kHeadThreads = kHeadWarps * 32;
constexpr int kHeadStages = 4;
constexpr int kHeadStageBytes = 32768;
constexpr int kHeadMaxRows = 64;

struct HeadArgs {
  const void* W;            // W_perm [V][d]
  const int32_t* perm;      // [V]
  const int32_t* offsets;   // [M+1]
  const int32_t* sel;       // [groups][M]
  const int32_t* sel_count; // [groups]
  const int32_t* sl_off;    // [groups][M+1]
  const void* h;            // [nrows][d]
  int32_t M, nrows, d, k_t, shared, lcap, stage_rows, pdl;
  int64_t max_shortlist;
  int32_t* top_ids;
  float* top_logits;
  float* top_logp;
  float* lse;
  float* z_out;
  int64_t z_stride;
  float* part;              // [G][nrows][2 + 2 k_t]
  unsigned* counter;
};

struct HeadLayout {
  uint32_t ring, bars, info, misc, sega, segn, h, zl, zid, total;
};

__host__ __device__ inline HeadLayout head_layout(int rows, int d, int esz, int lcap) {
  HeadLayout L;
  uint32_t o = 0;
  L.ring = o;
  o += kHeadStages * kHeadStageBytes;
  L.bars = o;
  o += 2 * kHeadStages * 8;
  L.info = o;
  o += kHeadStages * 16;
  L.misc = o;
  o += 16 * 4;
  L.sega = o;
  o += kHeadMaxRows * 8;
  L.segn = o;
  o += kHeadMaxRows * 4;
  o = (o + 127u) & ~127u;
  L.h = o;
  o += (uint32_t)rows * d * esz;
  o = (o + 15u) & ~15u;
  L.zl = o;
  o += (uint32_t)rows * lcap * 4;
  L.zid = o;
  o += (uint32_t)rows * lcap * 4;
  L.total = o;
  return L;
}

// One warp: fp32 dot of a staged W row with h (both in shared memory), lane-strided 16-byte
// chunks, two interleaved accumulators per lane (R18: lane-parallel partials + warp tree).
template <typename T>
__device__ __forceinline__ float dot_row(const T* __restrict__ w, const T* __restrict__ h, int d, int lane) {
  constexpr int E = Elem<T>::kPer16B;
  float acc0 = 0.f, acc1 = 0.f;
  int c = lane * E;
  for (; c + 32 * E < d; c += 64 * E) {
    const uint4 wv0 = *reinterpret_cast<const uint4*>(w + c);
    const uint4 hv0 = *reinterpret_cast<const uint4*>(h + c);
    const uint4 wv1 = *reinterpret_cast<const uint4*>(w + c + 32 * E);
    const uint4 hv1 = *reinterpret_cast<const uint4*>(h + c + 32 * E);
    float wf[E], hf[E];
    widen16(wv0, wf, w);
    widen16(hv0, hf, h);
#pragma unroll
    for (int j = 0; j < E; ++j) acc0 = fmaf(wf[j], hf[j], acc0);
    widen16(wv1, wf, w);
    widen16(hv1, hf, h);
#pragma unroll
    for (int j = 0; j < E; ++j) acc1 = fmaf(wf[j], hf[j], acc1);
  }
  if (c < d) {
    const uint4 wv = *reinterpret_cast<const uint4*>(w + c);
    const uint4 hv = *reinterpret_cast<const uint4*>(h + c);
    float wf[E], hf[E];
    widen16(wv, wf, w);
    widen16(hv, hf, h);
#pragma unroll
    for (int j = 0; j < E; ++j) acc0 = fmaf(wf[j], hf[j], acc0);
  }
  return acc0 + acc1;
}

__device__ __forceinline__ long long shortlist_len(const HeadArgs& a, int gi) {
  const int cnt = a.sel_count[gi];
  if (cnt < 1 || cnt > a.M) return -1;
  const long long N = a.sl_off[(size_t)gi * (a.M + 1) + cnt];
  return (N >= 1 && N <= a.max_shortlist) ? N : -1;
}

template <typename T>
__global__ void __launch_bounds__(kHeadThreads, 1) head_kernel(const HeadArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const HeadLayout L = head_layout(a.nrows, a.d, (int)sizeof(T), a.lcap);
  uint8_t* ring = smem + L.ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kHeadStages;
  int4* info = reinterpret_cast<int4*>(smem + L.info);
  int* misc = reinterpret_cast<int*>(smem + L.misc);
  long long* sega = reinterpret_cast<long long*>(smem + L.sega);
  int* segn = reinterpret_cast<int*>(smem + L.segn);
  T* hs = reinterpret_cast<T*>(smem + L.h);
  float* zl = reinterpret_cast<float*>(smem + L.zl);
  int* zid = reinterpret_cast<int*>(smem + L.zid);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, g = blockIdx.x;
  const int ngroups = a.shared ? 1 : a.nrows;

  if (tid == 0) {
    for (int s = 0; s < kHeadStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kHeadConsumerWarps);
    }
    fence_mbar_init();
  }
  if (a.pdl) pdl_wait();  // sel / sl_offsets / h_new come from upstream kernels
  for (int gi = tid; gi < ngroups; gi += kHeadThreads) {
    const long long N = shortlist_len(a, gi);
    if (N < 0) {
      sega[gi] = 0;
      segn[gi] = -1;
    } else {
      const long long s0 = N * g / G, s1 = N * (g + 1) / G;
      sega[gi] = s0;
      segn[gi] = (int)(s1 - s0);
    }
  }
  __syncthreads();

  if (warp == kHeadConsumerWarps) {
    // ---------------- producer: one lane streams this CTA's segments with TMA 1D bulk copies
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint32_t rowbytes = (uint32_t)a.d * (uint32_t)sizeof(T);
      const uint8_t* W = static_cast<const uint8_t*>(a.W);
      uint32_t it = 0;
      for (int gi = 0; gi < ngroups; ++gi) {
        const int nseg = segn[gi];
        if (nseg <= 0) continue;
        const long long s0 = sega[gi], s1 = s0 + nseg;
        const int32_t* so = a.sl_off + (size_t)gi * (a.M + 1);
        const int32_t* sl = a.sel + (size_t)gi * a.M;
        int i = 0;
        while (so[i + 1] <= s0) ++i;  // cluster holding virtual position s0
        long long pos = s0;
        while (pos < s1) {
          const long long cl_end = so[i + 1];
          const long long lim = cl_end < s1 ? cl_end : s1;
          const int n = (int)min((long long)a.stage_rows, lim - pos);
          const long long wrow = (long long)a.offsets[sl[i]] + (pos - so[i]);
          const uint32_t s = it % kHeadStages;
          mbar_wait(&empty[s], ((it / kHeadStages) & 1u) ^ 1u);
          info[s] = make_int4(gi, (int)(pos - s0), n, (int)wrow);
          mbar_arrive_expect_tx(&full[s], (uint32_t)n * rowbytes);
          bulk_g2s(ring + (size_t)s * kHeadStageBytes, W + (size_t)wrow * rowbytes, (uint32_t)n * rowbytes,
                   &full[s], pol);
          ++it;
          pos += n;
          if (pos == cl_end) ++i;
        }
      }
      const uint32_t s = it % kHeadStages;
      mbar_wait(&empty[s], ((it / kHeadStages) & 1u) ^ 1u);
      info[s] = make_int4(-1, 0, -1, 0);  // end of stream
      mbar_arrive(&full[s]);
    }
  } else {
    // ---------------- consumers: h_new -> smem once, then dot every staged row
    constexpr int kCT = kHeadConsumerWarps * 32;
    const size_t hvec = (size_t)a.nrows * a.d * sizeof(T) / 16;
    const uint4* hsrc = static_cast<const uint4*>(a.h);
    uint4* hdst = reinterpret_cast<uint4*>(hs);
    for (size_t i = tid; i < hvec; i += kCT) hdst[i] = hsrc[i];
    named_bar_sync(1, kCT);
    uint32_t q = 0;  // rows consumed so far: warp w takes rows q with q % 8 == w
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it % kHeadStages;
      mbar_wait(&full[s], (it / kHeadStages) & 1u);
      const int4 inf = info[s];
      if (inf.z < 0) break;
      const T* st = reinterpret_cast<const T*>(ring + (size_t)s * kHeadStageBytes);
      const int gi = inf.x;
      const int r_lo = a.shared ? 0 : gi, r_hi = a.shared ? a.nrows : gi + 1;
      const int first = (int)((warp - (int)(q % kHeadConsumerWarps) + kHeadConsumerWarps) % kHeadConsumerWarps);
      for (int rr = first; rr < inf.z; rr += kHeadConsumerWarps) {
        const T* wr = st + (size_t)rr * a.d;
        const int tok = __ldg(a.perm + inf.w + rr);
        const int local = inf.y + rr;
        for (int r = r_lo; r < r_hi; ++r) {
          float acc = dot_row<T>(wr, hs + (size_t)r * a.d, a.d, lane);
          acc = warp_sum(acc) + 0.0f;  // + 0.0f: -0 -> +0 (R23)
          if (lane == 0) {
            zl[r * a.lcap + local] = acc;
            zid[r * a.lcap + local] = tok;
            if (a.z_out) a.z_out[(size_t)r * a.z_stride + sega[gi] + local] = acc;
          }
        }
      }
      q += (uint32_t)inf.z;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (a.pdl) pdl_launch_dependents();

  // ---------------- per-CTA partial: top-k_t (logit desc, id asc), max, sum exp(z - max)
  const int rec = 2 + 2 * a.k_t;
  for (int r = warp; r < a.nrows; r += kHeadWarps) {
    const int gi = a.shared ? 0 : r;
    const int n = segn[gi];
    float* P = a.part + ((size_t)g * a.nrows + r) * rec;
    const float* zr = zl + r * a.lcap;
    const int* ir = zid + r * a.lcap;
    float pv = INFINITY, mx = -INFINITY;
    int pid = -1;
    for (int qq = 0; qq < a.k_t; ++qq) {
      float bv = -INFINITY;
      int bid = INT_MAX, aux = 0;
      for (int j = lane; j < n; j += 32) {
        const float v = zr[j];
        const int id = ir[j];
        if (beats(pv, pid, v, id) && beats(v, id, bv, bid)) {
          bv = v;
          bid = id;
        }
      }
      warp_best(bv, bid, aux);
      if (qq == 0) mx = bv;
      if (lane == 0) {
        P[2 + 2 * qq] = bv;
        P[3 + 2 * qq] = __int_as_float(bid);
      }
      pv = bv;
      pid = bid;
    }
    float se = 0.f;
    for (int j = lane; j < n; j += 32) se += expf(zr[j] - mx);
    se = warp_sum(se);
    if (lane == 0) {
      P[0] = mx;
      P[1] = se;
    }
  }

  // ---------------- last CTA merges the G partials in CTA order
  __threadfence();
  __syncthreads();
  if (tid == 0) misc[0] = (atomicAdd(a.counter, 1u) == (unsigned)(G - 1)) ? 1 : 0;
  __syncthreads();
  if (!misc[0]) return;
  __threadfence();

  const int per_row = G * rec;
  const int ring_bytes = kHeadStages * kHeadStageBytes;
  int batch = ring_bytes / (per_row * 4 + G);
  batch = batch < 1 ? 1 : (batch > kHeadWarps ? kHeadWarps : batch);
  float* mbuf = reinterpret_cast<float*>(ring);
  uint8_t* ptr_base = ring + (size_t)batch * per_row * 4;
  for (int r0 = 0; r0 < a.nrows; r0 += batch) {
    const int nb = min(batch, a.nrows - r0);
    for (int idx = tid; idx < nb * per_row; idx += kHeadThreads) {
      const int rb = idx / per_row, rem = idx - rb * per_row;
      const int gg = rem / rec, f = rem - gg * rec;
      mbuf[idx] = __ldcg(a.part + ((size_t)gg * a.nrows + r0 + rb) * rec + f);
    }
    __syncthreads();
    if (warp < nb) {
      const int r = r0 + warp;
      const float* R = mbuf + (size_t)warp * per_row;
      uint8_t* ptr = ptr_base + (size_t)warp * G;
      const bool ok = shortlist_len(a, a.shared ? 0 : r) >= 0;
      float mx = -INFINITY;
      for (int gg = lane; gg < G; gg += 32) {
        mx = fmaxf(mx, R[gg * rec]);
        ptr[gg] = 0;
      }
      mx = warp_max(mx);
      float S = 0.f;
      for (int gg = lane; gg < G; gg += 32) {
        const float m = R[gg * rec];
        if (m > -INFINITY) S += R[gg * rec + 1] * expf(m - mx);
      }
      S = warp_sum(S);
      const float lse = ok ? mx + logf(S) : __int_as_float(0x7fc00000);
      __syncwarp();
      float bv;
      int bid, bl;
      auto lane_best = [&]() {
        bv = -INFINITY;
        bid = INT_MAX;
        bl = -1;
        for (int gg = lane; gg < G; gg += 32) {
          const int p = ptr[gg];
          if (p >= a.k_t) continue;
          const float v = R[gg * rec + 2 + 2 * p];
          const int id = __float_as_int(R[gg * rec + 3 + 2 * p]);
          if (beats(v, id, bv, bid)) {
            bv = v;
            bid = id;
            bl = gg;
          }
        }
      };
      lane_best();
      for (int qq = 0; qq < a.k_t; ++qq) {
        float wv = bv;
        int wid = bid, wl = bl;
        warp_best(wv, wid, wl);
        if (lane == 0) {
          const bool valid = ok && wv > -INFINITY;
          a.top_ids[(size_t)r * a.k_t + qq] = valid ? wid : -1;
          a.top_logits[(size_t)r * a.k_t + qq] = valid ? wv : -INFINITY;
          a.top_logp[(size_t)r * a.k_t + qq] = valid ? wv - lse : -INFINITY;
        }
        if (wl >= 0 && (wl & 31) == lane) {
          ptr[wl] = (uint8_t)(ptr[wl] + 1);
          lane_best();
        }
        __syncwarp();
      }
      if (lane == 0) a.lse[r] = lse;
    }
    __syncthreads();
  }
  if (tid == 0) *a.counter = 0u;  // leave the ticket at zero for the next launch
}

// ------------------------------------------------------------------ host side

bool head_plan(const ds_clusters* c, int B, int k_t, int64_t max_shortlist, HeadPlan* p) {
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  const int rowbytes = c->d * esz;
  if (rowbytes > kHeadStageBytes || (rowbytes % 16) != 0) return false;
  p->stage_rows = std::min(kHeadStageBytes / rowbytes, 16);
  p->G = num_sms();
  const int64_t ms = (max_shortlist > 0 && max_shortlist < c->V) ? max_shortlist : c->V;
  p->lcap = (int)((ms + p->G - 1) / p->G);
  int dev = 0;
  cudaGetDevice(&dev);
  int max_smem = 232448;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const HeadLayout L0 = head_layout(0, c->d, esz, p->lcap);
  const int per_row = rowbytes + p->lcap * 8 + 16;
  int rows = (max_smem - (int)L0.total) / per_row;
  if (rows < 1) return false;
  rows = std::min(rows, kHeadMaxRows);
  p->rows_per_launch = std::max(1, std::min(B, rows));
  p->rec = 2 + 2 * k_t;
  p->smem = head_layout(p->rows_per_launch, c->d, esz, p->lcap).total;
  if (p->smem > (size_t)max_smem) return false;
  if ((int64_t)p->G * p->rec * 4 + p->G > kHeadStages * kHeadStageBytes) return false;
  p->part_bytes = (size_t)p->G * p->rows_per_launch * p->rec * sizeof(float);
  p->launches = (B + p->rows_per_launch - 1) / p->rows_per_launch;
  return true;
}

template <typename T>
static cudaError_t launch_head_t(const HeadArgs& a, const HeadPlan& p, cudaStream_t st, bool pdl) {
  static bool configured = false;  // idempotent attribute set; benign race
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(head_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(kHeadThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, head_kernel<T>, a);
}

cudaError_t launch_head(const ds_clusters* c, const HeadPlan& p, const void* h_new, int B, const int32_t* sel,
                        const int32_t* sel_count, const int32_t* sl_offsets, int shared, int k_t,
                        int64_t max_shortlist, int32_t* top_ids, float* top_logits, float* top_logp, float* lse,
                        float* z_out, int64_t z_stride, float* part, unsigned* counter, cudaStream_t st,
                        bool pdl) {
  const int esz = c->dtype == DS_BF16 ? 2 : 4;
  const int64_t ms = (max_shortlist > 0 && max_shortlist < c->V) ? max_shortlist : c->V;
  for (int r0 = 0; r0 < B; r0 += p.rows_per_launch) {
    const int nr = std::min(p.rows_per_launch, B - r0);
    HeadArgs a;
    a.W = c->W_perm;
    a.perm = c->perm;
    a.offsets = c->offsets;
    const int goff = shared ? 0 : r0;
    a.sel = sel + (size_t)goff * c->M;
    a.sel_count = sel_count + goff;
    a.sl_off = sl_offsets + (size_t)goff * (c->M + 1);
    a.h = static_cast<const uint8_t*>(h_new) + (size_t)r0 * c->d * esz;
    a.M = c->M;
    a.nrows = nr;
    a.d = c->d;
    a.k_t = k_t;
    a.shared = shared;
    a.lcap = p.lcap;
    a.stage_rows = p.stage_rows;
    a.pdl = pdl ? 1 : 0;
    a.max_shortlist = ms;
    a.top_ids = top_ids + (size_t)r0 * k_t;
    a.top_logits = top_logits + (size_t)r0 * k_t;
    a.top_logp = top_logp + (size_t)r0 * k_t;
    a.lse = lse + r0;
    a.z_out = z_out ? z_out + (size_t)r0 * z_stride : nullptr;
    a.z_stride = z_stride;
    a.part = part;
    a.counter = counter;
    HeadPlan pp = p;
    pp.smem = head_layout(nr, c->d, esz, p.lcap).total;
    cudaError_t e = c->dtype == DS_BF16 ? launch_head_t<__nv_bfloat16>(a, pp, st, pdl && r0 == 0)
                                        : launch_head_t<float>(a, pp, st, pdl && r0 == 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ds
