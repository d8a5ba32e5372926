// verify.cu — NEXT-4: lossless verification of drafted chains against the target's full-vocabulary
// logits (Eq. 3, and the speculative-sampling rule its footnote cites; SPEC S:454-464;
// reading R25), plus the shortlist-id materialisation (S4) that embeds the drafter's q in V.
//
// Two launches, both HBM-streaming over the target logits (no contraction: CUDA cores, 16 B loads).
// Every CTA is 16 independent warps; warp w of CTA c owns the contiguous vocabulary segment
// c * 16 + w of its row (segments in id order), streams it with 4-deep 16 B loads and keeps a
// per-lane online (max, sum exp) / residual sum — no block barrier on the streaming path, one
// fence + ticket per CTA.
//   verify_lse_kernel      grid (B (gamma+1), S1): per-segment (max, sum exp) of every target row;
//                          the last CTA of a row folds them into lse_p[row]; the last row of a chain
//                          takes the accept decisions u_i < p_i(x_i) / q_i(x_i), finds the first
//                          rejection j and scatters q_j into the chain's dense q buffer.
//   verify_residual_kernel grid (B, S3): per-segment sums of w = (p_j - q_j)_+ (the bonus case j =
//                          gamma has q = 0, so w = p_gamma); the last CTA of a chain finds the segment
//                          whose cumulative weight crosses u_res * Z, rescans it in id order for the
//                          token (R25) and clears the scattered q entries (the buffer stays zero).
#include <algorithm>

#include "head_impl.cuh"
#include "internal.h"

namespace ds {

constexpr int kVT = 512;             // threads per CTA
constexpr int kVW = kVT / 32;        // warps (= segments) per CTA

struct VerifyArgs {
  const void* p_logits;  // [B][gamma+1][V]
  int64_t V;
  int B, gamma;
  int s1, s3;            // CTAs per row (lse pass) / per chain (residual pass)
  int64_t L1, L3;        // segment lengths (multiples of 8)
  const int32_t* q_ids;
  const float* q_logits;
  int64_t q_stride;
  const int32_t* q_count;
  const float* q_lse;
  const int32_t* x;
  const int32_t* x_slot;
  const float* u_acc;
  const float* u_res;
  int32_t* accepted;
  int32_t* committed;
  float2* part;         // [B (gamma+1)][s1 * 16] (max, sum exp)
  float4* rowrec;       // [B (gamma+1)] decision inputs {l[x], log q(x), u, valid}
  int32_t* rowflag;     // [B (gamma+1)] 1 accept, 0 reject, -1 invalid proposal
  float* lse_p;         // [B (gamma+1)]
  float2* wpart;        // [B][s3 * 16] (sum w, sum p)
  int32_t* jrow;        // [B]
  float* qbuf;          // [B][V], zero between calls
  unsigned* ctr_row;    // [B (gamma+1)]
  unsigned* ctr_chain;  // [B]
  unsigned* ctr_res;    // [B]
  int pf;               // lse pass: L2 bulk-prefetch distance in batches (0 off; DS_VERIFY_PF)
};

constexpr float kLog2e = 1.4426950408889634f;
// 2^x on the SFU (ex2.approx.ftz: ~2 ulp; -inf -> +0).  exp(v - c) = ex2(v log2e - c log2e).
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe for x <= 0 (round-to-nearest split x = j + f, |f| <= 1/2, Taylor degree 6 of
// 2^f: relative error <= 1.3e-7, about ex2.approx's; x < -126 clamps to ~2^-126).  Moves part of the
// lse pass's exponentials off the SFU (DS_VERIFY_POLY = how many of each lane's 16 word pairs).
__device__ __forceinline__ float ex2_fma(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: the low mantissa bits hold round(x)
  const int j = __float_as_int(t) - 0x4B400000;
  const float f = x - (t - 12582912.f);
  float p = 1.5403530393381606e-4f;
  p = fmaf(p, f, 1.3333558146428443e-3f);
  p = fmaf(p, f, 9.6181291076284772e-3f);
  p = fmaf(p, f, 5.5504108664821580e-2f);
  p = fmaf(p, f, 2.4022650695910071e-1f);
  p = fmaf(p, f, 6.9314718055994531e-1f);
  p = fmaf(p, f, 1.f);
  return __int_as_float(__float_as_int(p) + (j << 23));
}

__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }

// ---- segment streaming: raw 16 B register buffers, the next batch's loads issued before the
// current batch is processed (software pipelining); U groups of 8 ids per lane per batch.
template <typename T> struct Raw { static constexpr int N = sizeof(T) == 2 ? 1 : 2; };  // uint4 per 8 ids
template <typename T> __device__ __forceinline__ uint32_t neg_inf_bits() {
  return sizeof(T) == 2 ? 0xFF80FF80u : 0xFF800000u;
}
__device__ __forceinline__ void widen8(const uint4* r, float* v, const __nv_bfloat16*) {
  widen16(r[0], v, (const __nv_bfloat16*)nullptr);
}
__device__ __forceinline__ void widen8(const uint4* r, float* v, const float*) {
  widen16(r[0], v, (const float*)nullptr);
  widen16(r[1], v + 4, (const float*)nullptr);
}

template <typename T, int U, bool Q, typename F>
__device__ __forceinline__ void stream_segment(const T* __restrict__ l, const float* __restrict__ qb, int lo, int hi,
                                               int lane, F&& f) {
  constexpr int R = Raw<T>::N, STEP = 32 * 8 * U;
  uint4 cl[U][R], cq[U][2];
  auto issue = [&](int x0, uint4 (&dl)[U][R], uint4 (&dq)[U][2]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int x = x0 + u * 256;
      if (x < hi) {
#pragma unroll
        for (int r = 0; r < R; ++r) dl[u][r] = reinterpret_cast<const uint4*>(l + x)[r];
        if (Q) {
          dq[u][0] = *reinterpret_cast<const uint4*>(qb + x);
          dq[u][1] = *reinterpret_cast<const uint4*>(qb + x + 4);
        }
      } else {
        const uint32_t ni = neg_inf_bits<T>();
#pragma unroll
        for (int r = 0; r < R; ++r) dl[u][r] = make_uint4(ni, ni, ni, ni);
        if (Q) dq[u][0] = dq[u][1] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
  };
  int x0 = lo + lane * 8;
  if (x0 >= hi) return;
  issue(x0, cl, cq);
  for (; x0 < hi; x0 += STEP) {
    uint4 nl[U][R], nq[U][2];
    const bool more = x0 + STEP < hi;
    if (more) issue(x0 + STEP, nl, nq);
    float v[U][8], q[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      widen8(cl[u], v[u], (const T*)nullptr);
      if (Q) {
        widen16(cq[u][0], q[u], (const float*)nullptr);
        widen16(cq[u][1], q[u] + 4, (const float*)nullptr);
      }
    }
    f(v, q);
    if (more) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int r = 0; r < R; ++r) cl[u][r] = nl[u][r];
        if (Q) {
          cq[u][0] = nq[u][0];
          cq[u][1] = nq[u][1];
        }
      }
    }
  }
}

// bf16 lse of a warp segment, lean inner loop: 4 x 16 B per lane per batch (1024 logits per warp),
// the next batch's loads in flight; the batch max by packed bf16x2 max (exact), then one
// exp2 per logit against the running max in two independent sums.  ~4.5 instructions per logit
// (the generic stream_segment path needs ~13).  Returns the first position it did not cover.
template <int NP>
__device__ __forceinline__ int lse_seg_bf16(const __nv_bfloat16* l, int lo, int hi, int lane, float& m, float& s,
                                            int pf) {
  constexpr int U = 4, STEP = 32 * 8 * U;
  const int nfull = (hi - lo) / STEP;
  if (nfull <= 0) return lo;
  const uint4* base = reinterpret_cast<const uint4*>(l + lo) + lane;
  if (pf > 0 && lane == 0) {  // batches 1 .. pf into L2 (one 2 KB bulk prefetch each; no registers)
    for (int q = 1; q <= pf && q < nfull; ++q)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(l + lo + (size_t)q * STEP), "r"(STEP * 2)
                   : "memory");
  }
  uint4 cur[U], nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cur[u] = __ldcs(base + u * 32);
  for (int bt = 0; bt < nfull; ++bt) {
    if (pf > 0 && lane == 0 && bt + 1 + pf < nfull)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(l + lo + (size_t)(bt + 1 + pf) * STEP),
                   "r"(STEP * 2)
                   : "memory");
    if (bt + 1 < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = __ldcs(base + (size_t)(bt + 1) * (STEP / 8) + u * 32);
    }
    uint32_t w[4 * U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      w[4 * u] = cur[u].x;
      w[4 * u + 1] = cur[u].y;
      w[4 * u + 2] = cur[u].z;
      w[4 * u + 3] = cur[u].w;
    }
    __nv_bfloat162 mx2 = *reinterpret_cast<const __nv_bfloat162*>(&w[0]);
#pragma unroll
    for (int i = 1; i < 4 * U; ++i) mx2 = __hmax2(mx2, *reinterpret_cast<const __nv_bfloat162*>(&w[i]));
    const float mx = fmaxf(m, fmaxf(__low2float(mx2), __high2float(mx2)));
    if (mx != -INFINITY) {
      const float mxl = mx * kLog2e;
      float acc0 = m == -INFINITY ? 0.f : s * ex2(fmaf(m, kLog2e, -mxl)), acc1 = 0.f;
#pragma unroll
      for (int i = 0; i < 4 * U; ++i) {
        acc0 += ex2(fmaf(__uint_as_float(w[i] << 16), kLog2e, -mxl));
        const float xh = fmaf(__uint_as_float(w[i] & 0xffff0000u), kLog2e, -mxl);
        acc1 += i < NP ? ex2_fma(xh) : ex2(xh);
      }
      s = acc0 + acc1;
      m = mx;
    }
    if (bt + 1 < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
  }
  return lo + nfull * STEP;
}

// Warp-wide (max, sum) combine, every lane returns the result (fixed xor-tree order).
__device__ __forceinline__ void warp_lse_pair(float& m, float& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_combine(m, s, m2, s2);
  }
}

// Decision inputs of drafted position i of chain b (row b (gamma+1) + i), loaded while the row
// streams: {target logit of x_i, log q_i(x_i), u_i, valid}.
template <typename T>
__device__ __forceinline__ void decision_inputs(const VerifyArgs& a, int b, int i) {
  const int g = a.gamma, pi = b * g + i;
  const int xi = a.x[pi], slot = a.x_slot[pi], cnt = a.q_count[pi];
  const bool ok = xi >= 0 && xi < a.V && slot >= 0 && slot < cnt;
  float lx = 0.f, lq = 0.f;
  bool valid = false;
  if (ok) {
    const int id = a.q_ids[(size_t)pi * a.q_stride + slot];
    const T* l = static_cast<const T*>(a.p_logits) + ((size_t)b * (g + 1) + i) * a.V;
    lx = to_f(l[xi]);
    lq = a.q_logits[(size_t)pi * a.q_stride + slot] - a.q_lse[pi];
    valid = id == xi;
  }
  a.rowrec[(size_t)b * (g + 1) + i] = make_float4(lx, lq, a.u_acc[pi], valid ? 1.f : 0.f);
}

// Chain b's first rejection from the per-row flags (warp 0), then the q_j scatter (whole CTA).
__device__ void verify_decide(const VerifyArgs& a, int b, int* sh) {
  const int lane = threadIdx.x & 31, g = a.gamma, g1 = g + 1;
  if (threadIdx.x < 32) {
    const int f = lane < g ? __ldcg(&a.rowflag[b * g1 + lane]) : 1;  // 1 accept, 0 reject, -1 invalid
    const int xl = lane < g ? a.x[b * g + lane] : 0;
    const unsigned stop = __ballot_sync(0xffffffffu, f != 1);
    const int j = stop ? __ffs(stop) - 1 : g;
    const bool bad = j < g && __shfl_sync(0xffffffffu, f, j & 31) < 0;
    if (!bad && lane < j) a.committed[(size_t)b * g1 + lane] = xl;
    if (lane == 0) {
      a.jrow[b] = bad ? -1 : j;
      a.accepted[b] = bad ? -1 : j;
      if (bad) a.committed[(size_t)b * g1] = -1;
      a.ctr_chain[b] = 0;
      sh[0] = bad ? -1 : j;
    }
  }
  __syncthreads();
  const int j = sh[0];
  if (j < 0 || j >= g) return;
  const int pi = b * g + j;
  const int n = a.q_count[pi];
  const float qs = a.q_lse[pi];
  const int32_t* __restrict__ ids = a.q_ids + (size_t)pi * a.q_stride;
  const float* __restrict__ ql = a.q_logits + (size_t)pi * a.q_stride;
  float* qb = a.qbuf + (size_t)b * a.V;
  for (int s0 = threadIdx.x; s0 < n; s0 += 8 * kVT) {  // loads first (8 in flight), then the stores
    int id[8];
    float z[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int s = s0 + u * kVT;
      id[u] = s < n ? ids[s] : -1;
      z[u] = s < n ? ql[s] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (id[u] >= 0) qb[id[u]] = expf(z[u] - qs);
  }
}

template <typename T, int NP>
__global__ void __launch_bounds__(kVT, 2) verify_lse_kernel(const VerifyArgs a) {
  __shared__ int sh[2];
  const int row = blockIdx.x, cta = blockIdx.y, g1 = a.gamma + 1, b = row / g1, i = row - b * g1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = cta * kVW + warp;
  pdl_launch_dependents();  // the residual pass may be scheduled now; it waits for this grid's completion
  const T* l = static_cast<const T*>(a.p_logits) + (size_t)row * a.V;
  const int V = (int)a.V, L1 = (int)a.L1;
  const int lo = (int)min((int64_t)seg * L1, (int64_t)V), hi = min(V, lo + L1);
  constexpr int U = sizeof(T) == 2 ? 2 : 1;  // groups of 8 ids per lane per batch (2 batches in flight)
  float m = -INFINITY, s = 0.f;
  int lo2 = lo;  // bf16 rows with 16-byte aligned segments: lean full batches, generic tail
  if (sizeof(T) == 2 && ((reinterpret_cast<uintptr_t>(l + lo) & 15u) == 0))
    lo2 = lse_seg_bf16<NP>(reinterpret_cast<const __nv_bfloat16*>(l), lo, hi, lane, m, s, a.pf);
  stream_segment<T, U, false>(l, nullptr, lo2, hi, lane, [&](float (&v)[U][8], float (&)[U][8]) {
    float mx = m;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < 8; ++e) mx = fmaxf(mx, v[u][e]);
    if (mx != -INFINITY) {
      const float mxl = mx * kLog2e;
      float acc = m == -INFINITY ? 0.f : s * ex2(fmaf(m, kLog2e, -mxl));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += ex2(fmaf(v[u][e], kLog2e, -mxl));
      s = acc;
      m = mx;
    }
  });
  __shared__ float2 wpart[kVW];
  warp_lse_pair(m, s);
  if (a.s1 == 1) {  // the row is this CTA's alone: fold the warp partials in shared memory
    if (lane == 0) wpart[warp] = make_float2(m, s);
  } else if (lane == 0) {
    a.part[(size_t)row * a.s1 * kVW + seg] = make_float2(m, s);
  }
  if (cta == 0 && threadIdx.x == 32 && i < a.gamma) decision_inputs<T>(a, b, i);
  __syncthreads();
  if (a.s1 > 1) {
    if (threadIdx.x == 0) {
      fence_acq_rel_gpu();
      sh[0] = atomicAdd(&a.ctr_row[row], 1u) == (unsigned)(a.s1 - 1);
    }
    __syncthreads();
    if (!sh[0]) return;
    fence_acq_rel_gpu();
  }
  if (warp == 0) {
    const int np = a.s1 * kVW;  // <= 512: 16 independent loads per lane
    float M = -INFINITY, S = 0.f;
    if (a.s1 == 1) {
      const float2 pp = lane < kVW ? wpart[lane] : make_float2(-INFINITY, 0.f);
      lse_combine(M, S, pp.x, pp.y);
    } else {
      for (int h = 0; h < np; h += 8 * 32) {  // 8 independent loads per lane per round
        float2 pp[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int c = h + k * 32 + lane;
          pp[k] = c < np ? __ldcg(&a.part[(size_t)row * np + c]) : make_float2(-INFINITY, 0.f);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) lse_combine(M, S, pp[k].x, pp[k].y);
      }
    }
    warp_lse_pair(M, S);
    if (lane == 0) {
      const float lse = M + logf(S);
      a.lse_p[row] = lse;
      if (i < a.gamma) {  // Eq. 3: accept iff u < p(x) / q(x)
        if (a.s1 == 1) fence_acq_rel_gpu();  // thread 32's rowrec store, ordered by the barrier
        const float4 r = __ldcg(&a.rowrec[row]);
        const float p = expf(r.x - lse), q = expf(r.y);
        a.rowflag[row] = r.w == 0.f ? -1 : (r.z < p / q ? 1 : 0);
      }
      a.ctr_row[row] = 0;
      fence_acq_rel_gpu();
      sh[1] = atomicAdd(&a.ctr_chain[b], 1u) == (unsigned)(g1 - 1);
    }
  }
  __syncthreads();
  if (!sh[1]) return;
  fence_acq_rel_gpu();
  verify_decide(a, b, sh);
}

template <typename T>
__global__ void __launch_bounds__(kVT, 2) verify_residual_kernel(const VerifyArgs a) {
  __shared__ int ish[2];
  __shared__ float wsum[kVW], fsh[3];
  const int b = blockIdx.x, cta = blockIdx.y, g1 = a.gamma + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();  // the lse pass (a programmatic dependency when DS_VERIFY_PDL is on; else a no-op)
  const int j = a.jrow[b];
  if (j < 0) return;
  const int row = b * g1 + j;
  const float lse = a.lse_p[row];
  const float lsel = lse * kLog2e;
  const T* l = static_cast<const T*>(a.p_logits) + (size_t)row * a.V;
  const float* qb = a.qbuf + (size_t)b * a.V;
  const int nseg = a.s3 * kVW;
  const int seg = cta * kVW + warp;
  const int V = (int)a.V, L3 = (int)a.L3;
  {
    const int lo = (int)min((int64_t)seg * L3, (int64_t)V), hi = min(V, lo + L3);
    constexpr int U = sizeof(T) == 2 ? 2 : 1;
    float sw = 0.f, sp = 0.f;
    stream_segment<T, U, true>(l, qb, lo, hi, lane, [&](float (&v)[U][8], float (&q)[U][8]) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float p = ex2(fmaf(v[u][e], kLog2e, -lsel));
          sp += p;
          sw += fmaxf(p - q[u][e], 0.f);
        }
    });
    sw = warp_sum(sw);
    sp = warp_sum(sp);
    if (lane == 0) a.wpart[(size_t)b * nseg + seg] = make_float2(sw, sp);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    ish[0] = atomicAdd(&a.ctr_res[b], 1u) == (unsigned)(a.s3 - 1);
  }
  __syncthreads();
  if (!ish[0]) return;
  fence_acq_rel_gpu();
  // ---- last CTA of the chain: inverse CDF in id order (R25).  Warp 0 finds the segment s* whose
  // cumulative weight first exceeds u_res Z; the 16 warps then split s* and the crossing warp
  // finds the token.
  if (warp == 0) {
    const float2* wp = a.wpart + (size_t)b * nseg;
    float2 t[16];  // nseg <= 512
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int c = k * 32 + lane;
      t[k] = c < nseg ? __ldcg(&wp[c]) : make_float2(0.f, 0.f);
    }
    float Zw = 0.f, Zp = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {  // fixed order: per 32 segments, the warp tree, then in k order
      Zw += warp_sum(t[k].x);
      Zp += warp_sum(t[k].y);
    }
    const bool usep = !(Zw > 0.f);  // R25: p == q numerically -> sample from p
    const float target = a.u_res[b] * (usep ? Zp : Zw);
    float base = 0.f, last_base = 0.f;
    int sstar = -1, last_pos = -1;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (sstar >= 0) break;
      const float w = usep ? t[k].y : t[k].x;
      float inc = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, w > 0.f && base + inc > target);
      const unsigned pos = __ballot_sync(0xffffffffu, w > 0.f);
      if (pos) {
        const int lp = 31 - __clz(pos);
        last_pos = k * 32 + lp;
        last_base = base + __shfl_sync(0xffffffffu, inc - w, lp);
      }
      if (hit) {
        const int f = __ffs(hit) - 1;
        sstar = k * 32 + f;
        base += __shfl_sync(0xffffffffu, inc - w, f);
      } else {
        base += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    if (sstar < 0) {
      sstar = last_pos >= 0 ? last_pos : 0;
      base = last_base;
    }
    if (lane == 0) {
      ish[1] = sstar | (usep ? (1 << 30) : 0);
      fsh[0] = base;
      fsh[1] = target;
    }
  }
  __syncthreads();
  const int sstar = ish[1] & ((1 << 30) - 1);
  const bool usep = (ish[1] >> 30) & 1;
  const float target = fsh[1];
  const int slo = (int)min((int64_t)sstar * L3, (int64_t)V), shi = min(V, slo + L3);
  const int sub = ((shi - slo + kVW - 1) / kVW + 7) / 8 * 8;  // per-warp sub-range of s*, multiple of 8
  const int wlo = min(shi, slo + warp * sub), whi = min(shi, wlo + sub);
  auto weights = [&](int x, float* w) -> float {  // w of 8 ids at x (0 past the segment)
    float tot = 0.f;
    if (x < whi) {
      float v[8], q[8];
      uint4 r[2];
#pragma unroll
      for (int k = 0; k < Raw<T>::N; ++k) r[k] = reinterpret_cast<const uint4*>(l + x)[k];
      widen8(r, v, (const T*)nullptr);
      widen16(*reinterpret_cast<const uint4*>(qb + x), q, (const float*)nullptr);
      widen16(*reinterpret_cast<const uint4*>(qb + x + 4), q + 4, (const float*)nullptr);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float p = ex2(fmaf(v[e], kLog2e, -lsel));
        w[e] = usep ? p : fmaxf(p - q[e], 0.f);
        tot += w[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) w[e] = 0.f;
    }
    return tot;
  };
  float mine = 0.f;
  for (int x0 = wlo; x0 < whi; x0 += 256) {
    float w[8];
    mine += weights(x0 + lane * 8, w);
  }
  mine = warp_sum(mine);
  if (lane == 0) wsum[warp] = mine;
  __syncthreads();
  float wb = fsh[0];
  int cw = -1;
  for (int k = 0; k < kVW; ++k) {  // the crossing warp (uniform across the CTA)
    if (cw < 0 && wsum[k] > 0.f && wb + wsum[k] > target) cw = k;
    if (cw < 0) wb += wsum[k];
  }
  if (cw < 0) {  // rounding: fall back to the last warp with weight
    float pre = 0.f, pre_last = 0.f;
    for (int k = 0; k < kVW; ++k) {
      if (wsum[k] > 0.f) {
        cw = k;
        pre_last = pre;
      }
      pre += wsum[k];
    }
    wb = fsh[0] + pre_last;
  }
  if (warp == (cw < 0 ? 0 : cw)) {
    int found = -1, lastx = -1;
    float base = wb;
    for (int x0 = wlo; x0 < whi && found < 0; x0 += 256) {
      const int x = x0 + lane * 8;
      float w[8];
      const float tot = weights(x, w);
      float inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      float cum = base + inc - tot;
      int f = -1, ml = -1;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cum += w[e];
        if (w[e] > 0.f) {
          ml = x + e;
          if (f < 0 && cum > target) f = x + e;
        }
      }
      const unsigned hit = __ballot_sync(0xffffffffu, f >= 0);
      if (hit) found = __shfl_sync(0xffffffffu, f, __ffs(hit) - 1);
      const unsigned pos = __ballot_sync(0xffffffffu, ml >= 0);
      if (pos) lastx = __shfl_sync(0xffffffffu, ml, 31 - __clz(pos));
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      a.committed[(size_t)b * g1 + j] = found >= 0 ? found : (lastx >= 0 ? lastx : slo);
      a.ctr_res[b] = 0;
    }
  }
  if (j < a.gamma) {  // leave the q buffer zero for the next call
    const int pi = b * a.gamma + j;
    const int n = a.q_count[pi];
    const int32_t* ids = a.q_ids + (size_t)pi * a.q_stride;
    float* qw = a.qbuf + (size_t)b * a.V;
    __syncthreads();  // the crossing warp's rescan reads the buffer
    for (int s0 = threadIdx.x; s0 < n; s0 += 8 * kVT) {
      int id[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) id[u] = s0 + u * kVT < n ? ids[s0 + u * kVT] : -1;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (id[u] >= 0) qw[id[u]] = 0.f;
    }
  }
}

// ------------------------------------------------------------------ shortlist ids (S4)

// One CTA per row, one warp per selected cluster: ids[r][sl_off[r][i] + u] = perm[offsets[m_i] + u].
__global__ void shortlist_ids_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ offsets, int M,
                                     const int32_t* __restrict__ sel, const int32_t* __restrict__ cnt,
                                     const int32_t* __restrict__ sl_off, int64_t stride, int32_t* __restrict__ ids) {
  const int r = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = cnt[r];
  for (int i = warp; i < n; i += nw) {
    const int m = sel[(size_t)r * M + i];
    const int o0 = offsets[m], sz = offsets[m + 1] - o0;
    const int base = sl_off[(size_t)r * (M + 1) + i];
    for (int u = lane; u < sz; u += 32) ids[(size_t)r * stride + base + u] = perm[o0 + u];
  }
}

// ------------------------------------------------------------------ host side

struct VerifyLayout {
  int s1, s3;
  int64_t L1, L3;
  size_t part, rowrec, rowflag, lse, wpart, jrow, ctr_row, ctr_chain, ctr_res, qbuf, total;
};

// Splits: at most one wave of two 512-thread CTAs per SM over the rows of each pass, <= 32 CTAs per
// row (<= 512 segments), warp segments >= 256 ids.
static int verify_split(int64_t V, int rows) {
  const char* ev = getenv("DS_VERIFY_SPLIT");  // tuning: CTAs per row
  if (ev && ev[0]) return std::max(1, std::min(32, atoi(ev)));
  const int64_t want = 2 * (int64_t)num_sms() / rows;  // floor: never a partial second wave
  return (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, 32), V / (kVW * 256)));
}
static int64_t verify_seg(int64_t V, int s) {
  const int64_t n = (V + (int64_t)s * kVW - 1) / ((int64_t)s * kVW);
  return (n + 7) / 8 * 8;
}

static VerifyLayout verify_layout(int64_t V, int B, int gamma) {
  const size_t rows = (size_t)B * (gamma + 1);
  VerifyLayout L;
  L.s1 = verify_split(V, (int)rows);
  L.s3 = verify_split(V, B);
  L.L1 = verify_seg(V, L.s1);
  L.L3 = verify_seg(V, L.s3);
  size_t o = 0;
  auto take = [&](size_t n) {
    const size_t at = o;
    o = align_up(o + n, 256);
    return at;
  };
  L.ctr_row = take(rows * 4);
  L.ctr_chain = take((size_t)B * 4);
  L.ctr_res = take((size_t)B * 4);
  L.qbuf = take((size_t)B * V * 4);
  L.part = take(rows * L.s1 * kVW * 8);
  L.rowrec = take(rows * 16);
  L.rowflag = take(rows * 4);
  L.lse = take(rows * 4);
  L.wpart = take((size_t)B * L.s3 * kVW * 8);
  L.jrow = take((size_t)B * 4);
  L.total = o;
  return L;
}

size_t verify_ws_bytes(int64_t V, int B, int gamma) { return verify_layout(V, B, gamma).total; }

cudaError_t launch_verify(const void* p_logits, int dtype, int64_t V, int B, int gamma, const int32_t* q_ids,
                          const float* q_logits, int64_t q_stride, const int32_t* q_count, const float* q_lse,
                          const int32_t* x, const int32_t* x_slot, const float* u_acc, const float* u_res,
                          int32_t* accepted, int32_t* committed, void* ws, cudaStream_t st) {
  const VerifyLayout L = verify_layout(V, B, gamma);
  uint8_t* w = static_cast<uint8_t*>(ws);
  VerifyArgs a;
  a.p_logits = p_logits;
  a.V = V;
  a.B = B;
  a.gamma = gamma;
  a.s1 = L.s1;
  a.s3 = L.s3;
  a.L1 = L.L1;
  a.L3 = L.L3;
  a.q_ids = q_ids;
  a.q_logits = q_logits;
  a.q_stride = q_stride;
  a.q_count = q_count;
  a.q_lse = q_lse;
  a.x = x;
  a.x_slot = x_slot;
  a.u_acc = u_acc;
  a.u_res = u_res;
  a.accepted = accepted;
  a.committed = committed;
  a.part = reinterpret_cast<float2*>(w + L.part);
  a.rowrec = reinterpret_cast<float4*>(w + L.rowrec);
  a.rowflag = reinterpret_cast<int32_t*>(w + L.rowflag);
  a.lse_p = reinterpret_cast<float*>(w + L.lse);
  a.wpart = reinterpret_cast<float2*>(w + L.wpart);
  a.jrow = reinterpret_cast<int32_t*>(w + L.jrow);
  a.qbuf = reinterpret_cast<float*>(w + L.qbuf);
  a.ctr_row = reinterpret_cast<unsigned*>(w + L.ctr_row);
  a.ctr_chain = reinterpret_cast<unsigned*>(w + L.ctr_chain);
  a.ctr_res = reinterpret_cast<unsigned*>(w + L.ctr_res);
  {
    const char* ev = getenv("DS_VERIFY_PF");
    a.pf = ev && ev[0] ? std::max(0, std::min(8, atoi(ev))) : 0;
  }
  const dim3 g1(B * (gamma + 1), L.s1), g2(B, L.s3);  // rows in x (no 65535 limit)
  const char* evp = getenv("DS_VERIFY_PDL");
  const bool pdl = evp && evp[0] == '1';  // A/B knob: no measurable gain (profiles/r2_probes), off
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g2;
  cfg.blockDim = dim3(kVT);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (dtype == DS_BF16) {
    const char* ev = getenv("DS_VERIFY_POLY");  // A/B knob: word pairs per lane on the FMA-pipe exp2
    const int np = ev && ev[0] ? atoi(ev) : 0;
    if (np >= 8)
      verify_lse_kernel<__nv_bfloat16, 8><<<g1, kVT, 0, st>>>(a);
    else if (np >= 6)
      verify_lse_kernel<__nv_bfloat16, 6><<<g1, kVT, 0, st>>>(a);
    else if (np >= 4)
      verify_lse_kernel<__nv_bfloat16, 4><<<g1, kVT, 0, st>>>(a);
    else if (np >= 2)
      verify_lse_kernel<__nv_bfloat16, 2><<<g1, kVT, 0, st>>>(a);
    else
      verify_lse_kernel<__nv_bfloat16, 0><<<g1, kVT, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, verify_residual_kernel<__nv_bfloat16>, a);
  } else {
    verify_lse_kernel<float, 0><<<g1, kVT, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, verify_residual_kernel<float>, a);
  }
}

cudaError_t launch_shortlist_ids(const ds_clusters* c, int rows, const int32_t* sel, const int32_t* cnt,
                                 const int32_t* sl_off, int64_t stride, int32_t* ids, cudaStream_t st) {
  shortlist_ids_kernel<<<rows, 256, 0, st>>>(c->perm, c->offsets, c->M, sel, cnt, sl_off, stride, ids);
  return cudaGetLastError();
}

}  // namespace ds
