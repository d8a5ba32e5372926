// meta_rows.cu — S1 + S3/S4 for a FEW rows (2 <= B <= 16, bf16) in ONE launch on all SMs.
//
// s_b = W2 ReLU(W1 [h_prev,b ‖ e_b] + b1) + b2   (§4.2 "Low-cost router"; R4, R5)
// K_b = TopK_k(s_b) (score desc, id asc; R7), ascending ids, sl_offsets
// shared (tree) mode: one union selection over the B rows                    (R9)
//
// Why: the split-K pair meta_l1 + meta_l2 (meta.cu) costs ~25 us for 10 tree rows (launch chain,
// split-K partials through L2, a row-CTA TopK, then a ticketed union) — a third of the Qwen tree
// step.  Here, as in the grid step (gstep.cu), the hidden units are spread over the grid:
//   * CTA g owns hidden unit u = g (h_r <= #SMs): its W1 row (2d bf16) is loaded into REGISTERS
//     before the dependency wait (router weights never depend on the upstream kernel; so is the
//     W2 row of each thread of the row CTAs); after the wait one thread stages the B rows of
//     x_b = [h_prev,b ‖ e_b] in shared memory with 2B bulk copies (one round trip), the CTA reduces
//     B dot products in a fixed order, and publishes a_bu = ReLU(. + b1_u) as ONE 64-bit word
//     (1 << 32 | bits) — value and "written" land together, no fence, no counter;
//   * CTA b < B (row CTAs) then polls the h_r unit words of row b (bounded spin), zeroes them
//     (it is their only reader), evaluates layer 2 (thread m: W2 row m from registers, fp32 a
//     from shared memory), writes the scores, and takes TopK_k by a rank count of 64-bit keys
//     (ord(score) << 32 | ~id, R7) over the M <= 256 scores; independent rows emit their
//     selection here;
//   * shared mode: row CTAs publish their TopK masks as tagged words; CTA B polls the B masks,
//     zeroes them, ORs them and emits the union (ascending ids, sl_offsets).
// Every spin is bounded (2 s) and raises DS_ERR_DEVICE_TIMEOUT in the workspace error word.  The
// unit / mask words live in the fixed workspace prefix (internal.h) and are left at zero.
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "select_impl.cuh"

namespace ds {

constexpr int kMrThreads = 256;
constexpr int kMrMaxRows = 16;
constexpr int kMrW1Chunks = 4;   // 16-byte W1 chunks per thread: 2d <= 4 x 256 x 8 = 8192
constexpr int kMrW2Chunks = 16;  // 16-byte W2 chunks per thread (row m): h_r <= 128
constexpr unsigned long long kMrSpinNs = 2000000000ull;

struct MrArgs {
  const __nv_bfloat16* W1;  // [h_r][2d]
  const float* b1;          // [h_r]
  const __nv_bfloat16* W2;  // [M][h_r]
  const float* b2;          // [M]
  const __nv_bfloat16* h_prev;  // [B][d]
  const __nv_bfloat16* e;       // [B][d]
  const int32_t* offsets;       // [M + 1]
  int32_t B, d, h_r, M, k, shared;
  int32_t RB;  // x rows staged per batch
  float* scores;      // [B][M]
  int32_t* sel;       // [B][M] (shared: one row)
  int32_t* sel_count;
  int32_t* sl_off;    // [B][M + 1]
  unsigned long long* units;  // [B][h_r] tagged words (workspace prefix)
  unsigned long long* masks;  // [B][32] tagged mask words (workspace prefix)
  unsigned* err;              // workspace error word
  int32_t pdl;
  int32_t defer_union;  // shared mode: the row masks stay in the workspace for the tree head (th.cu)
  unsigned long long* trace;
};

// spin (one thread) until *p != 0; 0 on timeout (error word raised)
__device__ __forceinline__ unsigned long long mr_poll(const unsigned long long* p, unsigned long long t0,
                                                      unsigned* err) {
  for (unsigned n = 1;; ++n) {
    const unsigned long long v = ld_relaxed_u64(p);
    if (v != 0ull) return v;
    if ((n & 63u) == 0u && globaltimer_ns() - t0 > kMrSpinNs) {
      atomicExch(err, (unsigned)DS_ERR_DEVICE_TIMEOUT);
      return 0ull;
    }
  }
}

__global__ void __launch_bounds__(kMrThreads, 1) meta_rows_kernel(const __grid_constant__ MrArgs a) {
  __shared__ float red[kMrThreads / 32][kMrMaxRows];
  __shared__ __align__(16) float a1[256];
  __shared__ unsigned long long keys[256 + 2];
  __shared__ uint32_t mask[32];
  __shared__ int32_t offs[kMaxM + 1];
  __shared__ int32_t tmp[kMaxM];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = blockIdx.x, B = a.B, d = a.d, dr = 2 * d, M = a.M, h_r = a.h_r;
  const int nch = dr / 8;  // 16-byte chunks of x

  extern __shared__ __align__(16) uint8_t mr_dyn[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(mr_dyn);  // [B][2d] staged x rows
  __shared__ __align__(8) uint64_t xbar;
  // ---- before the dependency wait: this CTA's W1 row and (row CTAs) W2 into L2
  if (tid == 0) {
    mbar_init(&xbar, 1);
    fence_mbar_init();
  }
  uint4 w1[kMrW1Chunks];
#pragma unroll
  for (int i = 0; i < kMrW1Chunks; ++i) {
    const int c = tid + i * kMrThreads;
    w1[i] = (g < h_r && c < nch) ? __ldg(reinterpret_cast<const uint4*>(a.W1 + (size_t)g * dr) + c)
                                  : make_uint4(0, 0, 0, 0);
  }
  const bool rowcta = g < B;
  uint4 w2[kMrW2Chunks];  // row CTAs: W2 row m of thread m, in registers before the dependency wait
#pragma unroll
  for (int i = 0; i < kMrW2Chunks; ++i)
    w2[i] = (rowcta && tid < M && i * 8 < h_r) ? __ldg(reinterpret_cast<const uint4*>(a.W2 + (size_t)tid * h_r) + i)
                                                : make_uint4(0, 0, 0, 0);
  const float b1u = g < h_r ? __ldg(a.b1 + g) : 0.f;
  const float b2m = (rowcta && tid < M) ? __ldg(a.b2 + tid) : 0.f;
  if (rowcta || (a.shared && g == B))
    for (int m = tid; m <= M; m += kMrThreads) offs[m] = __ldg(a.offsets + m);
  trace_mark(a.trace, 24);
  if (a.pdl) pdl_wait();
  trace_mark(a.trace, 25);
  __syncthreads();  // xbar initialised
  // ---- layer 1: unit g for every row.  x rows (produced upstream) staged in shared memory by 2 bulk
  // copies per row (h_prev_b, e_b), RB rows per batch (one batch when they fit: one round trip)
  if (g < h_r) {
    float acc[kMrMaxRows];
#pragma unroll
    for (int b = 0; b < kMrMaxRows; ++b) acc[b] = 0.f;
    float wf[kMrW1Chunks][8];
#pragma unroll
    for (int i = 0; i < kMrW1Chunks; ++i) widen16(w1[i], wf[i], a.W1);
    for (int b0 = 0, ph = 0; b0 < B; b0 += a.RB, ph ^= 1) {
      const int nb = min(a.RB, B - b0);
      if (b0 > 0) __syncthreads();  // the previous batch is consumed
      if (tid == 0) {
        mbar_arrive_expect_tx(&xbar, (uint32_t)(nb * dr * 2));
        for (int q = 0; q < nb; ++q) {
          bulk_g2s(xs + (size_t)q * dr, a.h_prev + (size_t)(b0 + q) * d, (uint32_t)(d * 2), &xbar, policy_evict_last());
          bulk_g2s(xs + (size_t)q * dr + d, a.e + (size_t)(b0 + q) * d, (uint32_t)(d * 2), &xbar, policy_evict_last());
        }
      }
      mbar_wait(&xbar, (uint32_t)ph);
#pragma unroll
      for (int b = 0; b < kMrMaxRows; ++b) {
        if (b >= b0 && b < b0 + nb) {
#pragma unroll
          for (int i = 0; i < kMrW1Chunks; ++i) {
            const int c = tid + i * kMrThreads;
            if (c < nch) {
              float xf[8];
              widen16(*reinterpret_cast<const uint4*>(xs + (size_t)(b - b0) * dr + c * 8), xf, a.W1);
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[b] = fmaf(wf[i][j], xf[j], acc[b]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kMrMaxRows; ++b) {
      const float v = warp_sum(acc[b]);
      if (lane == 0) red[warp][b] = v;
    }
    __syncthreads();
    if (tid < B) {  // fixed order over the warps (R19)
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kMrThreads / 32; ++w) s += red[w][tid];
      const float u = fmaxf(s + b1u, 0.f);
      st_relaxed_u64(a.units + (size_t)tid * h_r + g, (1ull << 32) | (unsigned long long)__float_as_uint(u));
    }
  }
  trace_mark(a.trace, 26);
  if (!rowcta && !(a.shared && !a.defer_union && g == B)) return;

  const unsigned long long t0 = globaltimer_ns();
  if (rowcta) {
    // ---- layer 2 + TopK for row b = g
    const int b = g;
    for (int u = tid; u < h_r; u += kMrThreads) {
      const unsigned long long v = mr_poll(a.units + (size_t)b * h_r + u, t0, a.err);
      a1[u] = __uint_as_float((uint32_t)v);
      st_relaxed_u64(a.units + (size_t)b * h_r + u, 0ull);  // its only reader: re-arm for the next launch
    }
    __syncthreads();
    trace_mark(a.trace, 27);
    unsigned long long key = 0ull;
    if (tid < M) {
      float e0 = 0.f, o0 = 0.f;
#pragma unroll
      for (int i = 0; i < kMrW2Chunks; ++i) {
        if (i * 8 < h_r) {
          float wf[8];
          widen16(w2[i], wf, a.W2);
          const float4 av0 = *reinterpret_cast<const float4*>(a1 + i * 8);
          const float4 av1 = *reinterpret_cast<const float4*>(a1 + i * 8 + 4);
          e0 = fmaf(wf[0], av0.x, e0);
          o0 = fmaf(wf[1], av0.y, o0);
          e0 = fmaf(wf[2], av0.z, e0);
          o0 = fmaf(wf[3], av0.w, o0);
          e0 = fmaf(wf[4], av1.x, e0);
          o0 = fmaf(wf[5], av1.y, o0);
          e0 = fmaf(wf[6], av1.z, e0);
          o0 = fmaf(wf[7], av1.w, o0);
        }
      }
      const float s = (e0 + o0) + b2m;
      a.scores[(size_t)b * M + tid] = s;
      key = ((unsigned long long)ord_key(s + 0.0f) << 32) | (unsigned long long)(~(uint32_t)tid);  // R7
    }
    keys[tid] = key;
    __syncthreads();
    {  // TopK_k: rank of each key among the M unique keys (one 64-bit compare per pair)
      int r0 = 0, r1 = 0;
#pragma unroll 8
      for (int j = 0; j < M; j += 2) {
        r0 += keys[j] > key ? 1 : 0;
        r1 += keys[j + 1] > key ? 1 : 0;
      }
      const bool selb = tid < M && r0 + r1 < a.k;
      const uint32_t bits = __ballot_sync(0xffffffffu, selb);
      if (lane == 0 && tid < ((M + 31) & ~31)) mask[warp] = bits;
    }
    __syncthreads();
    trace_mark(a.trace, 28);
    if (!a.shared) {
      emit_fast(mask, M, offs, a.sel + (size_t)b * M, a.sel_count + b, a.sl_off + (size_t)b * (M + 1), tmp);
      return;
    }
    const int words = (M + 31) >> 5;
    if (tid < words) st_relaxed_u64(a.masks + (size_t)b * 32 + tid, (1ull << 32) | mask[tid]);
    return;
  }
  // ---- shared mode, CTA B: the union of the B rows' TopK masks
  const int words = (M + 31) >> 5;
  if (tid < 32) {
    uint32_t acc = 0u;
    if (tid < words)
      for (int b = 0; b < B; ++b) {
        const unsigned long long v = mr_poll(a.masks + (size_t)b * 32 + tid, t0, a.err);
        acc |= (uint32_t)v;
        st_relaxed_u64(a.masks + (size_t)b * 32 + tid, 0ull);
      }
    mask[tid] = acc;
  }
  __syncthreads();
  emit_fast(mask, M, offs, a.sel, a.sel_count, a.sl_off, tmp);
  trace_mark(a.trace, 29);
}

bool meta_rows_supported(const ds_router* r, int B, int k, const int32_t* k_per_row) {
  const char* off = getenv("DS_META_ROWS");
  if (off && off[0] == '0') return false;
  const int G = num_sms();
  return r && r->dtype == DS_BF16 && r->h_r > 0 && B >= 2 && B <= kMrMaxRows && k_per_row == nullptr &&
         r->h_r <= G && r->h_r <= 8 * kMrW2Chunks && r->h_r % 8 == 0 && r->M <= kMrThreads && r->M <= 256 &&
         2 * r->d <= 8 * kMrThreads * kMrW1Chunks && r->d % 8 == 0 && G >= B + 1 && k >= 1 && k <= r->M &&
         (size_t)4 * r->d + 16 * 1024 <= (size_t)max_smem_optin();  // >= one x row staged in shared memory
  // (static arrays < 16 KB: see launch_meta_rows)
}

cudaError_t launch_meta_rows(const ds_router* r, const void* h_prev, const void* e, int B, float* scores,
                             const int32_t* offsets, int k, int shared, int32_t* sel, int32_t* sel_count,
                             int32_t* sl_offsets, void* ws, cudaStream_t st, bool pdl, bool defer_union) {
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  MrArgs a;
  a.W1 = static_cast<const __nv_bfloat16*>(r->W1);
  a.b1 = r->b1;
  a.W2 = static_cast<const __nv_bfloat16*>(r->W2);
  a.b2 = r->b2;
  a.h_prev = static_cast<const __nv_bfloat16*>(h_prev);
  a.e = static_cast<const __nv_bfloat16*>(e);
  a.offsets = offsets;
  a.B = B;
  a.d = r->d;
  a.h_r = r->h_r;
  a.M = r->M;
  a.k = k;
  a.shared = shared ? 1 : 0;
  a.scores = scores;
  a.sel = sel;
  a.sel_count = sel_count;
  a.sl_off = sl_offsets;
  a.units = reinterpret_cast<unsigned long long*>(w8 + kWsRowsUnits);
  a.masks = reinterpret_cast<unsigned long long*>(w8 + kWsRowsMasks);
  a.err = reinterpret_cast<unsigned*>(w8 + kWsErrorWord);
  a.pdl = pdl ? 1 : 0;
  a.defer_union = defer_union ? 1 : 0;
  a.trace = debug_trace();
  const int rb_fit = (int)(((size_t)max_smem_optin() - 16 * 1024) / ((size_t)4 * r->d));
  a.RB = std::max(1, std::min(B, rb_fit));
  const size_t smem = (size_t)a.RB * 2 * r->d * 2;
  static int configured[64] = {0};  // dynamic limit = opt-in maximum minus the static arrays (<= 16 KB)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!configured[dev]) {
    cudaError_t ce = cudaFuncSetAttribute(meta_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          max_smem_optin() - 16 * 1024);
    if (ce != cudaSuccess) return ce;
    configured[dev] = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(kMrThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, meta_rows_kernel, a);
}

}  // namespace ds
