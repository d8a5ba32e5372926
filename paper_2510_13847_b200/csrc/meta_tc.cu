// meta_tc.cu — S1 router layer 1 for MANY rows on the tensor cores (tcgen05 + TMEM).
//
// a = ReLU(W1 [h_prev ‖ e] + b1) (§4.2, R4, R5) for B rows is the GEMM
//   X [B x 2d] . W1^T [2d x h_r],   X = [h_prev ‖ e]
// which the CUDA-core split-K kernel (meta.cu) runs at ~2.8 TFLOP/s: 513 us of the Gemma-3 B = 512
// step (B 512 x 2d 10752 x h_r 256).  Here: M = 128 rows of X per tile, N = h_r (<= 256) hidden
// units, K = 64-wide chunks of the 2d input (chunks [0, d/64) from h_prev, the rest from e — two
// tensor maps, no concatenated copy), split over the grid so every SM has work; each CTA writes its
// fp32 partial sums to part[ks][b][u] — the layout meta_l2_kernel already reduces in fixed split
// order (bias, ReLU, layer 2, TopK), so no float atomics (R19).
//   warp 0 lane 0: TMA (128B swizzle) of the X tile and the W1 chunk per ring stage
//   warp 1 lane 0: tcgen05.mma 128 x h_r x 16 (4 per chunk), fp32 accumulator in TMEM
//   warps 2-5    : tcgen05.ld 32x32b (lane = row), partials to global memory
#include <algorithm>

#include "internal.h"
#include "tc_common.cuh"

namespace ds {

constexpr int kMtS = 4;
constexpr int kMtThreads = 192;
constexpr int kMtABytes = 128 * 128;  // 128 rows x 64 bf16

struct MtArgs {
  float* part;  // [KS][B][rows1]
  int32_t B, d, rows1, kc_total, kc_per, pdl;
};

__global__ void __launch_bounds__(kMtThreads, 1) meta_tc_l1_kernel(const __grid_constant__ CUtensorMap mh,
                                                                   const __grid_constant__ CUtensorMap me,
                                                                   const __grid_constant__ CUtensorMap mw,
                                                                   const MtArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int bbytes = a.rows1 * 128;
  uint8_t* sa = smem;
  uint8_t* sb = smem + kMtS * kMtABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + (size_t)kMtS * bbytes);
  uint64_t* empty = full + kMtS;
  uint64_t* tfull = empty + kMtS;
  uint32_t* slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt = blockIdx.x, ks = blockIdx.y;
  const int c0 = ks * a.kc_per, c1 = min(a.kc_total, c0 + a.kc_per), nch = max(0, c1 - c0);
  const int dch = a.d / 64;  // chunks of h_prev; chunks [dch, 2 dch) come from e
  int tcols = 32;
  while (tcols < a.rows1) tcols <<= 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMtS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&me)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mw)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (a.pdl) pdl_wait();  // h_prev / e come from the upstream kernel

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_first(), pol_w = policy_evict_last();
      for (int i = 0; i < nch; ++i) {
        const int kc = c0 + i, s = i % kMtS;
        mbar_wait(&empty[s], (uint32_t)((i / kMtS) & 1) ^ 1u);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(kMtABytes + bbytes));
        if (kc < dch) tma_load_2d(sa + (size_t)s * kMtABytes, &mh, kc * 64, rt * 128, &full[s], pol_x);
        else tma_load_2d(sa + (size_t)s * kMtABytes, &me, (kc - dch) * 64, rt * 128, &full[s], pol_x);
        tma_load_2d(sb + (size_t)s * bbytes, &mw, kc * 64, 0, &full[s], pol_w);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nch > 0) {
      // D f32, A / B bf16, both K-major, N = rows1 >> 3, M = 128 >> 4
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(a.rows1 >> 3) << 17) | (8u << 24);
      for (int i = 0; i < nch; ++i) {
        const int s = i % kMtS;
        mbar_wait(&full[s], (uint32_t)((i / kMtS) & 1));
        tc_fence_after();
        const uint32_t abase = smem_u32(sa + (size_t)s * kMtABytes), bbase = smem_u32(sb + (size_t)s * bbytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_bf16(tmem, sw128_desc(abase + k * 32), sw128_desc(bbase + k * 32), idesc, (i | k) != 0 ? 1u : 0u);
        tc_commit(&empty[s]);
      }
      tc_commit(tfull);
    }
    __syncwarp();
  } else {
    const int q = warp & 3, row = rt * 128 + 32 * q + lane;
    if (nch > 0) {
      mbar_wait(tfull, 0);
      tc_fence_after();
    }
    float* dst = a.part + ((size_t)ks * a.B + row) * a.rows1;
    for (int u0 = 0; u0 < a.rows1; u0 += 16) {
      float v[16];
      if (nch > 0) {
        tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)u0, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
      }
      if (row < a.B) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + u0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
  }
  if (a.pdl) pdl_launch_dependents();
}

// ---------------------------------------------------------------------------- host
// Used for bf16 routers with >= DS_META_TC_MIN_ROWS rows (default 32), d % 64 == 0, rows1 % 16 == 0
// and rows1 <= 256; the split count KS makes ceil(B / 128) x KS ~ one CTA per SM.
bool meta_tc_plan(const ds_router* r, int B, int* KS, int* kc_per) {
  const char* off = getenv("DS_META_TC");
  if (off && off[0] == '0') return false;
  const char* mr = getenv("DS_META_TC_MIN_ROWS");
  const int min_rows = mr && mr[0] ? atoi(mr) : 32;
  const int rows1 = r->h_r > 0 ? r->h_r : r->M;
  if (r->dtype != DS_BF16 || B < std::max(1, min_rows) || r->d % 64 != 0 || rows1 % 16 != 0 || rows1 > 256)
    return false;
  if (encode_fn() == nullptr) return false;
  const int tiles = (B + 127) / 128;
  const int kc_total = 2 * r->d / 64;
  const int want = std::max(1, std::min(kc_total, num_sms() / tiles));
  *kc_per = (kc_total + want - 1) / want;
  *KS = (kc_total + *kc_per - 1) / *kc_per;
  const size_t smem = (size_t)kMtS * (kMtABytes + rows1 * 128) + 256;
  return smem <= (size_t)max_smem_optin();
}

cudaError_t launch_meta_tc_l1(const ds_router* r, const void* h_prev, const void* e, int B, float* part, int KS,
                              int kc_per, cudaStream_t st, bool pdl) {
  const int rows1 = r->h_r > 0 ? r->h_r : r->M;
  CUtensorMap mh, me, mw;
  if (!make_map(&mh, h_prev, (uint64_t)B, (uint64_t)r->d, 128u) || !make_map(&me, e, (uint64_t)B, (uint64_t)r->d, 128u) ||
      !make_map(&mw, r->W1, (uint64_t)rows1, (uint64_t)(2 * r->d), (uint32_t)rows1))
    return cudaErrorInvalidValue;
  static int configured[64] = {0};
  cudaError_t err = configure_max_smem(reinterpret_cast<const void*>(meta_tc_l1_kernel), configured);
  if (err != cudaSuccess) return err;
  MtArgs a;
  a.part = part;
  a.B = B;
  a.d = r->d;
  a.rows1 = rows1;
  a.kc_total = 2 * r->d / 64;
  a.kc_per = kc_per;
  a.pdl = pdl ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((B + 127) / 128, KS);
  cfg.blockDim = dim3(kMtThreads);
  cfg.dynamicSmemBytes = (size_t)kMtS * (kMtABytes + rows1 * 128) + 256;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, meta_tc_l1_kernel, mh, me, mw, a);
}

}  // namespace ds
