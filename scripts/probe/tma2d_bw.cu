// Probe: HBM read rate of the tensor-core head's access pattern.  148 CTAs (one per SM) each stream
// tiles of 128 consecutive rows of a [rows][d] bf16 matrix (d = 3584, 1.09 GB) through a ring of
// 8 x 16 KB shared-memory stages, one 2-D TMA box per stage (64 columns x 128 rows, 128B swizzle):
//   (a) row-major W, K-chunk inner loop (what tc_head does): each box reads 128 B of 128 rows;
//   (b) K-blocked copy of W ([tile][chunk][128 rows][64]): each box is 16 KB contiguous;
//   (c) row-major W, 1-D bulk copies of whole rows (the CUDA-core head's pattern), for reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma2d_bw tma2d_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(su(b)),
               "r"(par)
               : "memory");
}

constexpr int S = 8, STAGE = 16384, D = 3584, KCH = D / 64;

// mode 0: row-major map, box (64, 128) at (kc*64, tile*128); mode 1: blocked map, box (64, 128) at
// (0, (tile*KCH + kc)*128); mode 2: 1-D bulk copies of 16 KB of consecutive rows; mode 3 (tree
// head): per K chunk 4 boxes of 16 rows (64-row tile, 16-row map) + one 16 x 64 box of H (hmap)
__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap m, const __grid_constant__ CUtensorMap m16,
                                           const __grid_constant__ CUtensorMap hm, const char* raw, int mode,
                                           int tiles_per_cta, float* sink) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nops = mode == 2 ? tiles_per_cta * 128 * D * 2 / STAGE : tiles_per_cta * KCH;
  if (mode == 3) {  // one 64-row tile per CTA: KCH stages of 4 x 2 KB + 2 KB (H)
    for (int c = 0; c < KCH; ++c) {
      const int s = c % S;
      if (c >= S) wait(&full[s], ((c / S) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(5 * 2048) : "memory");
      for (int b = 0; b < 5; ++b) {
        const CUtensorMap* mp = b < 4 ? &m16 : &hm;
        const int y = b < 4 ? blockIdx.x * 64 + b * 16 : 0;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su(sm + s * STAGE + b * 2048)),
            "l"(reinterpret_cast<uint64_t>(mp)), "r"(c * 64), "r"(y), "r"(su(&full[s]))
            : "memory");
      }
    }
    for (int c = KCH > S ? KCH - S : 0; c < KCH; ++c) wait(&full[c % S], (c / S) & 1);
    sink[blockIdx.x] = sm[5];
    return;
  }
  for (int c = 0; c < nops; ++c) {
    const int s = c % S;
    if (c >= S) wait(&full[s], ((c / S) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
    const int tile = blockIdx.x * tiles_per_cta + (mode == 2 ? 0 : c / KCH), kc = c % KCH;
    if (mode == 2) {
      const char* p = raw + ((size_t)blockIdx.x * tiles_per_cta * 128 * D * 2) + (size_t)c * STAGE;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su(sm + s * STAGE)),
                   "l"(p), "r"(STAGE), "r"(su(&full[s]))
                   : "memory");
    } else {
      const int x = mode == 0 ? kc * 64 : 0, y = mode == 0 ? tile * 128 : (tile * KCH + kc) * 128;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(su(sm + s * STAGE)),
          "l"(reinterpret_cast<uint64_t>(&m)), "r"(x), "r"(y), "r"(su(&full[s]))
          : "memory");
    }
  }
  for (int c = nops > S ? nops - S : 0; c < nops; ++c) wait(&full[c % S], (c / S) & 1);
  sink[blockIdx.x] = sm[5];
}

int main() {
  const int G = 148, tiles_per_cta = 8;  // 148 x 8 x 128 rows = 151552 rows (~Qwen V)
  const size_t rows = (size_t)G * tiles_per_cta * 128, bytes = rows * D * 2;
  char* w;
  float* sink;
  char* flush;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 1, bytes);
  cudaMalloc(&sink, 4096);
  cudaMalloc(&flush, 512 << 20);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  CUtensorMap mrow, mblk, m16, hmap;
  {
    const cuuint64_t dims[2] = {D, rows};
    const cuuint64_t str[1] = {D * 2};
    const cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    enc(&m16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const cuuint64_t hd[2] = {D, 16};
    enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, hd, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    const cuuint64_t dims[2] = {D, rows};
    const cuuint64_t str[1] = {D * 2};
    const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&mrow, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    const cuuint64_t dims[2] = {64, rows * KCH};
    const cuuint64_t str[1] = {128};
    const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&mblk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S * STAGE);
  const char* names[] = {"row-major, K-chunk boxes (tc_head)", "K-blocked copy, 16 KB boxes", "1-D bulk, whole rows",
                         "tree: 64-row tile, 4x16-row boxes + H, 1 tile"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaEventRecord(a);
      k<<<G, 64, S * STAGE>>>(mode == 1 ? mblk : mrow, m16, hmap, w, mode, tiles_per_cta, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    const double by = mode == 3 ? (double)G * KCH * 5 * 2048 : (double)bytes;
    printf("%-46s %8.1f us  %7.0f GB/s  %s\n", names[mode], best * 1e3, by / (best * 1e-3) / 1e9,
           cudaGetErrorString(e));
  }
  return 0;
}
