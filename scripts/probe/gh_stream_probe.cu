// gh_stream_probe.cu — HBM read rate of the grouped head's W access pattern at Gemma-3 shape
// (W [262144][5376] bf16, 2.8 GB; 148 CTAs, items = 256-row tiles, item i -> CTA i mod 148, a
// single TMA-issuing thread per CTA, clean L2 before each run):
//   A: per stage one 2-D box of 256 rows x 64 columns (128 B per row), S = 4 x 32 KB  (gh today)
//   B: same boxes, S = 6 x 32 KB (what a ring holding only W would allow)
//   C: per stage 4 boxes of 64 rows x 64 columns = K chunks kc..kc+3 of a 64-row tile (512 B per row)
//   D: 1-D bulk copies of 32 KB contiguous, S = 4
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gh_stream_probe gh_stream_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(su(b)), "r"(par)
               : "memory");
}
__device__ __forceinline__ void box(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(su(bar)) : "memory");
}
constexpr int D = 5376, KCH = D / 64, STAGE = 32768;
constexpr long long ROWS = 262144;

__device__ __forceinline__ bool test(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su(b)), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ void spin(uint64_t* b, uint32_t par) { while (!test(b, par)) { } }

// relay modes: warp 0 lane 0 = producer (waits empty[s]), warp 1 lane 0 = consumer (waits full[s], arrives empty[s])
__global__ void __launch_bounds__(64, 1) krelay(const __grid_constant__ CUtensorMap m256, int S, int use_spin, float* sink) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  const long long nst = 0;
  (void)nst;
  if (threadIdx.x == 0) {
    long long c = 0;
    for (int it = blockIdx.x; it < ROWS / 256; it += G)
      for (int kc = 0; kc < KCH; ++kc, ++c) {
        const int s = (int)(c % S);
        const uint32_t par = (uint32_t)(((c / S) & 1) ^ 1);
        if (use_spin) spin(&empty[s], par); else wait(&empty[s], par);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
        box(sm + s * STAGE, &m256, kc * 64, it * 256, &full[s]);
      }
  } else if (threadIdx.x == 32) {
    long long c = 0;
    for (int it = blockIdx.x; it < ROWS / 256; it += G)
      for (int kc = 0; kc < KCH; ++kc, ++c) {
        const int s = (int)(c % S);
        const uint32_t par = (uint32_t)((c / S) & 1);
        if (use_spin) spin(&full[s], par); else wait(&full[s], par);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
      }
    sink[blockIdx.x] = sm[5];
  }
}

__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap m256, const __grid_constant__ CUtensorMap m64,
                                           const char* raw, int mode, int S, float* sink) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t full[8];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int G = gridDim.x;
  long long c = 0;
  auto stage = [&]() -> int {
    const int s = (int)(c % S);
    if (c >= S) wait(&full[s], (uint32_t)(((c / S) - 1) & 1));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
    ++c;
    return s;
  };
  if (mode == 0 || mode == 1) {
    for (int it = blockIdx.x; it < ROWS / 256; it += G)
      for (int kc = 0; kc < KCH; ++kc) {
        const int s = stage();
        box(sm + s * STAGE, &m256, kc * 64, it * 256, &full[s]);
      }
  } else if (mode == 2) {
    for (int it = blockIdx.x; it < ROWS / 64; it += G)
      for (int kc = 0; kc < KCH; kc += 4) {
        const int s = stage();
        for (int j = 0; j < 4; ++j) box(sm + s * STAGE + j * 8192, &m64, (kc + j) * 64, it * 64, &full[s]);
      }
  } else {
    const long long nch = ROWS * D * 2 / STAGE;
    for (long long q = blockIdx.x; q < nch; q += G) {
      const int s = stage();
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su(sm + s * STAGE)), "l"(raw + q * STAGE), "r"(STAGE), "r"(su(&full[s])) : "memory");
    }
  }
  for (long long j = c > S ? c - S : 0; j < c; ++j) wait(&full[j % S], (uint32_t)((j / S) & 1));
  sink[blockIdx.x] = sm[5];
}

__global__ void k_read(const int4* p, long long n, int* out) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int4 v = p[i];
    acc.x ^= v.x;
  }
  if (acc.x == 0x12345) out[0] = 1;
}

int main() {
  const size_t bytes = (size_t)ROWS * D * 2;
  char* w;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 1, bytes);
  float* sink;
  cudaMalloc(&sink, 4096);
  char *flush, *clean;
  cudaMalloc(&flush, 512 << 20);
  cudaMalloc(&clean, 512 << 20);
  cudaMemset(clean, 2, 512 << 20);
  int* so;
  cudaMalloc(&so, 64);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  CUtensorMap m256, m64;
  const cuuint64_t dims[2] = {D, (cuuint64_t)ROWS};
  const cuuint64_t str[1] = {D * 2};
  const cuuint32_t es[2] = {1, 1};
  const cuuint32_t b256[2] = {64, 256}, b64[2] = {64, 64};
  enc(&m256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, b256, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, b64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * STAGE);
  const char* names[] = {"A 256x64 boxes, S=4 (gh)", "B 256x64 boxes, S=6", "C 4x(64x64) boxes/stage, S=4",
                         "D 1-D 32 KB bulk, S=4", "E 1-D 32 KB bulk, S=6"};
  const int modes[5] = {0, 1, 2, 3, 3};
  const int Ss[5] = {4, 6, 4, 4, 6};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) {
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      k_read<<<148 * 4, 512>>>((const int4*)clean, (512ll << 20) / 16, so);
      cudaEventRecord(a);
      k<<<148, 32, Ss[i] * STAGE>>>(m256, m64, w, modes[i], Ss[i], sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-34s %8.1f us  %7.0f GB/s  %s\n", names[i], best * 1e3, bytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(krelay, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * STAGE);
  for (int S : {4, 6})
    for (int sp : {0, 1}) {
      float best = 1e9f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flush, rep, 512 << 20);
        k_read<<<148 * 4, 512>>>((const int4*)clean, (512ll << 20) / 16, so);
        cudaEventRecord(a);
        krelay<<<148, 64, S * STAGE>>>(m256, S, sp, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("relay (producer <- consumer thread) S=%d %s %8.1f us  %7.0f GB/s  %s\n", S, sp ? "test_wait spin" : "try_wait      ",
             best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
