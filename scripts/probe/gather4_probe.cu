// gather4_probe.cu — TMA tile::gather4 (UTMALDG.2D.GATHER4) on sm_100a: (1) layout check: 4 arbitrary
// rows x 64 bf16 of a [R][D] tensor with SWIZZLE_128B land as smem rows 0..3 of a K-major SW128 tile;
// (2) issue throughput: one thread per CTA (148 CTAs) gathering 64 rows x 64 cols per stage from an
// L2-resident 5.5 MB tensor (16 gather4 ops per stage) into a ring of S stages.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* m, int col, int r0, int r1, int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok)
                 : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(par)
                 : "memory");
}

__global__ void k_layout(const __grid_constant__ CUtensorMap m, int col, int4 rows, uint8_t* out) {
  __shared__ __align__(1024) uint8_t buf[1024];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)),
                 "r"(512)
                 : "memory");
    g4(buf, &m, col, rows.x, rows.y, rows.z, rows.w, &bar);
    wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = buf[i];
}

__global__ void __launch_bounds__(32, 1) k_rate(const __grid_constant__ CUtensorMap m, const int* rows, int nrows,
                                                int kchunks, int S, int stages, unsigned long long* ts) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const unsigned long long t0 = gt();
  for (int it = 0; it < stages; ++it) {
    const int s = it % S;
    if (it >= S) wait(&full[s], ((it / S) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])),
                 "r"(nrows * 128)
                 : "memory");
    const int kc = (it + blockIdx.x) % kchunks;
    for (int r = 0; r < nrows; r += 4)
      g4(sm + (size_t)s * nrows * 128 + r * 128, &m, kc * 64, rows[r], rows[r + 1], rows[r + 2], rows[r + 3], &full[s]);
  }
  for (int it = (stages > S ? stages - S : 0); it < stages; ++it) wait(&full[it % S], (it / S) & 1);
  ts[2 * blockIdx.x] = t0;
  ts[2 * blockIdx.x + 1] = gt();
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int R = 512, D = 5376;
  std::vector<uint16_t> h((size_t)R * D);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < D; ++c) h[(size_t)r * D + c] = (uint16_t)((r * 131 + c) & 0xffff);
  uint16_t* dH;
  cudaMalloc(&dH, h.size() * 2);
  cudaMemcpy(dH, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)R};
  const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  const cuuint32_t box[2] = {64, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult e = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dH, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)e);
  uint8_t* dout;
  cudaMalloc(&dout, 512);
  const int4 rows = make_int4(7, 300, 2, 511);
  const int col = 128;
  k_layout<<<1, 128>>>(m, col, rows, dout);
  std::vector<uint8_t> out(512);
  cudaMemcpy(out.data(), dout, 512, cudaMemcpyDeviceToHost);
  printf("layout kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  const int rr[4] = {rows.x, rows.y, rows.z, rows.w};
  int bad_sw = 0, bad_lin = 0;
  for (int j = 0; j < 4; ++j)
    for (int c = 0; c < 8; ++c)
      for (int b = 0; b < 16; ++b) {
        const uint8_t* src = reinterpret_cast<const uint8_t*>(&h[(size_t)rr[j] * D + col]) + c * 16 + b;
        bad_sw += out[j * 128 + ((c ^ j) * 16) + b] != *src;   // SW128: chunk c of smem row j at c ^ (j % 8)
        bad_lin += out[j * 128 + c * 16 + b] != *src;
      }
  printf("layout: mismatches vs SW128 image %d, vs linear %d (of 512 bytes)\n", bad_sw, bad_lin);
  // rate
  int G = 0;
  cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
  std::vector<int> rws(128);
  for (int i = 0; i < 128; ++i) rws[i] = (i * 37 + 11) % R;
  int* drows;
  cudaMalloc(&drows, 128 * 4);
  cudaMemcpy(drows, rws.data(), 128 * 4, cudaMemcpyHostToDevice);
  unsigned long long* ts;
  cudaMallocManaged(&ts, 2 * 256 * 8);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nrows : {16, 64, 128}) {
    for (int S : {2, 4, 8}) {
      if ((size_t)S * nrows * 128 > 200 * 1024) continue;
      const int stages = 512;
      std::vector<double> r;
      for (int rep = 0; rep < 5; ++rep) {
        k_rate<<<G, 32, (size_t)S * nrows * 128>>>(m, drows, nrows, D / 64, S, stages, ts);
        cudaDeviceSynchronize();
        unsigned long long a = ~0ull, b = 0;
        for (int g = 0; g < G; ++g) {
          a = std::min(a, ts[2 * g]);
          b = std::max(b, ts[2 * g + 1]);
        }
        r.push_back((double)(b - a));
      }
      std::sort(r.begin(), r.end());
      const double ns = r[2];
      printf("gather4 rate: %3d rows/stage, S=%d: %.1f ns per stage per SM (%.2f ns per op), %.0f GB/s per SM\n", nrows,
             S, ns / stages, ns / stages / (nrows / 4), (double)stages * nrows * 128 / ns);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
