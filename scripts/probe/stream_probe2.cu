// stream_probe.cu — how fast can G CTAs (one per SM) stream B bytes of contiguous HBM into shared
// memory with a TMA bulk-copy ring, chunk c -> CTA c mod G (the grid-step assignment)?  In-kernel
// %globaltimer: start = min over CTAs of the first issue, end = max over CTAs of the last landing.
// Sizes 8 MB .. 1 GB, ring S x CH bytes.  Cold L2 (a 512 MB memset before each launch).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(64, 1) k_stream(const char* src, long long nbytes, int S, int CH,
                                                  unsigned long long* ts, int consume) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) unsigned long long full[48];
  const int G = gridDim.x, g = blockIdx.x;
  const long long nch = nbytes / CH;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0 = gt();
  if (consume & 1) {
    for (long long c = g; c < nch; c += G)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + c * CH), "r"(CH) : "memory");
  }
  long long it = 0;
  for (long long c = g; c < nch; c += G, ++it) {
    const int s = (int)(it % S);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[s]);
    if (it >= S) {
      unsigned ok = 0;
      const unsigned par = (unsigned)(((it / S) - 1) & 1);
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(sm + s * CH)),
                 "l"(src + c * CH), "r"(CH), "r"(bar)
                 : "memory");
  }
  for (long long j = (it > S ? it - S : 0); j < it; ++j) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[j % S]);
    unsigned ok = 0;
    const unsigned par = (unsigned)((j / S) & 1);
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  }
  ts[2 * g] = t0;
  ts[2 * g + 1] = gt();
  (void)consume;
}

int main() {
  int G0 = 0;
  cudaDeviceGetAttribute(&G0, cudaDevAttrMultiProcessorCount, 0);
  char* src;
  const size_t big = 1ull << 30;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  char* flush;
  cudaMalloc(&flush, 512ull << 20);
  unsigned long long* ts;
  cudaMallocManaged(&ts, 2 * 256 * 8);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int G, S, CH; };
  const Cfg cfgs[] = {{G0 - 1, 12, 16384}, {G0 - 1, 24, 8192}, {G0 - 1, 48, 4096}, {G0 - 1, 6, 32768}};
  const long long sizes[] = {8ll << 20, 33ll << 20, 131ll << 20, 1ll << 30};
  for (int mode = 0; mode < 2; ++mode)
  for (const Cfg& c : cfgs) {
    for (long long B : sizes) {
      std::vector<double> r;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 512ull << 20);
        k_stream<<<c.G, 64, (size_t)c.S * c.CH>>>(src, B, c.S, c.CH, ts, mode);
        cudaDeviceSynchronize();
        unsigned long long a = ~0ull, b = 0;
        for (int g = 0; g < c.G; ++g) {
          a = std::min(a, ts[2 * g]);
          b = std::max(b, ts[2 * g + 1]);
        }
        r.push_back((double)B / (double)(b - a));  // bytes per ns = GB/s
      }
      std::sort(r.begin(), r.end());
      printf("mode=%d G=%3d S=%2d CH=%5d  %5lld MB: %6.0f GB/s  (%.2f us)\n", mode, c.G, c.S, c.CH, B >> 20, r[2],
             (double)B / r[2] * 1e-3);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
