#include <algorithm>
// Probe: does a dependent shuffle chain on one warp run slower right after the chip streamed
// HBM at full rate (issue throttle), or after TMA bulk copies into shared memory?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void __launch_bounds__(416, 1) k(const uint4* src, size_t n_per_cta, long long* out, float* sink, int mode) {
  extern __shared__ uint4 sm[];
  float acc = 0.f;
  if (mode == 2 && blockIdx.x == 0) {  // CTA 0 only times chains while the others stream
    long long best = 1LL << 60, worst = 0;
    float v = threadIdx.x;
    for (int it = 0; it < 200; ++it) {
      long long a0 = clock64();
      if (threadIdx.x < 32)
        for (int r = 0; r < 10; ++r) v = warp_sum(v) * 1e-3f;
      long long a1 = clock64();
      best = min(best, a1 - a0);
      worst = max(worst, a1 - a0);
    }
    if (threadIdx.x == 0) { out[0] = best; out[1] = worst; sink[0] = v; }
    return;
  }
  if (mode == 3) {  // stream this CTA's slice with TMA bulk copies into a 12 x 16 KB ring (one producer lane)
    __shared__ __align__(8) unsigned long long bars[12];
    const int S = 12, CH = 16384;
    if (threadIdx.x == 0) {
      for (int i = 0; i < S; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bars[i])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const char* p = reinterpret_cast<const char*>(src + blockIdx.x * n_per_cta);
    const int nch = (int)(n_per_cta * 16 / CH);
    if (threadIdx.x == 0) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % S;
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[s]);
        if (c >= S) {  // wait for the slot's previous fill (consumed immediately)
          unsigned ok = 0;
          const unsigned par = ((c / S) - 1) & 1;
          while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(bar), "r"(par) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((unsigned)__cvta_generic_to_shared(reinterpret_cast<char*>(sm) + s * CH)),
                       "l"(p + (size_t)c * CH), "r"(CH), "r"(bar) : "memory");
      }
      for (int c = nch - S; c < nch; ++c) {
        const int s = c % S;
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[s]);
        unsigned ok = 0;
        const unsigned par = (c / S) & 1;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(bar), "r"(par) : "memory");
      }
      acc = __uint_as_float(sm[0].x & 0x3f800000u);
    }
  }
  if (mode == 1) {  // stream this CTA's slice of HBM with 16-byte loads
    const uint4* p = src + blockIdx.x * n_per_cta;
    for (size_t i = threadIdx.x; i < n_per_cta; i += blockDim.x) {
      const uint4 v = p[i];
      acc += __uint_as_float(v.x & 0x3f800000u);
    }
  }
  __syncthreads();
  long long t0 = clock64();
  float v = acc + threadIdx.x;
  if (threadIdx.x < 32)
    for (int r = 0; r < 10; ++r) v = warp_sum(v) * 1e-3f;
  long long t1 = clock64();
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x < 32)
    for (int r = 0; r < 10; ++r) v = warp_sum(v) * 1e-3f;
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t3 - t2;
    sink[blockIdx.x] = v;
  }
}
__global__ void __launch_bounds__(416, 1) kc(long long* out, float* sink, int mode) {
  // cluster launch; mode 1: CTAs with odd cluster rank exit immediately; then warp 0 times chains
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (mode == 1 && (rank & 1)) return;
  long long t0 = clock64();
  float v = threadIdx.x;
  if (threadIdx.x < 32)
    for (int r = 0; r < 10; ++r) v = warp_sum(v) * 1e-3f;
  long long t1 = clock64();
  if (mode == 2) {  // spin 20 us then time again
    long long w = clock64();
    while (clock64() - w < 40000) {}
  }
  long long t2 = clock64();
  if (threadIdx.x < 32)
    for (int r = 0; r < 10; ++r) v = warp_sum(v) * 1e-3f;
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = t3 - t2; sink[blockIdx.x] = v; }
}
int main() {
  const int G = 112;
  const size_t per = (size_t)(256 << 20) / 16 / G;  // 256 MB total
  uint4* src; long long* d; float* f;
  cudaMalloc(&src, per * G * 16); cudaMemset(src, 0, per * G * 16);
  cudaMalloc(&d, 16 * G); cudaMalloc(&f, 4 * G);
  long long h[2 * 112];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      k<<<G, 416, 200 * 1024>>>(src, per, d, f, mode);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, d, 16 * G, cudaMemcpyDeviceToHost);
    if (mode == 2) { printf("mode 2: idle CTA 0 chain during others' streaming: best %lld worst %lld\n", h[0], h[1]); continue; }
    long long mn = 1LL << 60, mx = 0;
    for (int i = 0; i < G; ++i) { mn = std::min(mn, h[2 * i]); mx = std::max(mx, h[2 * i]); }
    printf("  chain1 min %lld max %lld\n", mn, mx);
    long long a = 0, b = 0;
    for (int i = 0; i < G; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
    printf("mode %d (%s): chain1 %lld cycles, chain2 %lld cycles (mean over CTAs, 50 dependent shfl each)\n", mode,
           mode == 3 ? "after TMA streaming" : mode ? "after streaming 256 MB" : "no streaming", a / G, b / G);
  }
  cudaFuncSetAttribute(kc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 3; ++mode) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(112); cfg.blockDim = dim3(416); cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 16; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    for (int rep = 0; rep < 3; ++rep) { cudaLaunchKernelEx(&cfg, kc, d, f, mode); cudaDeviceSynchronize(); }
    cudaMemcpy(h, d, 16 * G, cudaMemcpyDeviceToHost);
    printf("cluster mode %d: CTA0 chain1 %lld chain2 %lld | CTA2 %lld %lld (%s)\n", mode, h[0], h[1], h[4], h[5],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
