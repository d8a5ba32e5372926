// Probe: HBM read bandwidth of G CTAs (1 per SM) streaming contiguous chunks, via (a) TMA bulk
// copies into a ring of S x 16 KB slots (one producer lane, consumers only wait), (b) LDG.128 by
// 384 threads with 8 loads in flight each.  Reports GB/s for G = 112 and 148.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(416, 1) k_tma(const char* src, size_t per_cta, int S, int CH, float* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long full[16];
  const char* p = src + blockIdx.x * per_cta;
  const int nch = (int)(per_cta / CH);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < nch; ++c) {
      const int s = c % S;
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[s]);
      if (c >= S) {
        unsigned ok = 0;
        const unsigned par = ((c / S) - 1) & 1;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(bar), "r"(par) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"((unsigned)__cvta_generic_to_shared(sm + s * CH)), "l"(p + (size_t)c * CH), "r"(CH), "r"(bar)
                   : "memory");
    }
    for (int c = (nch > S ? nch - S : 0); c < nch; ++c) {
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[c % S]);
      unsigned ok = 0;
      const unsigned par = (c / S) & 1;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    }
    sink[blockIdx.x] = sm[0];
  }
}
__global__ void __launch_bounds__(416, 1) k_ldg(const uint4* src, size_t per_cta_v, float* sink) {
  const uint4* p = src + blockIdx.x * per_cta_v;
  unsigned acc = 0;
  for (size_t i = threadIdx.x; i < per_cta_v; i += 8 * blockDim.x) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (i + u * blockDim.x < per_cta_v) ? __ldcs(p + i + u * blockDim.x) : make_uint4(0,0,0,0);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345) sink[blockIdx.x] = 1.f;
}
int main() {
  const size_t total = (size_t)1 << 30;
  char* src; float* sink; cudaMalloc(&src, total); cudaMemset(src, 1, total); cudaMalloc(&sink, 4096);
  char* flush; cudaMalloc(&flush, 512 << 20);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int G : {112, 148}) {
    for (int mode = 0; mode < 4; ++mode) {
      const size_t MB = (mode == 3) ? 35 : 131;   // per-step shortlist sizes (k = 8 / 32 at Llama-3)
      const size_t bytes = MB << 20;
      const size_t per = bytes / G / 16384 * 16384;
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 512 << 20);
        cudaEventRecord(a);
        if (mode == 0) k_tma<<<G, 416, 12 * 16384>>>(src, per, 12, 16384, sink);
        else if (mode == 1) k_tma<<<G, 416, 6 * 32768>>>(src, per, 6, 32768, sink);
        else k_ldg<<<G, 416>>>(reinterpret_cast<uint4*>(src), per / 16, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      const char* nm[] = {"tma 12x16KB", "tma 6x32KB", "ldg 8x16B x416", "ldg (35 MB)"};
      printf("G=%d %-15s %zu MB: %.1f us  %.0f GB/s\n", G, nm[mode], per * G >> 20, best * 1e3, per * G / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
