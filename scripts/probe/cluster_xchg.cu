// Probe: cost of one all-to-all exchange inside a 16-CTA cluster (one CTA per SM, 416 threads),
// (a) st.shared::cluster + barrier.cluster arrive.release / wait.acquire, (b) the same with a
// global store pending before the barrier, (c) st.async ... mbarrier::complete_tx (receiver waits
// on its own mbarrier for the expected bytes; no cluster-wide barrier).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_xchg cluster_xchg.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void bar_rel() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void bar_acq() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void mb_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}

constexpr int Q = 16, ITERS = 64;

__global__ void __cluster_dims__(1, 1, 1) k_dummy() {}

__global__ void k_probe(int mode, unsigned long long* out, float* gsink) {
  extern __shared__ __align__(16) uint8_t sm[];
  float* buf = reinterpret_cast<float*>(sm);           // [2][Q * 16]
  uint64_t* mb = reinterpret_cast<uint64_t*>(sm + 8192);  // [2]
  const uint32_t q = crank();
  if (threadIdx.x == 0) {
    mb_init(&mb[0], 1);
    mb_init(&mb[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  bar_rel();
  bar_acq();
  // each CTA sends 16 floats to every CTA (256 stores from 256 threads)
  const int t = threadIdx.x;
  const bool sender = t < Q * 16;
  const uint32_t dst = t / 16, slot = q * 16 + (t % 16);
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    const int p = it & 1;
    float* b = buf + p * Q * 16;
    if (mode == 0) {
      bar_rel();
      bar_acq();
    } else if (mode == 1 || mode == 2) {
      if (sender) asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(mapa(smem_u32(b + slot), dst)), "f"((float)it) : "memory");
      if (mode == 2 && t == 0) gsink[blockIdx.x] = (float)it;
      bar_rel();
      bar_acq();
    } else if (mode == 3) {
      // st.async: receiver's barrier p expects Q*16*4 bytes; thread 0 arms it for this phase
      if (t == 0) mb_expect(&mb[p], Q * 16 * 4);
      // the sender must know the receiver armed... expect_tx may come after complete_tx (tx count
      // goes negative transiently), so no ordering is needed
      if (sender) st_async(mapa(smem_u32(b + slot), dst), (float)it, mapa(smem_u32(&mb[p]), dst));
      mb_wait(&mb[p], (it >> 1) & 1);
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  bar_rel();
  bar_acq();
}

int main() {
  int G = 112;
  unsigned long long* d;
  float* g;
  cudaMalloc(&d, G * 8);
  cudaMalloc(&g, G * 4);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"bare barrier", "st.shared::cluster + barrier", "same + pending global store",
                         "st.async + mbarrier complete_tx (+__syncthreads)"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(416);
      cfg.dynamicSmemBytes = 200 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = Q;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_probe, mode, d, g);
      if (e != cudaSuccess) {
        printf("launch: %s\n", cudaGetErrorString(e));
        return 1;
      }
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("run: %s\n", cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[112];
      cudaMemcpy(h, d, G * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0, mn = ~0ull;
      for (int i = 0; i < G; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        mn = h[i] < mn ? h[i] : mn;
      }
      if (rep == 2) printf("%-50s cycles/exchange: min %.0f max %.0f\n", names[mode], (double)mn / ITERS, (double)mx / ITERS);
    }
  }
  return 0;
}
