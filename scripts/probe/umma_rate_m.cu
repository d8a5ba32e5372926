// Probe: issue rate of tcgen05.mma kind::f16 (bf16 in, fp32 accumulate in TMEM), M = 64 or 128, K = 16,
// for N = 16 .. 256, back-to-back into one accumulator, with and without a tcgen05.commit after
// every 4 MMAs (one 64-wide K chunk, as tc_head does per ring stage).  One CTA per SM, one issuing
// thread; operands are zero tiles in shared memory (the values do not matter for the rate).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(bar))
               : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(su(b)),
               "r"(par)
               : "memory");
}

__global__ void __launch_bounds__(128, 1) k(int M, int N, int iters, int commit_every, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* A = sm;            // 128 x 64 bf16, SW128 (16 KB)
  uint8_t* Bm = sm + 16384;   // N x 64 bf16 (<= 32 KB)
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = su(A), b0 = su(Bm);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma(tmem, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), idesc, (it | kk) != 0);
      if (commit_every == 1) {  // commit per chunk, no wait (the ring's release pattern)
        commit(&bar);
      } else if (commit_every == 2) {  // commit + wait per chunk (round trip per chunk)
        commit(&bar);
        wait(&bar, phase);
        phase ^= 1u;
      }
    }
    if (commit_every == 1) {  // every per-chunk commit arrived on the same barrier: count-1 phases
      commit(&bar);
      long long t1w = clock64();
      (void)t1w;
      // wait until all MMAs done: a final commit on a fresh phase is not separable here; wait
      // for the phase the last commit completes (iters + 1 arrivals -> parity of iters + 1)
      wait(&bar, (uint32_t)(iters & 1));
    } else {
      commit(&bar);
      wait(&bar, phase);
    }
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768);
  const int iters = 2000;
  printf("cycles per MMA (K=16), one CTA per SM x 148, no commit in the loop:\n");
  for (int M : {64, 128}) {
    for (int N : {8, 16, 32, 64, 128, 256}) {
      if (M == 128 && N == 8) continue;  // M = 128 needs N % 16 == 0
      k<<<148, 128, 16384 + 32768>>>(M, N, iters, 0, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("  M=%3d N=%3d: %7.1f cycles/MMA  %s\n", M, N, (double)mx / (iters * 4), cudaGetErrorString(e));
    }
  }
  return 0;
}
