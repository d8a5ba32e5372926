// lat_probe.cu — dependent-chain latencies (SM cycles per op) of the warp primitives the single-row
// step kernels are built from: SHFL.IDX, SHFL.BFLY, REDUX (__reduce_max_sync), VOTE+POPC, LDS.64,
// BAR.SYNC (16 warps), FFMA, FHFMA.BF16.  One CTA of 512 threads, chains of 256 ops.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256;

__global__ void probe(unsigned* out, unsigned long long* cyc, unsigned seed) {
  __shared__ unsigned long long sm[1024];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 1024; i += blockDim.x) sm[i] = (unsigned long long)(i * 7 + 1) & 1023;
  __syncthreads();
  unsigned v = seed + lane;
  unsigned long long t0, t1;
  // 0: SHFL.IDX chain
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (v + i) & 31) + 1u;
  t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  // 1: SHFL.BFLY chain
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1 + (i & 15)) + 1u;
  t1 = clock64();
  if (tid == 0) cyc[1] = t1 - t0;
  // 2: REDUX max chain
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) v = __reduce_max_sync(0xffffffffu, v ^ (unsigned)lane) + 1u;
  t1 = clock64();
  if (tid == 0) cyc[2] = t1 - t0;
  // 3: VOTE + POPC chain
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) v += __popc(__ballot_sync(0xffffffffu, ((v >> (lane & 7)) & 1u) != 0u));
  t1 = clock64();
  if (tid == 0) cyc[3] = t1 - t0;
  // 4: LDS.64 chain (pointer chase)
  unsigned long long p = (unsigned long long)(v & 1023);
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) p = sm[p & 1023];
  t1 = clock64();
  if (tid == 0) cyc[4] = t1 - t0;
  v += (unsigned)p;
  // 5: BAR.SYNC (all 16 warps)
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < 32; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0) * N / 32;
  // 6: FFMA chain
  float f = __uint_as_float(0x3f800000u + (v & 7));
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) f = fmaf(f, 0.999f, 0.001f);
  t1 = clock64();
  if (tid == 0) cyc[6] = t1 - t0;
  // 7: FHFMA.BF16 chain (bf16 x bf16 + f32)
  float h = f;
  const unsigned short b0 = (unsigned short)(0x3f80u + (v & 1)), b1 = 0x3f7fu;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(h) : "h"(b0), "h"(b1));
  t1 = clock64();
  if (tid == 0) cyc[7] = t1 - t0;
  // 8: loop back-edge cost: the FFMA chain again, not unrolled
  float g = f;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) g = fmaf(g, 0.999f, 0.001f);
  t1 = clock64();
  if (tid == 0) cyc[8] = t1 - t0;
  f += g;
  out[tid] = v + __float_as_uint(f) + __float_as_uint(h);
}

int main() {
  unsigned* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMallocManaged(&cyc, 16 * 8);
  const char* names[] = {"SHFL.IDX", "SHFL.BFLY", "REDUX.MAX", "VOTE+POPC", "LDS.64 chase", "BAR.SYNC x16 warps",
                         "FFMA", "FHFMA.BF16", "FFMA, unroll 1"};
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<1, 512>>>(out, cyc, rep);
    cudaDeviceSynchronize();
  }
  for (int i = 0; i < 9; ++i) printf("%-20s %6.1f cycles/op (chain of %d incl. loop)\n", names[i], (double)cyc[i] / N, N);
  return 0;
}
