// Probe: cycles of a warp-level (max, sum) combine of 12 pairs in shared memory, with the other
// warps of the block parked at __syncthreads (as in the cluster step's epilogue).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ void lse_pairs(const float* pm, const float* ps, int G, float& m, float& s) {
  const int lane = threadIdx.x & 31;
  float mx = -INFINITY;
  for (int g = lane; g < G; g += 32) mx = fmaxf(mx, pm[g]);
  mx = warp_max(mx);
  float sum = 0.f;
  if (mx > -INFINITY)
    for (int g = lane; g < G; g += 32)
      if (pm[g] > -INFINITY) sum += ps[g] * expf(pm[g] - mx);
  m = mx;
  s = warp_sum(sum);
}
__device__ __forceinline__ void lse_pairs_flat(const float* pm, const float* ps, int G, float& m, float& s) {
  const int lane = threadIdx.x & 31;
  const float a = lane < G ? pm[lane] : -INFINITY;
  const float b = lane < G ? ps[lane] : 0.f;
  const float mx = warp_max(a);
  const float e = a > -INFINITY ? b * expf(a - mx) : 0.f;
  m = mx;
  s = warp_sum(e);
}
__device__ __forceinline__ void lse_pairs_fast(const float* pm, const float* ps, int G, float& m, float& s) {
  const int lane = threadIdx.x & 31;
  const float a = lane < G ? pm[lane] : -INFINITY;
  const float b = lane < G ? ps[lane] : 0.f;
  const float mx = warp_max(a);
  const float e = a > -INFINITY ? b * __expf(a - mx) : 0.f;
  m = mx;
  s = warp_sum(e);
}
__global__ void k2(long long* out, float* sink, int G, int mode) {
  __shared__ float pm[64], ps[64];
  if (threadIdx.x < 64) { pm[threadIdx.x] = 0.1f * threadIdx.x; ps[threadIdx.x] = 1.f; }
  __syncthreads();
  float m = 0, s = 0;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int r = 0; r < 10; ++r) {
      float m2, s2;
      if (mode == 0) lse_pairs_flat(pm, ps, G, m2, s2); else lse_pairs_fast(pm, ps, G, m2, s2);
      m += m2; s += s2;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; sink[blockIdx.x] = m + s; }
}
__global__ void k3(long long* out, float* sink, int G) {  // empty timing
  long long t0 = clock64();
  float v = threadIdx.x;
  for (int r = 0; r < 10; ++r) v = warp_sum(v);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink[0] = v; }
}
__global__ void k(long long* out, float* sink, int G, int mode) {
  __shared__ float pm[64], ps[64];
  if (threadIdx.x < 64) { pm[threadIdx.x] = 0.1f * threadIdx.x; ps[threadIdx.x] = 1.f; }
  __syncthreads();
  float m = 0, s = 0;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int r = 0; r < 10; ++r) {
      float m2, s2;
      lse_pairs(pm, ps, G, m2, s2);
      m += m2; s += s2;
    }
  }
  long long t1 = clock64();
  if (mode == 1) __syncthreads();
  if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; sink[blockIdx.x] = m + s; }
}
__global__ void kglob(long long* out, float* sink, int G) {   // no shared data: registers only
  float m = 0, s = 0;
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int r = 0; r < 10; ++r) {
    float mx = warp_max(0.1f * lane + r);
    float e = expf(0.01f * lane - mx);
    m += mx; s += warp_sum(e);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink[0] = m + s; }
}
int main() {
  long long* d; float* f; cudaMalloc(&d, 8 * 1024); cudaMalloc(&f, 4 * 1024);
  long long h[4];
  for (int mode = 0; mode < 2; ++mode)
    for (int nt : {32, 416}) {
      k<<<1, nt>>>(d, f, 12, mode); cudaDeviceSynchronize();
      k<<<1, nt>>>(d, f, 12, mode); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      printf("mode %d threads %d: %lld cycles / 10 calls\n", mode, nt, h[0]);
    }
  for (int mode = 0; mode < 2; ++mode) {
    k2<<<1, 32>>>(d, f, 12, mode); cudaDeviceSynchronize();
    k2<<<1, 32>>>(d, f, 12, mode); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("flat %s: %lld cycles / 10 calls\n", mode ? "__expf" : "expf", h[0]);
  }
  k3<<<1, 32>>>(d, f, 12); cudaDeviceSynchronize();
  k3<<<1, 32>>>(d, f, 12); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("10 warp_sums: %lld cycles\n", h[0]);
  kglob<<<1, 32>>>(d, f, 12); cudaDeviceSynchronize();
  kglob<<<1, 32>>>(d, f, 12); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("register-only max+exp+sum: %lld cycles / 10\n", h[0]);
  return 0;
}
