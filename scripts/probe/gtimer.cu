// Probe: cost of reading %globaltimer vs clock64 (cycles per read, dependent use).
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned long long* out) {
  unsigned long long acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < 100; ++i) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    acc += t;
  }
  long long t1 = clock64();
  for (int i = 0; i < 100; ++i) acc += clock64();
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 100;
    out[1] = (t2 - t1) / 100;
    out[2] = acc;
  }
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 24);
  for (int r = 0; r < 3; ++r) k<<<1, 32>>>(d);
  unsigned long long h[3];
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("globaltimer read: %llu cycles, clock64 read: %llu cycles\n", h[0], h[1]);
}
