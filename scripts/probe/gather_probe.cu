// gather_probe.cu — TMA bulk streaming of a DynaSpec-like gathered shortlist: k selected clusters of a
// W_perm with Llama-3-like cluster sizes (449..558 rows of 8 KB), chunks of <= 2 rows that never cross
// a cluster; 147 CTAs, 12 x 16 KB ring, no consume.  Compares chunk -> CTA assignments:
//   A0: chunk c -> CTA c mod G (the grid step today)
//   A1: contiguous per-CTA segments of the chunk list
//   A2: chunk c -> CTA (c * 37) mod G... (a scrambled interleave)
// and the same bytes as ONE contiguous region.  Clean L2 before each launch (write + read flush).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather_probe gather_probe.cu
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

struct Chunk { long long off; int bytes; int pad; };

__global__ void __launch_bounds__(64, 1) k_gather(const char* src, const Chunk* ch, int nch, int S, int mode,
                                                  unsigned long long* ts) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) unsigned long long full[16];
  const int G = gridDim.x, g = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __shared__ Chunk my[512];
  long long lo = 0, hi = nch, step = 1, first = 0;
  if (mode == 0) { first = g; step = G; }
  else if (mode == 1) { lo = (long long)nch * g / G; hi = (long long)nch * (g + 1) / G; first = lo; }
  const int mine = (int)((hi - first + step - 1) / step);
  for (int j = threadIdx.x; j < mine && j < 512; j += blockDim.x) my[j] = ch[first + (long long)j * step];
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0 = gt();
  long long it = 0;
  for (long long i = first; i < hi; i += step, ++it) {
    const long long c = it;
    const int s = (int)(it % S);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[s]);
    if (it >= S) {
      unsigned ok = 0;
      const unsigned par = (unsigned)(((it / S) - 1) & 1);
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    }
    const Chunk k = my[c];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(k.bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(sm + s * 16384)),
                 "l"(src + k.off), "r"(k.bytes), "r"(bar)
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
}

__global__ void k_read(const int4* p, long long n, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int4 v = p[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) sink[0] = 1;
}

int main() {
  int G0 = 0;
  cudaDeviceGetAttribute(&G0, cudaDevAttrMultiProcessorCount, 0);
  const int G = G0 - 1, S = 12;
  const long long rowb = 8192;
  const int M = 256;
  std::vector<long long> off(M + 1, 0);
  unsigned long long x = 777;
  auto rnd = [&]() { x = x * 6364136223846793005ull + 1442695040888963407ull; return (unsigned)(x >> 33); };
  for (int m = 0; m < M; ++m) off[m + 1] = off[m] + 449 + rnd() % 110;
  const long long V = off[M];
  char* src;
  cudaMalloc(&src, V * rowb);
  cudaMemset(src, 1, V * rowb);
  char *flush, *clean;
  cudaMalloc(&flush, 512ull << 20);
  cudaMalloc(&clean, 512ull << 20);
  cudaMemset(clean, 3, 512ull << 20);
  int* sink;
  cudaMalloc(&sink, 64);
  unsigned long long* ts;
  cudaMallocManaged(&ts, 2 * 256 * 8);
  Chunk* ch;
  cudaMalloc(&ch, sizeof(Chunk) * 200000);
  std::vector<Chunk> hch(200000);
  cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, S * 16384);
  for (int k : {8, 32}) {
    for (int trial = 0; trial < 3; ++trial) {
      std::vector<int> ids(M);
      for (int i = 0; i < M; ++i) ids[i] = i;
      for (int i = M - 1; i > 0; --i) std::swap(ids[i], ids[rnd() % (i + 1)]);
      std::sort(ids.begin(), ids.begin() + k);
      for (int layout = 0; layout < 2; ++layout) {  // 0: gathered clusters, 1: same bytes contiguous
        int n = 0;
        long long bytes = 0, base = 0;
        for (int q = 0; q < k; ++q) {
          const int m = ids[q];
          const long long r0 = layout == 0 ? off[m] : base, sz = off[m + 1] - off[m];
          for (long long j = 0; j < sz; j += 2) {
            hch[n].off = (r0 + j) * rowb;
            hch[n].bytes = (int)(std::min(2ll, sz - j) * rowb);
            bytes += hch[n].bytes;
            ++n;
          }
          base += sz;
        }
        cudaMemcpy(ch, hch.data(), sizeof(Chunk) * n, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 2; ++mode) {
          std::vector<double> r;
          for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(flush, rep, 512ull << 20);
            k_read<<<G0 * 4, 512>>>((const int4*)clean, (512ll << 20) / 16, sink);
            k_gather<<<G, 64, S * 16384>>>(src, ch, n, S, mode, ts);
            cudaDeviceSynchronize();
            unsigned long long a = ~0ull, b = 0;
            for (int g = 0; g < G; ++g) {
              a = std::min(a, ts[2 * g]);
              b = std::max(b, ts[2 * g + 1]);
            }
            r.push_back((double)(b - a) * 1e-3);
          }
          std::sort(r.begin(), r.end());
          printf("k=%2d trial %d %s assign=%s: %6.1f MB in %6.2f us = %5.0f GB/s\n", k, trial,
                 layout ? "contig " : "gather ", mode ? "segment " : "c mod G ", bytes / 1e6, r[2],
                 bytes / (r[2] * 1e3));
        }
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
