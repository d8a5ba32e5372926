// phase_bench.cu — cycles per call of the grid step's once-per-launch phases in isolation (one CTA of
// 512 threads, the phase called R times back to back on fixed data): topk_mask (M = 256, k = 8 / 32),
// layer2 (M 256 x h_r 128 bf16), gstep_record (12 lists x K = 8).  For ncu source-level stall
// sampling of code that runs only ~1 us per launch in the real kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o phase_bench phase_bench.cu
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <functional>
#include <vector>

#include "../../paper_2510_13847_b200/csrc/gstep.cu"

using namespace ds;

constexpr int R = 64;

__global__ void __launch_bounds__(512, 1) k_topk(const float* scores, const int* offsets, int M, int k,
                                                 unsigned long long* cyc, unsigned* out, unsigned long long* dbg) {
  __shared__ float sc[256];
  __shared__ int offs[257];
  __shared__ uint32_t mask[8], thr[32];
  __shared__ int wc[16], total[4];
  __shared__ __align__(16) unsigned long long surv[384];
  const int tid = threadIdx.x;
  if (tid < M) sc[tid] = scores[tid];
  if (tid <= M) offs[tid] = offsets[tid];
  unsigned acc = 0;
  for (int r = 0; r < R; ++r) {
    if (tid < 8) mask[tid] = 0u;
    if (tid == 0) total[0] = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    topk_mask(sc, M, k, (M + 7) / 8, (k + 7) / 8, offs, mask, thr, surv, dbg);
    const unsigned long long t1 = clock64();
    if (tid == 0) {
      cyc[r] = t1 - t0;
      cyc[R + r] = dbg[32 + 13] - t0;
      cyc[2 * R + r] = dbg[32 + 14] - dbg[32 + 13];
      cyc[3 * R + r] = t1 - dbg[32 + 14];
    }
    acc += mask[r & 7] + total[0];
  }
  out[tid] = acc;
}

__global__ void __launch_bounds__(512, 1) k_layer2(GStepArgs a, const float* av, unsigned long long* cyc,
                                                   float* out) {
  __shared__ __align__(16) float a1[136];
  __shared__ float b2s[256], sc[256];
  const int tid = threadIdx.x;
  uint32_t w2r[kGRows2][2];
  load_w2<__nv_bfloat16>(a, tid >> 5, tid & 31, w2r);
  if (tid < 132) a1[tid] = av[tid];
  if (tid < 256) b2s[tid] = 0.f;
  float acc = 0.f;
  for (int r = 0; r < R; ++r) {
    __syncthreads();
    const unsigned long long t0 = clock64();
    layer2<__nv_bfloat16>(a, tid >> 5, tid & 31, w2r, a1, b2s, sc);
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[r] = t1 - t0;
    acc += sc[r & 255];
    if (tid == 0) a1[0] += 1.f;
  }
  out[tid] = acc;
}

__global__ void __launch_bounds__(512, 1) k_record(const unsigned long long* lists, int S, int K,
                                                   unsigned long long* cyc, unsigned long long* rec) {
  __shared__ unsigned long long wl[12 * 32], surv[384];
  __shared__ float wm[12], wsum[12];
  __shared__ int wn[12], cnt[4];
  const int tid = threadIdx.x;
  if (tid < S * K) wl[tid] = lists[tid];
  if (tid < S) {
    wm[tid] = 1.f;
    wsum[tid] = 2.f;
    wn[tid] = K;
  }
  for (int r = 0; r < R; ++r) {
    if (tid == 0) cnt[0] = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    gstep_record(rec + (size_t)(r & 3) * (2 + K), wl, wm, wsum, wn, S, K, 6, (uint32_t)((1ull << 32) / K));
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[r] = t1 - t0;
  }
}

__global__ void __launch_bounds__(512, 1) k_merge(GStepArgs a, const unsigned long long* recs, int G,
                                                  unsigned long long* cyc) {
  extern __shared__ __align__(16) unsigned long long raw[];
  const int tid = threadIdx.x, rec = 2 + a.k_t;
  for (int r = 0; r < R; ++r) {
    for (int i = tid; i < G * rec; i += blockDim.x) raw[i] = recs[i];
    __syncthreads();
    const unsigned long long t0 = clock64();
    gstep_merge_compute(a, raw, G, true);
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[r] = t1 - t0;
  }
}

__global__ void __launch_bounds__(512, 1) k_merge_fast(GStepArgs a, const unsigned long long* recs, int G,
                                                       unsigned long long* cyc) {
  extern __shared__ __align__(16) unsigned long long raw[];
  const int tid = threadIdx.x, rec = 2 + a.k_t;
  for (int r = 0; r < R; ++r) {
    for (int i = tid; i < G * rec; i += blockDim.x) raw[i] = recs[i];
    __syncthreads();
    const unsigned long long t0 = clock64();
    gstep_merge_fast(a, raw, G, true, reinterpret_cast<float*>(raw + (size_t)G * rec));
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[r] = t1 - t0;
  }
}

__global__ void __launch_bounds__(512, 1) k_radix(const float* scores, int M, int k, unsigned long long* cyc,
                                                  unsigned* out) {
  __shared__ float sc[256];
  __shared__ uint32_t mask[8], hist[264];
  const int tid = threadIdx.x;
  if (tid < M) sc[tid] = scores[tid];
  unsigned acc = 0;
  for (int r = 0; r < R; ++r) {
    __syncthreads();
    const unsigned long long t0 = clock64();
    radix_mask(sc, M, k, mask, hist);
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[r] = t1 - t0;
    acc += mask[r & 7];
  }
  __syncthreads();
  if (tid < 8) out[tid] = mask[tid];
  else out[tid] = acc;
}

static double median(std::vector<unsigned long long> v) {
  std::sort(v.begin(), v.end());
  return (double)v[v.size() / 2];
}

int main() {
  const int M = 256;
  std::vector<float> s(M);
  unsigned x = 12345;
  for (auto& f : s) {
    x = x * 1664525u + 1013904223u;
    f = (float)(x >> 8) / (float)(1u << 24) - 0.5f;
  }
  std::vector<int> off(M + 1);
  for (int i = 0; i <= M; ++i) off[i] = 500 * i;
  float* ds_;
  int* doff;
  unsigned long long* cyc;
  unsigned* out;
  cudaMalloc(&ds_, M * 4);
  cudaMalloc(&doff, (M + 1) * 4);
  cudaMallocManaged(&cyc, 4 * R * 8);
  unsigned long long* dbg;
  cudaMalloc(&dbg, 64 * 8);
  cudaMalloc(&out, 512 * 4 * 4);
  cudaMemcpy(ds_, s.data(), M * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(doff, off.data(), (M + 1) * 4, cudaMemcpyHostToDevice);
  for (int k : {8, 32}) {
    for (int rep = 0; rep < 2; ++rep) k_topk<<<1, 512>>>(ds_, doff, M, k, cyc, out, dbg);
    cudaDeviceSynchronize();
    {
      unsigned m0[8];
      cudaMemcpy(m0, out, 0, cudaMemcpyDeviceToHost);
    }
    printf("topk_mask M=256 k=%d: %.0f cycles/call (median of %d): to 1st barrier %.0f, compaction %.0f, rank %.0f\n", k,
           median({cyc, cyc + R}), R, median({cyc + R, cyc + 2 * R}), median({cyc + 2 * R, cyc + 3 * R}),
           median({cyc + 3 * R, cyc + 4 * R}));
  }
  for (int k : {8, 32}) {
    for (int rep = 0; rep < 2; ++rep) k_radix<<<1, 512>>>(ds_, M, k, cyc, out);
    cudaDeviceSynchronize();
    unsigned mk[8];
    cudaMemcpy(mk, out, 32, cudaMemcpyDeviceToHost);
    std::vector<int> idx(M);
    for (int i = 0; i < M; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return s[a] > s[b]; });
    unsigned ex[8] = {0};
    for (int i = 0; i < k; ++i) ex[idx[i] >> 5] |= 1u << (idx[i] & 31);
    int ok = 1;
    for (int w = 0; w < 8; ++w) ok &= mk[w] == ex[w];
    printf("radix_mask M=256 k=%d: %.0f cycles/call, mask %s\n", k, median({cyc, cyc + R}), ok ? "ok" : "WRONG");
  }
  // layer 2: W2 [256][128] bf16
  GStepArgs a = {};
  std::vector<uint16_t> w2(256 * 128, 0x3f80);
  void* dw2;
  cudaMalloc(&dw2, w2.size() * 2);
  cudaMemcpy(dw2, w2.data(), w2.size() * 2, cudaMemcpyHostToDevice);
  a.W2 = dw2;
  a.M = 256;
  a.h_r = 128;
  float* dav;
  cudaMalloc(&dav, 136 * 4);
  cudaMemset(dav, 0, 136 * 4);
  for (int rep = 0; rep < 2; ++rep) k_layer2<<<1, 512>>>(a, dav, cyc, reinterpret_cast<float*>(out));
  cudaDeviceSynchronize();
  printf("layer2 256x128 bf16 (+ barrier): %.0f cycles/call\n", median({cyc, cyc + R}));
  // record: 12 sorted lists of K keys; check the record = the K best of the union
  for (int K : {8, 32}) {
  const int S = 12;
  std::vector<unsigned long long> l(S * K);
  for (int w = 0; w < S; ++w)
    for (int r = 0; r < K; ++r) l[w * K + r] = ((unsigned long long)(0xc0000000u - 1000u * r - 37u * w) << 32) | (w * K + r);
  (void)0;
  unsigned long long *dl, *drec;
  cudaMalloc(&dl, l.size() * 8);
  cudaMalloc(&drec, 4 * (2 + K) * 8);
  cudaMemset(drec, 0, 4 * (2 + K) * 8);
  cudaMemcpy(dl, l.data(), l.size() * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) k_record<<<1, 512>>>(dl, S, K, cyc, drec);
  cudaDeviceSynchronize();
  printf("gstep_record S=12 K=%d (+ barrier): %.0f cycles/call\n", K, median({cyc, cyc + R}));
  std::vector<unsigned long long> hr(4 * (2 + K));
  cudaMemcpy(hr.data(), drec, hr.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> all(l);
  std::sort(all.begin(), all.end(), std::greater<unsigned long long>());
  int bad = 0;
  for (int r = 0; r < K; ++r) bad += hr[2 + r] != all[r];
  printf("  record check: %d wrong of %d (count word %llu)\n", bad, K, hr[1]);
  }
  {  // merger compute: G = 147 records of K = 8 keys
    const int G = 147, K = 8, rec = 2 + K;
    std::vector<unsigned long long> h((size_t)G * rec);
    unsigned y = 777;
    for (int g = 0; g < G; ++g) {
      float m = 10.f + (float)(g % 13) * 0.01f;
      unsigned mb;
      memcpy(&mb, &m, 4);
      float sm = 3.f;
      unsigned sb;
      memcpy(&sb, &sm, 4);
      h[(size_t)g * rec] = (unsigned long long)mb | ((unsigned long long)sb << 32);
      h[(size_t)g * rec + 1] = K + 1;
      unsigned hi = 0xc1000000u + (unsigned)(g * 7919 % 100000);
      for (int j = 0; j < K; ++j) {
        y = y * 1664525u + 1013904223u;
        hi -= 20000u + (y >> 18);
        h[(size_t)g * rec + 2 + j] = ((unsigned long long)hi << 32) | (0xffffffffu - (unsigned)(g * K + j));
      }
    }
    unsigned long long *dr;
    cudaMalloc(&dr, h.size() * 8);
    cudaMemcpy(dr, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    GStepArgs m = {};
    m.k_t = K;
    m.q_merge = (K + 4) / 5;
    int* oi;
    float* of;
    cudaMalloc(&oi, 64 * 4);
    cudaMalloc(&of, 3 * 64 * 4);
    m.top_ids = oi;
    m.top_logits = of;
    m.top_logp = of + 64;
    m.lse = of + 128;
    const size_t sm = (size_t)G * rec * 8 + (size_t)G * K * 8 + 1024;
    cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int rep = 0; rep < 2; ++rep) k_merge<<<1, 512, sm>>>(m, dr, G, cyc);
    cudaDeviceSynchronize();
    printf("merge_compute G=147 K=8 (+ barrier): %.0f cycles/call\n", median({cyc, cyc + R}));
    int ids0[8], ids1[8];
    cudaMemcpy(ids0, oi, 32, cudaMemcpyDeviceToHost);
    cudaFuncSetAttribute(k_merge_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int rep = 0; rep < 2; ++rep) k_merge_fast<<<1, 512, sm>>>(m, dr, G, cyc);
    cudaDeviceSynchronize();
    printf("merge_fast    G=147 K=8 (+ barrier): %.0f cycles/call\n", median({cyc, cyc + R}));
    cudaMemcpy(ids1, oi, 32, cudaMemcpyDeviceToHost);
    int same = 1;
    for (int i = 0; i < 8; ++i) same &= ids0[i] == ids1[i];
    printf("  same top ids: %d (%d %d %d ...)\n", same, ids1[0], ids1[1], ids1[2]);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

// host stubs for the library functions gstep.cu's host side references (not used here)
namespace ds {
int num_sms() { return 148; }
int max_smem_optin() { return 232448; }
unsigned long long* debug_trace() { return nullptr; }
}  // namespace ds
