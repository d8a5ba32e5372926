// Probe: cost of the cluster step's CTA-level warp merge in isolation (one CTA, fresh SM).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
// One warp, shared memory only (no shuffle trees: the epilogue runs them slowly): (M, sum_g s_g
// e^{m_g - M}) over G (max, sum) pairs.  Lane l owns pairs l, l + 32, ...; lane 0 folds the 32
// partials in lane order, so the result is run-to-run identical.  scr: 32 floats.
__device__ __forceinline__ void warp_lse_smem(const float* pm, const float* ps, int G, float& m, float& s,
                                              float* scr) {
  const int lane = threadIdx.x & 31;
  float mx = -INFINITY;
  for (int g = lane; g < G; g += 32) mx = fmaxf(mx, pm[g]);
  scr[lane] = mx;
  __syncwarp();
  float M = -INFINITY;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) M = fmaxf(M, scr[j]);
  float sum = 0.f;
  if (M > -INFINITY)
    for (int g = lane; g < G; g += 32)
      if (pm[g] > -INFINITY) sum += ps[g] * expf(pm[g] - M);
  __syncwarp();
  scr[lane] = sum;
  __syncwarp();
  float S = 0.f;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) S += scr[j];
  m = M;
  s = S;
  __syncwarp();
}

// One warp: the best K keys of G descending key lists ([G][K] in shared memory, 0-padded) ->
// out[0..K) descending, 0-padded.  Lower bounds on the K-th best key overall prune the candidates:
// T1 = the best of the lists' K-th entries (that list alone has K keys >= T1) and T2 = the K-th
// best of the first min(G, 32) list heads (K distinct keys >= T2).  Keys >= max(T1, T2) are
// compacted by ballot and rank-counted (keys are distinct).  surv: G*K keys, 16-byte aligned;
// scr: 32 keys.
__device__ __forceinline__ void warp_merge_lists(const unsigned long long* lists, int G, int K,
                                                 unsigned long long* surv, unsigned long long* out,
                                                 unsigned long long* scr) {
  const int lane = threadIdx.x & 31;
  unsigned long long T = 0;
  for (int g = lane; g < G; g += 32) T = max(T, lists[g * K + K - 1]);
  const int nh = min(G, 32);
  if (nh >= K && lane < nh) {
    const unsigned long long h = lists[lane * K];
    int rank = 0;
#pragma unroll 8
    for (int j = 0; j < nh; ++j) rank += lists[j * K] > h;
    if (h != 0ull && rank == K - 1) T = max(T, h);
  }
  scr[lane] = T;
  for (int r = lane; r < K; r += 32) out[r] = 0ull;
  __syncwarp();
#pragma unroll 8
  for (int j = 0; j < 32; ++j) T = max(T, scr[j]);
  const int n = G * K;
  int ns = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const unsigned long long x = i < n ? lists[i] : 0ull;
    const bool keep = x != 0ull && x >= T;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (keep) surv[ns + __popc(bal & ((1u << lane) - 1u))] = x;
    ns += __popc(bal);
  }
  __syncwarp();
  for (int t = lane; t < ns; t += 32) {
    const unsigned long long x = surv[t];
    int rank = 0, j = 0;
    for (; j + 8 <= ns; j += 8) {  // batched 16-byte loads: latency overlapped, not chained
      const ulonglong2 v0 = *reinterpret_cast<const ulonglong2*>(surv + j);
      const ulonglong2 v1 = *reinterpret_cast<const ulonglong2*>(surv + j + 2);
      const ulonglong2 v2 = *reinterpret_cast<const ulonglong2*>(surv + j + 4);
      const ulonglong2 v3 = *reinterpret_cast<const ulonglong2*>(surv + j + 6);
      rank += (v0.x > x) + (v0.y > x) + (v1.x > x) + (v1.y > x) + (v2.x > x) + (v2.y > x) + (v3.x > x) + (v3.y > x);
    }
    for (; j < ns; ++j) rank += surv[j] > x;
    if (rank < K) out[rank] = x;
  }
  __syncwarp();
}


__global__ void k(long long* out, unsigned long long* sink, int S, int K, int reps) {
  __shared__ __align__(16) unsigned long long wl[12 * 32], surv[12 * 32], out_s[32], scr[64];
  __shared__ float wm[32], ws[32];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < S * K; i += blockDim.x) {
    const int w = i / K, r = i % K;
    // warp lists: ~3 valid entries per warp (as at k = 8), descending
    wl[i] = r < 3 ? ((unsigned long long)(0x80000000u + 1000000u * (7 * w % 11) + 1000u * (10 - r)) << 32) | (unsigned)(~(w * 8 + r)) : 0ull;
  }
  for (int i = threadIdx.x; i < S; i += blockDim.x) { wm[i] = 0.1f * i; ws[i] = 1.f + i; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  float m = 0, s = 0;
  for (int r = 0; r < reps; ++r) {
    float m2, s2;
    warp_lse_smem(wm, ws, S, m2, s2, reinterpret_cast<float*>(scr));
    m += m2; s += s2;
  }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) warp_merge_lists(wl, S, K, surv, out_s, scr);
  long long t2 = clock64();
  if (lane == 0) { out[0] = t1 - t0; out[1] = t2 - t1; sink[0] = out_s[0] + (unsigned long long)(m + s); }
}
int main() {
  long long* d; unsigned long long* f; cudaMalloc(&d, 64); cudaMalloc(&f, 64);
  long long h[2];
  for (int reps : {1, 10}) {
    k<<<1, 416>>>(d, f, 12, 8, reps); cudaDeviceSynchronize();
    k<<<1, 416>>>(d, f, 12, 8, reps); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("reps %d: lse_smem %lld cycles, merge_lists %lld cycles (%s)\n", reps, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
