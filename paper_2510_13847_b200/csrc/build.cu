// build.cu — S0: offline vocabulary partition by spherical k-means (§4.2), in the
// integer-exact reading R12, so the GPU and the CPU oracle agree bit for bit in
// any thread order:
//   u_v = rint(2^14 w_v / ||w_v||), ||w_v||^2 a sequential fp64 sum (exact squares);
//   Forgy init from splitmix64(seed) (partial Fisher-Yates over token ids);
//   repeat: tau(v) = argmax_m <u_v, c_m> in int32 (|dot| < 2^31 by Cauchy-Schwarz; ties -> lower m);
//           stop if tau is unchanged;  S_m = sum u_v (int64, exact in any order);
//           c_m = rint(2^14 S_m / ||S_m||) with ||S_m||^2 a sequential fp64 sum of separately
//           rounded products (no FMA);  empty clusters reseeded in ascending m;
//   relabel clusters by their smallest token id; then the cluster-permuted layout (layout.cu).
// One 4-byte-ish D->H copy per iteration decides convergence (documented in dynaspec.h).
#include <math.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace ds {

constexpr int kNormThreads = 128;
constexpr int kNormChunk = 32;
constexpr int kAsgTok = 64;      // tokens per assignment CTA
constexpr int kAsgCen = 128;     // centroids per pass
constexpr int kAsgK = 32;        // K chunk
constexpr int kAsgThreads = 256; // 16 x 16 threads, 4 tokens x 8 centroids each

struct BuildWs {
  int16_t* U;      // [V][d]
  int16_t* C;      // [M][d]
  long long* S;    // [M][d]
  double* norm;    // [V]
  int32_t* tau_prev;
  int32_t* members;  // [V]
  int32_t* sims;     // [V]
  int32_t* sizes;    // [M]
  int32_t* starts;   // [M+1]
  int32_t* cursor;   // [M]
  int32_t* minid;    // [M]
  int32_t* stats;    // [4]: changed, degenerate, reseed v, pad
  size_t total;
};

static BuildWs build_ws(void* base, int64_t V, int d, int M) {
  BuildWs w;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  const size_t oU = take((size_t)V * d * 2), oC = take((size_t)M * d * 2), oS = take((size_t)M * d * 8),
               oN = take((size_t)V * 8), oT = take((size_t)V * 4), oMem = take((size_t)V * 4),
               oSim = take((size_t)V * 4), oSz = take((size_t)M * 4), oSt = take((size_t)(M + 1) * 4),
               oCur = take((size_t)M * 4), oMin = take((size_t)M * 4), oStat = take(16 * 4);
  const size_t oLay = take(layout_ws_bytes(V, M));
  uint8_t* b = static_cast<uint8_t*>(base);
  w.U = reinterpret_cast<int16_t*>(b + oU);
  w.C = reinterpret_cast<int16_t*>(b + oC);
  w.S = reinterpret_cast<long long*>(b + oS);
  w.norm = reinterpret_cast<double*>(b + oN);
  w.tau_prev = reinterpret_cast<int32_t*>(b + oT);
  w.members = reinterpret_cast<int32_t*>(b + oMem);
  w.sims = reinterpret_cast<int32_t*>(b + oSim);
  w.sizes = reinterpret_cast<int32_t*>(b + oSz);
  w.starts = reinterpret_cast<int32_t*>(b + oSt);
  w.cursor = reinterpret_cast<int32_t*>(b + oCur);
  w.minid = reinterpret_cast<int32_t*>(b + oMin);
  w.stats = reinterpret_cast<int32_t*>(b + oStat);
  (void)oLay;
  w.total = o;
  return w;
}

size_t build_ws_bytes(int64_t V, int d, int M) { return build_ws(nullptr, V, d, M).total; }

// ------------------------------------------------------------------ normalise + quantise

// ||w_v||^2 as a sequential fp64 sum over i (a 128-token x 32-column tile is staged through
// shared memory so the global reads are coalesced while each thread keeps its token's order).
template <typename T>
__global__ void __launch_bounds__(kNormThreads) row_norm_kernel(const T* __restrict__ W, int64_t V, int d,
                                                                double* __restrict__ norm, int32_t* stats) {
  __shared__ float tile[kNormThreads][kNormChunk + 1];
  const int64_t v0 = (int64_t)blockIdx.x * kNormThreads;
  const int64_t v = v0 + threadIdx.x;
  double acc = 0.0;
  for (int c0 = 0; c0 < d; c0 += kNormChunk) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kNormThreads * kNormChunk; idx += kNormThreads) {
      const int r = idx / kNormChunk, c = idx % kNormChunk;
      const int64_t vv = v0 + r;
      tile[r][c] = (vv < V && c0 + c < d) ? static_cast<float>(W[vv * d + c0 + c]) : 0.f;
    }
    __syncthreads();
    const int n = min(kNormChunk, d - c0);
    for (int c = 0; c < n; ++c) {
      const double x = (double)tile[threadIdx.x][c];
      acc = __dadd_rn(acc, __dmul_rn(x, x));   // x*x is exact in fp64 for bf16 / fp32 inputs
    }
  }
  if (v < V) {
    const double n = sqrt(acc);
    norm[v] = n;
    if (acc == 0.0) atomicExch(&stats[1], 1);
  }
}

template <typename T>
__global__ void quantise_kernel(const T* __restrict__ W, int64_t V, int d, const double* __restrict__ norm,
                                int16_t* __restrict__ U) {
  const int64_t n = V * (int64_t)d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / d;
    const double x = (double)static_cast<float>(W[i]);
    U[i] = (int16_t)rint(__dmul_rn(__ddiv_rn(x, norm[v]), 16384.0));
  }
}

__global__ void gather_centroids_kernel(const int16_t* __restrict__ U, const int32_t* __restrict__ ids, int M, int d,
                                        int16_t* __restrict__ C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)M * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / d), c = (int)(i % d);
    C[i] = U[(int64_t)ids[m] * d + c];
  }
}

// ------------------------------------------------------------------ assignment

// tau(v) = argmax_m <u_v, c_m> (exact int32), ties -> lower m; counts changes vs tau_prev.
__global__ void __launch_bounds__(kAsgThreads) assign_kernel(const int16_t* __restrict__ U,
                                                             const int16_t* __restrict__ C, int64_t V, int d, int M,
                                                             int32_t* __restrict__ tau,
                                                             const int32_t* __restrict__ tau_prev, int32_t* stats,
                                                             int first) {
  __shared__ int32_t su[kAsgK][kAsgTok + 1];   // [k][token]
  __shared__ int32_t sc[kAsgK][kAsgCen + 1];   // [k][centroid]
  __shared__ int32_t bestv[16][kAsgTok];
  __shared__ int32_t bestm[16][kAsgTok];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // ty: token group, tx: centroid group
  const int64_t v0 = (int64_t)blockIdx.x * kAsgTok;
  int32_t run_v[4], run_m[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    run_v[i] = INT32_MIN;
    run_m[i] = 0;
  }
  for (int m0 = 0; m0 < M; m0 += kAsgCen) {
    int32_t acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int k0 = 0; k0 < d; k0 += kAsgK) {
      __syncthreads();
      for (int idx = threadIdx.x; idx < kAsgTok * kAsgK; idx += kAsgThreads) {
        const int r = idx / kAsgK, c = idx % kAsgK;
        const int64_t v = v0 + r;
        su[c][r] = (v < V && k0 + c < d) ? (int32_t)U[v * d + k0 + c] : 0;
      }
      for (int idx = threadIdx.x; idx < kAsgCen * kAsgK; idx += kAsgThreads) {
        const int r = idx / kAsgK, c = idx % kAsgK;
        const int m = m0 + r;
        sc[c][r] = (m < M && k0 + c < d) ? (int32_t)C[(int64_t)m * d + k0 + c] : 0;
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < kAsgK; ++k) {
        int32_t a[4], b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = su[k][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] = sc[k][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] += a[i] * b[j];
      }
    }
    // fold this centroid block into the running best; j ascending => lower m wins ties
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int m = m0 + tx + 16 * j;
      if (m < M) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (acc[i][j] > run_v[i] || (acc[i][j] == run_v[i] && m < run_m[i])) {
            run_v[i] = acc[i][j];
            run_m[i] = m;
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bestv[tx][ty * 4 + i] = run_v[i];
    bestm[tx][ty * 4 + i] = run_m[i];
  }
  __syncthreads();
  if (threadIdx.x < kAsgTok) {
    const int r = threadIdx.x;
    int32_t bv = bestv[0][r], bm = bestm[0][r];
    for (int x = 1; x < 16; ++x) {
      const int32_t v = bestv[x][r], m = bestm[x][r];
      if (v > bv || (v == bv && m < bm)) {
        bv = v;
        bm = m;
      }
    }
    const int64_t v = v0 + r;
    if (v < V) {
      tau[v] = bm;
      if (!first && tau_prev[v] != bm) atomicAdd(&stats[0], 1);
    }
  }
}

// ------------------------------------------------------------------ update

__global__ void sizes_kernel(const int32_t* __restrict__ tau, int64_t V, int32_t* sizes) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&sizes[tau[v]], 1);
}

__global__ void members_kernel(const int32_t* __restrict__ tau, int64_t V, int32_t* cursor,
                               int32_t* __restrict__ members) {
  // slot order inside a cluster is arbitrary; only exact integer sums are taken over it
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    members[atomicAdd(&cursor[tau[v]], 1)] = (int32_t)v;
}

// S_m[c] = sum over members of U[v][c], int64 (exact, order-free).  grid (M, ceil(d/256)).
__global__ void sum_kernel(const int16_t* __restrict__ U, const int32_t* __restrict__ members,
                           const int32_t* __restrict__ starts, int d, long long* __restrict__ S) {
  const int m = blockIdx.x;
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= d) return;
  long long acc = 0;
  for (int j = starts[m]; j < starts[m + 1]; ++j) acc += U[(int64_t)members[j] * d + c];
  S[(int64_t)m * d + c] = acc;
}

// ||S_m|| = sqrt(sequential fp64 sum of separately rounded squares); one thread per cluster.
__global__ void cnorm_kernel(const long long* __restrict__ S, const int32_t* __restrict__ sizes, int M, int d,
                             double* __restrict__ cn) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  if (sizes[m] == 0) {
    cn[m] = 0.0;
    return;
  }
  double acc = 0.0;
  for (int i = 0; i < d; ++i) {
    const double x = (double)S[(int64_t)m * d + i];
    acc = __dadd_rn(acc, __dmul_rn(x, x));
  }
  cn[m] = sqrt(acc);
}

__global__ void centroid_kernel(const long long* __restrict__ S, const double* __restrict__ cn,
                                const int32_t* __restrict__ sizes, int M, int d, int16_t* __restrict__ C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)M * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / d);
    if (sizes[m] == 0) continue;
    C[i] = (int16_t)rint(__dmul_rn(__ddiv_rn((double)S[i], cn[m]), 16384.0));
  }
}

// sims[v] = <u_v, c_tau(v)> (updated centroids), warp per token.
__global__ void sims_kernel(const int16_t* __restrict__ U, const int16_t* __restrict__ C,
                            const int32_t* __restrict__ tau, int64_t V, int d, int32_t* __restrict__ sims) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); v < V; v += warps) {
    const int16_t* u = U + v * d;
    const int16_t* c = C + (int64_t)tau[v] * d;
    int32_t acc = 0;
    for (int i = lane; i < d; i += 32) acc += (int32_t)u[i] * (int32_t)c[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sims[v] = acc;
  }
}

// Reseed empty cluster m: v* = argmin (sims[v], v) over tokens whose cluster has > 1 member.
__global__ void __launch_bounds__(1024) reseed_kernel(const int32_t* __restrict__ sims, int32_t* tau, int64_t V,
                                                      int32_t* sizes, int m, const int16_t* __restrict__ U,
                                                      int16_t* C, int d) {
  __shared__ long long sbest[32];
  __shared__ long long winner;
  long long best = LLONG_MAX;   // key = (sim + 2^31) << 32 | v  : lexicographic (sim, v)
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
    if (sizes[tau[v]] > 1) {
      const long long key = ((long long)((int64_t)sims[v] + 2147483648LL) << 32) | (long long)v;
      best = key < best ? key : best;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other < best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) sbest[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long b = sbest[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) b = sbest[i] < b ? sbest[i] : b;
    winner = b;
    const int v = (int)(b & 0xffffffffLL);
    sizes[tau[v]] -= 1;
    tau[v] = m;
    sizes[m] = 1;
  }
  __syncthreads();
  const int64_t v = winner & 0xffffffffLL;
  for (int i = threadIdx.x; i < d; i += blockDim.x) C[(int64_t)m * d + i] = U[v * d + i];
}

__global__ void minid_kernel(const int32_t* __restrict__ tau, int64_t V, int32_t* minid) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    atomicMin(&minid[tau[v]], (int32_t)v);
}

__global__ void relabel_kernel(int32_t* tau, int64_t V, const int32_t* __restrict__ newlab) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    tau[v] = newlab[tau[v]];
}

// ------------------------------------------------------------------ host driver

static uint64_t splitmix64_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

#define DS_TRY(x)                                  \
  do {                                             \
    if ((x) != cudaSuccess) return DS_ERR_CUDA;    \
  } while (0)

ds_status run_build(const void* W, int dtype, int64_t V, int d, int M, uint64_t seed, int max_iters,
                    const int32_t* init_ids_host, int32_t* tau, int32_t* perm, int32_t* offsets, void* W_perm,
                    int32_t* iters_host, int32_t* sizes_host, void* ws, cudaStream_t st) {
  BuildWs w = build_ws(ws, V, d, M);
  const int sms = num_sms();
  DS_TRY(cudaMemsetAsync(w.stats, 0, 16 * sizeof(int32_t), st));
  // 1. normalise + quantise
  const int nb = (int)((V + kNormThreads - 1) / kNormThreads);
  if (dtype == DS_BF16) {
    row_norm_kernel<__nv_bfloat16><<<nb, kNormThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(W), V, d, w.norm,
                                                               w.stats);
  } else {
    row_norm_kernel<float><<<nb, kNormThreads, 0, st>>>(static_cast<const float*>(W), V, d, w.norm, w.stats);
  }
  DS_TRY(cudaGetLastError());
  int32_t stat_h[4];
  DS_TRY(cudaMemcpyAsync(stat_h, w.stats, sizeof(stat_h), cudaMemcpyDeviceToHost, st));
  DS_TRY(cudaStreamSynchronize(st));
  if (stat_h[1]) return DS_ERR_DEGENERATE_COLUMN;
  if (dtype == DS_BF16) {
    quantise_kernel<__nv_bfloat16><<<sms * 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(W), V, d, w.norm, w.U);
  } else {
    quantise_kernel<float><<<sms * 8, 256, 0, st>>>(static_cast<const float*>(W), V, d, w.norm, w.U);
  }
  DS_TRY(cudaGetLastError());
  // 2. Forgy init: partial Fisher-Yates over [0, V) driven by splitmix64(seed)
  std::vector<int32_t> ids(M);
  if (init_ids_host) {
    std::copy(init_ids_host, init_ids_host + M, ids.begin());
  } else {
    std::vector<int32_t> a(V);
    std::iota(a.begin(), a.end(), 0);
    uint64_t state = seed;
    for (int i = 0; i < M; ++i) {
      const uint64_t r = splitmix64_next(state);
      const int64_t j = i + (int64_t)(r % (uint64_t)(V - i));
      std::swap(a[i], a[j]);
    }
    std::copy(a.begin(), a.begin() + M, ids.begin());
  }
  DS_TRY(cudaMemcpyAsync(w.members, ids.data(), M * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  gather_centroids_kernel<<<sms * 4, 256, 0, st>>>(w.U, w.members, M, d, w.C);
  DS_TRY(cudaGetLastError());
  DS_TRY(cudaStreamSynchronize(st));  // ids[] is a host stack buffer
  // 3. Lloyd iterations
  std::vector<int32_t> sz(M), starts(M + 1);
  double* cn = w.norm;  // reuse (token norms no longer needed): M doubles
  int it = 0;
  const int asg_blocks = (int)((V + kAsgTok - 1) / kAsgTok);
  for (it = 1; it <= max_iters; ++it) {
    DS_TRY(cudaMemsetAsync(w.stats, 0, sizeof(int32_t), st));
    assign_kernel<<<asg_blocks, kAsgThreads, 0, st>>>(w.U, w.C, V, d, M, tau, w.tau_prev, w.stats, it == 1);
    DS_TRY(cudaGetLastError());
    DS_TRY(cudaMemsetAsync(w.sizes, 0, M * sizeof(int32_t), st));
    sizes_kernel<<<sms * 4, 256, 0, st>>>(tau, V, w.sizes);
    DS_TRY(cudaGetLastError());
    DS_TRY(cudaMemcpyAsync(stat_h, w.stats, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    DS_TRY(cudaMemcpyAsync(sz.data(), w.sizes, M * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    DS_TRY(cudaStreamSynchronize(st));
    if (it > 1 && stat_h[0] == 0) break;  // tau unchanged from the previous iteration's final tau
    // update: member lists, exact int64 sums, normalised centroids
    starts[0] = 0;
    for (int m = 0; m < M; ++m) starts[m + 1] = starts[m] + sz[m];
    DS_TRY(cudaMemcpyAsync(w.starts, starts.data(), (M + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    DS_TRY(cudaMemcpyAsync(w.cursor, starts.data(), M * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    members_kernel<<<sms * 4, 256, 0, st>>>(tau, V, w.cursor, w.members);
    DS_TRY(cudaGetLastError());
    sum_kernel<<<dim3(M, (d + 255) / 256), 256, 0, st>>>(w.U, w.members, w.starts, d, w.S);
    DS_TRY(cudaGetLastError());
    cnorm_kernel<<<(M + 127) / 128, 128, 0, st>>>(w.S, w.sizes, M, d, cn);
    DS_TRY(cudaGetLastError());
    centroid_kernel<<<sms * 4, 256, 0, st>>>(w.S, cn, w.sizes, M, d, w.C);
    DS_TRY(cudaGetLastError());
    // reseed empty clusters in ascending m
    bool any_empty = false;
    for (int m = 0; m < M; ++m) any_empty |= (sz[m] == 0);
    if (any_empty) {
      sims_kernel<<<sms * 8, 256, 0, st>>>(w.U, w.C, tau, V, d, w.sims);
      DS_TRY(cudaGetLastError());
      for (int m = 0; m < M; ++m) {
        if (sz[m] != 0) continue;
        reseed_kernel<<<1, 1024, 0, st>>>(w.sims, tau, V, w.sizes, m, w.U, w.C, d);
        DS_TRY(cudaGetLastError());
      }
    }
    DS_TRY(cudaMemcpyAsync(w.tau_prev, tau, V * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    DS_TRY(cudaStreamSynchronize(st));  // starts[] is reused next iteration
  }
  if (it > max_iters) it = max_iters;
  // 4. canonical relabel by smallest token id
  std::vector<int32_t> mins(M, INT32_MAX);
  DS_TRY(cudaMemcpyAsync(w.minid, mins.data(), M * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  minid_kernel<<<sms * 4, 256, 0, st>>>(tau, V, w.minid);
  DS_TRY(cudaGetLastError());
  DS_TRY(cudaMemcpyAsync(mins.data(), w.minid, M * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  DS_TRY(cudaStreamSynchronize(st));
  std::vector<int32_t> order(M), newlab(M);
  std::iota(order.begin(), order.end(), 0);
  for (int m = 0; m < M; ++m)
    if (mins[m] == INT32_MAX) return DS_ERR_EMPTY_SHORTLIST;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return mins[a] < mins[b]; });
  for (int i = 0; i < M; ++i) newlab[order[i]] = i;
  DS_TRY(cudaMemcpyAsync(w.cursor, newlab.data(), M * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  relabel_kernel<<<sms * 4, 256, 0, st>>>(tau, V, w.cursor);
  DS_TRY(cudaGetLastError());
  DS_TRY(cudaStreamSynchronize(st));
  if (iters_host) *iters_host = it;
  // 5. layout (perm, offsets, W_perm) — uses the tail of the workspace
  void* lay_ws = static_cast<uint8_t*>(ws) + (w.total - align_up(layout_ws_bytes(V, M), 256));
  return run_layout(tau, W, dtype, V, d, M, perm, offsets, W_perm, sizes_host, lay_ws, st);
}

}  // namespace ds
