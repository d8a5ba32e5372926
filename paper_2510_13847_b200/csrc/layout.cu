// layout.cu — S0 layout step: cluster-permuted LM head (R12 step 9).
//
// perm = stable sort of token ids by tau (cluster m = rows [offsets[m], offsets[m+1]) of
// W_perm, ascending token ids inside), offsets = exclusive scan of |C_m|,
// W_perm[i] = W[perm[i]].  This is what makes every cluster one contiguous HBM block, so the
// head streams V_S with bulk copies instead of per-token gathers.
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace ds {

constexpr int kLayThreads = 256;

__global__ void count_clusters_kernel(const int32_t* __restrict__ tau, int64_t V, int M, int32_t* sizes, int32_t* err) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int m = tau[v];
    if (m < 0 || m >= M) {
      atomicExch(err, 1);
    } else {
      atomicAdd(&sizes[m], 1);
    }
  }
}

// One CTA per cluster: ordered compaction of the tokens of cluster m (stable by construction).
__global__ void __launch_bounds__(kLayThreads) scatter_perm_kernel(const int32_t* __restrict__ tau, int64_t V,
                                                                   const int32_t* __restrict__ offsets,
                                                                   int32_t* __restrict__ perm) {
  __shared__ int scratch[kLayThreads / 32 + 1];
  const int m = blockIdx.x;
  int base = offsets[m];
  constexpr int kPer = 4;
  for (int64_t v0 = 0; v0 < V; v0 += (int64_t)kLayThreads * kPer) {
    int cnt = 0;
    int32_t f[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t v = v0 + (int64_t)threadIdx.x * kPer + j;
      f[j] = (v < V && tau[v] == m) ? 1 : 0;
      cnt += f[j];
    }
    int total;
    int pos = block_excl_scan<kLayThreads>(cnt, scratch, total);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (f[j]) perm[base + pos++] = (int32_t)(v0 + (int64_t)threadIdx.x * kPer + j);
    }
    base += total;
  }
}

// W_perm[i] = W[perm[i]]: one warp per row, 16-byte vectors.
__global__ void gather_rows_kernel(const uint8_t* __restrict__ W, const int32_t* __restrict__ perm, int64_t V,
                                   int rowbytes, uint8_t* __restrict__ Wp) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < V; i += warps) {
    const uint4* src = reinterpret_cast<const uint4*>(W + (size_t)perm[i] * rowbytes);
    uint4* dst = reinterpret_cast<uint4*>(Wp + (size_t)i * rowbytes);
    for (int c = lane; c < rowbytes / 16; c += 32) dst[c] = src[c];
  }
}

cudaError_t launch_gather_rows(const void* W, size_t rowb, const int32_t* ids, int64_t n, void* out, cudaStream_t st) {
  gather_rows_kernel<<<num_sms() * 8, 256, 0, st>>>(static_cast<const uint8_t*>(W), ids, n, (int)rowb,
                                                   static_cast<uint8_t*>(out));
  return cudaGetLastError();
}

size_t layout_ws_bytes(int64_t V, int M) {
  (void)V;
  return align_up((size_t)(M + 1) * sizeof(int32_t), 256) + 256;
}

ds_status run_layout(const int32_t* tau, const void* W, int dtype, int64_t V, int d, int M, int32_t* perm,
                     int32_t* offsets, void* W_perm, int32_t* sizes_host, void* ws, cudaStream_t st) {
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  int32_t* sizes = reinterpret_cast<int32_t*>(w8);
  int32_t* err = reinterpret_cast<int32_t*>(w8 + align_up((size_t)(M + 1) * sizeof(int32_t), 256));
  if (cudaMemsetAsync(sizes, 0, (size_t)(M + 1) * sizeof(int32_t), st) != cudaSuccess) return DS_ERR_CUDA;
  if (cudaMemsetAsync(err, 0, sizeof(int32_t), st) != cudaSuccess) return DS_ERR_CUDA;
  const int sms = num_sms();
  count_clusters_kernel<<<sms * 4, 256, 0, st>>>(tau, V, M, sizes, err);
  if (cudaGetLastError() != cudaSuccess) return DS_ERR_CUDA;
  std::vector<int32_t> hs(M + 1);
  int32_t herr = 0;
  if (cudaMemcpyAsync(hs.data(), sizes, (size_t)M * sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return DS_ERR_CUDA;
  if (cudaMemcpyAsync(&herr, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess) return DS_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return DS_ERR_CUDA;
  if (herr) return DS_ERR_INVALID_CLUSTER_ID;
  std::vector<int32_t> off(M + 1, 0);
  int32_t mn = INT32_MAX, mx = 0;
  for (int m = 0; m < M; ++m) {
    if (hs[m] == 0) return DS_ERR_EMPTY_SHORTLIST;
    off[m + 1] = off[m] + hs[m];
    mn = hs[m] < mn ? hs[m] : mn;
    mx = hs[m] > mx ? hs[m] : mx;
  }
  if (cudaMemcpyAsync(offsets, off.data(), (size_t)(M + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st) !=
      cudaSuccess)
    return DS_ERR_CUDA;
  scatter_perm_kernel<<<M, kLayThreads, 0, st>>>(tau, V, offsets, perm);
  if (cudaGetLastError() != cudaSuccess) return DS_ERR_CUDA;
  const int rowbytes = d * (dtype == DS_BF16 ? 2 : 4);
  if (W != nullptr && W_perm != nullptr) {
    gather_rows_kernel<<<sms * 8, 256, 0, st>>>(static_cast<const uint8_t*>(W), perm, V, rowbytes,
                                                static_cast<uint8_t*>(W_perm));
    if (cudaGetLastError() != cudaSuccess) return DS_ERR_CUDA;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return DS_ERR_CUDA;  // off[] lives on this stack frame
  if (sizes_host) {
    sizes_host[0] = mn;
    sizes_host[1] = mx;
  }
  return DS_OK;
}

}  // namespace ds
