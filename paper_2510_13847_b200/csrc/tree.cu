// tree.cu — NEXT-1: draft-tree bookkeeping of Algorithm 1 lines 12-18 on the device,
// so a whole gamma-step draft cycle stays graph-capturable (no host round trip between steps).
//   line 12  cu_scores = TopP_j + last_step_scores
//   line 13  d <- d + T~_j, d_scores <- d_scores + cu_scores      (node arrays, step-major)
//   line 14  TopC_j, last_step_scores <- TopK_{k_t}(cu_scores)    (ties -> lower flat index, R24)
//   lines 15-16  x_j <- T~_j[TopC_j]; parent beam of TopC_j selects h_j for the next step
//   line 18  re-rank d by d_scores (ties -> lower node index, R24)
#include "common.cuh"
#include "internal.h"

namespace ds {

__global__ void __launch_bounds__(256) tree_step_kernel(const int32_t* __restrict__ top_ids,
                                                        const float* __restrict__ top_logp, int R, int K,
                                                        const float* __restrict__ last_scores,
                                                        const int32_t* __restrict__ last_nodes, int step, int node_base,
                                                        int32_t* node_tok, float* node_score, int32_t* node_parent,
                                                        int32_t* node_step, int32_t* next_tok, float* next_score,
                                                        int32_t* next_node, int32_t* next_beam) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int n = R * K;
  float* cu = reinterpret_cast<float*>(sm);
  float* sv = cu + n;
  int* si = reinterpret_cast<int*>(sv + n);
  __shared__ int misc[4];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int b = i / K;
    const int tok = top_ids[i];
    const float c = top_logp[i] + (last_scores ? last_scores[b] : 0.f);   // line 12
    node_tok[node_base + i] = tok;                                          // line 13
    node_score[node_base + i] = tok >= 0 ? c : -INFINITY;
    node_parent[node_base + i] = last_nodes ? last_nodes[b] : -1;
    node_step[node_base + i] = step;
    cu[i] = tok >= 0 ? c : -INFINITY;
  }
  __syncthreads();
  block_topk(                                                               // line 14
      n, K, [&](int i, float& v, int& id) { v = cu[i]; id = i; },
      [&](int rank, float v, int id) {
        next_tok[rank] = top_ids[id];                                       // line 15
        next_score[rank] = v;
        next_node[rank] = node_base + id;
        next_beam[rank] = id / K;                                           // line 16
      },
      sv, si, misc);
  for (int q = misc[0] + threadIdx.x; q < K; q += blockDim.x) {
    next_tok[q] = -1;
    next_score[q] = -INFINITY;
    next_node[q] = -1;
    next_beam[q] = -1;
  }
}

__global__ void __launch_bounds__(1024) tree_rerank_kernel(const float* __restrict__ node_score,
                                                           const int32_t* __restrict__ node_tok, int n, int n_out,
                                                           int32_t* out_nodes) {
  extern __shared__ __align__(16) uint8_t sm[];
  float* sv = reinterpret_cast<float*>(sm);
  int* si = reinterpret_cast<int*>(sv + n);
  __shared__ int misc[4];
  block_topk(
      n, n_out,
      [&](int i, float& v, int& id) {
        v = node_tok[i] >= 0 ? node_score[i] : -INFINITY;
        id = i;
      },
      [&](int rank, float, int id) { out_nodes[rank] = id; }, sv, si, misc);
  for (int q = misc[0] + threadIdx.x; q < n_out; q += blockDim.x) out_nodes[q] = -1;
}

cudaError_t launch_tree_step(const int32_t* top_ids, const float* top_logp, int R, int K, const float* last_scores,
                             const int32_t* last_nodes, int step, int node_base, int32_t* node_tok, float* node_score,
                             int32_t* node_parent, int32_t* node_step, int32_t* next_tok, float* next_score,
                             int32_t* next_node, int32_t* next_beam, cudaStream_t st) {
  const size_t smem = (size_t)R * K * 12;
  if (smem > 40 * 1024) {  // opt in above the default (static smem counts too)
    cudaError_t e = cudaFuncSetAttribute(tree_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  tree_step_kernel<<<1, 256, smem, st>>>(top_ids, top_logp, R, K, last_scores, last_nodes, step, node_base, node_tok,
                                         node_score, node_parent, node_step, next_tok, next_score, next_node,
                                         next_beam);
  return cudaGetLastError();
}

cudaError_t launch_tree_rerank(const float* node_score, const int32_t* node_tok, int n, int n_out, int32_t* out_nodes,
                               cudaStream_t st) {
  const size_t smem = (size_t)n * 8;
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(tree_rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  tree_rerank_kernel<<<1, 1024, smem, st>>>(node_score, node_tok, n, n_out, out_nodes);
  return cudaGetLastError();
}

}  // namespace ds
