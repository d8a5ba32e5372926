// internal.h — launchers shared between the kernel translation units and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dynaspec.h"

namespace ds {

constexpr int kMaxM = 1024;      // largest cluster count the select kernels support
constexpr int kMaxMHost = kMaxM;
constexpr int kMaxKt = 64;       // largest token budget k_t

// Workspace prefix shared by every entry point (fixed offsets, so one workspace can serve any mix
// of calls): [0, 256) counters (left at zero by every kernel) with the device error word at 252;
// the polled-record regions of the single-row step kernels (0 = "not written yet", re-zeroed by
// their mergers, written by no other kernel); per-call scratch from kWsFixed on.
constexpr size_t kWsErrorWord = 252;
constexpr size_t kWsCstepRec = 256;                      // cluster step: [G][2 + k_t] u64 (<= 48 KB)
constexpr size_t kWsGstepRec = kWsCstepRec + 48 * 1024;  // grid step:    [G][2 + k_t] u64 (<= 48 KB)
constexpr size_t kWsGstepUnits = kWsGstepRec + 48 * 1024;  // grid step: [rows1] u64 layer-1 units (<= 4 KB)
constexpr size_t kWsRowsUnits = 112 * 1024;                // few-row router: [16][h_r <= 128] u64 units
constexpr size_t kWsRowsMasks = kWsRowsUnits + 16 * 1024;  // few-row router: [16][32] u64 TopK masks
constexpr size_t kWsFixed = kWsRowsMasks + 4 * 1024;       // 132 KB

int num_sms();
unsigned long long* debug_trace();   // device buffer set by dynaspec_debug_set_trace, or nullptr                 // SM count of the current device (cached per device)
size_t align_up(size_t x, size_t a);

// ---- meta-classifier (meta.cu)
struct MetaPlan {
  int KC;       // K-chunk per split (elements of the 2d input)
  int KS;       // number of K splits
  int rows1;    // layer-1 output rows (h_r, or M for a linear router)
  int RB;       // rows per layer-1 CTA (grid z = ceil(B / RB) row blocks)
  int tc;       // 1: layer 1 on tcgen05 (meta_tc.cu), KS_tc splits of kc_per_tc 64-wide chunks
  int KS_tc, kc_per_tc;
  size_t part_bytes;
};
bool meta_tc_plan(const ds_router* r, int B, int* KS, int* kc_per);
// Few rows (2 <= B <= 16, bf16, h_r <= #SMs, M <= 256): router + TopK (+ union) in ONE launch over all
// SMs (meta_rows.cu); ws = the workspace base (its unit / mask words live in the fixed prefix).
bool meta_rows_supported(const ds_router* r, int B, int k, const int32_t* k_per_row);
cudaError_t launch_meta_rows(const ds_router* r, const void* h_prev, const void* e, int B, float* scores,
                             const int32_t* offsets, int k, int shared, int32_t* sel, int32_t* sel_count,
                             int32_t* sl_offsets, void* ws, cudaStream_t st, bool pdl, bool defer_union = false);
cudaError_t launch_meta_tc_l1(const ds_router* r, const void* h_prev, const void* e, int B, float* part, int KS,
                              int kc_per, cudaStream_t st, bool pdl);
MetaPlan meta_plan(const ds_router* r, int B);
// Enqueue layer 1 (split-K partials) and layer 2 + (optionally) selection.
// sel == nullptr => scores only.
cudaError_t launch_meta(const ds_router* r, const void* h_prev, const void* e, int B, float* scores,
                        float* part, unsigned* counter, const int32_t* offsets, int k,
                        const int32_t* k_per_row, int shared, int32_t* sel, int32_t* sel_count,
                        int32_t* sl_offsets, cudaStream_t st, bool pdl);
cudaError_t launch_select(const float* scores, int B, int M, const int32_t* offsets, int k,
                          const int32_t* k_per_row, int shared, int32_t* sel, int32_t* sel_count,
                          int32_t* sl_offsets, unsigned* counter, cudaStream_t st);

// ---- head (head.cu)
struct HeadPlan {
  int G;               // CTAs per launch
  int rows_per_launch; // rows (per-row mode) / rows sharing the list (shared) per launch
  int lcap;            // logits capacity per row per CTA
  int rec;             // floats per partial record (2 + 2*k_t)
  int stage_rows;
  int stages;          // ring slots (= consumer warps)
  int stage_bytes;
  size_t smem;
  size_t part_bytes;   // workspace bytes for partials
  int launches;        // number of launches for B rows
};
bool head_plan(const ds_clusters* c, int B, int k_t, int64_t max_shortlist, HeadPlan* p);
bool head_plan_ex(const ds_clusters* c, int B, int k_t, int64_t max_shortlist, int extra_smem, int max_rows,
                  HeadPlan* p, int G = 0 /* CTAs per launch; 0 = one per SM */);
int max_smem_optin();
// cudaFuncAttributeMaxDynamicSharedMemorySize = max_smem_optin() for `fn`, once per device (done: [64]).
cudaError_t configure_max_smem(const void* fn, int* done);
cudaError_t launch_head(const ds_clusters* c, const HeadPlan& p, const void* h_new, int B, const int32_t* sel,
                        const int32_t* sel_count, const int32_t* sl_offsets, int shared, int k_t,
                        int64_t max_shortlist, int32_t* top_ids, float* top_logits, float* top_logp,
                        float* lse, float* z_out, int64_t z_stride, float* part, unsigned* counter,
                        cudaStream_t st, bool pdl, float* records = nullptr);

// ---- fused one-launch draft step (step.cu): router + select + head + epilogue
bool step_supported(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared, int64_t max_shortlist);
size_t step_ws_bytes(const ds_clusters* c, const ds_router* r, int B, int k_t);
// 2 <= B <= DS_GSTEP_ROWS_MAX (3) independent rows run as one grid step per row (launch_step)
bool step_rows_as_gsteps(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared);
cudaError_t launch_step(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                        const void* h_new, int B, int k, int k_t, int shared, int64_t max_shortlist, float* scores,
                        int32_t* sel, int32_t* sel_count, int32_t* sl_offsets, int32_t* top_ids, float* top_logits,
                        float* top_logp, float* lse, float* z_out, int64_t z_stride, void* ws, cudaStream_t st,
                        bool pdl);

// ---- cluster draft step (cstep.cu): B = 1, router per thread-block cluster (DSMEM), no grid barrier
bool cstep_supported(const ds_clusters* c, const ds_router* r, int B, int k_t, int shared, int64_t max_shortlist);
size_t cstep_ws_bytes(const ds_clusters* c, const ds_router* r, int B, int k_t);
bool cstep_pointers_ok(const ds_router* r, const void* h_prev, const void* e, const void* h_new);  // 16 B TMA
cudaError_t launch_cstep(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                         const void* h_new, int k, int k_t, int64_t max_shortlist, float* scores, int32_t* sel,
                         int32_t* sel_count, int32_t* sl_offsets, int32_t* top_ids, float* top_logits,
                         float* top_logp, float* lse, float* z_out, int64_t z_stride, void* ws, cudaStream_t st,
                         bool pdl);

bool cstep_head_supported(const ds_clusters* c, int k_t, int64_t max_shortlist);
size_t cstep_head_rec_bytes(const ds_clusters* c, int k_t);
cudaError_t launch_cstep_head(const ds_clusters* c, const void* h_new, const int32_t* sel, const int32_t* sel_count,
                              const int32_t* sl_offsets, int k_t, int64_t max_shortlist, int32_t* top_ids,
                              float* top_logits, float* top_logp, float* lse, float* z_out, int64_t z_stride,
                              void* rec, cudaStream_t st);

// ---- grid draft step (gstep.cu): B = 1, router units spread over every CTA, no clusters, no counters
bool gstep_supported(const ds_clusters* c, const ds_router* r /* nullptr: head only */, int B, int k_t, int shared);
bool gstep_pointers_ok(const ds_router* r, const void* h_prev, const void* e, const void* h_new);
cudaError_t launch_gstep(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                         const void* h_new, int k, int k_t, int64_t max_shortlist, float* scores, int32_t* sel,
                         int32_t* sel_count, int32_t* sl_offsets, int32_t* top_ids, float* top_logits,
                         float* top_logp, float* lse, float* z_out, void* ws, cudaStream_t st, bool pdl);
cudaError_t launch_gstep_head(const ds_clusters* c, const void* h_new, const int32_t* sel, const int32_t* sel_count,
                              const int32_t* sl_offsets, int k_t, int64_t max_shortlist, int32_t* top_ids,
                              float* top_logits, float* top_logp, float* lse, float* z_out, void* ws,
                              cudaStream_t st);

// ---- tcgen05 shared-shortlist head (tc_head.cu), bf16, R <= 64 rows sharing one shortlist
bool tc_head_supported(const ds_clusters* c, int R, int k_t, int64_t max_shortlist);
size_t tc_head_part_bytes(const ds_clusters* c, int R, int k_t);
cudaError_t launch_tc_head(const ds_clusters* c, const void* h_new, int R, const int32_t* sel,
                           const int32_t* sel_count, const int32_t* sl_offsets, int k_t, int64_t max_shortlist,
                           int32_t* top_ids, float* top_logits, float* top_logp, float* lse, float* z_out,
                           int64_t z_stride, float* part, unsigned* counter, cudaStream_t st, bool pdl);
// ---- balanced tree head (th.cu): <= 16 rows sharing one shortlist, k_t <= 16 (dispatched by launch_tc_head)
bool th_supported(const ds_clusters* c, int R, int k_t);
size_t th_ws_bytes(const ds_clusters* c, int R, int k_t);
cudaError_t launch_th(const ds_clusters* c, const void* h_new, int R, const int32_t* sel, const int32_t* sel_count,
                      const int32_t* sl_offsets, int k_t, int64_t max_shortlist, int32_t* top_ids,
                      float* top_logits, float* top_logp, float* lse, float* z_out, int64_t z_stride, void* ws,
                      unsigned* counter, cudaStream_t st, bool pdl, int rows = 0,
                      const void* umask_ws = nullptr /* workspace base: deferred tree union (meta_rows) */);
// independent rows (shared = 0) on the tree head: 2 <= B <= 16, no z_out (dispatch in api.cu)
bool use_th_rows(const ds_clusters* c, int B, int k_t, int shared, bool z_out);
bool use_tc_head(const ds_clusters* c, int B, int k_t, int shared, int64_t max_shortlist);
// batched per-row rows (each with its own selection), streamed once as their union on tcgen05
bool tc_batched_supported(const ds_clusters* c, int B, int k_t);
size_t tc_batched_ws_bytes(const ds_clusters* c, int B, int k_t);
cudaError_t launch_tc_batched(const ds_clusters* c, const void* h_new, int B, const int32_t* sel,
                              const int32_t* sel_count, int k_t, int32_t* top_ids, float* top_logits,
                              float* top_logp, float* lse, void* ws, unsigned* counter, cudaStream_t st);
bool use_tc_batched(const ds_clusters* c, int B, int k_t, int shared, bool z_out);
// ---- grouped (cluster-major) tcgen05 head for many independent rows (gh.cu)
bool gh_supported(const ds_clusters* c, int B, int k_t, int kmax);
bool gh_wide_grouping(int B, int shared);  // grouping by three grid-wide kernels instead of one CTA
size_t gh_ws_bytes(const ds_clusters* c, int B, int k_t, int kmax);
cudaError_t launch_gh(const ds_clusters* c, const void* h_new, int B, const int32_t* sel, const int32_t* sel_count,
                      int shared, int k_t, int kmax, int32_t* top_ids, float* top_logits, float* top_logp, float* lse, void* ws,
                      cudaStream_t st);
bool use_gh(const ds_clusters* c, int B, int k_t, int shared, bool z_out, int kmax);

// ---- cluster sharding (shard.cu)
cudaError_t launch_restrict(const int32_t* sel, const int32_t* cnt, int rows, int M, const int32_t* offsets, int m_lo,
                            int m_hi, int32_t* osel, int32_t* ocnt, int32_t* ooff, cudaStream_t st);
cudaError_t launch_merge_records(const float* records, int G, int B, int K, int32_t* top_ids, float* top_logits,
                                 float* top_logp, float* lse, cudaStream_t st);

// ---- draft-tree bookkeeping (tree.cu)
cudaError_t launch_tree_step(const int32_t* top_ids, const float* top_logp, int R, int K, const float* last_scores,
                             const int32_t* last_nodes, int step, int node_base, int32_t* node_tok, float* node_score,
                             int32_t* node_parent, int32_t* node_step, int32_t* next_tok, float* next_score,
                             int32_t* next_node, int32_t* next_beam, cudaStream_t st);
cudaError_t launch_tree_rerank(const float* node_score, const int32_t* node_tok, int n, int n_out, int32_t* out_nodes,
                               cudaStream_t st);

// ---- lossless verification + shortlist ids (verify.cu)
size_t verify_ws_bytes(int64_t V, int B, int gamma);
cudaError_t launch_verify(const void* p_logits, int dtype, int64_t V, int B, int gamma, const int32_t* q_ids,
                          const float* q_logits, int64_t q_stride, const int32_t* q_count, const float* q_lse,
                          const int32_t* x, const int32_t* x_slot, const float* u_acc, const float* u_res,
                          int32_t* accepted, int32_t* committed, void* ws, cudaStream_t st);
cudaError_t launch_shortlist_ids(const ds_clusters* c, int rows, const int32_t* sel, const int32_t* cnt,
                                 const int32_t* sl_off, int64_t stride, int32_t* ids, cudaStream_t st);

// ---- row gather (layout.cu): out[i] = W[ids[i]], rows of rowb bytes (a multiple of 16)
cudaError_t launch_gather_rows(const void* W, size_t rowb, const int32_t* ids, int64_t n, void* out, cudaStream_t st);

// ---- offline partition (build.cu)
size_t build_ws_bytes(int64_t V, int d, int M);
size_t layout_ws_bytes(int64_t V, int M);
ds_status run_layout(const int32_t* tau, const void* W, int dtype, int64_t V, int d, int M, int32_t* perm,
                     int32_t* offsets, void* W_perm, int32_t* sizes_host, void* ws, cudaStream_t st);
ds_status run_build(const void* W, int dtype, int64_t V, int d, int M, uint64_t seed, int max_iters,
                    const int32_t* init_ids_host, int32_t* tau, int32_t* perm, int32_t* offsets, void* W_perm,
                    int32_t* iters_host, int32_t* sizes_host, void* ws, cudaStream_t st);

}  // namespace ds
