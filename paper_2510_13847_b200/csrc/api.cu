// api.cu — the C ABI (include/dynaspec.h): synchronous validation, workspace carving, launches.
#include <cuda_runtime.h>

#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "../../include/dynaspec.h"
#include "internal.h"

namespace ds {

static unsigned long long* g_trace = nullptr;
unsigned long long* debug_trace() { return g_trace; }

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// Tree / shared shortlist with >= 4 rows in bf16: the contraction goes to tcgen05 (S5').
bool use_tc_head(const ds_clusters* c, int B, int k_t, int shared, int64_t max_shortlist) {
  const char* off = getenv("DS_DISABLE_TC");
  if (off && off[0] == '1') return false;
  return shared && c->dtype == DS_BF16 && B >= 4 && tc_head_supported(c, B, k_t, max_shortlist);
}

bool use_tc_batched(const ds_clusters* c, int B, int k_t, int shared, bool z_out) {
  const char* off = getenv("DS_DISABLE_TC");
  if (off && off[0] == '1') return false;
  return !shared && !z_out && c->dtype == DS_BF16 && B >= 8 && tc_batched_supported(c, B, k_t);
}

// A few independent bf16 rows: the union of their clusters streamed once on the balanced tree head
// with per-row cluster masks (th.cu rows mode).  Measured at Llama-3 (us per draft step, rows mode vs
// the default; with 8 stored H rows for R <= 8): B = 4 71.8 vs 71.1 (multi-row fused step), B = 5
// 80.6 vs 82.1, B = 6 85.0 vs 92.6, B = 8 88.8 vs 105.4 (grouped head), B = 9 101.0 vs 108.4,
// B = 10 114.7 vs 111.4, B = 12 136.0 vs 117.7 — so by default for 5 <= B <= 9 (DS_TH_ROWS_MIN /
// _MAX; "0" in DS_TH_ROWS disables it).
bool use_th_rows(const ds_clusters* c, int B, int k_t, int shared, bool z_out) {
  const char* off = getenv("DS_TH_ROWS");
  if (off && off[0] == '0') return false;
  const char* tc = getenv("DS_DISABLE_TC");
  if (tc && tc[0] == '1') return false;
  const char* lo = getenv("DS_TH_ROWS_MIN");
  const char* hi = getenv("DS_TH_ROWS_MAX");
  const int bmin = lo && lo[0] ? std::max(2, atoi(lo)) : 5;
  const int bmax = hi && hi[0] ? std::min(16, atoi(hi)) : 9;
  return !shared && !z_out && B >= bmin && B <= bmax && th_supported(c, B, k_t);
}

// Many independent rows in bf16: the grouped cluster-major head (gh.cu) reads every selected cluster
// block once for all the rows that chose it.  DS_GH_MIN_ROWS (default 8) is the smallest batch.
bool use_gh(const ds_clusters* c, int B, int k_t, int shared, bool z_out, int kmax) {
  const char* off = getenv("DS_DISABLE_TC");
  if (off && off[0] == '1') return false;
  const char* mr = getenv("DS_GH_MIN_ROWS");
  const int min_rows = mr && mr[0] ? atoi(mr) : 8;
  // shared (tree) mode: every row streams the one union shortlist, >= 2 rows
  return !z_out && c->dtype == DS_BF16 && B >= (shared ? 2 : std::max(2, min_rows)) && gh_supported(c, B, k_t, kmax);
}

static bool dtype_ok(int dt) { return dt == DS_BF16 || dt == DS_F32; }

// S1 + S3/S4 for B rows: the few-row one-launch router (meta_rows.cu) when it applies, else the
// split-K pair (meta.cu).  ws = the workspace base.
static bool rows_router(const ds_router* r, const void* h_prev, const void* e, int B, int k) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(h_prev) | reinterpret_cast<uintptr_t>(e) |
                         reinterpret_cast<uintptr_t>(r->W1) | reinterpret_cast<uintptr_t>(r->W2)) & 15u) == 0;
  return aligned && meta_rows_supported(r, B, k, nullptr);
}
// defer_union (tree rows + tree head): the router leaves the rows' masks in the workspace and the
// tree head forms the union (one kernel boundary less on the path)
static cudaError_t route_rows(const ds_router* r, const ds_clusters* c, const void* h_prev, const void* e, int B,
                              float* scores, float* part, unsigned* counter, int k, int shared, int32_t* sel,
                              int32_t* sel_count, int32_t* sl_offsets, void* ws, cudaStream_t st, bool pdl,
                              bool defer_union = false) {
  if (rows_router(r, h_prev, e, B, k))
    return launch_meta_rows(r, h_prev, e, B, scores, c->offsets, k, shared, sel, sel_count, sl_offsets, ws, st, pdl,
                            defer_union);
  return launch_meta(r, h_prev, e, B, scores, part, counter, c->offsets, k, nullptr, shared, sel, sel_count,
                     sl_offsets, st, pdl);
}

static ds_status check_clusters(const ds_clusters* c) {
  if (!c || !c->perm || !c->offsets || !c->W_perm) return DS_ERR_SHAPE;
  if (!dtype_ok(c->dtype)) return DS_ERR_DTYPE;
  if (c->V < 1 || c->V > INT32_MAX || c->d < 1) return DS_ERR_SHAPE;
  if (c->M < 1 || c->M > c->V || c->M > kMaxMHost) return DS_ERR_INVALID_CLUSTER_COUNT;
  if (c->d % 8 != 0) return DS_ERR_UNSUPPORTED;
  if (c->min_size < 1 || c->max_size < c->min_size) return DS_ERR_SHAPE;
  return DS_OK;
}

static ds_status check_router(const ds_router* r) {
  if (!r || !r->W1 || !r->b1) return DS_ERR_SHAPE;
  if (!dtype_ok(r->dtype)) return DS_ERR_DTYPE;
  if (r->d < 1 || r->d % 8 != 0) return r->d < 1 ? DS_ERR_SHAPE : DS_ERR_UNSUPPORTED;
  if (r->M < 1 || r->M > kMaxMHost) return DS_ERR_INVALID_CLUSTER_COUNT;
  if (r->h_r < 0 || r->h_r > kMaxMHost) return DS_ERR_SHAPE;
  if (r->h_r > 0 && (!r->W2 || !r->b2)) return DS_ERR_SHAPE;
  if (r->h_r % 8 != 0) return DS_ERR_UNSUPPORTED;
  return DS_OK;
}

// Workspace carving: [counters 256 B][meta partials][head partials]
struct WsLayout {
  size_t counters, meta, head, total;
};
static WsLayout ws_layout(size_t meta_bytes, size_t head_bytes) {
  WsLayout L;
  L.counters = 0;
  L.meta = kWsFixed;  // after the counters and the polled-record regions (internal.h)
  L.head = align_up(L.meta + meta_bytes, 256);
  L.total = align_up(L.head + head_bytes, 256);
  return L;
}

}  // namespace ds

using namespace ds;

extern "C" {

const char* dynaspec_status_string(ds_status s) {
  switch (s) {
    case DS_OK: return "ok";
    case DS_ERR_SHAPE: return "shape error: inconsistent sizes or NULL required pointer";
    case DS_ERR_DTYPE: return "dtype error";
    case DS_ERR_INVALID_BUDGET: return "invalid budget (k or k_t out of range)";
    case DS_ERR_INVALID_CLUSTER_COUNT: return "invalid cluster count";
    case DS_ERR_INVALID_CLUSTER_ID: return "invalid cluster id";
    case DS_ERR_INVALID_TOKEN: return "invalid token id";
    case DS_ERR_DEGENERATE_COLUMN: return "degenerate (zero-norm) LM-head column";
    case DS_ERR_EMPTY_SHORTLIST: return "empty cluster / shortlist";
    case DS_ERR_WORKSPACE: return "workspace missing or too small";
    case DS_ERR_CUDA: return "CUDA error";
    case DS_ERR_UNSUPPORTED: return "unsupported shape";
    case DS_ERR_DEVICE_TIMEOUT: return "device timeout: a CTA waited > 2 s for its grid (SMs held by a concurrent kernel)";
  }
  return "unknown status";
}

ds_status dynaspec_debug_set_trace(void* dev_buf) {
  g_trace = static_cast<unsigned long long*>(dev_buf);
  return DS_OK;
}

int32_t dynaspec_budget(int32_t t, int32_t k_max, int32_t k_min) {
  if (t < 0 || k_min < 1 || k_max < k_min) return -1;
  if (t <= 1) return k_max;
  const int32_t k = k_max / ((t + 1) * 2);
  return k > k_min ? k : k_min;
}

int32_t dynaspec_pa_fr_budget(int32_t t, int32_t K_max) {
  if (t < 0 || K_max < 1) return -1;
  if (t <= 1) return K_max;
  const int32_t k = K_max / (t + 1);
  return k > 1 ? k : 1;
}

ds_status dynaspec_gather_rows(const void* W, int32_t dtype, int64_t V, int32_t d, const int32_t* ids, int64_t n,
                               void* out, ds_stream_t stream) {
  if (!W || !ids || !out || V < 1 || d < 1 || n < 0) return DS_ERR_SHAPE;
  if (!dtype_ok(dtype)) return DS_ERR_DTYPE;
  const size_t rowb = (size_t)d * (dtype == DS_BF16 ? 2 : 4);
  if (rowb % 16 != 0) return DS_ERR_UNSUPPORTED;
  if (n == 0) return DS_OK;
  return launch_gather_rows(W, rowb, ids, n, out, (cudaStream_t)stream) == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

int64_t dynaspec_max_shortlist(const ds_clusters* c, int32_t k) {
  if (!c || k < 1) return 0;
  const int64_t b = (int64_t)k * c->max_size;
  return b < c->V ? b : c->V;
}

ds_status dynaspec_ws_init(void* ws, size_t ws_bytes, ds_stream_t stream) {
  if (!ws || ws_bytes < 256) return DS_ERR_WORKSPACE;
  return cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream) == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

ds_status dynaspec_ws_error(void* ws, size_t ws_bytes, int32_t* code_host, ds_stream_t stream) {
  if (!ws || ws_bytes < kWsFixed || !code_host) return DS_ERR_WORKSPACE;
  unsigned v = 0;
  uint8_t* w = static_cast<uint8_t*>(ws) + kWsErrorWord;
  if (cudaMemcpyAsync(&v, w, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess) return DS_ERR_CUDA;
  if (cudaMemsetAsync(w, 0, 4, (cudaStream_t)stream) != cudaSuccess) return DS_ERR_CUDA;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return DS_ERR_CUDA;
  *code_host = (int32_t)v;
  return DS_OK;
}

size_t dynaspec_layout_ws(int64_t V, int32_t M) { return layout_ws_bytes(V, M); }

ds_status dynaspec_layout(const int32_t* tau, const void* W, int32_t dtype, int64_t V, int32_t d, int32_t M,
                          int32_t* perm, int32_t* offsets, void* W_perm, int32_t* sizes_host, void* ws,
                          size_t ws_bytes, ds_stream_t stream) {
  if (!tau || !perm || !offsets) return DS_ERR_SHAPE;
  if ((W == nullptr) != (W_perm == nullptr)) return DS_ERR_SHAPE;
  if (!dtype_ok(dtype)) return DS_ERR_DTYPE;
  if (V < 1 || V > INT32_MAX || d < 1) return DS_ERR_SHAPE;
  if (M < 1 || M > V || M > kMaxMHost) return DS_ERR_INVALID_CLUSTER_COUNT;
  if (d % 8 != 0) return DS_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < layout_ws_bytes(V, M)) return DS_ERR_WORKSPACE;
  return run_layout(tau, W, dtype, V, d, M, perm, offsets, W_perm, sizes_host, ws, (cudaStream_t)stream);
}

size_t dynaspec_build_clusters_ws(int64_t V, int32_t d, int32_t M) { return build_ws_bytes(V, d, M); }

ds_status dynaspec_build_clusters(const void* W, int32_t dtype, int64_t V, int32_t d, int32_t M, uint64_t seed,
                                  int32_t max_iters, const int32_t* init_ids_host, int32_t* tau, int32_t* perm,
                                  int32_t* offsets, void* W_perm, int32_t* iters_run_host, int32_t* sizes_host,
                                  void* ws, size_t ws_bytes, ds_stream_t stream) {
  if (!W || !tau || !perm || !offsets || !W_perm) return DS_ERR_SHAPE;
  if (!dtype_ok(dtype)) return DS_ERR_DTYPE;
  if (V < 1 || V > INT32_MAX || d < 1 || max_iters < 1) return DS_ERR_SHAPE;
  if (M < 1 || M > V || M > kMaxMHost) return DS_ERR_INVALID_CLUSTER_COUNT;
  if (d % 8 != 0) return DS_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < build_ws_bytes(V, d, M)) return DS_ERR_WORKSPACE;
  if (init_ids_host) {
    for (int m = 0; m < M; ++m)
      if (init_ids_host[m] < 0 || init_ids_host[m] >= V) return DS_ERR_INVALID_TOKEN;
  }
  return run_build(W, dtype, V, d, M, seed, max_iters, init_ids_host, tau, perm, offsets, W_perm, iters_run_host,
                   sizes_host, ws, (cudaStream_t)stream);
}

size_t dynaspec_meta_score_ws(const ds_router* r, int32_t B) {
  if (!r || B < 1) return 0;
  return ws_layout(meta_plan(r, B).part_bytes, 0).total;
}

ds_status dynaspec_meta_score(const ds_router* r, const void* h_prev, const void* e, int32_t B, float* scores,
                              void* ws, size_t ws_bytes, ds_stream_t stream) {
  ds_status s = check_router(r);
  if (s != DS_OK) return s;
  if (!h_prev || !e || !scores || B < 1) return DS_ERR_SHAPE;
  const WsLayout L = ws_layout(meta_plan(r, B).part_bytes, 0);
  if (!ws || ws_bytes < L.total) return DS_ERR_WORKSPACE;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  cudaError_t err = launch_meta(r, h_prev, e, B, scores, reinterpret_cast<float*>(w8 + L.meta),
                                reinterpret_cast<unsigned*>(w8 + L.counters), nullptr, 0, nullptr, 0, nullptr,
                                nullptr, nullptr, (cudaStream_t)stream, false);
  return err == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

ds_status dynaspec_select(const float* scores, int32_t B, const ds_clusters* c, int32_t k, const int32_t* k_per_row,
                          int32_t shared, int32_t* sel, int32_t* sel_count, int32_t* sl_offsets,
                          ds_stream_t stream) {
  if (!c || !c->offsets) return DS_ERR_SHAPE;
  if (c->M < 1 || c->M > kMaxMHost || c->M > c->V) return DS_ERR_INVALID_CLUSTER_COUNT;
  if (!scores || !sel || !sel_count || !sl_offsets || B < 1) return DS_ERR_SHAPE;
  if (!k_per_row && (k < 1 || k > c->M)) return DS_ERR_INVALID_BUDGET;
  cudaError_t err = launch_select(scores, B, c->M, c->offsets, k, k_per_row, shared ? 1 : 0, sel, sel_count,
                                  sl_offsets, nullptr, (cudaStream_t)stream);
  return err == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

// Head scratch for B rows: the largest of the head kernels' partials (the single-row step kernels'
// records live in the fixed prefix, internal.h).
static size_t head_scratch(const ds_clusters* c, int32_t B, int32_t k_t, const HeadPlan& pmax) {
  const size_t gh = gh_supported(c, B, k_t, c->M) ? gh_ws_bytes(c, B, k_t, c->M) : 0;
  return std::max(std::max(std::max(pmax.part_bytes, tc_head_part_bytes(c, B, k_t)), tc_batched_ws_bytes(c, B, k_t)),
                  gh);
}

size_t dynaspec_head_forward_ws(const ds_clusters* c, int32_t B, int32_t k_t) {
  HeadPlan p;
  if (!c || B < 1 || k_t < 1 || k_t > kMaxKt) return 0;
  if (!head_plan(c, B, k_t, 0, &p)) return 0;
  return ws_layout(0, head_scratch(c, B, k_t, p)).total;
}

ds_status dynaspec_head_forward(const ds_clusters* c, const void* h_new, int32_t B, const int32_t* sel,
                                const int32_t* sel_count, const int32_t* sl_offsets, int32_t shared, int32_t k_t,
                                int64_t max_shortlist, int32_t* top_ids, float* top_logits, float* top_logp,
                                float* lse, float* z_out, int64_t z_stride, void* ws, size_t ws_bytes,
                                ds_stream_t stream) {
  ds_status s = check_clusters(c);
  if (s != DS_OK) return s;
  if (!h_new || !sel || !sel_count || !sl_offsets || !top_ids || !top_logits || !top_logp || !lse || B < 1)
    return DS_ERR_SHAPE;
  if (k_t < 1 || k_t > kMaxKt) return DS_ERR_INVALID_BUDGET;
  if (max_shortlist < 0) return DS_ERR_SHAPE;
  if (z_out && z_stride < (max_shortlist > 0 ? std::min<int64_t>(max_shortlist, c->V) : c->V)) return DS_ERR_SHAPE;
  HeadPlan p;
  if (!head_plan(c, B, k_t, max_shortlist, &p)) return DS_ERR_UNSUPPORTED;
  // the workspace is sized for the largest plan (max_shortlist = V); smaller bounds need less
  const WsLayout L = ws_layout(0, p.part_bytes);
  if (!ws || ws_bytes < L.total) return DS_ERR_WORKSPACE;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  cudaError_t err;
  if (use_th_rows(c, B, k_t, shared, z_out != nullptr)) {
    if (ws_bytes < ws_layout(0, tc_head_part_bytes(c, B, k_t)).total) return DS_ERR_WORKSPACE;
    err = launch_th(c, h_new, B, sel, sel_count, sl_offsets, k_t, max_shortlist, top_ids, top_logits, top_logp, lse,
                    nullptr, 0, w8 + L.head, reinterpret_cast<unsigned*>(w8 + L.counters), (cudaStream_t)stream,
                    false, 1);
  } else if (!use_tc_head(c, B, k_t, shared, max_shortlist) && use_gh(c, B, k_t, shared, z_out != nullptr, c->M)) {
    if (ws_bytes < ws_layout(0, gh_ws_bytes(c, B, k_t, c->M)).total) return DS_ERR_WORKSPACE;
    err = launch_gh(c, h_new, B, sel, sel_count, shared, k_t, c->M, top_ids, top_logits, top_logp, lse, w8 + L.head,
                    (cudaStream_t)stream);
  } else if (use_tc_batched(c, B, k_t, shared, z_out != nullptr)) {
    if (ws_bytes < ws_layout(0, tc_batched_ws_bytes(c, B, k_t)).total) return DS_ERR_WORKSPACE;
    err = launch_tc_batched(c, h_new, B, sel, sel_count, k_t, top_ids, top_logits, top_logp, lse, w8 + L.head,
                            reinterpret_cast<unsigned*>(w8 + L.counters), (cudaStream_t)stream);
  } else if (use_tc_head(c, B, k_t, shared, max_shortlist)) {
    if (ws_bytes < ws_layout(0, tc_head_part_bytes(c, B, k_t)).total) return DS_ERR_WORKSPACE;
    err = launch_tc_head(c, h_new, B, sel, sel_count, sl_offsets, k_t, max_shortlist, top_ids, top_logits,
                         top_logp, lse, z_out, z_stride, reinterpret_cast<float*>(w8 + L.head),
                         reinterpret_cast<unsigned*>(w8 + L.counters), (cudaStream_t)stream, false);
  } else if (B == 1 && gstep_supported(c, nullptr, 1, k_t, 0) && (reinterpret_cast<uintptr_t>(h_new) & 15u) == 0) {
    // one row (shared == per-row): one CTA per SM streams chunk c of the shortlist on CTA c mod G
    err = launch_gstep_head(c, h_new, sel, sel_count, sl_offsets, k_t, max_shortlist, top_ids, top_logits, top_logp,
                            lse, z_out, ws, (cudaStream_t)stream);
  } else if (B == 1 && cstep_head_supported(c, k_t, max_shortlist)) {
    err = launch_cstep_head(c, h_new, sel, sel_count, sl_offsets, k_t, max_shortlist, top_ids, top_logits, top_logp,
                            lse, z_out, z_stride, ws, (cudaStream_t)stream);
  } else {
    err = launch_head(c, p, h_new, B, sel, sel_count, sl_offsets, shared ? 1 : 0, k_t, max_shortlist, top_ids,
                      top_logits, top_logp, lse, z_out, z_stride, reinterpret_cast<float*>(w8 + L.head),
                      reinterpret_cast<unsigned*>(w8 + L.counters), (cudaStream_t)stream, false);
  }
  return err == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

ds_status dynaspec_restrict_selection(const int32_t* sel, const int32_t* sel_count, const int32_t* sl_offsets,
                                      int32_t rows, const ds_clusters* c, int32_t m_lo, int32_t m_hi, int32_t* out_sel,
                                      int32_t* out_count, int32_t* out_sl_offsets, ds_stream_t stream) {
  if (!c || !c->offsets || !sel || !sel_count || !sl_offsets || !out_sel || !out_count || !out_sl_offsets || rows < 1)
    return DS_ERR_SHAPE;
  if (c->M < 1 || c->M > kMaxMHost) return DS_ERR_INVALID_CLUSTER_COUNT;
  if (m_lo < 0 || m_hi > c->M || m_lo > m_hi) return DS_ERR_INVALID_CLUSTER_ID;
  return launch_restrict(sel, sel_count, rows, c->M, c->offsets, m_lo, m_hi, out_sel, out_count, out_sl_offsets,
                         (cudaStream_t)stream) == cudaSuccess
             ? DS_OK
             : DS_ERR_CUDA;
}

ds_status dynaspec_head_partial(const ds_clusters* c, const void* h_new, int32_t B, const int32_t* sel,
                                const int32_t* sel_count, const int32_t* sl_offsets, int32_t shared, int32_t k_t,
                                int64_t max_shortlist, float* records, void* ws, size_t ws_bytes, ds_stream_t stream) {
  ds_status s = check_clusters(c);
  if (s != DS_OK) return s;
  if (!h_new || !sel || !sel_count || !sl_offsets || !records || B < 1) return DS_ERR_SHAPE;
  if (k_t < 1 || k_t > kMaxKt) return DS_ERR_INVALID_BUDGET;
  if (max_shortlist < 0) return DS_ERR_SHAPE;
  HeadPlan p;
  if (!head_plan(c, B, k_t, max_shortlist, &p)) return DS_ERR_UNSUPPORTED;
  const WsLayout L = ws_layout(0, p.part_bytes);
  if (!ws || ws_bytes < L.total) return DS_ERR_WORKSPACE;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  // the final-output pointers are unused in record mode; pass the record buffer as a harmless target
  cudaError_t err = launch_head(c, p, h_new, B, sel, sel_count, sl_offsets, shared ? 1 : 0, k_t, max_shortlist,
                                reinterpret_cast<int32_t*>(records), records, records, records, nullptr, 0,
                                reinterpret_cast<float*>(w8 + L.head), reinterpret_cast<unsigned*>(w8 + L.counters),
                                (cudaStream_t)stream, false, records);
  return err == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

ds_status dynaspec_merge_records(const float* records, int32_t G, int32_t B, int32_t k_t, int32_t* top_ids,
                                 float* top_logits, float* top_logp, float* lse, ds_stream_t stream) {
  if (!records || !top_ids || !top_logits || !top_logp || !lse || G < 1 || G > 64 || B < 1) return DS_ERR_SHAPE;
  if (k_t < 1 || k_t > kMaxKt) return DS_ERR_INVALID_BUDGET;
  return launch_merge_records(records, G, B, k_t, top_ids, top_logits, top_logp, lse, (cudaStream_t)stream) ==
                 cudaSuccess
             ? DS_OK
             : DS_ERR_CUDA;
}

ds_status dynaspec_tree_step(const int32_t* top_ids, const float* top_logp, int32_t R, int32_t k_t,
                             const float* last_scores, const int32_t* last_nodes, int32_t step, int32_t node_base,
                             int32_t* node_tok, float* node_score, int32_t* node_parent, int32_t* node_step,
                             int32_t* next_tok, float* next_score, int32_t* next_node, int32_t* next_beam,
                             ds_stream_t stream) {
  if (!top_ids || !top_logp || !node_tok || !node_score || !node_parent || !node_step || !next_tok || !next_score ||
      !next_node || !next_beam || R < 1 || R > 64)
    return DS_ERR_SHAPE;
  if (k_t < 1 || k_t > kMaxKt) return DS_ERR_INVALID_BUDGET;
  if (step < 0 || node_base < 0) return DS_ERR_SHAPE;
  return launch_tree_step(top_ids, top_logp, R, k_t, last_scores, last_nodes, step, node_base, node_tok, node_score,
                          node_parent, node_step, next_tok, next_score, next_node, next_beam,
                          (cudaStream_t)stream) == cudaSuccess
             ? DS_OK
             : DS_ERR_CUDA;
}

ds_status dynaspec_tree_rerank(const float* node_score, const int32_t* node_tok, int32_t n_nodes, int32_t n_out,
                               int32_t* out_nodes, ds_stream_t stream) {
  if (!node_score || !node_tok || !out_nodes || n_nodes < 1 || n_out < 1) return DS_ERR_SHAPE;
  if (n_nodes > 16384) return DS_ERR_UNSUPPORTED;
  return launch_tree_rerank(node_score, node_tok, n_nodes, n_out, out_nodes, (cudaStream_t)stream) == cudaSuccess
             ? DS_OK
             : DS_ERR_CUDA;
}

ds_status dynaspec_shortlist_ids(const ds_clusters* c, int32_t rows, const int32_t* sel, const int32_t* sel_count,
                                 const int32_t* sl_offsets, int64_t stride, int32_t* ids, ds_stream_t stream) {
  ds_status s = check_clusters(c);
  if (s != DS_OK) return s;
  if (!sel || !sel_count || !sl_offsets || !ids || rows < 1 || stride < 1) return DS_ERR_SHAPE;
  return launch_shortlist_ids(c, rows, sel, sel_count, sl_offsets, stride, ids, (cudaStream_t)stream) == cudaSuccess
             ? DS_OK
             : DS_ERR_CUDA;
}

size_t dynaspec_verify_ws(int64_t V, int32_t B, int32_t gamma) {
  if (V < 1 || B < 1 || gamma < 0 || gamma > 32) return 0;
  return verify_ws_bytes(V, B, gamma);
}

ds_status dynaspec_verify_chain(const void* p_logits, int32_t dtype, int64_t V, int32_t B, int32_t gamma,
                                const int32_t* q_ids, const float* q_logits, int64_t q_stride, const int32_t* q_count,
                                const float* q_lse, const int32_t* x, const int32_t* x_slot, const float* u_acc,
                                const float* u_res, int32_t* accepted, int32_t* committed, void* ws, size_t ws_bytes,
                                ds_stream_t stream) {
  if (!dtype_ok(dtype)) return DS_ERR_DTYPE;
  if (!p_logits || !u_res || !accepted || !committed || B < 1 || V < 1 || V > INT32_MAX || gamma < 0)
    return DS_ERR_SHAPE;
  if (gamma > 32 || V % 8 != 0) return DS_ERR_UNSUPPORTED;
  if (gamma > 0 && (!q_ids || !q_logits || !q_count || !q_lse || !x || !x_slot || !u_acc || q_stride < 1))
    return DS_ERR_SHAPE;
  if (!ws || ws_bytes < verify_ws_bytes(V, B, gamma)) return DS_ERR_WORKSPACE;
  return launch_verify(p_logits, dtype, V, B, gamma, q_ids, q_logits, q_stride, q_count, q_lse, x, x_slot, u_acc,
                       u_res, accepted, committed, ws, (cudaStream_t)stream) == cudaSuccess
             ? DS_OK
             : DS_ERR_CUDA;
}

ds_status dynaspec_step_route(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e, int32_t B,
                              int32_t t, int32_t k_max, int32_t k_min, int32_t shared, const ds_step_outputs* out,
                              void* ws, size_t ws_bytes, ds_stream_t s_meta) {
  ds_status s = check_clusters(c);
  if (s != DS_OK) return s;
  if ((s = check_router(r)) != DS_OK) return s;
  if (r->M != c->M || r->d != c->d) return DS_ERR_SHAPE;
  if (!h_prev || !e || !out || !out->sel || !out->sel_count || !out->sl_offsets || B < 1) return DS_ERR_SHAPE;
  const int32_t k = dynaspec_budget(t, k_max, k_min);
  if (k < 1 || k_max > c->M) return DS_ERR_INVALID_BUDGET;
  const size_t meta_bytes = meta_plan(r, B).part_bytes;
  const size_t score_bytes = (size_t)B * r->M * sizeof(float);
  const WsLayout L = ws_layout(align_up(meta_bytes, 256) + align_up(score_bytes, 256), 0);
  if (!ws || ws_bytes < L.total) return DS_ERR_WORKSPACE;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  float* scores = out->scores ? out->scores : reinterpret_cast<float*>(w8 + L.meta + align_up(meta_bytes, 256));
  return route_rows(r, c, h_prev, e, B, scores, reinterpret_cast<float*>(w8 + L.meta),
                    reinterpret_cast<unsigned*>(w8 + L.counters) + 1, k, shared ? 1 : 0, out->sel, out->sel_count,
                    out->sl_offsets, ws, (cudaStream_t)s_meta, false) == cudaSuccess
             ? DS_OK
             : DS_ERR_CUDA;
}

ds_status dynaspec_step_head(const ds_clusters* c, const void* h_new, int32_t B, int32_t t, int32_t k_max,
                             int32_t k_min, int32_t k_t, int32_t shared, const ds_step_outputs* out, void* ws,
                             size_t ws_bytes, ds_stream_t s_draft) {
  ds_status s = check_clusters(c);
  if (s != DS_OK) return s;
  if (!h_new || !out || B < 1) return DS_ERR_SHAPE;
  const int32_t k = dynaspec_budget(t, k_max, k_min);
  if (k < 1 || k_max > c->M) return DS_ERR_INVALID_BUDGET;
  if (k_t < 1 || k_t > kMaxKt || (int64_t)k_t > (int64_t)k * c->min_size) return DS_ERR_INVALID_BUDGET;
  // shared (tree) mode: the union of B rows' k clusters has at most min(M, B k) clusters
  const int64_t ms = dynaspec_max_shortlist(c, shared ? (int32_t)std::min<int64_t>(c->M, (int64_t)B * k) : k);
  if (out->z_out && out->z_stride < ms) return DS_ERR_SHAPE;
  return dynaspec_head_forward(c, h_new, B, out->sel, out->sel_count, out->sl_offsets, shared, k_t, ms, out->top_ids,
                               out->top_logits, out->top_logp, out->lse, out->z_out, out->z_stride, ws, ws_bytes,
                               s_draft);
}

size_t dynaspec_draft_step_ws(const ds_clusters* c, const ds_router* r, int32_t B, int32_t k_t) {
  HeadPlan p;
  if (!c || !r || B < 1 || k_t < 1 || k_t > kMaxKt) return 0;
  if (!head_plan(c, B, k_t, 0, &p)) return 0;
  const size_t meta = meta_plan(r, B).part_bytes;
  const size_t scores = (size_t)B * r->M * sizeof(float);
  return std::max(ws_layout(align_up(meta, 256) + align_up(scores, 256), head_scratch(c, B, k_t, p)).total,
                  step_ws_bytes(c, r, B, k_t));
}

int32_t dynaspec_draft_step_launches(const ds_clusters* c, const ds_router* r, int32_t B, int32_t k_t,
                                     int32_t shared, int32_t two_streams, int32_t z_out) {
  HeadPlan p;
  if (!c || !r || !head_plan(c, B, k_t, 0, &p)) return 0;
  const int64_t ms = shared ? c->V : 0;
  // router: one launch (few rows, meta_rows.cu; 16-byte aligned inputs assumed) or layer 1 + layer 2
  const int meta = meta_rows_supported(r, B, 1, nullptr) ? 1 : 2;
  if (use_tc_head(c, B, k_t, shared, ms)) return meta + 1;  // router (+union), tcgen05 tree head
  if (use_th_rows(c, B, k_t, shared, z_out != 0)) return meta + 1;  // router, tree head (rows mode)
  if (use_gh(c, B, k_t, shared, z_out != 0, c->M))  // router, grouping (1 or 3), grouped tcgen05 head, merge
    return meta + (gh_wide_grouping(B, shared) ? 5 : 3);
  if (use_tc_batched(c, B, k_t, shared, z_out != 0))
    return meta + 2 * ((B + 127) / 128);  // router, then (union + tcgen05 head) per 128 rows
  if (!two_streams && step_supported(c, r, B, k_t, shared, 0))  // fused single-stream step
    return step_rows_as_gsteps(c, r, B, k_t, shared) ? B : 1;      // (a couple of rows: a grid step each)
  return meta + p.launches;  // router (+select), head chunks
}

const char* dynaspec_draft_step_kernel(const ds_clusters* c, const ds_router* r, int32_t B, int32_t k_t,
                                       int32_t shared, int32_t two_streams, int32_t z_out) {
  HeadPlan p;
  if (!c || !r || !head_plan(c, B, k_t, 0, &p)) return "?";
  const int64_t ms = shared ? c->V : 0;
  if (use_tc_head(c, B, k_t, shared, ms))
    return th_supported(c, B, k_t) ? "ds::th_kernel (tcgen05 balanced tree head: one cluster per CTA, 3-D TMA boxes)"
                                   : "ds::tc_head_kernel (tcgen05, shared shortlist)";
  if (use_th_rows(c, B, k_t, shared, z_out != 0))
    return "ds::th_kernel (tcgen05 balanced tree head, rows mode: the rows' union once, per-row cluster masks)";
  if (use_gh(c, B, k_t, shared, z_out != 0, c->M))
    return "ds::gh_head_kernel (tcgen05 grouped head: every selected cluster block once for the rows that chose it)";
  if (use_tc_batched(c, B, k_t, shared, z_out != 0))
    return "ds::tc_head_kernel (tcgen05, batched rows over the union)";
  if (!two_streams && step_supported(c, r, B, k_t, shared, 0)) {
    if (step_rows_as_gsteps(c, r, B, k_t, shared))
      return "ds::gstep_kernel (one grid step per row, PDL-chained)";
    if (gstep_supported(c, r, B, k_t, shared))
      return "ds::gstep_kernel (grid step: router units over all CTAs + select + gathered head + epilogue, one launch)";
    if (cstep_supported(c, r, B, k_t, shared, 0))
      return "ds::cstep_kernel (cluster step: router per 16-CTA cluster + select + gathered head + epilogue, one launch)";
    return "ds::step_kernel (router + select + gathered head + epilogue, one launch)";
  }
  if (B == 1 && !shared && gstep_supported(c, nullptr, 1, k_t, 0)) return "ds::gstep_kernel (head only, after the router on S_m)";
  if (B == 1 && !shared && cstep_head_supported(c, k_t, 0)) return "ds::cstep_kernel (head only, after the router on S_m)";
  return "ds::head_kernel (gathered head + epilogue, after the router on S_m)";
}

ds_status dynaspec_draft_step(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                              const void* h_new, int32_t B, int32_t t, int32_t k_max, int32_t k_min, int32_t k_t,
                              int32_t shared, const ds_step_outputs* out, void* ws, size_t ws_bytes,
                              ds_stream_t s_draft, ds_stream_t s_meta, ds_event_t ev_fork, ds_event_t ev_join,
                              ds_event_t head_begin, ds_event_t head_end) {
  ds_status s = check_clusters(c);
  if (s != DS_OK) return s;
  if ((s = check_router(r)) != DS_OK) return s;
  if (r->M != c->M || r->d != c->d) return DS_ERR_SHAPE;
  if (r->dtype != c->dtype) return DS_ERR_DTYPE;
  if (!h_prev || !e || !h_new || !out || B < 1) return DS_ERR_SHAPE;
  if (!out->sel || !out->sel_count || !out->sl_offsets || !out->top_ids || !out->top_logits || !out->top_logp ||
      !out->lse)
    return DS_ERR_SHAPE;
  const int32_t k = dynaspec_budget(t, k_max, k_min);
  if (k < 1 || k_max > c->M) return DS_ERR_INVALID_BUDGET;
  if (k_t < 1 || k_t > kMaxKt || (int64_t)k_t > (int64_t)k * c->min_size) return DS_ERR_INVALID_BUDGET;
  // shared (tree) mode: the union of B rows' k clusters has at most min(M, B k) clusters
  const int64_t ms = dynaspec_max_shortlist(c, shared ? (int32_t)std::min<int64_t>(c->M, (int64_t)B * k) : k);
  if (out->z_out && out->z_stride < ms) return DS_ERR_SHAPE;
  const bool two_streams = s_meta != nullptr && s_meta != s_draft;
  if (two_streams && (!ev_fork || !ev_join)) return DS_ERR_SHAPE;
  // tree rows (shared): the shared-shortlist tcgen05 head (Qwen tree 90 vs 127 us per step with the
  // grouped head, whose router / grouping / merge launches dominate at 10 rows); independent rows: the
  // grouped head.  Supported-ness with kmax = M (what dynaspec_draft_step_ws sized the workspace for).
  const char* gt = getenv("DS_GH_TREE");  // "1": tree rows on the grouped head too (A/B)
  const bool gh_tree = gt && gt[0] == '1';
  const bool tc = !gh_tree && use_tc_head(c, B, k_t, shared, ms);
  const bool thr = !tc && use_th_rows(c, B, k_t, shared, out->z_out != nullptr);
  const bool gh = !tc && !thr && use_gh(c, B, k_t, shared, out->z_out != nullptr, c->M);
  const bool tcb = !tc && !thr && !gh && use_tc_batched(c, B, k_t, shared, out->z_out != nullptr);
  const bool fused = !tc && !thr && !tcb && !gh && !two_streams && step_supported(c, r, B, k_t, shared, ms);
  if (fused) {  // one persistent launch: router + select + head + epilogue (step.cu)
    const size_t need = step_ws_bytes(c, r, B, k_t);
    if (!ws || need == 0 || ws_bytes < need) return DS_ERR_WORKSPACE;
    cudaStream_t sd = (cudaStream_t)s_draft;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(sd, &cap);
    const unsigned evflags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (head_begin && cudaEventRecordWithFlags((cudaEvent_t)head_begin, sd, evflags) != cudaSuccess)
      return DS_ERR_CUDA;
    cudaError_t err = launch_step(c, r, h_prev, e, h_new, B, k, k_t, shared ? 1 : 0, ms, out->scores, out->sel,
                                  out->sel_count, out->sl_offsets, out->top_ids, out->top_logits, out->top_logp,
                                  out->lse, out->z_out, out->z_stride, ws, sd, head_begin == nullptr);
    if (err != cudaSuccess) return DS_ERR_CUDA;
    if (head_end && cudaEventRecordWithFlags((cudaEvent_t)head_end, sd, evflags) != cudaSuccess) return DS_ERR_CUDA;
    return DS_OK;
  }
  HeadPlan p;
  if (!head_plan(c, B, k_t, ms, &p)) return DS_ERR_UNSUPPORTED;
  HeadPlan pmax;
  if (!head_plan(c, B, k_t, 0, &pmax)) return DS_ERR_UNSUPPORTED;
  const size_t meta_bytes = meta_plan(r, B).part_bytes;
  const size_t score_bytes = (size_t)B * r->M * sizeof(float);
  const WsLayout L = ws_layout(align_up(meta_bytes, 256) + align_up(score_bytes, 256), pmax.part_bytes);
  if (!ws || ws_bytes < L.total) return DS_ERR_WORKSPACE;
  if ((tc || thr) && ws_bytes < ws_layout(align_up(meta_bytes, 256) + align_up(score_bytes, 256),
                                          tc_head_part_bytes(c, B, k_t)).total)
    return DS_ERR_WORKSPACE;
  if (gh && ws_bytes < ws_layout(align_up(meta_bytes, 256) + align_up(score_bytes, 256),
                                 gh_ws_bytes(c, B, k_t, k)).total)
    return DS_ERR_WORKSPACE;
  if (tcb && ws_bytes < ws_layout(align_up(meta_bytes, 256) + align_up(score_bytes, 256),
                                  tc_batched_ws_bytes(c, B, k_t)).total)
    return DS_ERR_WORKSPACE;  // checked before anything is enqueued
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  unsigned* counters = reinterpret_cast<unsigned*>(w8 + L.counters);
  float* meta_part = reinterpret_cast<float*>(w8 + L.meta);
  float* scores = out->scores ? out->scores : reinterpret_cast<float*>(w8 + L.meta + align_up(meta_bytes, 256));

  cudaStream_t sd = (cudaStream_t)s_draft;
  cudaStream_t sm = two_streams ? (cudaStream_t)s_meta : sd;
  if (two_streams) {  // S_m forks off S_d (its inputs h_prev, e were produced upstream on S_d)
    if (cudaEventRecord((cudaEvent_t)ev_fork, sd) != cudaSuccess) return DS_ERR_CUDA;
    if (cudaStreamWaitEvent(sm, (cudaEvent_t)ev_fork, 0) != cudaSuccess) return DS_ERR_CUDA;
  }
  const char* du = getenv("DS_DEFER_UNION");  // "0": the router forms the tree union (A/B)
  const bool defer = tc && shared && !two_streams && !(du && du[0] == '0') && th_supported(c, B, k_t) &&
                     rows_router(r, h_prev, e, B, k);
  cudaError_t err = route_rows(r, c, h_prev, e, B, scores, meta_part, counters + 1, k, shared ? 1 : 0, out->sel,
                               out->sel_count, out->sl_offsets, ws, sm, !two_streams, defer);
  if (err != cudaSuccess) return DS_ERR_CUDA;
  if (two_streams) {  // Alg. 1 line 10: "sync S_m, S_d"
    if (cudaEventRecord((cudaEvent_t)ev_join, sm) != cudaSuccess) return DS_ERR_CUDA;
    if (cudaStreamWaitEvent(sd, (cudaEvent_t)ev_join, 0) != cudaSuccess) return DS_ERR_CUDA;
  }
  // measurement events: recorded as real event nodes when the stream is being captured into a graph
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(sd, &cap);
  const unsigned evflags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (head_begin && cudaEventRecordWithFlags((cudaEvent_t)head_begin, sd, evflags) != cudaSuccess) return DS_ERR_CUDA;
  if (gh) {
    // shared (tree) mode: the union of the rows' k clusters has up to min(M, B k) clusters
    const int kmax = shared ? (int)std::min<int64_t>(c->M, (int64_t)B * k) : k;
    err = launch_gh(c, h_new, B, out->sel, out->sel_count, shared, k_t, kmax, out->top_ids, out->top_logits, out->top_logp,
                    out->lse, w8 + L.head, sd);
  } else if (tcb) {
    err = launch_tc_batched(c, h_new, B, out->sel, out->sel_count, k_t, out->top_ids, out->top_logits,
                            out->top_logp, out->lse, w8 + L.head, counters, sd);
  } else if (thr) {
    err = launch_th(c, h_new, B, out->sel, out->sel_count, out->sl_offsets, k_t, ms, out->top_ids, out->top_logits,
                    out->top_logp, out->lse, nullptr, 0, w8 + L.head, counters, sd,
                    !two_streams && head_begin == nullptr, 1);
  } else if (defer) {
    err = launch_th(c, h_new, B, out->sel, out->sel_count, out->sl_offsets, k_t, ms, out->top_ids, out->top_logits,
                    out->top_logp, out->lse, out->z_out, out->z_stride, w8 + L.head, counters, sd,
                    head_begin == nullptr, 0, ws);
  } else if (tc) {
    err = launch_tc_head(c, h_new, B, out->sel, out->sel_count, out->sl_offsets, k_t, ms, out->top_ids,
                         out->top_logits, out->top_logp, out->lse, out->z_out, out->z_stride,
                         reinterpret_cast<float*>(w8 + L.head), counters, sd, !two_streams && head_begin == nullptr);
  } else if (B == 1 && !shared && gstep_supported(c, nullptr, 1, k_t, 0) &&
             (reinterpret_cast<uintptr_t>(h_new) & 15u) == 0) {
    err = launch_gstep_head(c, h_new, out->sel, out->sel_count, out->sl_offsets, k_t, ms, out->top_ids,
                            out->top_logits, out->top_logp, out->lse, out->z_out, ws, sd);
  } else if (B == 1 && !shared && cstep_head_supported(c, k_t, ms)) {
    err = launch_cstep_head(c, h_new, out->sel, out->sel_count, out->sl_offsets, k_t, ms, out->top_ids,
                            out->top_logits, out->top_logp, out->lse, out->z_out, out->z_stride, ws, sd);
  } else {
    err = launch_head(c, p, h_new, B, out->sel, out->sel_count, out->sl_offsets, shared ? 1 : 0, k_t, ms,
                      out->top_ids, out->top_logits, out->top_logp, out->lse, out->z_out, out->z_stride,
                      reinterpret_cast<float*>(w8 + L.head), counters, sd, !two_streams && head_begin == nullptr);
  }
  if (err != cudaSuccess) return DS_ERR_CUDA;
  if (head_end && cudaEventRecordWithFlags((cudaEvent_t)head_end, sd, evflags) != cudaSuccess) return DS_ERR_CUDA;
  return DS_OK;
}

}  // extern "C"
