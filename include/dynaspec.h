/*
 * dynaspec.h — C ABI of the B200-native DynaSpec dynamic drafter LM head.
 *
 * Paper: "DynaSpec: Context-aware Dynamic Speculative Sampling for Large-Vocabulary
 * Language Models", arXiv 2510.13847.  Citations are PAPER.md line numbers (P:n) with
 * the section / equation / Algorithm-1 line they fall in; R<n> are the readings of
 * ambiguous passages listed in DESIGN.md §2.
 *
 * One draft step of Algorithm 1 for one position t is
 *   k   = k_c(t)                                   (line 7)   dynaspec_budget
 *   s   = r_theta([h_prev || e])                   (line 8)       dynaspec_meta_score
 *   K   = TopK_k(s);  I = indices(U_{m in K} C_m)  (line 8)   dynaspec_select
 *   z   = FUSED_INDEX_GEMM(h_new, W_LM, I)         (line 10)      dynaspec_head_forward
 *   p   = log_softmax(z); T, TopP = TopK_{k_t}(p); T~ = remap2realid(T)
 *                                                  (line 11)  (fused into head_forward)
 * and dynaspec_draft_step runs the whole step on two streams (S_m and S_d).
 * The clusters C_m come from dynaspec_build_clusters (offline spherical k-means).
 *
 * ------------------------------------------------------------------------------------
 * Conventions (all calls)
 *  - Tensor pointers are DEVICE pointers unless the name ends in _host.  They are owned by
 *    the caller, row-major and contiguous, and must stay alive until the enqueued work has
 *    completed on the given stream(s).  16-byte alignment is required for weights and
 *    hidden states.
 *  - Every call validates its arguments synchronously (on the host, before any launch)
 *    and returns a ds_status; on any error nothing is enqueued and no output is written.
 *    Calls only ENQUEUE work and return (except dynaspec_build_clusters, which
 *    synchronises its stream once per k-means iteration and documents it).
 *  - No call allocates device memory.  Scratch comes from a caller-provided workspace
 *    whose size is queried with the matching *_ws() function and which must be
 *    zero-filled once by dynaspec_ws_init() before its first use (the library leaves the
 *    counters it uses back at zero after each call).  One workspace must not be used by
 *    two calls that may run concurrently.
 *  - Co-residency: the draft-step and head kernels launch at most one CTA per SM and their
 *    CTAs wait on each other (the single-row steps poll published words and records; the
 *    last-CTA merges wait on a grid counter).  A concurrent kernel that keeps SMs busy delays
 *    them; the single-row step kernels bound every wait (2 s) and then raise
 *    DS_ERR_DEVICE_TIMEOUT in the workspace error word (dynaspec_ws_error) instead of hanging.
 *  - Workspace layout: the first 132 KB of every workspace are a fixed prefix (counters, the
 *    device error word, the polled-record / unit / mask words of the single-row step and
 *    few-row router kernels, written by no other kernel), so one workspace may serve any
 *    sequence of calls on one stream.
 *  - Precision: weights and activations are bf16 (DS_BF16) or fp32 (DS_F32), one dtype per
 *    call; every dot product accumulates in fp32; all floating outputs are fp32.
 *  - Determinism: no floating-point atomics; every reduction has a fixed order, so two
 *    runs with the same inputs and launch configuration produce identical bytes.
 *  - Total orders (R7, R23): clusters by (score desc, cluster id asc); tokens by
 *    (logit desc, vocabulary id asc); -0.0 and +0.0 compare equal.  NaN/Inf inputs are a
 *    precondition violation (not checked on the hot path).
 *  - CUDA errors raised while launching are returned as DS_ERR_CUDA.
 * ------------------------------------------------------------------------------------
 */
#ifndef DYNASPEC_H
#define DYNASPEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ds_stream_t; /* == cudaStream_t (NULL = legacy default stream) */
typedef struct CUevent_st* ds_event_t;   /* == cudaEvent_t */

typedef enum {
  DS_OK = 0,
  DS_ERR_SHAPE = 1,                 /* inconsistent d / M / V / B / h_r, or a required pointer is NULL */
  DS_ERR_DTYPE = 2,                 /* dtype not DS_BF16 / DS_F32, or mixed dtypes */
  DS_ERR_INVALID_BUDGET = 3,        /* k < 1, k > M, k_min > k_max, k_t < 1 or k_t > 64 (SPEC InvalidBudget) */
  DS_ERR_INVALID_CLUSTER_COUNT = 4, /* M < 1, M > V or M > 1024 (SPEC InvalidClusterCount) */
  DS_ERR_INVALID_CLUSTER_ID = 5,    /* a cluster id outside [0, M) (SPEC InvalidClusterId) */
  DS_ERR_INVALID_TOKEN = 6,         /* a token id outside [0, V) (SPEC InvalidToken) */
  DS_ERR_DEGENERATE_COLUMN = 7,     /* a zero-norm token vector in build_clusters (SPEC DegenerateColumn) */
  DS_ERR_EMPTY_SHORTLIST = 8,       /* a cluster would be empty (SPEC EmptyShortlist) */
  DS_ERR_WORKSPACE = 9,             /* workspace NULL or smaller than the *_ws() size */
  DS_ERR_CUDA = 10,                 /* a CUDA runtime error while launching */
  DS_ERR_UNSUPPORTED = 11,          /* shape outside what the kernels support (e.g. d % 8 != 0) */
  DS_ERR_DEVICE_TIMEOUT = 12        /* (device error word) a CTA of a single-row step kernel waited > 2 s for
                                       another CTA of its grid: SMs held by a concurrent kernel; outputs invalid */
} ds_status;

typedef enum { DS_BF16 = 0, DS_F32 = 1 } ds_dtype;

/* Vocabulary partition Pi = {C_1..C_M}, tau: V -> [M], in the cluster-permuted
 * layout: cluster m occupies rows [offsets[m], offsets[m+1]) of W_perm, tokens ascending
 * inside a cluster; perm[i] is the vocabulary id of row i of W_perm (remap2realid).
 * Filled by dynaspec_build_clusters or dynaspec_layout. */
typedef struct {
  int64_t V;               /* vocabulary size |V| */
  int32_t d;               /* hidden size */
  int32_t M;               /* number of clusters, 1 <= M <= min(V, 1024) */
  int32_t dtype;           /* ds_dtype of W_perm */
  int32_t min_size;        /* HOST: smallest |C_m| (>= 1) */
  int32_t max_size;        /* HOST: largest |C_m| */
  const int32_t* tau;      /* device [V]   cluster of each token (may be NULL on the hot path) */
  const int32_t* perm;     /* device [V]   W_perm row -> vocabulary id */
  const int32_t* offsets;  /* device [M+1] exclusive scan of cluster sizes */
  const void* W_perm;      /* device [V][d] LM-head rows (W_LM columns) in cluster order */
} ds_clusters;

/* Router r_theta: R^{2d} -> R^M, input x = [h_prev || e] (R4).
 * h_r > 0: s = W2 * ReLU(W1 x + b1) + b2, W1 [h_r][2d], b1 [h_r], W2 [M][h_r], b2 [M]  (R5).
 * h_r == 0: linear router s = W1 x + b1 with W1 [M][2d], b1 [M]; W2, b2 unused.
 * Biases are fp32; W1/W2 have the router dtype.  Scores are pre-sigmoid logits (R6). */
typedef struct {
  int32_t d;
  int32_t h_r;
  int32_t M;
  int32_t dtype;
  const void* W1;
  const float* b1;
  const void* W2;
  const float* b2;
} ds_router;

/* Outputs of one draft step (all device pointers).  B_sel = 1 in shared mode, else B. */
typedef struct {
  float* scores;       /* [B][M]       router scores s (may be NULL: then the workspace holds them) */
  int32_t* sel;        /* [B_sel][M]   selected cluster ids, ascending, first sel_count[r] valid */
  int32_t* sel_count;  /* [B_sel]      |K| */
  int32_t* sl_offsets; /* [B_sel][M+1] exclusive scan of |C_m| over sel; |V_S| = sl_offsets[r][sel_count[r]] */
  int32_t* top_ids;    /* [B][k_t]     vocabulary ids of TopK_{k_t}, (logit desc, id asc); -1 padding */
  float* top_logits;   /* [B][k_t]     z at those ids; -inf padding */
  float* top_logp;     /* [B][k_t]     log_softmax(z) at those ids = z - lse; -inf padding */
  float* lse;          /* [B]          log sum_{v in V_S} exp(z_v) */
  float* z_out;        /* nullable [B][z_stride]: z over V_S in shortlist order (tau(v), v) (R8) */
  int64_t z_stride;    /* >= dynaspec_max_shortlist(c, k) when z_out != NULL */
} ds_step_outputs;

/* ---------------------------------------------------------------- helpers (host only) */

const char* dynaspec_status_string(ds_status s);

/* k_c(t) = k_max for t in {0,1}, floor(k_max / ((t+1)*2)) for t >= 2 (Alg. 1
 * line 7, with i read as the step index, R2), clamped below by k_min (R1).
 * Returns -1 if t < 0, k_min < 1 or k_max < k_min. */
int32_t dynaspec_budget(int32_t t, int32_t k_max, int32_t k_min);

/* PA-FR position-aware frequency budget (App. A.1): K_fr(t) = K_max for t in {0,1},
 * floor(K_max / (t + 1)) for t >= 2, clamped below by 1 (reading R26).  Returns -1 if t < 0 or
 * K_max < 1. */
int32_t dynaspec_pa_fr_budget(int32_t t, int32_t K_max);

/* Upper bound on |V_S| for k selected clusters of one row: min(V, k * max_size). */
int64_t dynaspec_max_shortlist(const ds_clusters* c, int32_t k);

/* Zero-fill a workspace (once, before its first use). */
ds_status dynaspec_ws_init(void* ws, size_t ws_bytes, ds_stream_t stream);

/* Data-dependent device errors raised after a call returned are written to the workspace's error
 * word (today: DS_ERR_DEVICE_TIMEOUT from a bounded inter-CTA wait).  Copies it to *code_host
 * (DS_OK if none) and clears it.  SYNCHRONISES `stream`. */
ds_status dynaspec_ws_error(void* ws, size_t ws_bytes, int32_t* code_host, ds_stream_t stream);

/* ---------------------------------------------------------------- S0: offline partition */

/* Workspace bytes for dynaspec_build_clusters. */
size_t dynaspec_build_clusters_ws(int64_t V, int32_t d, int32_t M);

/* Spherical k-means on column-normalised W_LM columns, no balance constraint,
 * in the integer-exact reading R12: u_v = rint(2^14 w_v/||w_v||) with the
 * norm a sequential fp64 sum; Forgy init from splitmix64(seed) (or init_ids_host);
 * assignment argmax_m <u_v, c_m> in exact integers (ties -> lower m); centroids
 * rint(2^14 S_m/||S_m||); empty clusters reseeded in ascending m with the lowest-similarity
 * token of a cluster of size > 1; stop when tau repeats or after max_iters assignment
 * passes; clusters relabelled by their smallest token id; then the layout of ds_clusters.
 *   W        device [V][d] (dtype)                  input LM-head rows (W_LM columns)
 *   init_ids_host  NULL or host [M] distinct token ids (replaces the Forgy draw)
 *   tau      device [V] out;  perm device [V] out;  offsets device [M+1] out
 *   W_perm   device [V][d] out (dtype), W_perm[i] = W[perm[i]]  (a drafter-side copy, R21)
 *   iters_run_host   host out: assignment passes run;  sizes_host: host [2] out (min, max |C_m|), nullable
 * SYNCHRONISES `stream` once per iteration (one 4-byte D->H copy).  Errors:
 * DS_ERR_INVALID_CLUSTER_COUNT, DS_ERR_DEGENERATE_COLUMN, DS_ERR_SHAPE, DS_ERR_WORKSPACE. */
ds_status dynaspec_build_clusters(const void* W, int32_t dtype, int64_t V, int32_t d, int32_t M,
                                  uint64_t seed, int32_t max_iters, const int32_t* init_ids_host,
                                  int32_t* tau, int32_t* perm, int32_t* offsets, void* W_perm,
                                  int32_t* iters_run_host, int32_t* sizes_host,
                                  void* ws, size_t ws_bytes, ds_stream_t stream);

/* Layout from a given partition tau (device [V], values in [0,M), every cluster non-empty):
 * perm = stable sort of token ids by tau, offsets = exclusive scan of sizes, W_perm[i] =
 * W[perm[i]] (R12 step 9).  SYNCHRONISES `stream` once (to validate and to return sizes).
 * Errors: DS_ERR_INVALID_CLUSTER_ID (tau out of range), DS_ERR_EMPTY_SHORTLIST (empty cluster). */
size_t dynaspec_layout_ws(int64_t V, int32_t M);
ds_status dynaspec_layout(const int32_t* tau, const void* W, int32_t dtype, int64_t V, int32_t d, int32_t M,
                          int32_t* perm, int32_t* offsets, void* W_perm, int32_t* sizes_host,
                          void* ws, size_t ws_bytes, ds_stream_t stream);

/* ---------------------------------------------------------------- S1: meta-classifier */

/* Workspace bytes for dynaspec_meta_score with B rows. */
size_t dynaspec_meta_score_ws(const ds_router* r, int32_t B);

/* s = r_theta([h_prev || e]) for B independent rows (Alg. 1 line 3 / line 8).
 *   h_prev  device [B][d]  drafter hidden of the previous position (h_{c[-1]} at j = 0, R11)
 *   e       device [B][d]  embedding E(x_t) of the current input token (R10)
 *   scores  device [B][M]  out, fp32 */
ds_status dynaspec_meta_score(const ds_router* r, const void* h_prev, const void* e, int32_t B,
                              float* scores, void* ws, size_t ws_bytes, ds_stream_t stream);

/* ---------------------------------------------------------------- S3/S4: selection */

/* K_r = TopK_k(s_r) under (score desc, id asc), emitted in ascending id (R7, R8),
 * and sl_offsets_r = exclusive scan of |C_m| over K_r (|V_S| = sum |C_m|).
 * shared = 0: one selection per row (independent requests).  shared = 1: ONE output row, the
 * ascending union over the B rows of their TopK sets (tree depth, one I for all rows, R9).
 * k_per_row: nullable device [B] per-row budgets (each in [1, M]); else every row uses k.
 *   scores device [B][M]; sel device [B_sel][M] out; sel_count device [B_sel] out;
 *   sl_offsets device [B_sel][M+1] out.  Errors: DS_ERR_INVALID_BUDGET. */
ds_status dynaspec_select(const float* scores, int32_t B, const ds_clusters* c, int32_t k,
                          const int32_t* k_per_row, int32_t shared, int32_t* sel, int32_t* sel_count,
                          int32_t* sl_offsets, ds_stream_t stream);

/* ---------------------------------------------------------------- S5/S6: head + epilogue */

/* Workspace bytes for dynaspec_head_forward with B rows and token budget k_t. */
size_t dynaspec_head_forward_ws(const ds_clusters* c, int32_t B, int32_t k_t);

/* z_r[j] = <h_new_r, W_LM[:, V_S,r[j]]> over the shortlist only (Alg. 1 line 10),
 * fp32 accumulation, then log_softmax over V_S (R14), TopK_{k_t} by (z desc, id asc) and
 * remap2realid through perm (line 11) — one fused pass.
 *   h_new        device [B][d]          head input (as-is, no norm/bias/temperature, R22)
 *   sel, sel_count, sl_offsets          as produced by dynaspec_select (shared: one row)
 *   max_shortlist  upper bound on every row's |V_S| (0 => V); sizes the on-chip buffers
 *   outputs      as in ds_step_outputs (top_*: [B][k_t]; lse: [B]; z_out nullable)
 * Rows whose |V_S| < k_t get -1 / -inf padding.  A row whose |V_S| exceeds max_shortlist
 * is not computed: its top_ids are -1 and lse is NaN.  Errors: DS_ERR_INVALID_BUDGET
 * (k_t < 1 or > 64), DS_ERR_SHAPE, DS_ERR_WORKSPACE, DS_ERR_UNSUPPORTED (d % 8 != 0). */
ds_status dynaspec_head_forward(const ds_clusters* c, const void* h_new, int32_t B, const int32_t* sel,
                                const int32_t* sel_count, const int32_t* sl_offsets, int32_t shared,
                                int32_t k_t, int64_t max_shortlist, int32_t* top_ids, float* top_logits,
                                float* top_logp, float* lse, float* z_out, int64_t z_stride,
                                void* ws, size_t ws_bytes, ds_stream_t stream);

/* ---------------------------------------------------------------- S7: one draft step */

/* Workspace bytes for dynaspec_draft_step. */
size_t dynaspec_draft_step_ws(const ds_clusters* c, const ds_router* r, int32_t B, int32_t k_t);

/* One DynaSpec draft position t (Alg. 1 lines 7-11):
 *   host:   k = dynaspec_budget(t, k_max, k_min)                     (line 7)
 *   s_meta: meta_score(h_prev, e) -> select(k)                       (line 8, stream S_m)
 *   s_draft: [caller's drafter core already enqueued]                (line 9, stream S_d)
 *            wait(meta) -> head_forward(h_new)                       (lines 10-11, after "sync S_m,S_d")
 * ev_fork / ev_join: caller-owned events used to fork s_meta off s_draft and join it back
 * (both required when s_meta != s_draft; ignored otherwise).  head_begin / head_end:
 * nullable events recorded on s_draft around the head kernel (for measurement).
 * On return all work is enqueued; the outputs are complete when s_draft reaches this point.
 * Errors: as the individual calls, plus DS_ERR_INVALID_BUDGET if k_t > k * min_size. */
ds_status dynaspec_draft_step(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e,
                              const void* h_new, int32_t B, int32_t t, int32_t k_max, int32_t k_min,
                              int32_t k_t, int32_t shared, const ds_step_outputs* out,
                              void* ws, size_t ws_bytes, ds_stream_t s_draft, ds_stream_t s_meta,
                              ds_event_t ev_fork, ds_event_t ev_join, ds_event_t head_begin,
                              ds_event_t head_end);

/* The two halves of a draft step, for callers that overlap the router with their drafter core
 * (Alg. 1 lines 8-10: "the router runs on a separate parallel CUDA stream and completes
 * while the drafter's attention/MLP is executing"):
 *   caller: record an event on S_d; make s_meta wait on it; dynaspec_step_route(.., s_meta);
 *           enqueue the drafter core on S_d (producing h_new); record an event on s_meta and make
 *           S_d wait on it ("sync S_m, S_d"); dynaspec_step_head(.., S_d).
 * route: router + TopK + sl_offsets into out->scores / sel / sel_count / sl_offsets (2 launches).
 * head:  the gathered head + epilogue over that selection into out->top_* / lse / z_out.
 * Workspaces: route needs dynaspec_draft_step_ws bytes of its own; head needs its own workspace
 * of dynaspec_head_forward_ws bytes (the two may run concurrently, so they must not share). */
ds_status dynaspec_step_route(const ds_clusters* c, const ds_router* r, const void* h_prev, const void* e, int32_t B,
                              int32_t t, int32_t k_max, int32_t k_min, int32_t shared, const ds_step_outputs* out,
                              void* ws, size_t ws_bytes, ds_stream_t s_meta);
ds_status dynaspec_step_head(const ds_clusters* c, const void* h_new, int32_t B, int32_t t, int32_t k_max,
                             int32_t k_min, int32_t k_t, int32_t shared, const ds_step_outputs* out, void* ws,
                             size_t ws_bytes, ds_stream_t s_draft);

/* Number of kernel launches one dynaspec_draft_step enqueues (for launch accounting):
 * 1 for the fused single-stream step, 2 + head chunks for the two-stream path, 5 for the grouped
 * tcgen05 head (router x2, grouping, head, merge).  z_out: whether the call passes out->z_out. */
int32_t dynaspec_draft_step_launches(const ds_clusters* c, const ds_router* r, int32_t B, int32_t k_t,
                                     int32_t shared, int32_t two_streams, int32_t z_out);

/* Name of the dominant kernel one dynaspec_draft_step runs for this shape (for measurement
 * bookkeeping: the kernel a roofline is quoted on).  Static string, never NULL ("?" on bad
 * arguments).  Assumes 16-byte aligned inputs (the unaligned fallbacks are not named). */
const char* dynaspec_draft_step_kernel(const ds_clusters* c, const ds_router* r, int32_t B, int32_t k_t,
                                       int32_t shared, int32_t two_streams, int32_t z_out);

/* ---------------------------------------------------------------- draft tree (Alg. 1 lines 12-18) */

/* One step of the draft-tree bookkeeping for R current beams (R = 1 at j = 0):
 *   cu[b][q] = top_logp[b][q] + last_scores[b]                       (line 12; last_scores NULL => 0)
 *   node arrays at [node_base, node_base + R k_t): token, cu, parent node (last_nodes[b], or -1
 *   when NULL), step                                                  (line 13: d, d_scores)
 *   next_* [k_t]: the k_t best expansions by (cu desc, flat index b k_t + q asc) (R24): token
 *   (x_j, line 15), score (last_step_scores, line 14), node index, parent beam b (h_j, line 16).
 * top_ids / top_logp are the head outputs [R][k_t] (-1 / -inf padding is skipped; next_* are padded
 * with -1 / -inf).  R <= 64, k_t <= 64.  One CTA; all device pointers. */
ds_status dynaspec_tree_step(const int32_t* top_ids, const float* top_logp, int32_t R, int32_t k_t,
                             const float* last_scores, const int32_t* last_nodes, int32_t step, int32_t node_base,
                             int32_t* node_tok, float* node_score, int32_t* node_parent, int32_t* node_step,
                             int32_t* next_tok, float* next_score, int32_t* next_node, int32_t* next_beam,
                             ds_stream_t stream);

/* Re-rank the draft list d by d_scores (line 18): out_nodes[0..n_out) = the node indices of
 * the n_out best valid nodes by (score desc, node index asc) (R24), -1 padded.  n_nodes <= 16384. */
ds_status dynaspec_tree_rerank(const float* node_score, const int32_t* node_tok, int32_t n_nodes, int32_t n_out,
                               int32_t* out_nodes, ds_stream_t stream);

/* ---------------------------------------------------------------- cluster sharding (multi-GPU) */

/* Keep, for each of `rows` selection rows, only the selected clusters in [m_lo, m_hi) (the
 * cluster range a rank owns), preserving ascending order, and rebuild sl_offsets over them.
 * Same layouts as dynaspec_select.  Errors: DS_ERR_INVALID_CLUSTER_ID for a bad range. */
ds_status dynaspec_restrict_selection(const int32_t* sel, const int32_t* sel_count, const int32_t* sl_offsets,
                                      int32_t rows, const ds_clusters* c, int32_t m_lo, int32_t m_hi, int32_t* out_sel,
                                      int32_t* out_count, int32_t* out_sl_offsets, ds_stream_t stream);

/* As dynaspec_head_forward (same workspace size), but instead of the final outputs emit one
 * record per row: records[r] = {max z, sum exp(z - max), (z, id) of the top-k_t by (z desc,
 * id asc), padded with (-inf, INT_MAX)} as 2 + 2 k_t floats (ids bit-cast).  A rank holding
 * only rows [offsets[m_lo], offsets[m_hi]) of W_perm passes a ds_clusters whose W_perm points
 * offsets[m_lo] rows before its slice and a selection restricted to [m_lo, m_hi). */
ds_status dynaspec_head_partial(const ds_clusters* c, const void* h_new, int32_t B, const int32_t* sel,
                                const int32_t* sel_count, const int32_t* sl_offsets, int32_t shared, int32_t k_t,
                                int64_t max_shortlist, float* records, void* ws, size_t ws_bytes, ds_stream_t stream);

/* Merge G per-rank records (device [G][B][2 + 2 k_t], rank-major as an all-gather produces them)
 * in rank order into lse / top_ids / top_logits / top_logp exactly as dynaspec_head_forward
 * defines them (softmax over the union of the ranks' shortlists).  G <= 64. */
ds_status dynaspec_merge_records(const float* records, int32_t G, int32_t B, int32_t k_t, int32_t* top_ids,
                                 float* top_logits, float* top_logp, float* lse, ds_stream_t stream);

/* ---------------------------------------------------------------- static frequency heads (NEXT-3) */

/* Row gather out[i] = W[ids[i]] for i < n (W [V][d] of dtype, out [n][d]; device pointers): the
 * frequency-ordered copy of W_LM that FR-Spec / PA-FR heads stream as one contiguous prefix
 * (App. A.1; ids = pi_f, tokens by descending corpus count, R26).  Errors: DS_ERR_SHAPE,
 * DS_ERR_DTYPE, DS_ERR_UNSUPPORTED (d * sizeof(dtype) not a multiple of 16).  The ids are not
 * range-checked on the device (an id outside [0, V) is a precondition violation). */
ds_status dynaspec_gather_rows(const void* W, int32_t dtype, int64_t V, int32_t d, const int32_t* ids, int64_t n,
                               void* out, ds_stream_t stream);

/* ---------------------------------------------------------------- lossless verification (NEXT-4) */

/* Materialise the shortlist V_S as vocabulary ids in shortlist order (S4): for each of `rows`
 * selection rows (B per-row, or 1 for a shared selection), ids[r][sl_offsets[r][i] + u] =
 * perm[offsets[sel[r][i]] + u] for u < |C_{sel[r][i]}|.  `stride` (int32 elements between rows) must
 * be >= the row's shortlist length.  This is the id list that pairs with z_out of the head. */
ds_status dynaspec_shortlist_ids(const ds_clusters* c, int32_t rows, const int32_t* sel, const int32_t* sel_count,
                                 const int32_t* sl_offsets, int64_t stride, int32_t* ids, ds_stream_t stream);

/* Workspace bytes of dynaspec_verify_chain.  The workspace must be zeroed once (dynaspec_ws_init)
 * before its first use; every call leaves it zeroed again (it holds a dense [B][V] q buffer). */
size_t dynaspec_verify_ws(int64_t V, int32_t B, int32_t gamma);

/* Speculative-sampling verification of B drafted chains (Eq. 3, via the rule its footnote
 * cites; reading R25 in DESIGN.md).  All pointers are device memory.
 *   p_logits [B][gamma+1][V] (dtype DS_BF16 / DS_F32): the target's logits at the gamma+1 positions.
 *   q_ids / q_logits [B][gamma][q_stride]: drafter shortlist ids and logits z (the head's z_out and
 *     dynaspec_shortlist_ids), q_count [B][gamma] valid entries, q_lse [B][gamma] the head's lse:
 *     q_i(v) = exp(z - lse) on the shortlist, 0 off it.
 *   x / x_slot [B][gamma]: drafted tokens and their slot in the shortlist (q_ids[..][slot] == x).
 *   u_acc [B][gamma], u_res [B]: uniforms in [0, 1) (the caller's random numbers).
 * Position i is accepted iff u_acc < p_i(x_i) / q_i(x_i); at the first rejection j the corrective token
 * is the first v (id order) whose cumulative (p_j - q_j)_+ exceeds u_res * sum; with no rejection the
 * bonus token is drawn the same way from p_gamma (R25).  Outputs: accepted[b] = j and committed[b][0..j]
 * (accepted tokens, then the corrective / bonus token); accepted[b] = -1 and committed[b][0] = -1 when
 * the first non-accepted position has x_slot / x inconsistent with q_ids (InvalidProposal).
 * Limits: gamma in [0, 32], V a multiple of 8 (16-byte rows).  Two launches on `stream`. */
ds_status dynaspec_verify_chain(const void* p_logits, int32_t dtype, int64_t V, int32_t B, int32_t gamma,
                                const int32_t* q_ids, const float* q_logits, int64_t q_stride, const int32_t* q_count,
                                const float* q_lse, const int32_t* x, const int32_t* x_slot, const float* u_acc,
                                const float* u_res, int32_t* accepted, int32_t* committed, void* ws, size_t ws_bytes,
                                ds_stream_t stream);

/* Debugging: when dev_buf != NULL, the fused step kernel records %globaltimer nanosecond
 * timestamps of its phases into dev_buf[cta * 64 + slot] and the SM clock64() into
 * dev_buf[cta * 64 + 32 + slot] (uint64, >= #SM * 64 entries):
 * 0 start, 1 after PDL wait, 2 router layer 1 done, 3 selection visible, 4 segments ready,
 * 5 head streamed, 6 partials written, 7 merge done (last CTA), 8..13 selection phases,
 * 14 ticket won, 16..20 merge phases.
 * Pass NULL to disable (the default).  Not for concurrent use from several threads. */
ds_status dynaspec_debug_set_trace(void* dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* DYNASPEC_H */
