"""DynaSpec dynamic drafter LM head — CPU ORACLE (test infrastructure only).

THIS IS TEST INFRASTRUCTURE.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The product
path (`paper_2510_13847_b200/`, `include/`, the CUDA library) never imports, links
or calls anything here, and this file shares no code with it.

What it computes is the plain definition of the method (arXiv 2510.13847, PAPER.md,
cited as P:<line>), written in fp64 / int64 with numpy, with no blocking, fusion or
reordering beyond what the definition states.  Where the paper is silent the
readings R1..R23 of SURVEY.md §8(c) are taken (listed in DESIGN.md §2).

Steps:
  O0 budget            k_c(t)                                   P:201-211 (§4.2), R1/R2
  O1 build_clusters    spherical k-means, integer-exact reading P:193-196 (§4.2), R12
  O2 meta_score        s = r_theta([h_prev || e])               P:198-199 (§4.2), R4/R5/R6
  O3 select            K = TopK_k(s), ascending ids             P:212-213 (§4.2), R7/R8
  O4 shortlist         V_S = U_{m in K} C_m in (tau(v), v) order P:214 (§4.2), R8/R9
  O5 head              z = <h_new, W[v]> for v in V_S           P:262 (Alg. 1 line 10)
  O6 epilogue          log_softmax, TopK_{k_t}, remap2realid    P:263-264 (Alg. 1 line 11), R14/R7
  O7 dense             full-vocabulary head p = softmax(H W_LM)  P:182 (§4.1)
  NEXT-1 tree_step / tree_rerank   beam bookkeeping + re-rank    P:265-271 (Alg. 1 lines 12-18), R24
  NEXT-3 frequency_ranking, fr_head  FR-Spec / PA-FR prefix heads P:184-192, App. A.1
  NEXT-4 verify_chain      lossless acceptance + residual sampling  Eq. 3, R25

Pins: tests/test_oracle_*.py (golden values from SPEC/the worked example E2E-1,
closed forms, brute force on tiny inputs, invariants).  Every function below is
pinned; see DESIGN.md §4 for the pin of each.
"""
from __future__ import annotations

import math

import numpy as np

Q_SCALE = 16384.0  # 2^14: quantisation scale of unit vectors (R12)
MASK64 = (1 << 64) - 1


class OracleError(ValueError):
    """Error vocabulary of SPEC used by the oracle."""


# ---------------------------------------------------------------------------
# O0  position-aware budget   (Alg. 1 line 7; reading R1, R2)
# ---------------------------------------------------------------------------


def budget(t: int, k_max: int, k_min: int = 1) -> int:
    """k_c(t) = k_max for t in {0,1}; floor(k_max / ((t+1)*2)) for t >= 2,
    clamped below by k_min (the paper's range {k_min..k_max}; R1)."""
    if t < 0 or k_min < 1 or k_max < k_min:
        raise OracleError("InvalidBudget")
    if t in (0, 1):
        return k_max
    return max(k_min, k_max // ((t + 1) * 2))


def budget_pa_fr(t: int, k_max: int) -> int:
    """PA-FR K_fr(t) (App. A.1): k_max for t in {0,1}, floor(k_max/(t+1)) after, >= 1."""
    if t in (0, 1):
        return k_max
    return max(1, k_max // (t + 1))


# ---------------------------------------------------------------------------
# O1  offline vocabulary partition by spherical k-means   (reading R12)
# ---------------------------------------------------------------------------


def normalize_quantize(W: np.ndarray) -> np.ndarray:
    """Column-normalised LM-head weights W_LM[:,v]/||W_LM[:,v]||_2, quantised.

    W is [V][d] (row v = token v's column of W_LM).  For each v:
      n_v = sqrt(sum_i w_vi^2), the sum taken sequentially in i in fp64 (w^2 is exact in
      fp64 for bf16/fp32 inputs), then u_vi = rint(2^14 * w_vi / n_v) (round half to even).
    A zero-norm column is SPEC's DegenerateColumn.
    """
    W = np.asarray(W, dtype=np.float64)
    V, d = W.shape
    U = np.empty((V, d), dtype=np.int64)
    step = max(1, (1 << 24) // max(d, 1))
    for a in range(0, V, step):
        blk = W[a:a + step]
        n2 = np.cumsum(blk * blk, axis=1)[:, -1]          # sequential left-to-right sum
        n = np.sqrt(n2)
        if np.any(n == 0.0):
            raise OracleError("DegenerateColumn")
        U[a:a + step] = np.rint(blk / n[:, None] * Q_SCALE).astype(np.int64)
    return U


def splitmix64_stream(seed: int):
    """splitmix64 (Steele, Lea, Flood 2014): the counter-based generator both sides implement."""
    state = seed & MASK64
    while True:
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def forgy_init(V: int, M: int, seed: int) -> np.ndarray:
    """Forgy initialisation (R12 step 2): M distinct token ids from a partial Fisher-Yates
    shuffle of [0, V) driven by splitmix64(seed): for i < M, j = i + r_i mod (V - i), swap."""
    a = list(range(V))
    rnd = splitmix64_stream(seed)
    for i in range(M):
        j = i + next(rnd) % (V - i)
        a[i], a[j] = a[j], a[i]
    return np.array(a[:M], dtype=np.int64)


def centroid_from_sum(S: np.ndarray) -> np.ndarray:
    """c_m = rint(2^14 * S_m / ||S_m||) (R12 step 4): ||S_m||^2 is the sequential fp64 sum of
    the fp64 products S_mi*S_mi, each rounded separately (no fused multiply-add)."""
    Sf = S.astype(np.float64)                    # exact: |S_mi| <= V * 2^14 < 2^53
    sq = Sf * Sf                                 # one rounding per product
    n = math.sqrt(float(np.cumsum(sq)[-1]))      # sequential sum, then IEEE sqrt
    return np.rint(Sf / n * Q_SCALE).astype(np.int64)


def _dots(U: np.ndarray, C: np.ndarray) -> np.ndarray:
    """All <u_v, c_m> as int64.  Computed with an fp64 matmul, which is EXACT here: every
    partial sum is bounded by sum_i |u_vi c_mi| <= ||u|| ||c|| < (2^14 + sqrt(d)/2)^2 < 2^31
    (Cauchy-Schwarz), far below 2^53, so any summation order gives the integer result."""
    return (U.astype(np.float64) @ C.astype(np.float64).T).astype(np.int64)


def spherical_kmeans(W: np.ndarray, M: int, seed: int = 2, max_iters: int = 20,
                     init_ids=None, U: np.ndarray | None = None):
    """Spherical k-means on column-normalised W_LM columns, no balance constraint.

    Integer-exact reading R12, in this order per iteration:
      1. assign every token: tau(v) = argmax_m <u_v, c_m> (ties -> lower m);
      2. stop if tau equals the previous iteration's final tau;
      3. recompute c_m = rint(2^14 S_m/||S_m||), S_m = sum_{tau(v)=m} u_v, for non-empty m;
      4. reseed empty clusters in ascending m: the token with the lowest <u_v, c_tau(v)>
         (updated centroids; ties -> lower v) among tokens whose cluster has > 1 member
         moves to m and c_m = u_v.
    max_iters counts assignment passes.  Returns (tau int64[V], iterations run).
    """
    if U is None:
        U = normalize_quantize(W)
    V = U.shape[0]
    if not (1 <= M <= V):
        raise OracleError("InvalidClusterCount")
    ids = forgy_init(V, M, seed) if init_ids is None else np.asarray(init_ids, dtype=np.int64)
    C = U[ids].copy()
    tau_prev = None
    tau = None
    it = 0
    for it in range(1, max_iters + 1):
        tau = np.argmax(_dots(U, C), axis=1).astype(np.int64)   # argmax returns the lowest m on ties
        if tau_prev is not None and np.array_equal(tau, tau_prev):
            break
        sizes = np.bincount(tau, minlength=M)
        for m in range(M):
            if sizes[m] > 0:
                C[m] = centroid_from_sum(U[tau == m].sum(axis=0))
        if np.any(sizes == 0):
            sims = np.einsum("vd,vd->v", U.astype(np.float64), C[tau].astype(np.float64)).astype(np.int64)
            for m in range(M):
                if sizes[m] != 0:
                    continue
                cand = np.nonzero(sizes[tau] > 1)[0]
                v = int(cand[np.argmin(sims[cand])])          # argmin: lowest v among ties
                sizes[tau[v]] -= 1
                tau[v] = m
                sizes[m] = 1
                C[m] = U[v]
        tau_prev = tau.copy()
    return tau, it


def canonical_relabel(tau: np.ndarray, M: int) -> np.ndarray:
    """Relabel clusters by their minimum token id (R12 step 8): the cluster holding the
    smallest token id becomes 0, and so on."""
    tau = np.asarray(tau, dtype=np.int64)
    first = np.full(M, np.iinfo(np.int64).max)
    np.minimum.at(first, tau, np.arange(tau.size))
    if np.any(first == np.iinfo(np.int64).max):
        raise OracleError("EmptyCluster")
    new_label = np.empty(M, dtype=np.int64)
    new_label[np.argsort(first, kind="stable")] = np.arange(M)
    return new_label[tau]


def layout(tau: np.ndarray, M: int):
    """Cluster-permuted layout (R12 step 9): perm = stable sort of v by tau(v) (so cluster m
    occupies rows [offsets[m], offsets[m+1]) of W_perm, tokens ascending inside), offsets =
    exclusive scan of cluster sizes.  perm is remap2realid (Alg. 1 line 11)."""
    tau = np.asarray(tau, dtype=np.int64)
    perm = np.argsort(tau, kind="stable").astype(np.int64)
    offsets = np.zeros(M + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(np.bincount(tau, minlength=M))
    return perm, offsets


def build_clusters(W, M, seed=2, max_iters=20, init_ids=None):
    """O1: k-means -> canonical relabel -> layout.  Returns dict(tau, perm, offsets, iters)."""
    tau, iters = spherical_kmeans(W, M, seed, max_iters, init_ids)
    tau = canonical_relabel(tau, M)
    perm, offsets = layout(tau, M)
    return {"tau": tau, "perm": perm, "offsets": offsets, "iters": iters}


def kmeans_objective(U: np.ndarray, tau: np.ndarray, M: int) -> float:
    """Spherical k-means objective of a partition with optimal (mean-direction) centroids:
    sum_m ||sum_{v in C_m} u_v|| / 2^14  (= sum_v cos(u_v, c_tau(v)))."""
    tot = 0.0
    for m in range(M):
        mem = U[tau == m]
        if len(mem):
            tot += float(np.linalg.norm(mem.sum(axis=0).astype(np.float64)))
    return tot / Q_SCALE


# ---------------------------------------------------------------------------
# O2  meta-classifier (router)   (§4.2; Alg. 1 lines 3 and 8)
# ---------------------------------------------------------------------------


def meta_score(W1, b1, W2, b2, h_prev, e):
    """s = r_theta([h_prev || e]) over M clusters, input order per R4.

    Two-layer MLP (R5): a = max(0, W1 x + b1), s = W2 a + b2; W2 None => linear router
    s = W1 x + b1.  Rows of h_prev/e are independent rows.  fp64 throughout; scores are
    pre-sigmoid logits (R6)."""
    x = np.concatenate([np.atleast_2d(h_prev), np.atleast_2d(e)], axis=1).astype(np.float64)
    a = x @ np.asarray(W1, np.float64).T + np.asarray(b1, np.float64)
    if W2 is None:
        return a
    a = np.maximum(a, 0.0)
    return a @ np.asarray(W2, np.float64).T + np.asarray(b2, np.float64)


# ---------------------------------------------------------------------------
# O3/O4  selection and shortlist   (Alg. 1 line 8)
# ---------------------------------------------------------------------------


def top_k_order(values, k, tiebreak=None):
    """Indices of the k largest values, ordered (value desc, tiebreak asc) (R7).
    tiebreak defaults to the index itself.  -0.0 and +0.0 compare equal (R23)."""
    values = np.asarray(values, dtype=np.float64) + 0.0
    n = values.size
    if not (1 <= k <= n):
        raise OracleError("InvalidBudget")
    tb = np.arange(n) if tiebreak is None else np.asarray(tiebreak)
    order = np.lexsort((tb, -values))
    return order[:k]


def select(scores_row, k):
    """K = TopK_k(s), emitted in ascending cluster id (R8)."""
    return np.sort(top_k_order(scores_row, k)).astype(np.int64)


def select_shared(scores, k):
    """Shared (tree) mode (R9): ascending union over the rows of one depth of each row's TopK_k."""
    sel = set()
    for r in range(scores.shape[0]):
        sel.update(int(m) for m in top_k_order(scores[r], k))
    return np.array(sorted(sel), dtype=np.int64)


def shortlist_offsets(sel, offsets):
    """sl_offsets: exclusive scan of |C_m| over the selected ids in ascending order."""
    sizes = np.array([offsets[m + 1] - offsets[m] for m in sel], dtype=np.int64)
    out = np.zeros(len(sel) + 1, dtype=np.int64)
    out[1:] = np.cumsum(sizes)
    return out


def shortlist(sel, perm, offsets):
    """V_S = U_{m in K} C_m, in (tau(v), v) order = concatenated perm blocks (R8)."""
    if len(sel) == 0:
        raise OracleError("EmptyShortlist")
    return np.concatenate([perm[offsets[m]:offsets[m + 1]] for m in sel]).astype(np.int64)


def cluster_union_sorted(sel, tau):
    """SPEC cluster_union: sorted token ids whose cluster is selected."""
    return np.nonzero(np.isin(tau, np.asarray(sel)))[0]


# ---------------------------------------------------------------------------
# O5/O6  gathered head and epilogue   (Alg. 1 lines 10-11)
# ---------------------------------------------------------------------------


def head(h_new, W, V_S):
    """z_j = <h_new, W_LM[:, V_S[j]]> (FUSED_INDEX_GEMM, Alg. 1 line 10) in fp64.
    W is [V][d]; rows of h_new are independent."""
    return np.atleast_2d(np.asarray(h_new, np.float64)) @ np.asarray(W[V_S], np.float64).T


def log_softmax(z):
    """p = log_softmax(z) (Alg. 1 line 11) with max subtraction; returns (logp, lse)."""
    z = np.asarray(z, dtype=np.float64)
    if z.size == 0:
        raise OracleError("EmptyInput")
    mx = z.max()
    lse = mx + math.log(float(np.sum(np.exp(z - mx))))
    return z - lse, lse


def epilogue(z_row, V_S, k_t):
    """log_softmax over V_S (R14), TopK_{k_t} by (logit desc, token id asc) (R7), and
    remap2realid: shortlist position -> vocabulary id."""
    logp, lse = log_softmax(z_row)
    order = top_k_order(z_row, k_t, tiebreak=V_S)
    return {"top_ids": V_S[order], "top_logits": np.asarray(z_row)[order], "top_logp": logp[order],
            "lse": lse, "top_pos": order}


# ---------------------------------------------------------------------------
# O7  dense full-vocabulary head   (§4.1)
# ---------------------------------------------------------------------------


def dense_head(h_new, W, k_t):
    """Full-vocabulary drafter head p = softmax(H~ W_LM) with the same epilogue."""
    V = W.shape[0]
    ids = np.arange(V)
    z = head(h_new, W, ids)
    return [dict(epilogue(z[r], ids, k_t), z=z[r]) for r in range(z.shape[0])]


# ---------------------------------------------------------------------------
# One DynaSpec draft step (Alg. 1 lines 7-11 for one position t)
# ---------------------------------------------------------------------------


def draft_step(part, router, W, h_prev, e, h_new, t, k_max, k_min, k_t, shared=False, sel_override=None):
    """One draft position: budget (line 7) -> meta score + TopK + indices (line 8) ->
    gathered head (line 10) -> log_softmax, TopK_{k_t}, remap (line 11).

    part = dict(perm, offsets); router = (W1, b1, W2, b2).  Rows are independent requests
    (per-row shortlists) unless shared=True (one union shortlist per depth, R9).
    sel_override: list of per-row selections (conditional parity: reuse a given selection).
    Returns a list of per-row dicts.
    """
    k = budget(t, k_max, k_min)
    scores = meta_score(*router, h_prev, e)
    B = scores.shape[0]
    if shared:
        sels = [select_shared(scores, k)] * B
    else:
        sels = [select(scores[r], k) for r in range(B)]
    if sel_override is not None:
        sels = [np.asarray(s, dtype=np.int64) for s in sel_override]
    out = []
    hn = np.atleast_2d(np.asarray(h_new, np.float64))
    for r in range(B):
        V_S = shortlist(sels[r], part["perm"], part["offsets"])
        z = head(hn[r], W, V_S)[0]
        res = epilogue(z, V_S, min(k_t, len(V_S)))
        res.update(k=k, scores=scores[r], sel=sels[r], sl_offsets=shortlist_offsets(sels[r], part["offsets"]),
                   V_S=V_S, z=z)
        out.append(res)
    return out


# ---------------------------------------------------------------------------
# NEXT-1  tree / beam bookkeeping   (Alg. 1 lines 12-18; reading R24 in DESIGN.md)
# ---------------------------------------------------------------------------


def tree_step(top_ids, top_logp, last_scores, last_nodes, step, node_base, k_t):
    """One step of Alg. 1 lines 12-16 for R current beams (R = 1 at j = 0):
      line 12: cu_scores[b, q] = TopP_j[b, q] + last_step_scores[b]
      line 13: d <- d + T~_j (all R x k_t expansions, with their cu_scores, step and parent node)
      line 14: TopC_j, last_step_scores <- TopK_{k_t}(cu_scores) over the flattened (b, q) expansions,
               ties -> lower flat index b * k_t + q (R24)
      line 15: x_j = T~_j[TopC_j];  line 16: h_j <- h~[beam of TopC_j]
    top_ids / top_logp: [R][k_t] from the head (id -1 / -inf padding is skipped).
    Returns (nodes, next) with nodes = list of (token, score, parent_node, step) appended at
    node_base + b * k_t + q, and next = dict(tok, score, node, beam) for the k_t kept expansions."""
    top_ids = np.atleast_2d(np.asarray(top_ids))
    top_logp = np.atleast_2d(np.asarray(top_logp, dtype=np.float64))
    R, K = top_ids.shape
    last_scores = np.zeros(R) if last_scores is None else np.asarray(last_scores, dtype=np.float64)
    last_nodes = np.full(R, -1) if last_nodes is None else np.asarray(last_nodes)
    cu = top_logp + last_scores[:, None]
    nodes = []
    for b in range(R):
        for q in range(K):
            nodes.append((int(top_ids[b, q]), float(cu[b, q]), int(last_nodes[b]), step))
    flat = cu.reshape(-1)
    valid = top_ids.reshape(-1) >= 0
    keys = [(-flat[i], i) for i in range(R * K) if valid[i]]
    keys.sort()
    keep = [i for _, i in keys[:k_t]]
    nxt = {"tok": np.array([int(top_ids.reshape(-1)[i]) for i in keep]),
           "score": np.array([flat[i] for i in keep]),
           "node": np.array([node_base + i for i in keep]),
           "beam": np.array([i // K for i in keep])}
    return nodes, nxt


def tree_rerank(nodes, n_out):
    """Alg. 1 line 18: re-rank the draft list d by d_scores (descending); ties -> lower node index
    (nodes are numbered step-major, so earlier steps win, then beam order; R24).  Returns the
    indices of the best n_out valid nodes."""
    keyed = [(-sc, i) for i, (tok, sc, par, st) in enumerate(nodes) if tok >= 0]
    keyed.sort()
    return np.array([k[1] for k in keyed[:n_out]], dtype=np.int64)


# ---------------------------------------------------------------------------
# NEXT-3  static frequency-ranked heads: FR-Spec and PA-FR (App. A.1)
# ---------------------------------------------------------------------------


def frequency_ranking(counts):
    """pi_f: token ids by descending corpus count, ties -> lower token id."""
    counts = np.asarray(counts)
    return np.lexsort((np.arange(counts.size), -counts)).astype(np.int64)


def fr_head(h_new, W, pi_f, K, k_t):
    """p_stat = softmax(H~ W~), W~[:, j] = W_LM[:, V_high[j]], V_high = pi_f[:K];
    the shortlist is the K most frequent tokens in frequency order."""
    V_S = np.asarray(pi_f[:K], dtype=np.int64)
    out = []
    for h in np.atleast_2d(np.asarray(h_new, np.float64)):
        z = head(h, W, V_S)[0]
        out.append(dict(epilogue(z, V_S, min(k_t, K)), z=z, V_S=V_S))
    return out


# ---------------------------------------------------------------------------
# NEXT-4  lossless verification of a drafted chain   (Eq. 3 P:82-89 and its footnote to
#         Leviathan et al. §3; reading R25 in DESIGN.md)
# ---------------------------------------------------------------------------


def softmax_full(logits):
    """p = softmax(l) over the full vocabulary, fp64."""
    l = np.asarray(logits, dtype=np.float64)
    m = l.max()
    e = np.exp(l - m)
    return e / e.sum()


def embed_q(V, q_ids, q_logits, q_lse):
    """q over the full vocabulary: exp(z - lse) on the shortlist tokens, 0 off V_S."""
    q = np.zeros(V, dtype=np.float64)
    q[np.asarray(q_ids, dtype=np.int64)] = np.exp(np.asarray(q_logits, np.float64) - float(q_lse))
    return q


def sample_inverse_cdf(w, u):
    """R25: the first token x (id order) whose cumulative weight exceeds u * sum(w)."""
    c = np.cumsum(np.asarray(w, dtype=np.float64))
    return int(np.searchsorted(c, u * c[-1], side="right"))


def verify_chain(p_logits, q_ids, q_logits, q_lse, x, u_acc, u_res):
    """Speculative-sampling verification of one chain of gamma drafted tokens x.

    p_logits: (gamma+1, V) target logits at the gamma+1 positions; q_i (i < gamma) is the drafter's
    shortlist distribution embedded in V.  Position i is accepted iff u_acc[i] < min(1, p_i(x_i)/q_i(x_i))
    (Eq. 3); at the first rejection the corrective token is drawn from the normalised residual
    (p_i - q_i)_+ with u_res; if all gamma are accepted, a bonus token is drawn from p_gamma with u_res.
    Returns (accepted_count, committed tokens (accepted_count + 1 of them))."""
    p_logits = np.asarray(p_logits, dtype=np.float64)
    gamma = len(x)
    V = p_logits.shape[1]
    for i in range(gamma):
        p = softmax_full(p_logits[i])
        q = embed_q(V, q_ids[i], q_logits[i], q_lse[i])
        xi = int(x[i])
        if q[xi] <= 0.0:
            raise OracleError("InvalidProposal")
        if u_acc[i] < min(1.0, p[xi] / q[xi]):
            continue
        r = np.maximum(p - q, 0.0)
        if r.sum() <= 0.0:  # R25: p == q numerically -> sample from p
            r = p
        return i, [int(t) for t in x[:i]] + [sample_inverse_cdf(r, u_res)]
    return gamma, [int(t) for t in x] + [sample_inverse_cdf(softmax_full(p_logits[gamma]), u_res)]
