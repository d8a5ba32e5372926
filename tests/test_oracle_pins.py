"""Pins for the CPU oracle (-m "not gpu").

Each test pins oracle/ against something other than itself: golden values printed in
SPEC.md / the worked example E2E-1 (tests/golden/e2e1.json), closed forms, brute force
on tiny inputs, special cases that reduce to textbook results, and invariants the
paper states.  Citation per test: P:<line> = PAPER.md, S:<line> = SPEC.md.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import dynaspec_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "e2e1.json")))


# ----------------------------------------------------------------- O0 budget

def test_budget_spec_golden():
    # S:255-256 (k_max=16): 16,16,2,2,1 — direct evaluation of P:205-210.
    assert [O.budget(t, 16, 1) for t in range(5)] == [16, 16, 2, 2, 1]
    # S:257 clamp: k_max=4, k_min=1, t=5 -> floor(4/12)=0 -> 1.
    assert O.budget(5, 4, 1) == 1


def test_budget_config_strings():
    # BASELINE.json configs: "16->4" and "32->8" reproduced with k_min = 4 / 8 (reading R1).
    assert [O.budget(t, 16, 4) for t in range(8)] == [16, 16, 4, 4, 4, 4, 4, 4]
    assert [O.budget(t, 32, 8) for t in range(8)] == [32, 32, 8, 8, 8, 8, 8, 8]
    # Without the clamp the raw formula: 32 -> 5,4,3,2,2,2.
    assert [O.budget(t, 32, 1) for t in range(2, 8)] == [5, 4, 3, 2, 2, 2]


def test_budget_monotone_and_pa_fr():
    for kmax in (1, 4, 16, 32, 64):
        ks = [O.budget(t, kmax, 1) for t in range(40)]
        assert ks[0] == ks[1] == kmax
        assert all(a >= b for a, b in zip(ks[1:], ks[2:]))
    assert O.budget_pa_fr(2, 32768) == 10922
    with pytest.raises(O.OracleError):
        O.budget(0, 4, 0)


# ----------------------------------------------------------------- O1 partition

def test_normalize_golden():
    # column [3,4] -> [0.6, 0.8]; quantised at 2^14: rint(9830.4)=9830, rint(13107.2)=13107.
    assert O.normalize_quantize(np.array([[3.0, 4.0]])).tolist() == [[9830, 13107]]
    assert O.normalize_quantize(np.array([[1.0, 0.0]])).tolist() == [[16384, 0]]   # already unit
    assert O.normalize_quantize(np.array([[0.0, -2.0]])).tolist() == [[0, -16384]]
    with pytest.raises(O.OracleError):
        O.normalize_quantize(np.array([[0.0, 0.0]]))


def test_normalize_invariants():
    rng = np.random.default_rng(5)
    W = rng.standard_normal((50, 64)).astype(np.float32).astype(np.float64)
    U = O.normalize_quantize(W)
    n = np.linalg.norm(U.astype(np.float64), axis=1)
    assert np.all(np.abs(n - 16384.0) <= 0.5 * math.sqrt(64) + 1e-9)   # unit norm within rounding
    assert np.array_equal(O.normalize_quantize(8.0 * W), U)           # scale invariance (exact: 2^3)
    assert np.array_equal(O.normalize_quantize(-W), -U)               # odd symmetry of rint
    # cosine check against an independent computation of the direction
    direc = W / np.linalg.norm(W, axis=1, keepdims=True)
    assert np.max(np.abs(U / 16384.0 - direc)) <= 0.5 / 16384 + 1e-12


def test_splitmix64_reference_vector():
    # splitmix64 reference output for seed 0 (Vigna's splitmix64.c): first value 0xE220A8397B1DCDAF.
    g = O.splitmix64_stream(0)
    assert next(g) == 0xE220A8397B1DCDAF
    assert next(g) == 0x6E789E6AA1B965F4
    assert next(g) == 0x06C45D188009454F


def test_forgy_distinct():
    for V, M, seed in [(10, 10, 0), (100, 7, 3), (5, 1, 9)]:
        ids = O.forgy_init(V, M, seed)
        assert len(set(ids.tolist())) == M and ids.min() >= 0 and ids.max() < V


def test_forgy_hand_draw():
    """R12 step 2 by hand from the published splitmix64 reference vector (seed 0):
    r0 = 16294208416658607535 (0xE220A8397B1DCDAF): r0 mod 10 = 5 (last digit) -> swap a[0], a[5];
    r1 = 7960286522194355700: digit sum 90, so r1 mod 9 = 0 -> j = 1, no swap;
    r2 = 487617019471545679: 679 mod 8 = 7 -> j = 2 + 7 = 9 -> swap a[2], a[9].
    a = [0..9] becomes [5, 1, 9, ...]: the first M = 3 entries are the Forgy ids."""
    assert O.forgy_init(10, 3, 0).tolist() == [5, 1, 9]
    assert O.forgy_init(10, 1, 0).tolist() == [5]
    assert O.forgy_init(10, 2, 0).tolist() == [5, 1]


def _W_e2e():
    return np.array(GOLD["W_rows"], dtype=np.float64)


def test_e2e1_quantised_and_golden_inits():
    W = _W_e2e()
    assert O.normalize_quantize(W).tolist() == GOLD["U_quantised"]
    for key, exp in GOLD["golden_inits"].items():
        init = [int(x) for x in key.split(",")]
        tau, iters = O.spherical_kmeans(W, 3, init_ids=init, max_iters=20)
        tau = O.canonical_relabel(tau, 3)
        assert tau.tolist() == GOLD["partition"]["tau"], key
        assert iters == exp["iters"], key
    perm, off = O.layout(np.array(GOLD["partition"]["tau"]), 3)
    assert perm.tolist() == GOLD["partition"]["perm"] and off.tolist() == GOLD["partition"]["offsets"]


def test_kmeans_four_angles_all_inits():
    # unit vectors at 1,3,88,91 degrees, M=2 -> {0,1},{2,3}, for every ordered Forgy pair.
    ang = np.deg2rad([1, 3, 88, 91])
    W = np.stack([np.cos(ang), np.sin(ang)], axis=1)
    for init in itertools.permutations(range(4), 2):
        tau, _ = O.spherical_kmeans(W, 2, init_ids=list(init))
        tau = O.canonical_relabel(tau, 2)
        assert tau.tolist() == [0, 0, 1, 1], init


def test_kmeans_trivial_M():
    rng = np.random.default_rng(1)
    W = rng.standard_normal((9, 5))
    tau, _ = O.spherical_kmeans(W, 9, seed=4)         # S:184 M=|V| -> singletons, objective 1 each
    assert sorted(tau.tolist()) == list(range(9))
    U = O.normalize_quantize(W)
    assert abs(O.kmeans_objective(U, tau, 9) - 9.0) < 9 * 1e-3
    tau1, _ = O.spherical_kmeans(W, 1, seed=4)        # S:185 M=1 -> one cluster
    assert set(tau1.tolist()) == {0}


def _partitions(n, M):
    """All surjections [n] -> [M] up to relabelling (set partitions into exactly M blocks)."""
    for labels in itertools.product(range(M), repeat=n):
        if labels[0] != 0:
            continue
        seen, ok = [], True
        for l in labels:                               # canonical: first occurrences in order
            if l not in seen:
                if l != len(seen):
                    ok = False
                    break
                seen.append(l)
        if ok and len(seen) == M:
            yield np.array(labels)


def test_kmeans_brute_force_tiny():
    # Brute force over all partitions (V<=7, M<=3): Lloyd's objective <= the optimum, and a
    # converged run is a Lloyd fixed point (every token at the argmax of its final centroid).
    rng = np.random.default_rng(11)
    for trial in range(12):
        V, M = int(rng.integers(3, 8)), int(rng.integers(1, 4))
        M = min(M, V)
        W = rng.standard_normal((V, 3))
        U = O.normalize_quantize(W)
        best = max(O.kmeans_objective(U, p, M) for p in _partitions(V, M))
        tau, iters = O.spherical_kmeans(W, M, seed=trial, max_iters=50)
        assert np.all(np.bincount(tau, minlength=M) > 0)
        assert O.kmeans_objective(U, tau, M) <= best + 1e-9
        if iters < 50:
            C = np.stack([O.centroid_from_sum(U[tau == m].sum(0)) for m in range(M)])
            dots = U @ C.T
            assert np.array_equal(np.argmax(dots, axis=1), tau)
    # Some seeds must reach the optimum on the E2E example (36/120 inits do).
    W = _W_e2e()
    U = O.normalize_quantize(W)
    hits = 0
    for init in itertools.permutations(range(6), 3):
        tau, _ = O.spherical_kmeans(W, 3, init_ids=list(init))
        if abs(O.kmeans_objective(U, tau, 3) - GOLD["optimum_objective"]) < 1e-6:
            hits += 1
    assert hits == 36


def test_partition_invariants_and_determinism():
    rng = np.random.default_rng(3)
    W = rng.standard_normal((300, 16)).astype(np.float32).astype(np.float64)
    a = O.build_clusters(W, 12, seed=7, max_iters=15)
    b = O.build_clusters(W, 12, seed=7, max_iters=15)
    assert all(np.array_equal(a[k], b[k]) for k in ("tau", "perm", "offsets"))
    tau, perm, off = a["tau"], a["perm"], a["offsets"]
    assert sorted(perm.tolist()) == list(range(300))
    assert off[0] == 0 and off[-1] == 300 and np.all(np.diff(off) > 0)
    for m in range(12):
        blk = perm[off[m]:off[m + 1]]
        assert np.all(tau[blk] == m) and np.all(np.diff(blk) > 0)    # contiguous, ascending ids
    # canonical labels: cluster minima increase with the label
    mins = [perm[off[m]:off[m + 1]].min() for m in range(12)]
    assert mins == sorted(mins)


# ----------------------------------------------------------------- O2 router

def test_meta_score_examples():
    d = 3
    z = O.meta_score(np.zeros((5, 2 * d)), np.zeros(5), np.zeros((4, 5)), np.zeros(4),
                     np.ones(d), np.ones(d))
    assert np.all(z == 0)
    R = np.array(GOLD["router_linear_rows"], dtype=np.float64)
    s = O.meta_score(R, np.zeros(3), None, None, np.array(GOLD["h_prev"]), np.array(GOLD["e"]))
    assert s[0].tolist() == GOLD["scores"]
    # hand example of the 2-layer form: a = relu([3, -3]) = [3, 0]; s = [[1,1],[2,-1]] a + [0.5, 0]
    s2 = O.meta_score(np.array([[1.0, 0.0], [-1.0, 0.0]]), np.zeros(2), np.array([[1.0, 1.0], [2.0, -1.0]]),
                      np.array([0.5, 0.0]), np.array([3.0]), np.array([5.0]))
    assert s2[0].tolist() == [3.5, 6.0]
    # input order [h_prev || e] (R4): W1 acting only on e
    s3 = O.meta_score(np.array([[0.0, 1.0]]), np.zeros(1), None, None, np.array([7.0]), np.array([2.0]))
    assert s3[0].tolist() == [2.0]


# ----------------------------------------------------------------- O3/O4 select + union

def test_select_spec_examples():
    assert O.top_k_order([0.1, 0.9, 0.5], 2).tolist() == [1, 2]
    assert O.top_k_order([0.5, 0.5], 1).tolist() == [0]
    assert O.select(np.array([3.0, 2.0, 1.0, 0.0]), 3).tolist() == [0, 1, 2]
    assert O.select(np.array([0.0, 5.0, 1.0]), 3).tolist() == [0, 1, 2]       # S:265 k=M
    assert O.select(np.array(GOLD["tie_variants"]["router_row0_2"]["scores"], float), 1).tolist() == [0]
    assert O.select(np.array([-0.0, 0.0, -1.0]), 1).tolist() == [0]           # R23: -0 == +0
    with pytest.raises(O.OracleError):
        O.select(np.array([1.0]), 2)


def test_select_brute_force():
    rng = np.random.default_rng(2)
    for _ in range(200):
        M = int(rng.integers(1, 9))
        s = rng.integers(-3, 4, size=M).astype(float)                 # many ties
        k = int(rng.integers(1, M + 1))
        sel = O.select(s, k)
        # brute force: the unique k-subset that dominates its complement under (score desc, id asc)
        dom = [c for c in itertools.combinations(range(M), k)
               if all(s[i] > s[j] or (s[i] == s[j] and i < j) for i in c for j in range(M) if j not in c)]
        assert len(dom) == 1 and sel.tolist() == list(dom[0])


def test_shortlist_invariants():
    rng = np.random.default_rng(4)
    V, M = 200, 17
    tau = rng.integers(0, M, V)
    tau[:M] = np.arange(M)
    perm, off = O.layout(tau, M)
    for _ in range(20):
        k = int(rng.integers(1, M + 1))
        sel = np.sort(rng.choice(M, k, replace=False))
        VS = O.shortlist(sel, perm, off)
        assert len(VS) == sum(off[m + 1] - off[m] for m in sel)
        assert O.shortlist_offsets(sel, off)[-1] == len(VS)
        assert sorted(VS.tolist()) == O.cluster_union_sorted(sel, tau).tolist()
        assert set(tau[VS].tolist()) == set(sel.tolist())              # closure under cluster-mates S:361
        assert np.all(np.diff(tau[VS]) >= 0)                           # (tau(v), v) order, R8
    assert sorted(O.shortlist(np.arange(M), perm, off).tolist()) == list(range(V))
    with pytest.raises(O.OracleError):
        O.shortlist([], perm, off)


# ----------------------------------------------------------------- O5/O6 head + epilogue

def test_head_spec_examples():
    W = np.eye(3)                                  # W_LM = I3, our rows = columns
    assert O.head(np.array([1.0, 2, 3]), W, np.array([2, 0]))[0].tolist() == [3.0, 1.0]
    WLM = np.array([[1.0, 2, 3], [4, 5, 6]])       # d=2 x n=3
    assert O.head(np.array([1.0, 1.0]), WLM.T, np.array([1]))[0].tolist() == [7.0]


def test_head_equals_dense_at_ids():
    rng = np.random.default_rng(6)
    W = rng.standard_normal((8, 16))
    h = rng.standard_normal(16)
    dense = W @ h                                   # textbook matvec
    assert np.allclose(O.head(h, W, np.arange(8))[0], dense, rtol=0, atol=1e-12)
    ids = np.array([5, 1, 6])
    assert np.allclose(O.head(h, W, ids)[0], dense[ids], rtol=0, atol=1e-12)


def test_log_softmax_examples():
    lp, _ = O.log_softmax(np.array([0.0, 0.0]))
    assert np.allclose(lp, [-math.log(2)] * 2, atol=1e-15)
    lp, _ = O.log_softmax(np.array([1000.0, 0.0]))
    assert np.all(np.isfinite(lp)) and abs(lp[0]) < 1e-300 + 1e-12
    z = np.random.default_rng(0).standard_normal(1000) * 5
    lp, lse = O.log_softmax(z)
    assert abs(np.exp(lp).sum() - 1.0) <= 1e-12
    lp2, _ = O.log_softmax(z + 123.25)
    assert np.allclose(lp, lp2, atol=1e-12)                            # shift invariance S:47
    lp1, _ = O.log_softmax(np.array([4.2]))
    assert lp1.tolist() == [0.0]                                       # |V_S| = 1 => p = 1
    # lse against the closed form ln(sum e^z) for small z
    assert abs(O.log_softmax(np.array([1.0, 2.0, 3.0]))[1] - math.log(math.e + math.e ** 2 + math.e ** 3)) < 1e-14


def test_e2e1_pipeline_golden():
    W = _W_e2e()
    part = O.build_clusters(W, 3, init_ids=[0, 5, 2])
    R = np.array(GOLD["router_linear_rows"], dtype=np.float64)
    router = (R, np.zeros(3), None, None)
    for case in GOLD["cases"]:
        k = case["k"]
        out = O.draft_step(part, router, W, np.array(GOLD["h_prev"], float), np.array(GOLD["e"], float),
                           np.array(GOLD["h_new"], float), t=0, k_max=k, k_min=1, k_t=len(case["V_S"]))[0]
        assert out["scores"].tolist() == GOLD["scores"]
        assert out["sel"].tolist() == case["sel"]
        assert out["sl_offsets"].tolist() == case["sl_offsets"]
        assert out["V_S"].tolist() == case["V_S"]
        assert out["z"].tolist() == case["z"]
        assert abs(out["lse"] - case["lse"]) < 1e-11
        assert out["top_ids"].tolist() == case["top_ids"]
        assert np.allclose(out["top_logp"], np.array(case["z"])[out["top_pos"]] - case["lse"], atol=1e-11)
    tv = GOLD["tie_variants"]["h_new_3_2"]
    out = O.draft_step(part, router, W, np.array(GOLD["h_prev"], float), np.array(GOLD["e"], float),
                       np.array(tv["h_new"], float), t=0, k_max=2, k_min=1, k_t=4)[0]
    assert out["z"].tolist() == tv["z"] and out["top_ids"].tolist() == tv["top_ids"]


def test_k_equals_M_is_dense():
    # north star: with k = M the output equals the full-vocabulary head's argmax and logits.
    rng = np.random.default_rng(8)
    V, d, M = 120, 12, 7
    W = rng.standard_normal((V, d)).astype(np.float32).astype(np.float64)
    part = O.build_clusters(W, M, seed=1, max_iters=10)
    router = (rng.standard_normal((4, 2 * d)), np.zeros(4), rng.standard_normal((M, 4)), np.zeros(M))
    h = rng.standard_normal((3, d))
    outs = O.draft_step(part, router, W, h, h, h, t=0, k_max=M, k_min=1, k_t=5)
    dense = O.dense_head(h, W, 5)
    for o, dn in zip(outs, dense):
        assert o["top_ids"].tolist() == dn["top_ids"].tolist()
        assert abs(o["lse"] - dn["lse"]) < 1e-12
        z_at = dn["z"][o["V_S"]]
        assert np.allclose(o["z"], z_at, atol=1e-12)


def test_shared_mode_hand_example():
    """R9 (one index set I for all rows of a depth) by hand.  M = 5 clusters of one
    token each (tau = id), k = 2:
      row 0 scores [5, 4, 1, 0, 0] -> TopK {0, 1};  row 1 [0, 1, 9, 8, 0] -> {2, 3};
      row 2 [3, 3, 3, 0, 0] -> ties, lower id first (R7) -> {0, 1}.
    Shared selection = ascending union [0, 1, 2, 3]; every row's logits, lse and top ids range over
    tokens 0..3 (not over its own clusters only): W rows e_0..e_4 of R^5 give z_r = h_r[0..3]."""
    s = np.array([[5, 4, 1, 0, 0], [0, 1, 9, 8, 0], [3, 3, 3, 0, 0]], dtype=np.float64)
    assert O.select_shared(s, 2).tolist() == [0, 1, 2, 3]
    assert O.select(s[2], 2).tolist() == [0, 1]
    part = {"perm": np.arange(5), "offsets": np.arange(6)}
    W = np.eye(5)
    # a linear router that reproduces the scores: s = W1 [h_prev || e] + b1 with W1 = 0, b1 per row is
    # not expressible (b1 is shared), so feed the rows through h_prev with W1 = [I | 0]
    W1 = np.hstack([np.eye(5), np.zeros((5, 5))])
    router = (W1, np.zeros(5), None, None)
    h_new = np.array([[1.0, 0, 0, 0, 7.0], [0, 2.0, 0, 0, 0], [0, 0, 0, 3.0, 0]])
    out = O.draft_step(part, router, W, s, np.zeros_like(s), h_new, t=0, k_max=2, k_min=1, k_t=2, shared=True)
    for r, o in enumerate(out):
        assert o["V_S"].tolist() == [0, 1, 2, 3]
        z = h_new[r, :4]
        assert np.array_equal(o["z"], z)                      # token 4 (z = 7 in row 0) is not in I
        assert abs(o["lse"] - math.log(np.exp(z).sum())) < 1e-12
    assert out[0]["top_ids"].tolist() == [0, 1]               # z = [1, 0, 0, 0]: then id order
    assert out[1]["top_ids"].tolist() == [1, 0]
    assert out[2]["top_ids"].tolist() == [3, 0]


def test_shared_mode_union():
    rng = np.random.default_rng(9)
    s = rng.standard_normal((4, 10))
    u = O.select_shared(s, 3)
    ref = sorted(set().union(*[set(O.select(s[r], 3).tolist()) for r in range(4)]))
    assert u.tolist() == ref


# ----------------------------------------------------------------- NEXT-1 tree bookkeeping

def test_tree_greedy_chain_closed_form():
    # k_t = 1: one chain; scores are the running sums of the chosen log-probs.
    logps = [-0.1, -0.7, -0.2]
    toks = [5, 9, 2]
    last, lastn, base, chain = None, None, 0, []
    for j, (tk, lp) in enumerate(zip(toks, logps)):
        nodes, nxt = O.tree_step([[tk]], [[lp]], last, lastn, j, base, 1)
        base += 1
        last, lastn = nxt["score"], nxt["node"]
        chain.append((int(nxt["tok"][0]), float(nxt["score"][0])))
    assert [c[0] for c in chain] == toks
    assert np.allclose([c[1] for c in chain], np.cumsum(logps))


def test_tree_step_hand_example():
    # two beams, k_t = 2: cu = TopP + last; keep the 2 best of 4 expansions (ties -> lower index)
    nodes, nxt = O.tree_step([[3, 1], [7, 2]], [[-0.5, -1.0], [-0.1, -0.5]], [-1.0, -1.2], [10, 11], 1, 20, 2)
    assert [n[1] for n in nodes] == [-1.5, -2.0, -1.3, -1.7]
    assert [n[2] for n in nodes] == [10, 10, 11, 11]
    assert nxt["tok"].tolist() == [7, 3] and nxt["node"].tolist() == [22, 20] and nxt["beam"].tolist() == [1, 0]
    _, nx2 = O.tree_step([[3, 1]], [[-0.5, -0.5]], [0.0], [-1], 0, 0, 1)
    assert nx2["tok"].tolist() == [3]                                  # tie -> lower flat index


def _enumerate_paths(logp_of, V, depth):
    """All token paths of length `depth` with their summed log-probs (brute force)."""
    paths = [((), 0.0)]
    for _ in range(depth):
        paths = [(p + (v,), s + logp_of(p, v)) for p, s in paths for v in range(V)]
    return paths


def test_tree_beam_equals_exhaustive_when_nothing_is_pruned():
    # with k_t >= (number of expansions), beam search keeps every path, so the
    # draft list d equals the exhaustive enumeration of all paths with the same scores.
    V, depth, K = 3, 3, 27
    rng = np.random.default_rng(4)
    table = {}

    def logp_of(prefix, v):
        if prefix not in table:
            z = rng.standard_normal(V)
            table[prefix] = z - np.log(np.exp(z).sum())
        return table[prefix][v]

    exhaustive = {}
    for dpt in range(1, depth + 1):
        for p, sc in _enumerate_paths(logp_of, V, dpt):
            exhaustive[p] = sc
    beams = [()]
    last, lastn, base = None, None, 0
    allnodes, paths_of_node = [], {}
    for j in range(depth):
        ids = [[v for v in range(V)] + [-1] * (K - V) for _ in beams]
        lps = [[logp_of(b, v) for v in range(V)] + [-np.inf] * (K - V) for b in beams]
        nodes, nxt = O.tree_step(ids, lps, last, lastn, j, base, K)
        for i, nd in enumerate(nodes):
            if nd[0] >= 0:
                paths_of_node[base + i] = beams[i // K] + (nd[0],)
        allnodes += nodes
        beams = [beams[b] + (int(t),) for b, t in zip(nxt["beam"], nxt["tok"])]
        base += len(nodes)
        last, lastn = nxt["score"], nxt["node"]
    got = {paths_of_node[i]: allnodes[i][1] for i in paths_of_node}
    assert set(got) == set(exhaustive)
    assert all(abs(got[p] - exhaustive[p]) < 1e-12 for p in got)
    # re-rank: the best n nodes are closed under parents (scores never increase along a path)
    top = O.tree_rerank(allnodes, 10)
    chosen = set(top.tolist())
    for i in chosen:
        par = allnodes[i][2]
        assert par == -1 or par in chosen


# ----------------------------------------------------------------- NEXT-3 static frequency heads

def test_frequency_ranking_and_fr_head():
    assert O.frequency_ranking([0, 5, 5, 1]).tolist() == [1, 2, 3, 0]          # ties -> lower id
    assert O.frequency_ranking([3, 3, 3]).tolist() == [0, 1, 2]                # uniform -> identity
    rng = np.random.default_rng(2)
    W = rng.standard_normal((50, 8))
    h = rng.standard_normal(8)
    pi = O.frequency_ranking(rng.integers(0, 100, 50))
    full = O.fr_head(h, W, pi, 50, 5)[0]
    dense = O.dense_head(h, W, 5)[0]
    assert full["top_ids"].tolist() == dense["top_ids"].tolist()               # K = |V| -> dense
    assert abs(full["lse"] - dense["lse"]) < 1e-12
    small = O.fr_head(h, W, pi, 10, 3)[0]
    assert set(small["V_S"].tolist()) <= set(O.fr_head(h, W, pi, 20, 3)[0]["V_S"].tolist())   # nesting S:359
    assert [O.budget_pa_fr(t, 32768) for t in range(4)] == [32768, 32768, 10922, 8192]     # App. A.1


# ----------------------------------------------------------------- NEXT-4 lossless verification

def test_sample_inverse_cdf_brute():
    w = [0.0, 1.0, 0.0, 3.0]
    assert O.sample_inverse_cdf(w, 0.0) == 1                 # zero-weight tokens are never drawn
    assert O.sample_inverse_cdf(w, 0.2499) == 1
    assert O.sample_inverse_cdf(w, 0.25) == 3                # first cumulative strictly above u*Z (R25)
    assert O.sample_inverse_cdf(w, 0.999999) == 3


def test_verify_two_token_example():
    """|V|=2, p=[.6,.4], q=[.5,.5]: beta = 0.9; rejecting token 1 leaves all residual on 0."""
    pl = np.log([[0.6, 0.4], [0.3, 0.7]])
    qi, ql, qs = [[0, 1]], [[0.0, 0.0]], [math.log(2.0)]
    assert O.verify_chain(pl, qi, ql, qs, [1], [0.85], 0.99) == (0, [0])      # 0.85 >= 0.4/0.5 -> reject
    assert O.verify_chain(pl, qi, ql, qs, [1], [0.79], 0.2) == (1, [1, 0])    # accept; bonus from p_1
    assert O.verify_chain(pl, qi, ql, qs, [1], [0.79], 0.5) == (1, [1, 1])
    grid = (np.arange(1000) + 0.5) / 1000
    acc = [np.mean([O.verify_chain(pl, qi, ql, qs, [x], [u], 0.5)[0] for u in grid]) for x in (0, 1)]
    assert abs(0.5 * acc[0] + 0.5 * acc[1] - 0.9) < 1e-12                     # Eq. 3: sum min(p, q)


def test_verify_q_equals_p_accepts_everything():
    rng = np.random.default_rng(4)
    pl = rng.standard_normal((4, 16)) * 2
    lse = [float(np.log(np.exp(r).sum())) for r in pl]
    ids = [np.arange(16)] * 3
    for u in (0.0, 0.5, 0.999999):
        n, com = O.verify_chain(pl, ids, pl[:3], lse[:3], [3, 7, 1], [u] * 3, 0.3)
        assert n == 3 and com[:3] == [3, 7, 1] and len(com) == 4


def test_verify_invalid_proposal():
    with pytest.raises(O.OracleError):
        O.verify_chain(np.zeros((2, 4)), [[0, 1]], [[0.0, 0.0]], [math.log(2)], [3], [0.1], 0.1)


def test_verify_monte_carlo_exactness():
    """the committed tokens follow the target law (TV < 0.02-0.03) even though q is zero off its
    shortlist; position 1 given acceptance at 0 follows p_1."""
    rng = np.random.default_rng(5)
    V, n = 8, 30000
    pl = rng.standard_normal((3, V)) * 1.5
    p = [O.softmax_full(r) for r in pl]
    S = [np.array([0, 2, 3, 5, 6]), np.array([1, 2, 4, 7])]
    ql = [rng.standard_normal(len(s)) for s in S]
    qs = [float(np.log(np.exp(z).sum())) for z in ql]
    q = [O.embed_q(V, S[i], ql[i], qs[i]) for i in range(2)]
    first, second = np.zeros(V), np.zeros(V)
    for _ in range(n):
        x = [int(rng.choice(V, p=q[i])) for i in range(2)]
        k, com = O.verify_chain(pl, S, ql, qs, x, rng.random(2), rng.random())
        first[com[0]] += 1
        if k >= 1:
            second[com[1]] += 1
    assert 0.5 * np.abs(first / n - p[0]).sum() < 0.02
    assert 0.5 * np.abs(second / second.sum() - p[1]).sum() < 0.03
