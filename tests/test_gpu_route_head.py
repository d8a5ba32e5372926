"""NEXT-2 split of one draft step through the C ABI: dynaspec_step_route
(router + TopK + offsets, Alg. 1 line 8) on a side stream S_m while a stand-in drafter core runs on
S_d, the event join ("sync S_m, S_d", Alg. 1 line 10), then dynaspec_step_head (gathered head +
log-softmax + top-k_t, lines 10-11) on S_d -- compared with the oracle's draft step."""
import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S
from tests.parity import Rows, check_topk, f64, score_tol, selection_certified

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _run_split(Dy, st, hp, e, hn, t, k_max, k_min):
    """route on S_m || a core stand-in on S_d (it writes h_new), join, head on S_d."""
    cur = torch.cuda.current_stream()
    s_meta = torch.cuda.Stream()
    ev_f, ev_j = torch.cuda.Event(), torch.cuda.Event()
    h_new = torch.empty_like(hn)
    ev_f.record(cur)
    s_meta.wait_event(ev_f)
    st.route(hp, e, t, k_max, k_min, s_meta)
    h_new.copy_(hn * 1.0)          # the caller's drafter core on S_d produces the head input
    ev_j.record(s_meta)
    cur.wait_event(ev_j)
    st.head(h_new, t, k_max, k_min, cur)


# bf16 B in 2..16 takes the few-row one-launch router (meta_rows.cu), f32 / B = 1 the split-K pair
@pytest.mark.parametrize("dtype,shared,B", [("bf16", False, 1), ("f32", False, 1), ("bf16", False, 3),
                                            ("bf16", True, 3), ("bf16", True, 10), ("bf16", False, 16),
                                            ("f32", True, 10)])
def test_route_head_exact_regime(dtype, shared, B):
    """Exact regime (every fp32 sum exact): scores, selection, offsets, every logit and the top-k
    are bit-exact against the oracle."""
    from paper_2510_13847_b200 import dynaspec as Dy
    V, d, M, h_r, k_t = 5003, 256, 24, 16, 8
    W = S.lm_head(V, d, 0, dtype, "exact")
    rt = S.router(d, h_r, M, 1, dtype, "exact")
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, k_t, shared=shared, z_out=True)
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for t in range(4):
        hp, e, hn = S.step_inputs(B, d, t, dtype, "exact", h_r=h_r)
        _run_split(Dy, st, hp.to(DEV), e.to(DEV), hn.to(DEV), t, 8, 2)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 8, 2, k_t, shared=shared)
        sc = st.scores.cpu().numpy()
        for b in range(B):
            assert np.array_equal(sc[b], ref[b]["scores"].astype(np.float32))
        for b in range(1 if shared else B):
            cnt = st.sel_count[b].item()
            assert st.sel[b, :cnt].cpu().tolist() == ref[b]["sel"].tolist()
            assert st.sl_offsets[b, :cnt + 1].cpu().tolist() == ref[b]["sl_offsets"].tolist()
        for b in range(B):
            n = len(ref[b]["V_S"])
            assert np.array_equal(st.z[b, :n].cpu().numpy(), ref[b]["z"].astype(np.float32))
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), ref[b]["z"], ref[b]["V_S"], k_t, torch.float32, exact=True)


@pytest.mark.parametrize("B", [1, 4])
def test_route_head_llama3_random(B):
    """Llama-3 head at full size (V 128256, d 4096, M 256, bf16), random regime, the bench's
    NEXT-2 launch configuration: scores within 1e-5 rms, selections bit-exact when certified,
    every shortlist logit within 2e-2, top-k valid."""
    from paper_2510_13847_b200 import dynaspec as Dy
    C = S.CONFIGS["llama3"]
    W = S.lm_head(C.V, C.d, 0, "bf16")
    rt = S.router(C.d, C.h_r, C.M, 1, "bf16")
    tau = S.random_partition(C.V, C.M, 2)
    perm, off = O.layout(tau, C.M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), C.M)
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, C.k_t, z_out=True)
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for t in (0, 3):
        hp, e, hn = S.step_inputs(B, C.d, t, "bf16")
        _run_split(Dy, st, hp.to(DEV), e.to(DEV), hn.to(DEV), t, C.k_max, C.k_min)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t)
        for b in range(B):
            rb = ref[b]
            assert np.max(np.abs(st.scores[b].cpu().numpy() - rb["scores"])) <= score_tol(rb["scores"])
            cnt = st.sel_count[b].item()
            sel = st.sel[b, :cnt].cpu().numpy()
            if selection_certified(rb["scores"], rb["k"]):
                assert sel.tolist() == rb["sel"].tolist()
            else:
                rb = O.draft_step(part, ro, Wo, f64(hp[b:b + 1]), f64(e[b:b + 1]), f64(hn[b:b + 1]), t, C.k_max,
                                  C.k_min, C.k_t, sel_override=[sel])[0]
            assert st.sl_offsets[b, :cnt + 1].cpu().tolist() == rb["sl_offsets"].tolist()
            n = len(rb["V_S"])
            assert np.max(np.abs(st.z[b, :n].cpu().numpy().astype(np.float64) - rb["z"])) <= 2e-2
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), rb["z"], rb["V_S"], C.k_t, torch.bfloat16)


@pytest.mark.parametrize("B,split", [(8, False), (8, True), (3, False)])
def test_th_rows_mode_exact_regime(B, split, monkeypatch):
    """Independent rows on the balanced tree head (th.cu rows mode: the union of the rows' clusters
    streamed once, each row reduced over its OWN clusters only): selection, offsets, top-k ids /
    logits (bit-exact) and lse against the oracle, through draft_step and the route/head split."""
    from paper_2510_13847_b200 import dynaspec as Dy
    monkeypatch.setenv("DS_TH_ROWS_MIN", "2")
    V, d, M, h_r, k_t = 5003, 256, 24, 16, 8
    W = S.lm_head(V, d, 0, "bf16", "exact")
    rt = S.router(d, h_r, M, 1, "bf16", "exact")
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, k_t)
    assert st.kernel.startswith("ds::th_kernel"), st.kernel
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for t in range(4):
        hp, e, hn = S.step_inputs(B, d, t, "bf16", "exact", h_r=h_r)
        if split:
            _run_split(Dy, st, hp.to(DEV), e.to(DEV), hn.to(DEV), t, 8, 2)
        else:
            st(hp.to(DEV), e.to(DEV), hn.to(DEV), t, 8, 2)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 8, 2, k_t)
        for b in range(B):
            cnt = st.sel_count[b].item()
            assert st.sel[b, :cnt].cpu().tolist() == ref[b]["sel"].tolist()
            assert st.sl_offsets[b, :cnt + 1].cpu().tolist() == ref[b]["sl_offsets"].tolist()
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), ref[b]["z"], ref[b]["V_S"], k_t, torch.float32, exact=True)


def test_th_rows_mode_llama3_b8_sampled_rows():
    """Llama-3 at full size, the bench's B = 8 (rows mode is the default there): sampled rows
    against the oracle (scores, selection, top-k, lse) in the random regime."""
    from paper_2510_13847_b200 import dynaspec as Dy
    C = S.CONFIGS["llama3"]
    B = 8
    W = S.lm_head(C.V, C.d, 0, "bf16", device=DEV)
    tau = S.random_partition(C.V, C.M, 2)
    perm, off = O.layout(tau, C.M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W, torch.as_tensor(tau, dtype=torch.int32, device=DEV), C.M)
    rt = S.router(C.d, C.h_r, C.M, 1, "bf16")
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, C.k_t)
    assert st.kernel.startswith("ds::th_kernel"), st.kernel
    for t in (0, 3):
        hp, e, hn = S.step_inputs(B, C.d, t, "bf16")
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=C.k_max, k_min=C.k_min)
        torch.cuda.synchronize()
        Wo, ro = Rows(W), tuple(f64(x) for x in rt)
        for b in (0, 5):
            cnt = st.sel_count[b].item()
            sel = np.array(st.sel[b, :cnt].cpu().tolist(), dtype=np.int32)
            ref = O.draft_step(part, ro, Wo, f64(hp[b:b + 1]), f64(e[b:b + 1]), f64(hn[b:b + 1]), t, C.k_max,
                               C.k_min, C.k_t, sel_override=[sel])[0]
            assert np.max(np.abs(st.scores[b].cpu().numpy() - ref["scores"])) <= score_tol(ref["scores"])
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), ref["z"], ref["V_S"], C.k_t, torch.bfloat16)


@pytest.mark.parametrize("defer", ["1", "0"])
def test_tree_rows_exact_regime_deferred_union(defer, monkeypatch):
    """Tree rows (shared, 8 rows) through draft_step on the few-row router + the tree head; with
    DS_DEFER_UNION=1 the union is formed by the tree head from the rows' published masks.  Scores,
    the union selection and its offsets, every logit and the top-k are bit-exact against the oracle,
    several steps in a row on one workspace (the masks must be cleared between steps)."""
    from paper_2510_13847_b200 import dynaspec as Dy
    monkeypatch.setenv("DS_DEFER_UNION", defer)
    V, d, M, h_r, k_t, B = 5003, 256, 24, 16, 8, 8
    W = S.lm_head(V, d, 0, "bf16", "exact")
    rt = S.router(d, h_r, M, 1, "bf16", "exact")
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, k_t, shared=True, z_out=True)
    assert st.kernel.startswith("ds::th_kernel"), st.kernel
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for t in range(5):
        hp, e, hn = S.step_inputs(B, d, t, "bf16", "exact", h_r=h_r)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t, 8, 2)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 8, 2, k_t, shared=True)
        sc = st.scores.cpu().numpy()
        for b in range(B):
            assert np.array_equal(sc[b], ref[b]["scores"].astype(np.float32))
        cnt = st.sel_count[0].item()
        assert st.sel[0, :cnt].cpu().tolist() == ref[0]["sel"].tolist()
        assert st.sl_offsets[0, :cnt + 1].cpu().tolist() == ref[0]["sl_offsets"].tolist()
        for b in range(B):
            n = len(ref[b]["V_S"])
            assert np.array_equal(st.z[b, :n].cpu().numpy(), ref[b]["z"].astype(np.float32))
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), ref[b]["z"], ref[b]["V_S"], k_t, torch.float32, exact=True)


def test_few_row_router_batched_staging_exact():
    """The few-row router with the x rows staged in two batches (B = 16 rows of 2d = 8192 bf16 do not
    fit shared memory at once): scores, selection and offsets bit-exact against the oracle."""
    from paper_2510_13847_b200 import dynaspec as Dy
    V, d, M, h_r, k_t, B = 2003, 4096, 24, 16, 8, 16
    W = S.lm_head(V, d, 0, "bf16", "exact")
    rt = S.router(d, h_r, M, 1, "bf16", "exact")
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, k_t)
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for t in (0, 3):
        hp, e, hn = S.step_inputs(B, d, t, "bf16", "exact", h_r=h_r)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t, 8, 2)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 8, 2, k_t)
        sc = st.scores.cpu().numpy()
        for b in range(B):
            assert np.array_equal(sc[b], ref[b]["scores"].astype(np.float32)), (t, b)
            cnt = st.sel_count[b].item()
            assert st.sel[b, :cnt].cpu().tolist() == ref[b]["sel"].tolist()
            assert st.sl_offsets[b, :cnt + 1].cpu().tolist() == ref[b]["sl_offsets"].tolist()
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), ref[b]["z"], ref[b]["V_S"], k_t, torch.float32, exact=True)


def test_th_rows_mode_per_row_shortlist_bound(monkeypatch):
    """Rows mode with a shortlist bound that some rows exceed: those rows get the documented sentinel
    (ids -1, lse NaN), the others are computed exactly (head_forward on the tree head's rows mode)."""
    from paper_2510_13847_b200 import dynaspec as Dy
    monkeypatch.setenv("DS_TH_ROWS_MIN", "2")
    V, d, M, k_t, B = 3001, 128, 20, 4, 6
    q = max(1, min(127, int((2 ** 21 / d) ** 0.5)))
    W = S.lm_head(V, d, 0, "bf16", "exact", q=q)
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    hn = S.hidden(B, d, 7, "bf16", "exact", q=q)
    rng = np.random.default_rng(1)
    sizes = np.diff(off)
    ks = [1, 2, 3, 1, 4, 2]
    sel = torch.zeros((B, M), dtype=torch.int32)
    cnt = torch.zeros(B, dtype=torch.int32)
    slo = torch.zeros((B, M + 1), dtype=torch.int32)
    sels = []
    for b in range(B):
        sb = np.sort(rng.choice(M, ks[b], replace=False)).astype(np.int32)
        sels.append(sb)
        sel[b, :ks[b]] = torch.as_tensor(sb)
        cnt[b] = ks[b]
        slo[b, :ks[b] + 1] = torch.as_tensor(O.shortlist_offsets(sb, off), dtype=torch.int32)
    tot = [int(sizes[sb].sum()) for sb in sels]
    bound = sorted(tot)[B // 2]  # about half the rows exceed it
    out = Dy.head_forward(c, hn.to(DEV), sel.to(DEV), cnt.to(DEV), slo.to(DEV), k_t, max_shortlist=bound)
    for b in range(B):
        if tot[b] > bound:
            assert (out["top_ids"][b].cpu() == -1).all() and np.isnan(out["lse"][b].item())
        else:
            V_S = O.shortlist(sels[b], perm, off)
            zref = O.head(f64(hn[b:b + 1]), f64(W), V_S)[0]
            check_topk(out["top_ids"][b].cpu().numpy(), out["top_logits"][b].cpu().numpy(),
                       out["top_logp"][b].cpu().numpy(), out["lse"][b].item(), zref, V_S, k_t, torch.float32,
                       exact=True)
