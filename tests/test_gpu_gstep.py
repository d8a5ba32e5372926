"""GPU parity of the grid draft step (gstep.cu: B = 1, router layer-1 units spread over every CTA and
published as tagged words, layer 2 + TopK evaluated redundantly in every CTA, all SMs streaming,
per-warp online top-k / log-sum-exp, polled record merge) against the CPU oracle.

Exact regime (integer-grid inputs): every fp32 dot product is exact in any summation
order, so scores, selections, offsets, every shortlist logit and the top-k_t ids and logits must be
bit-identical to the oracle's.  Random regime at the Llama-3 head's full size.  Also: the head-only
variant behind dynaspec_step_route + dynaspec_step_head (the S_m / S_d split), the
max_shortlist sentinel, workspace reuse across entry points, PDL-chained steps in one CUDA graph.
"""
import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S
from tests.parity import Rows, check_topk, f64, score_tol, selection_certified

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _dyn():
    from paper_2510_13847_b200 import dynaspec
    return dynaspec


def _setup(V, d, M, h_r, dtype, regime, seed_part=2):
    D = _dyn()
    W = S.lm_head(V, d, 0, dtype, regime)
    rt = S.router(d, h_r, M, 1, dtype, regime)
    tau = S.random_partition(V, M, seed_part)
    perm, off = O.layout(tau, M)
    c = D.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = D.Router(*[None if x is None else x.to(DEV) for x in rt])
    return W, rt, {"perm": perm, "offsets": off}, c, r


def _ran_gstep(D, fn):
    """Run fn() with the phase trace on; True iff the launch was the grid step (512-thread CTAs)."""
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(G * 64, dtype=torch.int64, device=DEV)
    D.debug_set_trace(buf)
    try:
        fn()
        torch.cuda.synchronize()
    finally:
        D.debug_set_trace(None)
    t = buf.view(G, 64).cpu()
    # the grid step runs one 512-thread CTA on every SM but one (gstep.cu: gstep_grid)
    return bool((t[:G - 1, 30] == 512).all() and (t[:G - 1, 0] > 0).all())


def _exact_check(st, ref, k_t):
    assert np.array_equal(st.scores[0].cpu().numpy(), ref["scores"].astype(np.float32)), "scores"
    cnt = st.sel_count[0].item()
    assert st.sel[0, :cnt].cpu().tolist() == ref["sel"].tolist()
    assert st.sl_offsets[0, :cnt + 1].cpu().tolist() == ref["sl_offsets"].tolist()
    n = len(ref["V_S"])
    assert np.array_equal(st.z[0, :n].cpu().numpy(), ref["z"].astype(np.float32)), "logits"
    check_topk(st.top_ids[0].cpu().numpy(), st.top_logits[0].cpu().numpy(), st.top_logp[0].cpu().numpy(),
               st.lse[0].item(), ref["z"], ref["V_S"], k_t, torch.float32, exact=True)


@pytest.mark.parametrize("dtype,h_r,k_t", [("bf16", 16, 8), ("f32", 16, 1), ("bf16", 0, 32), ("f32", 8, 32),
                                           ("bf16", 128, 8), ("f32", 64, 4)])
@pytest.mark.parametrize("M,k_max,k_min", [(40, 16, 4), (40, 40, 33), (3, 3, 1), (256, 32, 8), (200, 64, 8)])
def test_grid_step_exact_bit_exact(dtype, h_r, k_t, M, k_max, k_min):
    D = _dyn()
    V, d = 7919, 384       # prime V, ragged clusters
    W, rt, part, c, r = _setup(V, d, M, h_r, dtype, "exact")
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    k_t = min(k_t, k_min * c.min_size)  # the ABI requires k_t <= k * min |C_m| (<= |V_S|)
    st = D.DraftStep(c, r, 1, k_t, z_out=True)
    assert st.launches == 1
    for t in range(4):
        hp, e, hn = S.step_inputs(1, d, t, dtype, "exact", h_r=h_r)
        hp, e, hn = hp.to(DEV), e.to(DEV), hn.to(DEV)
        used = _ran_gstep(D, lambda: st(hp, e, hn, t=t, k_max=k_max, k_min=k_min))
        assert used, "the B = 1 draft step did not run the grid step"
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, k_max, k_min, k_t)[0]
        _exact_check(st, ref, k_t)
    assert st.ws.error() == "DS_OK"


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_grid_step_ties(dtype):
    """Injected exact ties: two router rows duplicated (score tie -> lower cluster id, R7) and two
    token rows duplicated (logit tie -> lower token id, R7)."""
    D = _dyn()
    V, d, M, h_r, k_t = 5003, 256, 64, 32, 16
    W = S.lm_head(V, d, 0, dtype, "exact")
    rt = list(S.router(d, h_r, M, 1, dtype, "exact"))
    tau = S.random_partition(V, M, 2)
    perm, off = O.layout(tau, M)
    # the two best-scoring clusters at t = 0 get identical W2 rows and b2 (an exact score tie at the
    # selection boundary is then likely); duplicate token rows inside one cluster
    W2, b2 = rt[2].clone(), rt[3].clone()
    W2[7] = W2[3]
    b2[7] = b2[3]
    W2[11] = W2[3]
    b2[11] = b2[3]
    rt[2], rt[3] = W2, b2
    members = np.nonzero(tau == tau[0])[0]
    if len(members) > 1:
        W[int(members[1])] = W[int(members[0])]
    c = D.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = D.Router(*[x.to(DEV) for x in rt])
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    k_t = min(k_t, c.min_size)  # k = 1 below: k_t <= |C_m| for every cluster
    st = D.DraftStep(c, r, 1, k_t, z_out=True)
    for t, (kmax, kmin) in enumerate([(1, 1), (2, 2), (4, 1), (8, 8), (12, 12)]):
        hp, e, hn = S.step_inputs(1, d, t, dtype, "exact", h_r=h_r)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=0, k_max=kmax, k_min=kmin)
        torch.cuda.synchronize()
        ref = O.draft_step(part_of(perm, off), ro, Wo, f64(hp), f64(e), f64(hn), 0, kmax, kmin, k_t)[0]
        _exact_check(st, ref, k_t)


def part_of(perm, off):
    return {"perm": perm, "offsets": off}


def test_grid_step_llama3_random_full_size():
    """Llama-3 head (V 128256, d 4096, M 256, h_r 128) at k = 32 and 8, random regime, bf16; scores
    within 1e-5 rms (the fp32 router error measured in SURVEY §8(c) O2 is 3.9e-7 at this shape)."""
    D = _dyn()
    C = S.CONFIGS["llama3"]
    W, rt, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    st = D.DraftStep(c, r, 1, C.k_t, z_out=True)
    for t in (0, 1, 2, 5, 7):
        hp, e, hn = [x.to(DEV) for x in S.step_inputs(1, C.d, t, "bf16")]
        assert _ran_gstep(D, lambda: st(hp, e, hn, t=t, k_max=C.k_max, k_min=C.k_min))
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t)[0]
        s_ref = ref["scores"]
        assert np.max(np.abs(st.scores[0].cpu().numpy() - s_ref)) <= score_tol(s_ref)
        cnt = st.sel_count[0].item()
        sel = np.array(st.sel[0, :cnt].cpu().tolist())
        if selection_certified(s_ref, ref["k"]):
            assert sel.tolist() == ref["sel"].tolist()
            rb = ref
        else:
            rb = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t,
                              sel_override=[sel])[0]
        assert st.sl_offsets[0, :cnt + 1].cpu().tolist() == rb["sl_offsets"].tolist()
        n = len(rb["V_S"])
        assert np.max(np.abs(st.z[0, :n].cpu().double().numpy() - rb["z"])) <= 2e-2
        check_topk(st.top_ids[0].cpu().numpy(), st.top_logits[0].cpu().numpy(), st.top_logp[0].cpu().numpy(),
                   st.lse[0].item(), rb["z"], rb["V_S"], C.k_t, torch.bfloat16)


@pytest.mark.parametrize("regime", ["exact", "random"])
def test_route_then_head_matches_oracle(regime):
    """dynaspec_step_route on S_m (router + TopK, Alg. 1 line 8) || nothing on S_d, join,
    dynaspec_step_head (line 10-11): the two-call split equals the oracle."""
    D = _dyn()
    if regime == "exact":
        V, d, M, h_r, k_t, kmax, kmin, dt = 7919, 512, 64, 32, 8, 16, 4, "bf16"
    else:
        C = S.CONFIGS["llama3"]
        V, d, M, h_r, k_t, kmax, kmin, dt = C.V, C.d, C.M, C.h_r, C.k_t, C.k_max, C.k_min, "bf16"
    W, rt, part, c, r = _setup(V, d, M, h_r, dt, regime)
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    st = D.DraftStep(c, r, 1, k_t, z_out=True)
    s_meta = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    for t in (0, 3):
        hp, e, hn = [x.to(DEV) for x in S.step_inputs(1, d, t, dt, regime, h_r=h_r)]
        ev0, ev1 = torch.cuda.Event(), torch.cuda.Event()
        ev0.record(cur)
        s_meta.wait_event(ev0)
        st.route(hp, e, t, kmax, kmin, s_meta)
        ev1.record(s_meta)
        cur.wait_event(ev1)
        used = _ran_gstep(D, lambda: st.head(hn, t, kmax, kmin, cur))
        assert used, "the B = 1 head did not run the grid-step kernel (head-only mode)"
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, kmax, kmin, k_t)[0]
        cnt = st.sel_count[0].item()
        sel = st.sel[0, :cnt].cpu().numpy()
        if regime == "exact":
            _exact_check(st, ref, k_t)
            continue
        rb = ref if sel.tolist() == ref["sel"].tolist() else O.draft_step(
            part, ro, Wo, f64(hp), f64(e), f64(hn), t, kmax, kmin, k_t, sel_override=[sel])[0]
        if selection_certified(ref["scores"], ref["k"]):
            assert sel.tolist() == ref["sel"].tolist()
        n = len(rb["V_S"])
        assert np.max(np.abs(st.z[0, :n].cpu().double().numpy() - rb["z"])) <= 2e-2
        check_topk(st.top_ids[0].cpu().numpy(), st.top_logits[0].cpu().numpy(), st.top_logp[0].cpu().numpy(),
                   st.lse[0].item(), rb["z"], rb["V_S"], k_t, torch.bfloat16)


def test_head_only_max_shortlist_sentinel():
    """A row whose |V_S| exceeds max_shortlist is not computed: top ids -1, lse NaN (dynaspec.h)."""
    D = _dyn()
    V, d, M = 4099, 256, 16
    W, rt, part, c, r = _setup(V, d, M, 8, "bf16", "exact")
    sel = torch.arange(M, dtype=torch.int32, device=DEV).view(1, M)
    cnt = torch.tensor([M], dtype=torch.int32, device=DEV)
    off = c.offsets.view(1, M + 1).contiguous()
    hn = S.hidden(1, d, 5, "bf16", "exact").to(DEV)
    out = D.head_forward(c, hn, sel, cnt, off, 8, max_shortlist=V - 1, z_out=True)
    torch.cuda.synchronize()
    assert (out["top_ids"] == -1).all() and torch.isnan(out["lse"]).all()
    out = D.head_forward(c, hn, sel, cnt, off, 8, max_shortlist=V, z_out=True)   # fits: computed
    torch.cuda.synchronize()
    z = out["z"][0, :V].cpu().double().numpy()
    ref = O.head(f64(hn)[0], f64(W), part["perm"])[0]
    assert np.array_equal(z, ref), "k = M: every logit of the dense head"


def test_workspace_shared_across_entry_points():
    """One workspace serves a B = 4 fused step (grid-wide step kernel), a B = 1 grid step, a head-only
    call and another B = 1 step in any order (fixed polled-record prefix, internal.h)."""
    D = _dyn()
    V, d, M, h_r, k_t = 7919, 384, 40, 16, 8
    W, rt, part, c, r = _setup(V, d, M, h_r, "bf16", "exact")
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    st1 = D.DraftStep(c, r, 1, k_t, z_out=True)
    st4 = D.DraftStep(c, r, 4, k_t, z_out=True)
    ws = D.Workspace(max(st1.ws.nbytes, st4.ws.nbytes), DEV)
    st1.ws = st4.ws = ws
    for it in range(3):
        hp4, e4, hn4 = [x.to(DEV) for x in S.step_inputs(4, d, 10 + it, "bf16", "exact", h_r=h_r)]
        st4(hp4, e4, hn4, t=0, k_max=8, k_min=8)
        hp, e, hn = [x.to(DEV) for x in S.step_inputs(1, d, it, "bf16", "exact", h_r=h_r)]
        st1(hp, e, hn, t=it, k_max=16, k_min=4)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), it, 16, 4, k_t)[0]
        _exact_check(st1, ref, k_t)
        refs4 = O.draft_step(part, ro, Wo, f64(hp4), f64(e4), f64(hn4), 0, 8, 8, k_t)
        for b in range(4):
            cnt = st4.sel_count[b].item()
            assert st4.sel[b, :cnt].cpu().tolist() == refs4[b]["sel"].tolist()
            check_topk(st4.top_ids[b].cpu().numpy(), st4.top_logits[b].cpu().numpy(),
                       st4.top_logp[b].cpu().numpy(), st4.lse[b].item(), refs4[b]["z"], refs4[b]["V_S"], k_t,
                       torch.float32, exact=True)
        out = D.head_forward(c, hn, st1.sel[:1], st1.sel_count[:1], st1.sl_offsets[:1], k_t, ws=ws)
        torch.cuda.synchronize()
        assert out["top_ids"][0].tolist() == st1.top_ids[0].tolist()
    assert ws.error() == "DS_OK"


def test_grid_step_pdl_chain_in_graph_matches_eager():
    """Eight PDL-chained steps (early launch_dependents, zero-polled words re-zeroed by the merger) in
    one CUDA graph give the same bytes as eight eagerly launched steps, over repeated replays."""
    D = _dyn()
    C = S.CONFIGS["llama2"]
    W, rt, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    P = C.positions
    steps = [D.DraftStep(c, r, 1, C.k_t) for _ in range(P)]
    ins = [[x.to(DEV) for x in S.step_inputs(1, C.d, t, "bf16")] for t in range(P)]
    eager = []
    for t in range(P):
        steps[t](*ins[t], t, C.k_max, C.k_min)
        torch.cuda.synchronize()
        eager.append({k: v.clone() for k, v in steps[t].outputs().items() if v is not None})
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for t in range(P):
            steps[t](*ins[t], t, C.k_max, C.k_min)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for t in range(P):
            steps[t](*ins[t], t, C.k_max, C.k_min)
    for rep in range(5):
        for st in steps:
            st.top_ids.fill_(-7)
        g.replay()
        torch.cuda.synchronize()
        for t in range(P):
            o = steps[t].outputs()
            for k, v in eager[t].items():
                assert torch.equal(o[k].view(torch.uint8), v.view(torch.uint8)), (rep, t, k)
    for st in steps:
        assert st.ws.error() == "DS_OK"
