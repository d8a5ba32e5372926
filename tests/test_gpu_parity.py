"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bar (task rule ③, BASELINE.json north star): bit-exact for cluster ids, selections,
offsets and token ids; logits within 2e-2 (bf16) / 1e-5 relative (fp32); in the exact
regime (integer-grid inputs) scores and logits are bit-exact too.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import dynaspec_oracle as O
from synth import inputs as S
from tests.parity import Rows, check_topk, f64, score_tol, selection_certified

pytestmark = pytest.mark.gpu

D = None


def _dyn():
    global D
    if D is None:
        from paper_2510_13847_b200 import dynaspec
        D = dynaspec
    return D


DEV = "cuda"
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "e2e1.json")))


def _partition(V, M, seed=2):
    tau = S.random_partition(V, M, seed)
    perm, off = O.layout(tau, M)
    return tau, {"perm": perm, "offsets": off}


def _setup(V, d, M, h_r, dtype, regime, seed_part=2):
    W = S.lm_head(V, d, 0, dtype, regime)
    rt = S.router(d, h_r, M, 1, dtype, regime)
    tau, part = _partition(V, M, seed_part)
    c = _dyn().Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = _dyn().Router(*[None if x is None else x.to(DEV) for x in rt])
    return W, rt, tau, part, c, r


def _oracle_router(rt):
    return tuple(f64(x) for x in rt)


# ------------------------------------------------------------------ golden worked example

@pytest.mark.parametrize("cstep_head", ["1", "0"])  # head-only cluster kernel (B = 1) or the grid head
def test_e2e1_golden_on_gpu(cstep_head, monkeypatch):
    monkeypatch.setenv("DS_CSTEP_HEAD", cstep_head)
    Dy = _dyn()
    d = 8  # pad the 2-D example with zero dimensions (kernels need d % 8 == 0); dot products unchanged
    W = torch.zeros((6, d), dtype=torch.float32)
    W[:, :2] = torch.tensor(GOLD["W_rows"], dtype=torch.float32)
    tau = torch.tensor(GOLD["partition"]["tau"], dtype=torch.int32)
    c = Dy.Clusters.from_tau(W.to(DEV), tau.to(DEV), 3)
    assert c.perm.cpu().tolist() == GOLD["partition"]["perm"]
    assert c.offsets.cpu().tolist() == GOLD["partition"]["offsets"]
    R = torch.zeros((3, 2 * d))
    rows = torch.tensor(GOLD["router_linear_rows"], dtype=torch.float32)
    R[:, 0:2] = rows[:, 0:2]            # acts on h_prev
    R[:, d:d + 2] = rows[:, 2:4]        # acts on e
    r = Dy.Router(R.to(DEV), torch.zeros(3, device=DEV))
    hp = torch.zeros((1, d)); hp[0, :2] = torch.tensor(GOLD["h_prev"], dtype=torch.float32)
    e = torch.zeros((1, d)); e[0, :2] = torch.tensor(GOLD["e"], dtype=torch.float32)
    hn = torch.zeros((1, d)); hn[0, :2] = torch.tensor(GOLD["h_new"], dtype=torch.float32)
    s = Dy.meta_score(r, hp.to(DEV), e.to(DEV))
    assert s.cpu()[0].tolist() == GOLD["scores"]
    for case in GOLD["cases"]:
        k = case["k"]
        sel, cnt, off = Dy.select(s, c, k)
        assert cnt.item() == k and sel.cpu()[0, :k].tolist() == case["sel"]
        assert off.cpu()[0, :k + 1].tolist() == case["sl_offsets"]
        kt = len(case["V_S"])
        out = Dy.head_forward(c, hn.to(DEV), sel, cnt, off, kt, z_out=True)
        assert out["z"].cpu()[0, :kt].tolist() == case["z"]
        assert out["top_ids"].cpu()[0].tolist() == case["top_ids"]
        assert abs(out["lse"].item() - case["lse"]) < 1e-6
        # draft_step (two streams, and the fused one-launch step) reproduces the same step
        for two in (True, False):
            st = Dy.DraftStep(c, r, 1, kt, two_streams=two)
            st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=0, k_max=k, k_min=1)
            torch.cuda.synchronize()
            assert st.top_ids.cpu()[0].tolist() == case["top_ids"]
            assert st.sel.cpu()[0, :k].tolist() == case["sel"]
            assert abs(st.lse.item() - case["lse"]) < 1e-6
    # tie variants: lower cluster id / lower token id win (R7)
    R2 = R.clone(); R2[0, 0] = 2.0
    s2 = Dy.meta_score(Dy.Router(R2.to(DEV), torch.zeros(3, device=DEV)), hp.to(DEV), e.to(DEV))
    sel, cnt, _ = Dy.select(s2, c, 1)
    assert sel.cpu()[0, 0].item() == 0
    tv = GOLD["tie_variants"]["h_new_3_2"]
    hn2 = torch.zeros((1, d)); hn2[0, :2] = torch.tensor(tv["h_new"], dtype=torch.float32)
    sel, cnt, off = Dy.select(s, c, 2)
    out = Dy.head_forward(c, hn2.to(DEV), sel, cnt, off, 4, z_out=True)
    assert out["z"].cpu()[0, :4].tolist() == tv["z"]
    assert out["top_ids"].cpu()[0].tolist() == tv["top_ids"]


# ------------------------------------------------------------------ exact regime: bit-exact

@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("shared", [False, True])
@pytest.mark.parametrize("cstep_head", ["1", "0"])  # head-only cluster kernel (B = 1) or the grid head
def test_exact_regime_pipeline(dtype, shared, fused, cstep_head, monkeypatch):
    monkeypatch.setenv("DS_CSTEP_HEAD", cstep_head)
    Dy = _dyn()
    V, d, M, h_r, B = 5003, 256, 24, 16, 3   # ragged V (prime), several tiles, ragged clusters
    W, rt, tau, part, c, r = _setup(V, d, M, h_r, dtype, "exact")
    Wo = Rows(W)
    ro = _oracle_router(rt)
    k_t = 8
    st = Dy.DraftStep(c, r, B, k_t, shared=shared, z_out=True, two_streams=not fused)
    # fused: one launch, or one grid step per row (B <= DS_GSTEP_ROWS_MAX); two streams: router + head
    assert (st.launches in (1, B)) if fused else st.launches >= 2
    for t in range(4):
        hp, e, hn = S.step_inputs(B, d, t, dtype, "exact", h_r=h_r)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=8, k_min=2)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, 8, 2, k_t, shared=shared)
        scores = st.scores.cpu().numpy()
        for b in range(B):
            assert np.array_equal(scores[b], ref[b]["scores"].astype(np.float32)), "scores not bit-exact"
        rows = 1 if shared else B
        for b in range(rows):
            cnt = st.sel_count[b].item()
            assert st.sel[b, :cnt].cpu().tolist() == ref[b]["sel"].tolist()
            assert st.sl_offsets[b, :cnt + 1].cpu().tolist() == ref[b]["sl_offsets"].tolist()
        for b in range(B):
            n = len(ref[b]["V_S"])
            z = st.z[b, :n].cpu().numpy()
            assert np.array_equal(z, ref[b]["z"].astype(np.float32)), "logits not bit-exact"
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), ref[b]["z"], ref[b]["V_S"], k_t, torch.float32, exact=True)


@pytest.mark.parametrize("cstep_head", ["1", "0"])  # head-only cluster kernel (B = 1) or the grid head
def test_exact_ties_injected(cstep_head, monkeypatch):
    monkeypatch.setenv("DS_CSTEP_HEAD", cstep_head)
    """Duplicated router rows (score ties -> lower cluster id) and duplicated W rows
    (logit ties -> lower token id), exact regime."""
    Dy = _dyn()
    V, d, M = 2000, 64, 10
    W = S.lm_head(V, d, 0, "bf16", "exact")
    hn0 = S.step_inputs(2, d, 0, "bf16", "exact", h_r=0)[2]
    top = (torch.sign(hn0[0].float()) * 127 * 2.0 ** -6).to(torch.bfloat16)
    W[7] = top; W[901] = top; W[1500] = top   # the maximal logit for row 0 at t=0, tied 3 ways
    rt = list(S.router(d, 0, M, 1, "bf16", "exact"))
    rt[0][6] = rt[0][2]; rt[1][6] = rt[1][2]   # clusters 2 and 6: identical scores
    tau, part = _partition(V, M)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    r = Dy.Router(rt[0].to(DEV), rt[1].to(DEV))
    for t in range(6):
        hp, e, hn = S.step_inputs(2, d, t, "bf16", "exact", h_r=0)
        hn = hn.clone()
        for kk in range(1, M + 1):
            s = Dy.meta_score(r, hp.to(DEV), e.to(DEV))
            sel, cnt, off = Dy.select(s, c, kk)
            ref_s = O.meta_score(f64(rt[0]), f64(rt[1]), None, None, f64(hp), f64(e))
            for b in range(2):
                assert sel[b, :kk].cpu().tolist() == O.select(ref_s[b], kk).tolist()
        sel_all = torch.arange(M, dtype=torch.int32, device=DEV).repeat(2, 1)
        cnt_all = torch.full((2,), M, dtype=torch.int32, device=DEV)
        off_all = c.offsets.repeat(2, 1)
        out = Dy.head_forward(c, hn.to(DEV), sel_all, cnt_all, off_all, 64)
        dense = O.dense_head(f64(hn), f64(W), 64)
        for b in range(2):
            assert out["top_ids"][b].cpu().tolist() == dense[b]["top_ids"].tolist()
        if t == 0:
            assert out["top_ids"][0, :3].cpu().tolist() == [7, 901, 1500]


# ------------------------------------------------------------------ random regime

@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("cfg,dtype,B", [("tiny", "bf16", 1), ("tiny", "f32", 1), ("llama2", "bf16", 1),
                                         ("tiny", "bf16", 8), ("llama3", "bf16", 4)])
def test_random_regime_config(cfg, dtype, B, fused):
    Dy = _dyn()
    C = S.CONFIGS[cfg]
    W, rt, tau, part, c, r = _setup(C.V, C.d, C.M, C.h_r, dtype, "random")
    Wo, ro = Rows(W), _oracle_router(rt)
    k_t = C.k_t
    st = Dy.DraftStep(c, r, B, k_t, z_out=True, two_streams=not fused)
    tdt = S.TORCH_DTYPES[dtype]
    for t in range(min(C.positions, 4)):
        hp, e, hn = S.step_inputs(B, C.d, t, dtype)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=C.k_max, k_min=C.k_min)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, k_t)
        s_gpu = st.scores.cpu().numpy()
        for b in range(B):
            s_ref = ref[b]["scores"]
            assert np.max(np.abs(s_gpu[b] - s_ref)) <= score_tol(s_ref)
            cnt = st.sel_count[b].item()
            sel_gpu = np.array(st.sel[b, :cnt].cpu().tolist())
            if selection_certified(s_ref, ref[b]["k"]):
                assert sel_gpu.tolist() == ref[b]["sel"].tolist()
                rb = ref[b]
            else:   # conditional parity: feed the GPU's selection back to the oracle
                rb = O.draft_step(part, ro, Wo, f64(hp[b:b + 1]), f64(e[b:b + 1]), f64(hn[b:b + 1]), t, C.k_max,
                                  C.k_min, k_t, sel_override=[sel_gpu])[0]
            assert st.sl_offsets[b, :cnt + 1].cpu().tolist() == rb["sl_offsets"].tolist()
            n = len(rb["V_S"])
            z = st.z[b, :n].cpu().numpy().astype(np.float64)
            if tdt == torch.bfloat16:
                assert np.max(np.abs(z - rb["z"])) <= 2e-2
            else:
                rms = np.sqrt(np.mean(rb["z"] ** 2))
                assert np.all(np.abs(z - rb["z"]) <= 1e-5 * np.maximum(np.abs(rb["z"]), rms))
            check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                       st.lse[b].item(), rb["z"], rb["V_S"], k_t, tdt)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("positions", [(0, 2)])
@pytest.mark.parametrize("cstep_head", ["1", "0"])  # head-only cluster kernel (B = 1) or the grid head
def test_llama3_full_size(positions, fused, cstep_head, monkeypatch):
    monkeypatch.setenv("DS_CSTEP_HEAD", cstep_head)
    """BASELINE configs[2] at full size (V=128256, d=4096, M=256, bf16), the bench's launch
    configuration (two streams, B=1); every logit of V_S compared with the oracle."""
    Dy = _dyn()
    C = S.CONFIGS["llama3"]
    W, rt, tau, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    Wo, ro = Rows(W), _oracle_router(rt)
    st = Dy.DraftStep(c, r, 1, C.k_t, z_out=True, two_streams=not fused)
    for t in positions:
        hp, e, hn = S.step_inputs(1, C.d, t, "bf16")
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=C.k_max, k_min=C.k_min)
        torch.cuda.synchronize()
        ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t)[0]
        cnt = st.sel_count[0].item()
        assert cnt == ref["k"]
        sel_gpu = st.sel[0, :cnt].cpu().numpy()
        if not selection_certified(ref["scores"], ref["k"]):
            ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t,
                               sel_override=[sel_gpu])[0]
        assert sel_gpu.tolist() == ref["sel"].tolist()
        n = len(ref["V_S"])
        assert st.sl_offsets[0, cnt].item() == n
        z = st.z[0, :n].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(z - ref["z"])) <= 2e-2
        check_topk(st.top_ids[0].cpu().numpy(), st.top_logits[0].cpu().numpy(), st.top_logp[0].cpu().numpy(),
                   st.lse[0].item(), ref["z"], ref["V_S"], C.k_t, torch.bfloat16)


@pytest.mark.parametrize("fused", [True, False])
def test_shared_tree_mode_qwen_shape(fused):
    """Tree mode (R9): R=10 sibling rows share the union shortlist (Qwen-2.5 head shape)."""
    Dy = _dyn()
    C = S.CONFIGS["qwen25"]
    W, rt, tau, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    Wo, ro = Rows(W), _oracle_router(rt)
    st = Dy.DraftStep(c, r, C.B, C.k_t, shared=True, z_out=True, two_streams=not fused)
    t = 2
    hp, e, hn = S.step_inputs(C.B, C.d, t, "bf16", sibling_eps=0.1)
    st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=C.k_max, k_min=C.k_min)
    torch.cuda.synchronize()
    cnt = st.sel_count[0].item()
    sel_gpu = st.sel[0, :cnt].cpu().numpy()
    ref = O.draft_step(part, ro, Wo, f64(hp), f64(e), f64(hn), t, C.k_max, C.k_min, C.k_t, shared=True,
                       sel_override=[sel_gpu] * C.B)
    scores_ref = ref[0]["scores"]
    ok = all(selection_certified(O.meta_score(*ro, f64(hp), f64(e))[b], ref[0]["k"]) for b in range(C.B))
    if ok:
        assert sel_gpu.tolist() == O.select_shared(O.meta_score(*ro, f64(hp), f64(e)), ref[0]["k"]).tolist()
    for b in range(C.B):
        n = len(ref[b]["V_S"])
        z = st.z[b, :n].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(z - ref[b]["z"])) <= 2e-2
        check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                   st.lse[b].item(), ref[b]["z"], ref[b]["V_S"], C.k_t, torch.bfloat16)
    del scores_ref


# ------------------------------------------------------------------ invariants / edge cases

def test_k_equals_M_is_dense():
    Dy = _dyn()
    V, d, M = 7001, 512, 16
    W, rt, tau, part, c, r = _setup(V, d, M, 8, "bf16", "random")
    hn = S.hidden(2, d, 77, "bf16")
    sel = torch.arange(M, dtype=torch.int32, device=DEV).repeat(2, 1)
    cnt = torch.full((2,), M, dtype=torch.int32, device=DEV)
    off = c.offsets.repeat(2, 1)
    out = Dy.head_forward(c, hn.to(DEV), sel, cnt, off, 16, z_out=True)
    dense = O.dense_head(f64(hn), f64(W), 16)
    perm = c.perm.cpu().numpy()
    for b in range(2):
        z = out["z"][b].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(z - dense[b]["z"][perm])) <= 2e-2     # shortlist logits == dense logits at ids
        assert out["top_ids"][b, 0].item() == dense[b]["top_ids"][0]
        assert abs(out["lse"][b].item() - dense[b]["lse"]) <= 2e-2


@pytest.mark.parametrize("cstep_head", ["1", "0"])  # head-only cluster kernel (B = 1) or the grid head
def test_edge_cases_small_clusters_padding_and_singletons(cstep_head, monkeypatch):
    monkeypatch.setenv("DS_CSTEP_HEAD", cstep_head)
    Dy = _dyn()
    V, d, M = 40, 8, 20
    W = S.lm_head(V, d, 3, "f32", "exact")
    tau = np.arange(V) % M
    tau[0] = 5                                    # cluster 0 = {20}, size 1 ... sizes 1..3
    part_perm, part_off = O.layout(tau, M)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    assert c.min_size == 1
    hn = S.hidden(1, d, 5, "f32", "exact")
    for m in range(M):
        sel = torch.tensor([[m] + [0] * (M - 1)], dtype=torch.int32, device=DEV)
        cnt = torch.tensor([1], dtype=torch.int32, device=DEV)
        off = torch.zeros((1, M + 1), dtype=torch.int32, device=DEV)
        size = int(part_off[m + 1] - part_off[m])
        off[0, 1] = size
        out = Dy.head_forward(c, hn.to(DEV), sel, cnt, off, 5, z_out=True)
        V_S = O.shortlist([m], part_perm, part_off)
        z = O.head(f64(hn)[0], f64(W), V_S)[0]
        check_topk(out["top_ids"][0].cpu().numpy(), out["top_logits"][0].cpu().numpy(),
                   out["top_logp"][0].cpu().numpy(), out["lse"][0].item(), z, V_S, 5, torch.float32, exact=True)
        if size == 1:
            assert out["top_logp"][0, 0].item() == 0.0          # |V_S| = 1 => p = 1


def test_single_cluster_M1_and_d8():
    Dy = _dyn()
    V, d = 333, 8
    W = S.lm_head(V, d, 4, "bf16", "random")
    c = Dy.Clusters.from_tau(W.to(DEV), torch.zeros(V, dtype=torch.int32, device=DEV), 1)
    hn = S.hidden(1, d, 9, "bf16")
    sel, cnt, off = Dy.select(torch.zeros((1, 1), device=DEV), c, 1)
    out = Dy.head_forward(c, hn.to(DEV), sel, cnt, off, 64, z_out=True)
    dense = O.dense_head(f64(hn), f64(W), 64)[0]
    assert out["top_ids"][0].cpu().tolist()[:3] == dense["top_ids"][:3].tolist()


def test_determinism_bytes():
    Dy = _dyn()
    C = S.CONFIGS["tiny"]
    W, rt, tau, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    hp, e, hn = S.step_inputs(4, C.d, 0, "bf16")
    outs = []
    for two in (True, True, False, False):
        st = Dy.DraftStep(c, r, 4, 16, z_out=True, two_streams=two)
        st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=0, k_max=8, k_min=8)
        torch.cuda.synchronize()
        outs.append({k: v.clone() for k, v in st.outputs().items() if v is not None})
    for k in outs[0]:
        assert torch.equal(outs[0][k].view(torch.uint8), outs[1][k].view(torch.uint8)), k
        assert torch.equal(outs[2][k].view(torch.uint8), outs[3][k].view(torch.uint8)), k


def test_error_codes():
    Dy = _dyn()
    V, d, M = 100, 16, 4
    W = S.lm_head(V, d, 0, "bf16").to(DEV)
    tau = torch.as_tensor(np.arange(V) % M, dtype=torch.int32, device=DEV)
    c = Dy.Clusters.from_tau(W, tau, M)
    r = Dy.Router(*[x.to(DEV) for x in S.router(d, 8, M, 1, "bf16")])
    s = torch.zeros((1, M), device=DEV)
    with pytest.raises(Dy.DynaspecError) as ei:
        Dy.select(s, c, M + 1)
    assert ei.value.name == "DS_ERR_INVALID_BUDGET"
    with pytest.raises(Dy.DynaspecError) as ei:
        Dy.select(s, c, 0)
    assert ei.value.name == "DS_ERR_INVALID_BUDGET"
    sel, cnt, off = Dy.select(s, c, 1)
    with pytest.raises(Dy.DynaspecError) as ei:
        Dy.head_forward(c, torch.zeros((1, d), dtype=torch.bfloat16, device=DEV), sel, cnt, off, 65)
    assert ei.value.name == "DS_ERR_INVALID_BUDGET"
    bad = torch.full((V,), M, dtype=torch.int32, device=DEV)
    with pytest.raises(Dy.DynaspecError) as ei:
        Dy.Clusters.from_tau(W, bad, M)
    assert ei.value.name == "DS_ERR_INVALID_CLUSTER_ID"
    gap = torch.zeros(V, dtype=torch.int32, device=DEV)
    with pytest.raises(Dy.DynaspecError) as ei:
        Dy.Clusters.from_tau(W, gap, M)
    assert ei.value.name == "DS_ERR_EMPTY_SHORTLIST"
    st = Dy.DraftStep(c, r, 1, 8)
    z = torch.zeros((1, d), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(Dy.DynaspecError) as ei:
        st(z, z, z, t=0, k_max=M + 1, k_min=1)
    assert ei.value.name == "DS_ERR_INVALID_BUDGET"
    with pytest.raises(Dy.DynaspecError) as ei:   # k_t > k * min_size
        Dy.DraftStep(c, r, 1, 64)(z, z, z, t=0, k_max=1, k_min=1)
    assert ei.value.name == "DS_ERR_INVALID_BUDGET"


# ------------------------------------------------------------------ tcgen05 shared-shortlist head (S5')

@pytest.mark.parametrize("th", ["1", "0"])  # balanced tree head (th.cu, R <= 16) / general tc_head
@pytest.mark.parametrize("R,d", [(4, 256), (10, 200), (16, 128), (17, 512), (64, 128)])
def test_tc_head_exact_bit_exact(R, d, th, monkeypatch):
    """Tree rows sharing one shortlist on the tensor cores: every logit bit-exact vs the oracle
    (exact regime keeps partial sums < 2^21 units), and identical to the CUDA-core path."""
    Dy = _dyn()
    monkeypatch.setenv("DS_TH", th)
    V, M = 6007, 24
    q = max(1, min(127, int((2 ** 21 / d) ** 0.5)))
    W = S.lm_head(V, d, 0, "bf16", "exact", q=q)
    tau, part = _partition(V, M)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    hn = S.hidden(R, d, 11, "bf16", "exact", q=q)
    rng = np.random.default_rng(R)
    for k in (1, 5, M):
        sel = np.sort(rng.choice(M, k, replace=False)).astype(np.int32)
        selt = torch.zeros((1, M), dtype=torch.int32)
        selt[0, :k] = torch.as_tensor(sel)
        off = torch.zeros((1, M + 1), dtype=torch.int32)
        off[0, :k + 1] = torch.as_tensor(O.shortlist_offsets(sel, part["offsets"]), dtype=torch.int32)
        cnt = torch.tensor([k], dtype=torch.int32)
        outs = {}
        for mode in ("tc", "cuda"):
            monkeypatch.setenv("DS_DISABLE_TC", "0" if mode == "tc" else "1")
            outs[mode] = Dy.head_forward(c, hn.to(DEV), selt.to(DEV), cnt.to(DEV), off.to(DEV), 8, shared=True,
                                         z_out=True)
        V_S = O.shortlist(sel, part["perm"], part["offsets"])
        zref = O.head(f64(hn), f64(W), V_S)
        n = len(V_S)
        for r in range(R):
            ztc = outs["tc"]["z"][r, :n].cpu().numpy()
            assert np.array_equal(ztc, zref[r].astype(np.float32)), f"tc logits not exact (R={R}, d={d}, k={k})"
            assert np.array_equal(ztc, outs["cuda"]["z"][r, :n].cpu().numpy())
            check_topk(outs["tc"]["top_ids"][r].cpu().numpy(), outs["tc"]["top_logits"][r].cpu().numpy(),
                       outs["tc"]["top_logp"][r].cpu().numpy(), outs["tc"]["lse"][r].item(), zref[r], V_S, 8,
                       torch.float32, exact=True)
            assert outs["tc"]["top_ids"][r].cpu().tolist() == outs["cuda"]["top_ids"][r].cpu().tolist()


@pytest.mark.parametrize("th,tc", [("1", "0"), ("0", "0"), ("0", "1")])
def test_tc_head_random_regime_qwen_full_size(th, tc, monkeypatch):
    """Qwen-2.5 head at full size (V=151936, d=3584, M=256), 10 tree rows, vs the oracle: the
    balanced tree head, the general tcgen05 head, and (DS_DISABLE_TC=1) the CUDA-core fused step —
    whose workspace is sized from a bounded plan (the full-vocabulary bound does not fit its
    shared memory at this shape)."""
    Dy = _dyn()
    monkeypatch.setenv("DS_DISABLE_TC", tc)
    monkeypatch.setenv("DS_TH", th)
    C = S.CONFIGS["qwen25"]
    W, rt, tau, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    st = Dy.DraftStep(c, r, C.B, C.k_t, shared=True, z_out=True)
    if tc == "0":
        assert st.launches == 2  # few-row router + tree head
    hp, e, hn = S.step_inputs(C.B, C.d, 0, "bf16", sibling_eps=0.1)
    st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=0, k_max=C.k_max, k_min=C.k_min)
    torch.cuda.synchronize()
    cnt = st.sel_count[0].item()
    sel_gpu = st.sel[0, :cnt].cpu().numpy()
    ref = O.draft_step(part, _oracle_router(rt), Rows(W), f64(hp), f64(e), f64(hn), 0, C.k_max, C.k_min, C.k_t,
                       shared=True, sel_override=[sel_gpu] * C.B)
    for b in range(C.B):
        n = len(ref[b]["V_S"])
        z = st.z[b, :n].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(z - ref[b]["z"])) <= 2e-2
        check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                   st.lse[b].item(), ref[b]["z"], ref[b]["V_S"], C.k_t, torch.bfloat16)


@pytest.mark.parametrize("R,kt", [(4, 1), (16, 16), (7, 5)])
def test_th_tree_head_ragged_exact(R, kt, monkeypatch):
    """Balanced tree head (th.cu): clusters of every size mod 8 (1..37 rows: pieces ending inside an
    8-row group, singletons, runs of adjacent selected clusters), k in {1, 3, M}; ids, logits and the
    token order bit-exact against the oracle, lse within the exact-regime bound; a shortlist bound
    below the union gives the documented sentinel (ids -1, lse NaN)."""
    Dy = _dyn()
    monkeypatch.setenv("DS_DISABLE_TC", "0")
    monkeypatch.setenv("DS_TH", "1")
    d, M = 192, 40
    sizes = np.array([1 + (7 * m) % 37 for m in range(M)])
    V = int(sizes.sum())
    tau = np.repeat(np.arange(M), sizes)
    np.random.default_rng(3).shuffle(tau)
    tau = O.canonical_relabel(tau, M) if hasattr(O, "canonical_relabel") else tau
    perm, offs = O.layout(tau, M)
    part = {"perm": perm, "offsets": offs}
    q = max(1, min(127, int((2 ** 21 / d) ** 0.5)))
    W = S.lm_head(V, d, 0, "bf16", "exact", q=q)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    hn = S.hidden(R, d, 17, "bf16", "exact", q=q)
    rng = np.random.default_rng(R + kt)
    for k in (1, 3, M):
        sel = np.sort(rng.choice(M, k, replace=False)).astype(np.int32)
        if int(sizes[sel].sum()) < kt:
            continue
        selt = torch.zeros((1, M), dtype=torch.int32)
        selt[0, :k] = torch.as_tensor(sel)
        off = torch.zeros((1, M + 1), dtype=torch.int32)
        off[0, :k + 1] = torch.as_tensor(O.shortlist_offsets(sel, part["offsets"]), dtype=torch.int32)
        cnt = torch.tensor([k], dtype=torch.int32)
        out = Dy.head_forward(c, hn.to(DEV), selt.to(DEV), cnt.to(DEV), off.to(DEV), kt, shared=True, z_out=True)
        V_S = O.shortlist(sel, part["perm"], part["offsets"])
        zref = O.head(f64(hn), f64(W), V_S)
        n = len(V_S)
        for r in range(R):
            assert np.array_equal(out["z"][r, :n].cpu().numpy(), zref[r].astype(np.float32)), (R, kt, k, r)
            check_topk(out["top_ids"][r].cpu().numpy(), out["top_logits"][r].cpu().numpy(),
                       out["top_logp"][r].cpu().numpy(), out["lse"][r].item(), zref[r], V_S, kt, torch.float32,
                       exact=True)
        if n > kt:
            out = Dy.head_forward(c, hn.to(DEV), selt.to(DEV), cnt.to(DEV), off.to(DEV), kt, shared=True,
                                  max_shortlist=n - 1)
            assert (out["top_ids"].cpu() == -1).all() and torch.isnan(out["lse"].cpu()).all()


# ------------------------------------------------------------------ batched per-row rows on tcgen05 (K5/S5')

@pytest.mark.parametrize("B", [8, 13, 64, 130])
def test_tc_batched_per_row_exact(B, monkeypatch):
    """Independent rows with their own selections, streamed once as their union on the tensor cores
    with per-row cluster masks and online (max, sum, top-k): top ids / logits / lse equal the oracle
    (exact regime) and the CUDA-core per-row path."""
    Dy = _dyn()
    V, d, M, k, kt = 9001, 256, 32, 6, 10
    q = max(1, min(127, int((2 ** 21 / d) ** 0.5)))
    W = S.lm_head(V, d, 0, "bf16", "exact", q=q)
    tau, part = _partition(V, M)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    hn = S.hidden(B, d, 17, "bf16", "exact", q=q)
    rng = np.random.default_rng(B)
    sel = torch.zeros((B, M), dtype=torch.int32)
    off = torch.zeros((B, M + 1), dtype=torch.int32)
    cnt = torch.full((B,), k, dtype=torch.int32)
    sels = []
    for b in range(B):
        sb = np.sort(rng.choice(M, k, replace=False))
        sels.append(sb)
        sel[b, :k] = torch.as_tensor(sb)
        off[b, :k + 1] = torch.as_tensor(O.shortlist_offsets(sb, part["offsets"]))
    outs = {}
    for mode in ("tc", "cuda"):
        monkeypatch.setenv("DS_DISABLE_TC", "0" if mode == "tc" else "1")
        outs[mode] = Dy.head_forward(c, hn.to(DEV), sel.to(DEV), cnt.to(DEV), off.to(DEV), kt)
    torch.cuda.synchronize()
    for b in range(B):
        V_S = O.shortlist(sels[b], part["perm"], part["offsets"])
        z = O.head(f64(hn)[b], f64(W), V_S)[0]
        check_topk(outs["tc"]["top_ids"][b].cpu().numpy(), outs["tc"]["top_logits"][b].cpu().numpy(),
                   outs["tc"]["top_logp"][b].cpu().numpy(), outs["tc"]["lse"][b].item(), z, V_S, kt, torch.float32,
                   exact=True)
    assert torch.equal(outs["tc"]["top_ids"], outs["cuda"]["top_ids"])
    assert torch.equal(outs["tc"]["top_logits"], outs["cuda"]["top_logits"])


@pytest.mark.parametrize("gh", ["1", "0"])  # grouped cluster-major head (gh.cu) / union-batched tc_head
def test_tc_batched_draft_step_llama3_b16(gh, monkeypatch):
    """Draft step at Llama-3 size with 16 independent rows (tcgen05 paths) vs the oracle."""
    Dy = _dyn()
    monkeypatch.setenv("DS_DISABLE_TC", "0")
    monkeypatch.setenv("DS_GH", gh)
    C = S.CONFIGS["llama3"]
    B = 16
    W, rt, tau, part, c, r = _setup(C.V, C.d, C.M, C.h_r, "bf16", "random")
    st = Dy.DraftStep(c, r, B, C.k_t)
    # router: one launch (meta_rows.cu) when the 16 rows' x fit its shared-memory staging, else two;
    # then gh (3) / union + tc head (2)
    assert st.launches in ((4, 5) if gh == "1" else (3, 4))
    hp, e, hn = S.step_inputs(B, C.d, 2, "bf16")
    st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=2, k_max=C.k_max, k_min=C.k_min)
    torch.cuda.synchronize()
    Wo, ro = Rows(W), _oracle_router(rt)
    for b in range(B):
        cnt = st.sel_count[b].item()
        sel_gpu = st.sel[b, :cnt].cpu().numpy()
        ref = O.draft_step(part, ro, Wo, f64(hp[b:b + 1]), f64(e[b:b + 1]), f64(hn[b:b + 1]), 2, C.k_max, C.k_min,
                           C.k_t, sel_override=[sel_gpu])[0]
        check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                   st.lse[b].item(), ref["z"], ref["V_S"], C.k_t, torch.bfloat16)


# ------------------------------------------------------------------ static frequency heads (NEXT-3)

@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_frequency_heads_fr_and_pa_fr(dtype):
    """FR-Spec (fixed K) and PA-FR (K_fr(t)) prefix heads vs the oracle at the Llama-3 shape."""
    Dy = _dyn()
    C = S.CONFIGS["llama3"]
    W = S.lm_head(C.V, C.d, 0, dtype)
    pi = O.frequency_ranking(S.zipf_token_counts(C.V))
    fh = Dy.FrequencyHead(W.to(DEV), pi)
    hn = S.hidden(2, C.d, 9, dtype)
    Wo = Rows(W)
    for t in (0, 2, 5):
        for K in (32768, O.budget_pa_fr(t, 32768)):
            out = fh.forward(hn.to(DEV), K, 8, z_out=True)
            ref = O.fr_head(f64(hn), Wo, pi, K, 8)
            tdt = S.TORCH_DTYPES[dtype]
            for b in range(2):
                z = out["z"][b, :K].cpu().numpy().astype(np.float64)
                if dtype == "bf16":
                    assert np.max(np.abs(z - ref[b]["z"])) <= 2e-2
                else:
                    rms = np.sqrt(np.mean(ref[b]["z"] ** 2))
                    assert np.all(np.abs(z - ref[b]["z"]) <= 1e-5 * np.maximum(np.abs(ref[b]["z"]), rms))
                check_topk(out["top_ids"][b].cpu().numpy(), out["top_logits"][b].cpu().numpy(),
                           out["top_logp"][b].cpu().numpy(), out["lse"][b].item(), ref[b]["z"], ref[b]["V_S"], 8,
                           tdt)


def test_router_many_rows_row_blocks():
    """B = 512 rows (the Gemma config's batch on one GPU): the layer-1 router kernel stages x in
    row blocks (grid z); scores and selections of sampled rows match the oracle."""
    Dy = _dyn()
    V, d, M, h_r, B = 20011, 512, 64, 32, 512
    W, rt, tau, part, c, r = _setup(V, d, M, h_r, "bf16", "random")
    hp, e, hn = S.step_inputs(B, d, 7, "bf16")
    st = Dy.DraftStep(c, r, B, 8)
    st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=2, k_max=16, k_min=4)
    torch.cuda.synchronize()
    ro = _oracle_router(rt)
    for b in (0, 1, 191, 192, 300, 511):
        ref = O.draft_step(part, ro, Rows(W), f64(hp[b:b + 1]), f64(e[b:b + 1]), f64(hn[b:b + 1]), 2, 16, 4, 8)[0]
        s_ref = ref["scores"]
        assert np.max(np.abs(st.scores[b].cpu().numpy() - s_ref)) <= score_tol(s_ref)
        if selection_certified(s_ref, ref["k"]):
            cnt = st.sel_count[b].item()
            assert st.sel[b, :cnt].cpu().tolist() == ref["sel"].tolist()


@pytest.mark.parametrize("online,th", [("1", "0"), ("0", "0"), ("0", "1")])
def test_tc_head_shared_online_epilogue_exact(online, th, monkeypatch):
    """Tree rows on the tensor cores without z_out and a per-CTA logit bound above 4 tiles: the
    online per-tile (max, sum, top-k) epilogue (and, forced off, the on-chip partial) give the
    oracle's top ids / logits exactly and its lse (exact regime)."""
    Dy = _dyn()
    monkeypatch.setenv("DS_DISABLE_TC", "0")
    monkeypatch.setenv("DS_TC_ONLINE", online)
    monkeypatch.setenv("DS_TH", th)  # th.cu: several 128-row tiles per CTA (double-buffered TMEM)
    V, d, M, R, kt = 80021, 256, 24, 10, 8
    q = max(1, min(127, int((2 ** 21 / d) ** 0.5)))
    W = S.lm_head(V, d, 0, "bf16", "exact", q=q)
    tau, part = _partition(V, M)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    hn = S.hidden(R, d, 13, "bf16", "exact", q=q)
    rng = np.random.default_rng(5)
    for k in (3, M):
        sel = np.sort(rng.choice(M, k, replace=False)).astype(np.int32)
        selt = torch.zeros((1, M), dtype=torch.int32)
        selt[0, :k] = torch.as_tensor(sel)
        off = torch.zeros((1, M + 1), dtype=torch.int32)
        off[0, :k + 1] = torch.as_tensor(O.shortlist_offsets(sel, part["offsets"]), dtype=torch.int32)
        cnt = torch.tensor([k], dtype=torch.int32)
        out = Dy.head_forward(c, hn.to(DEV), selt.to(DEV), cnt.to(DEV), off.to(DEV), kt, shared=True)
        V_S = O.shortlist(sel, part["perm"], part["offsets"])
        zref = O.head(f64(hn), f64(W), V_S)
        for r in range(R):
            check_topk(out["top_ids"][r].cpu().numpy(), out["top_logits"][r].cpu().numpy(),
                       out["top_logp"][r].cpu().numpy(), out["lse"][r].item(), zref[r], V_S, kt, torch.float32,
                       exact=True)


def test_gemma3_batched_full_size_sampled_rows(monkeypatch):
    """Gemma-3 head at full size (V 262144, d 5376, M 512, h_r 256) and the bench's batch (B = 64
    independent rows -> router + union + batched tcgen05 head), k = 16 (t = 2): sampled rows
    against the oracle (scores, selection, shortlist offsets, top-k, lse)."""
    Dy = _dyn()
    monkeypatch.setenv("DS_DISABLE_TC", "0")
    C = S.CONFIGS["gemma3"]
    B, t = 64, 2
    W = S.lm_head(C.V, C.d, 0, "bf16", device=DEV)
    tau = S.random_partition(C.V, C.M, 2)
    perm, off = O.layout(tau, C.M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W, torch.as_tensor(tau, dtype=torch.int32, device=DEV), C.M)
    rt = S.router(C.d, C.h_r, C.M, 1, "bf16")
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, C.k_t)
    hp, e, hn = S.step_inputs(B, C.d, t, "bf16")
    st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=C.k_max, k_min=C.k_min)
    torch.cuda.synchronize()
    Wo, ro = Rows(W), _oracle_router(rt)
    for b in (0, 37, 63):
        ref = O.draft_step(part, ro, Wo, f64(hp[b:b + 1]), f64(e[b:b + 1]), f64(hn[b:b + 1]), t, C.k_max, C.k_min,
                           C.k_t)[0]
        s_ref = ref["scores"]
        assert np.max(np.abs(st.scores[b].cpu().numpy() - s_ref)) <= score_tol(s_ref)
        cnt = st.sel_count[b].item()
        sel = np.array(st.sel[b, :cnt].cpu().tolist())
        if selection_certified(s_ref, ref["k"]):
            assert sel.tolist() == ref["sel"].tolist()
            rb = ref
        else:
            rb = O.draft_step(part, ro, Wo, f64(hp[b:b + 1]), f64(e[b:b + 1]), f64(hn[b:b + 1]), t, C.k_max,
                              C.k_min, C.k_t, sel_override=[sel])[0]
        assert st.sl_offsets[b, :cnt + 1].cpu().tolist() == rb["sl_offsets"].tolist()
        check_topk(st.top_ids[b].cpu().numpy(), st.top_logits[b].cpu().numpy(), st.top_logp[b].cpu().numpy(),
                   st.lse[b].item(), rb["z"], rb["V_S"], C.k_t, torch.bfloat16)
