"""The grouped cluster-major tcgen05 head (gh.cu, S5 for many independent rows)
through the C ABI against the oracle: exact regime bit-exact (ids, logits), ragged clusters of more
than one 256-token tile, more than 128 rows per cluster (row blocks), every k_t bound (register
lists of 8 / 16 / 32), and the Gemma-3 / Llama-3 batches at full size on sampled rows."""
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


def _exact_setup(V, d, M, seed=2):
    Dy = _dyn()
    W = S.lm_head(V, d, 0, "bf16", "exact")
    tau = S.random_partition(V, M, seed)
    perm, off = O.layout(tau, M)
    c = Dy.Clusters.from_tau(W.to(DEV), torch.as_tensor(tau, dtype=torch.int32, device=DEV), M)
    return W, tau, perm, off, c


def _random_selection(B, M, k, seed):
    rng = np.random.default_rng(seed)
    sel = np.zeros((B, M), dtype=np.int32)
    for b in range(B):
        sel[b, :k] = np.sort(rng.choice(M, size=k, replace=False))
    return sel


@pytest.mark.parametrize("B,k,k_t", [(16, 8, 8), (300, 16, 8), (12, 5, 1), (40, 6, 16), (9, 7, 32)])
def test_gh_exact_regime(B, k, k_t, monkeypatch):
    """Exact regime (every fp32 sum exact): every row's top-k_t ids and logits bit-exact and its lse
    within fp32 rounding of the oracle's, through dynaspec_head_forward's grouped path (B >= 8)."""
    monkeypatch.setenv("DS_GH_MIN_ROWS", "2")
    Dy = _dyn()
    V, d, M = 5003, 256, 24   # ragged V, clusters of ~100-400 tokens (1-2 vocabulary tiles)
    W, tau, perm, off, c = _exact_setup(V, d, M)
    assert max(np.diff(off)) > 256, "the partition must have clusters of more than one 256-token tile"
    hn = S.step_inputs(B, d, 0, "bf16", "exact")[2]
    sel = _random_selection(B, M, k, 11)
    cnt = np.full(B, k, dtype=np.int32)
    sl = np.zeros((B, M + 1), dtype=np.int32)
    for b in range(B):
        sl[b, :k + 1] = O.shortlist_offsets(sel[b, :k], off)
    out = Dy.head_forward(c, hn.to(DEV), torch.as_tensor(sel, device=DEV), torch.as_tensor(cnt, device=DEV),
                          torch.as_tensor(sl, device=DEV), k_t)
    torch.cuda.synchronize()
    Wo = Rows(W)
    for b in range(B):
        VS = O.shortlist(sel[b, :k], perm, off)
        z = O.head(f64(hn[b]), Wo, VS)[0]
        check_topk(out["top_ids"][b].cpu().numpy(), out["top_logits"][b].cpu().numpy(),
                   out["top_logp"][b].cpu().numpy(), out["lse"][b].item(), z, VS, k_t, torch.float32, exact=True)


def test_gh_matches_other_heads_exact(monkeypatch):
    """Exact regime: the grouped head and the CUDA-core head give identical bytes (ids, logits)."""
    Dy = _dyn()
    V, d, M, B, k, k_t = 4099, 128, 16, 24, 5, 8
    W, tau, perm, off, c = _exact_setup(V, d, M, seed=5)
    hn = S.step_inputs(B, d, 1, "bf16", "exact")[2].to(DEV)
    sel = _random_selection(B, M, k, 3)
    sl = np.zeros((B, M + 1), dtype=np.int32)
    for b in range(B):
        sl[b, :k + 1] = O.shortlist_offsets(sel[b, :k], off)
    args = (torch.as_tensor(sel, device=DEV), torch.full((B,), k, dtype=torch.int32, device=DEV),
            torch.as_tensor(sl, device=DEV), k_t)
    monkeypatch.setenv("DS_GH", "1")
    a = Dy.head_forward(c, hn, *args)
    monkeypatch.setenv("DS_GH", "0")
    monkeypatch.setenv("DS_DISABLE_TC", "1")
    b_ = Dy.head_forward(c, hn, *args)
    torch.cuda.synchronize()
    assert torch.equal(a["top_ids"], b_["top_ids"])
    assert torch.equal(a["top_logits"], b_["top_logits"])
    assert torch.allclose(a["lse"], b_["lse"], rtol=2e-6, atol=1e-6)


def test_gh_determinism():
    """Same inputs, same launch configuration -> identical bytes (R19: no float atomics)."""
    Dy = _dyn()
    C = S.CONFIGS["llama3"]
    W = S.lm_head(C.V, C.d, 0, "bf16", device=DEV)
    tau = torch.as_tensor(S.random_partition(C.V, C.M, 2), dtype=torch.int32, device=DEV)
    c = Dy.Clusters.from_tau(W, tau, C.M)
    r = Dy.Router(*[x.to(DEV) for x in S.router(C.d, C.h_r, C.M, 1, "bf16")])
    st = Dy.DraftStep(c, r, 32, C.k_t)
    assert st.kernel.startswith("ds::gh_head_kernel"), st.kernel
    hp, e, hn = [x.to(DEV) for x in S.step_inputs(32, C.d, 0, "bf16")]
    outs = []
    for _ in range(3):
        st(hp, e, hn, t=0, k_max=C.k_max, k_min=C.k_min)
        torch.cuda.synchronize()
        outs.append((st.top_ids.clone(), st.top_logp.clone(), st.lse.clone()))
    for o in outs[1:]:
        assert all(torch.equal(x, y) for x, y in zip(o, outs[0]))


@pytest.mark.parametrize("cfg,B,t", [("llama3", 16, 0), ("llama3", 64, 3), ("gemma3", 512, 0), ("gemma3", 512, 2)])
def test_gh_full_size_sampled_rows(cfg, B, t):
    """BASELINE configs at full size and the bench's batches (Llama-3 B = 16 / 64; Gemma-3 B = 512,
    k = 64 at t = 0 and 16 at t = 2): router + select + grouped head through dynaspec_draft_step;
    sampled rows against the oracle (scores, selection, offsets, top-k, lse)."""
    Dy = _dyn()
    C = S.CONFIGS[cfg]
    W = S.lm_head(C.V, C.d, 0, "bf16", device=DEV)
    tau = S.random_partition(C.V, C.M, 2)
    perm, off = O.layout(tau, C.M)
    part = {"perm": perm, "offsets": off}
    c = Dy.Clusters.from_tau(W, torch.as_tensor(tau, dtype=torch.int32, device=DEV), C.M)
    rt = S.router(C.d, C.h_r, C.M, 1, "bf16")
    r = Dy.Router(*[x.to(DEV) for x in rt])
    st = Dy.DraftStep(c, r, B, C.k_t)
    assert st.kernel.startswith("ds::gh_head_kernel"), st.kernel
    hp, e, hn = S.step_inputs(B, C.d, t, "bf16")
    st(hp.to(DEV), e.to(DEV), hn.to(DEV), t=t, k_max=C.k_max, k_min=C.k_min)
    torch.cuda.synchronize()
    Wo, ro = Rows(W), tuple(f64(x) for x in rt)
    for b in sorted({0, B // 3, B - 1}):
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


@pytest.mark.parametrize("B", [2, 3])
def test_gh_shared_tree_rows_exact(B):
    """Tree mode (R9: one index set for all rows of a depth) on the grouped head: every row streams
    the one union selection; bit-exact top-k against the oracle over the union shortlist."""
    Dy = _dyn()
    V, d, M, k, k_t = 5003, 256, 24, 6, 8
    W, tau, perm, off, c = _exact_setup(V, d, M)
    hn = S.step_inputs(B, d, 2, "bf16", "exact")[2]
    union = np.sort(np.random.default_rng(7).choice(M, size=k, replace=False)).astype(np.int32)
    sel = np.zeros((1, M), dtype=np.int32)
    sel[0, :k] = union
    sl = np.zeros((1, M + 1), dtype=np.int32)
    sl[0, :k + 1] = O.shortlist_offsets(union, off)
    out = Dy.head_forward(c, hn.to(DEV), torch.as_tensor(sel, device=DEV),
                          torch.tensor([k], dtype=torch.int32, device=DEV), torch.as_tensor(sl, device=DEV), k_t,
                          shared=True)
    torch.cuda.synchronize()
    VS = O.shortlist(union, perm, off)
    Wo = Rows(W)
    for b in range(B):
        z = O.head(f64(hn[b]), Wo, VS)[0]
        check_topk(out["top_ids"][b].cpu().numpy(), out["top_logits"][b].cpu().numpy(),
                   out["top_logp"][b].cpu().numpy(), out["lse"][b].item(), z, VS, k_t, torch.float32, exact=True)
